"""The C-ABI library loads and exports every symbol include/vpb200.h declares.

No compute calls here (no GPU in the build container); argument validation
that fails before any device work is exercised.
"""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vpb200.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vpb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1803_02143_b200 import _build, _lib

    _build.build()
    return _lib.load()


def test_header_declares_the_plugin_entry_points():
    syms = declared_symbols()
    for name in ("vpb_dg_sweep_contig", "vpb_dg_sweep_strided", "vpb_spline_sweep_contig",
                 "vpb_spline_sweep_strided", "vpb_dg_tables", "vpb_dg_sweep_axis",
                 "vpb_spline_sweep_axis", "vpb_density", "vpb_field_solve", "vpb_diagnostics"):
        assert name in syms


def test_every_declared_symbol_is_exported(lib):
    from paper_1803_02143_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.lib_path())],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (vpb_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and every exported vpb_ symbol is typed in the ctypes binding
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_version_and_error_strings(lib):
    assert lib.vpb_version().startswith(b"vpb200")
    assert lib.vpb_strerror(0) == b"ok"
    assert lib.vpb_strerror(1) == b"invalid argument"
    assert lib.vpb_strerror(3) == b"unsupported"


def test_argument_validation_without_device(lib):
    from paper_1803_02143_b200 import _lib

    dims = _lib.dims((48, 48, 48, 48))
    # axis out of range: rejected before touching the device
    rc = lib.vpb_dg_sweep_axis(7, 1, 2, dims, 3, None, None, None, None, None, None)
    assert rc == 1
    assert b"axis" in lib.vpb_last_error()
    # src aliases dst
    rc = lib.vpb_dg_sweep_axis(0, 16, 16, dims, 3, None, None, None, None, None, None)
    assert rc == 1
    # non-positive cell width (dg.py:109-110)
    rc = lib.vpb_dg_tables(None, 0, 1.0, -1.0, 3, None, None, None, None, None)
    assert rc == 1
    with pytest.raises(ValueError, match="cell width"):
        _lib.check(rc, "vpb_dg_tables")
    # ragged line (dg.py:169-171)
    rc = lib.vpb_dg_sweep_contig(1, 2, 1, 7, 3, None, None, None, None, 1, 2, 3, None)
    assert rc == 1
    rc = lib.vpb_spline_sweep_contig(1, 2, 1, 1, 3, 4, 1, 0.5, None)
    assert rc == 1
    assert lib.vpb_density_work_len(dims) > 0
    assert lib.vpb_diag_work_len(dims) == 3 * 48 * 48
    # merged x passes: aliasing, orders, qmul, halo widths (all host-side checks)
    rc = lib.vpb_dg_sweep_xcomp(16, 16, dims, 3, 1, 2, 3, 4, 5, 6, None, None)
    assert rc == 1 and b"distinct" in lib.vpb_last_error()
    rc = lib.vpb_dg_sweep_xcomp(16, 32, dims, 12, 1, 2, 3, 4, 5, 6, None, None)
    assert rc == 1 and b"order" in lib.vpb_last_error()
    rc = lib.vpb_dg_compose_tables(1, 2, 5, 0, 3, None)
    assert rc == 1
    rc = lib.vpb_dg_sweep_xstencil(16, 32, dims, 3, 1, 2, 3, 4, 5, 6, 3, None, 0, None, 0,
                                   None, None)
    assert rc == 1 and b"qmul" in lib.vpb_last_error()
    # odd order: halo blocks must stay 16-byte multiples (even widths)
    rc = lib.vpb_dg_sweep_xstencil(16, 32, dims, 3, 1, 2, 3, 4, 5, 6, 2, 64, 1, 64, 2,
                                   None, None)
    assert rc == 1 and b"16-byte" in lib.vpb_last_error()
    rc = lib.vpb_dg_sweep_xstencil(16, 32, dims, 3, 1, 2, 3, 4, 5, 6, 2, 64, 20, 64, 2,
                                   None, None)
    assert rc == 1 and b"wider than the shard" in lib.vpb_last_error()
    # spline double sweep: axis range
    rc = lib.vpb_spline_sweep_axis2(5, 16, 32, dims, 1, 0.1, 0.5, None, None)
    assert rc == 1


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200._lib import VpbError

    grid = vpb.make_grid(vpb.problem_spec("landau4d"), "dg", 12, dg_order=3)
    with pytest.raises(VpbError, match="CUDA device"):
        vpb.initialize(vpb.problem_spec("landau4d"), grid)


def test_library_has_no_torch_dependency():
    from paper_1803_02143_b200 import _lib

    out = subprocess.run(["ldd", str(_lib.lib_path())], capture_output=True, text=True).stdout
    assert "torch" not in out and "c10" not in out
    ctypes.CDLL(str(_lib.lib_path()))
