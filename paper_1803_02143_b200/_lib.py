"""ctypes binding of the vpb200 C ABI (``include/vpb200.h``).

This is the only way the package reaches the GPU.  There is no CPU
fallback: if the shared library is missing or no CUDA device is visible,
every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libvpb200.so"
_lib = None

VPB_OK = 0


class VpbError(RuntimeError):
    """A nonzero status from the C ABI."""


class FieldGeom(ctypes.Structure):
    """Mirror of ``vpb_field_geom``."""

    _fields_ = [
        ("n1", c_int64),
        ("n2", c_int64),
        ("c1", c_int64),
        ("c2", c_int64),
        ("ncomp", c_int32),
        ("g1", c_void_p),
        ("g2", c_void_p),
        ("m1", c_void_p),
        ("m2", c_void_p),
        ("kmul", c_void_p),
        ("wx1", c_void_p),
        ("wx2", c_void_p),
        ("volume", c_double),
        ("r1", c_int64),
        ("r2", c_int64),
    ]


Dims = c_int64 * 4

# name -> (restype, argtypes)
SIGNATURES = {
    "vpb_version": (c_char_p, []),
    "vpb_strerror": (c_char_p, [c_int]),
    "vpb_last_error": (c_char_p, []),
    "vpb_launch_count": (ctypes.c_ulonglong, []),
    "vpb_dg_sweep_contig": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32,
                                    c_void_p]),
    "vpb_dg_sweep_strided": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64), c_void_p,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                     c_int32, c_void_p]),
    "vpb_spline_sweep_contig": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                        c_void_p, c_int64, c_double, c_void_p]),
    "vpb_spline_sweep_strided": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64),
                                         c_void_p, c_void_p, c_int64, c_double, c_void_p]),
    "vpb_dg_tables": (c_int, [c_void_p, c_int64, c_double, c_double, c_int32, c_void_p,
                              c_void_p, c_void_p, c_void_p, c_void_p]),
    "vpb_dg_sweep_axis": (c_int, [c_int32, c_void_p, c_void_p, POINTER(c_int64), c_int32,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "vpb_dg_sweep_xplane": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p]),
    "vpb_dg_sweep_vplane": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p]),
    "vpb_dg_xplane_density_work_len": (c_int64, [POINTER(c_int64), c_int32]),
    "vpb_dg_sweep_xplane_density": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32,
                                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_double, c_void_p, c_void_p, c_void_p, c_void_p]),
    "vpb_dg_sweep_xplane_moments": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                                    + [c_void_p] * 17 + [c_double] + [c_void_p] * 5),
    "vpb_dg_sweep_xplane2": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                             + [c_void_p] * 13),
    "vpb_dg_xplane2_density_work_len": (c_int64, [POINTER(c_int64), c_int32]),
    "vpb_dg_sweep_xplane2_density": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                                     + [c_void_p] * 17 + [c_double] + [c_void_p] * 4),
    "vpb_dg_compose_tables": (c_int, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "vpb_dg_sweep_xcomp": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                           + [c_void_p] * 8),
    "vpb_dg_xcomp_density_work_len": (c_int64, [POINTER(c_int64), c_int32]),
    "vpb_dg_sweep_xcomp_density": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                                   + [c_void_p] * 12 + [c_double] + [c_void_p] * 4),
    "vpb_dg_single_tables": (c_int, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "vpb_dg_sweep_xstencil": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                              + [c_void_p] * 6 + [c_int32, c_void_p, c_int32, c_void_p, c_int32,
                                                  c_void_p, c_void_p]),
    "vpb_dg_xstencil_density_work_len": (c_int64, [POINTER(c_int64), c_int32, c_int32,
                                                   c_int32]),
    "vpb_dg_sweep_xstencil_density": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                                      + [c_void_p] * 6
                                      + [c_int32, c_void_p, c_int32, c_void_p, c_int32]
                                      + [c_void_p] * 6 + [c_double] + [c_void_p] * 4),
    "vpb_dg_sweep_xcomp_rows": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32,
                                        c_int64, c_int64] + [c_void_p] * 6
                                + [c_void_p] * 6 + [c_double] + [c_void_p] * 3
                                + [c_int32, c_void_p]),
    "vpb_dg_sweep_xstencil2": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32]
                               + [c_void_p] * 6
                               + [c_int32, c_void_p, c_int32, c_void_p, c_int32]
                               + [c_int32, c_void_p, c_int32, c_void_p]
                               + [c_void_p] * 6 + [c_double] + [c_void_p] * 4),
    "vpb_dg_sweep_xstencil_rows": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32,
                                           c_int64, c_int64]
                                   + [c_void_p] * 6
                                   + [c_int32, c_void_p, c_int32, c_void_p, c_int32]
                                   + [c_void_p] * 6 + [c_double] + [c_void_p] * 3
                                   + [c_int32, c_void_p]),
    "vpb_dg_sweep_vplane_v2halo": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_int32,
                                           c_int32, c_int32] + [c_void_p] * 12),
    "vpb_dg_sweep_vplane_v2peer": (c_int, [c_void_p, c_int32, c_int32, c_void_p, c_int32,
                                           c_int32, c_void_p, c_int32, c_int32, c_int32,
                                           c_void_p, POINTER(c_int64), c_int32]
                                   + [c_void_p] * 12),
    "vpb_slab_copy": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "vpb_spline_sweep_axis": (c_int, [c_int32, c_void_p, c_void_p, POINTER(c_int64), c_void_p,
                                      c_double, c_double, c_void_p, c_void_p]),
    "vpb_spline_sweep_axis2": (c_int, [c_int32, c_void_p, c_void_p, POINTER(c_int64), c_void_p,
                                       c_double, c_double, c_void_p, c_void_p]),
    "vpb_spline_density_part_len": (c_int64, [POINTER(c_int64)]),
    "vpb_spline_sweep_x1dbl_density": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_void_p,
                                               c_double, c_double, c_void_p, c_void_p, c_void_p,
                                               c_void_p]),
    "vpb_density_work_len": (c_int64, [POINTER(c_int64)]),
    "vpb_density": (c_int, [c_void_p, POINTER(c_int64), c_void_p, c_void_p, c_void_p, c_void_p,
                            c_void_p]),
    "vpb_field_work_len": (c_int64, [POINTER(FieldGeom)]),
    "vpb_field_solve": (c_int, [c_void_p, POINTER(FieldGeom), c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p]),
    "vpb_diag_work_len": (c_int64, [POINTER(c_int64)]),
    "vpb_diagnostics": (c_int, [c_void_p, POINTER(c_int64), c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
                                c_void_p]),
    "vpb_electric_energy": (c_int, [c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_void_p]),
    "vpb_fill_separable": (c_int, [c_void_p, POINTER(c_int64), c_void_p, c_void_p, c_void_p,
                                   c_void_p]),
    "vpb_halo_pack": (c_int, [c_int32, c_void_p, POINTER(c_int64), c_int32, c_int64, c_int64,
                              c_void_p, c_void_p]),
    "vpb_dg_sweep_axis_halo": (c_int, [c_int32, c_void_p, c_void_p, POINTER(c_int64), c_int32,
                                       c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p]),
}


def lib_path() -> Path:
    return _LIB_PATH


def load(path: Path | None = None):
    """Load (once) and type the shared library.  Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # VPB_LIB: load another build of the same ABI (A/B timing of kernel variants)
    p = Path(path) if path else Path(os.environ.get("VPB_LIB") or _LIB_PATH)
    if not p.exists():
        raise VpbError(
            f"vpb200 CUDA library not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    lib = ctypes.CDLL(str(p))
    override = not path and bool(os.environ.get("VPB_LIB"))
    for name, (res, args) in SIGNATURES.items():
        if override and not hasattr(lib, name):
            continue  # an older build under A/B timing: entry points it lacks stay unbound
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != VPB_OK:
        lib = load()
        detail = lib.vpb_last_error().decode(errors="replace")
        kind = lib.vpb_strerror(status).decode()
        if status == 1:
            raise ValueError(f"{what}: {detail}")
        raise VpbError(f"{what}: {kind}: {detail}")


def dims(shape4) -> "ctypes.Array":
    return Dims(*[int(v) for v in shape4])
