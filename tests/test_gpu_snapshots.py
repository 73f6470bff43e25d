"""VLF1 snapshot byte parity (reference field.py:246-295, test_grid.py:26-31,
309-333) against files WRITTEN BY THE REFERENCE (tests/golden/snapshots.npz,
made by tests/golden/make_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1803_02143_b200 as vpb
from vpb_testutil import max_rel

pytestmark = pytest.mark.gpu

# tests/test_grid.py:26-31 of the reference: magic, axis count, two axis
# records (lower, upper, count, kind), method, degree of a 4x4 spline grid
VLF1_HEADER_4X4 = bytes.fromhex(
    "564c463102000000"
    "000000000000000000000000000000400400000000"
    "000000000000f0bf000000000000f03f0400000001"
    "0000"
)

CASES = [("landau4d_dg3", "landau4d", "dg", 12, 3), ("landau4d_spline", "landau4d", "spline", 8, 0),
         ("landau2d_dg2", "landau2d", "dg", 16, 2)]


def _grid_4x4():
    return vpb.GridSpec((vpb.Axis(0.0, 2.0, 4, "space"), vpb.Axis(-1.0, 1.0, 4, "velocity")),
                        "spline")


def test_header_and_payload_order_4x4(golden, tmp_path):
    z = golden("snapshots")
    field = vpb.DistributionField.from_values(_grid_4x4(), np.arange(16.0).reshape(4, 4))
    path = tmp_path / "h.vlf"
    vpb.write_snapshot(field, path)
    blob = path.read_bytes()
    assert blob[: len(VLF1_HEADER_4X4)] == VLF1_HEADER_4X4
    assert len(blob) == len(VLF1_HEADER_4X4) + 16 * 8
    payload = np.frombuffer(blob[len(VLF1_HEADER_4X4):], dtype="<f8")
    np.testing.assert_array_equal(payload[:4], np.arange(16.0).reshape(4, 4)[:, 0])
    # the whole file is byte-identical to the one the reference wrote
    assert blob == z["h4x4_bytes"].tobytes()


@pytest.mark.parametrize("tag,prob,method,dofs,order", CASES)
def test_reads_reference_written_snapshots_exactly(golden, tmp_path, tag, prob, method, dofs,
                                                   order):
    z = golden("snapshots")
    path = tmp_path / f"{tag}.vlf"
    path.write_bytes(z[tag + "_bytes"].tobytes())
    field = vpb.read_snapshot(path)
    assert field.grid.method == method
    assert field.grid.dg_degree == (order - 1 if method == "dg" else 0)
    assert np.array_equal(field.numpy(), z[tag + "_array"])
    # and writes the same bytes back
    again = tmp_path / f"{tag}_again.vlf"
    vpb.write_snapshot(field, again)
    assert again.read_bytes() == path.read_bytes()


@pytest.mark.parametrize("tag,prob,method,dofs,order", CASES)
def test_written_snapshots_match_reference_bytes(golden, tmp_path, tag, prob, method, dofs, order):
    """Same grid and state: the header bytes are identical and the payload is
    the reference's state in the same order (bitwise for the initial state,
    within the parity bar after steps)."""
    z = golden("snapshots")
    ref = z[tag + "_bytes"].tobytes()
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    field = vpb.initialize(problem, grid)
    for _ in range(int(z[tag + "_steps"])):
        field = vpb.strang_step(field, 0.1, consume=True)
    path = tmp_path / f"{tag}.vlf"
    vpb.write_snapshot(field, path)
    blob = path.read_bytes()
    head = len(ref) - 8 * grid.total_dof
    assert blob[:head] == ref[:head]
    got = np.frombuffer(blob[head:], dtype="<f8")
    want = np.frombuffer(ref[head:], dtype="<f8")
    assert max_rel(got, want) <= 1e-12
    # payload order: canonical (x1 fastest, dG nodes innermost)
    canon = np.ascontiguousarray(z[tag + "_array"].transpose(*reversed(range(grid.ndim))))
    assert np.array_equal(want, canon.ravel())


def test_initial_state_snapshot_is_byte_identical(tmp_path):
    """Initial state (bitwise equal to the reference's, test_gpu_step) ->
    the whole VLF1 file equals what the reference writes for it."""
    from oracle import refstep

    slvp = refstep.load()
    for prob, method, dofs, order in (("landau4d", "dg", 12, 3), ("landau2d", "spline", 16, 0)):
        ours = tmp_path / "ours.vlf"
        theirs = tmp_path / "theirs.vlf"
        problem = vpb.problem_spec(prob)
        vpb.write_snapshot(vpb.initialize(problem, vpb.make_grid(problem, method, dofs,
                                                                 dg_order=order)), ours)
        rp = slvp.problem_spec(prob)
        slvp.write_snapshot(slvp.initialize(rp, slvp.make_grid(rp, method, dofs, dg_order=order)),
                            theirs)
        assert ours.read_bytes() == theirs.read_bytes(), (prob, method)
