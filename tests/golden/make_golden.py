"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference package is copied to a scratch directory and its Cython
kernels are built there (its source tree is read-only), then imported and
driven through its public API.  Outputs:

  kernels.npz  projection_pairs, spline factors, dg/spline line sweeps on
               seeded random lines (compiled backend)
  steps.npz    short trajectories (f after each step + diagnostics) on small
               2x2v / 1x1v grids for every method/order the tests cover
  series.npz   diagnostics time series at BASELINE config 1 (48^4, 20 steps)
               and reduced-size configs 3 (200 steps) and 4 (50 steps), plus
               per-step f checksums
  snapshots.npz  VLF1 files written by the reference's write_snapshot (raw
               bytes) and the arrays they hold

Nothing here is used at run time on the GPU box; the .npz files are.
"""

from __future__ import annotations

import math
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path(os.environ.get("SLVP_REFERENCE", "/root/reference/pkg"))


def load_reference():
    scratch = Path(tempfile.mkdtemp(prefix="slvp_ref_"))
    pkg = scratch / "pkg"
    shutil.copytree(REF, pkg, ignore=shutil.ignore_patterns("frontend"))
    env = dict(os.environ, CC="/usr/bin/gcc", LDSHARED="/usr/bin/gcc -shared")
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=pkg, env=env,
                   check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, str(pkg / "src"))
    import slvp  # noqa: E402

    assert slvp.backend_name() == "compiled", slvp.backend_name()
    return slvp


def records_array(records) -> np.ndarray:
    keys = ("time", "electric_energy", "mass", "l1_norm", "l2_norm", "kinetic_energy",
            "total_energy")
    return np.array([[getattr(r, k) for k in keys] for r in records])


def baseline_twostream_values(grid) -> np.ndarray:
    """BASELINE.json config 3 initial data in logical order (same expression
    as oracle.core.initialize('twostream4d_baseline'))."""
    eps, k, d = 1e-3, 0.2, 2.4
    pts = [grid.axis_points(a) for a in range(4)]
    root = math.sqrt(2.0 * math.pi)
    space = 1.0 + eps * (np.cos(k * pts[1])[:, None] + np.cos(k * pts[0])[None, :])
    g1 = 0.5 * (np.exp(-0.5 * (pts[2] - d) ** 2) + np.exp(-0.5 * (pts[2] + d) ** 2)) / root
    g2 = np.exp(-0.5 * pts[3] ** 2) / root
    phys = (g2[:, None] * g1[None, :])[:, :, None, None] * space[None, None, :, :]
    return np.ascontiguousarray(phys.transpose(3, 2, 1, 0))


def kernels_fixture(slvp) -> dict:
    from slvp import _kernels as ck
    from slvp import _kernels_py as pk
    from slvp.dg import projection_pairs

    out = {}
    rng = np.random.default_rng(20260419)
    shifts = np.concatenate([
        [0.0, 1e-12, -1e-12, 0.3, -0.3, 0.7 * 3, -0.7 * 3, 1.0 - 1e-12, 2.5, -2.75, 7.0, -11.0,
         123.456],
        rng.uniform(-3.0, 3.0, 40),
    ])
    for h in (0.7, 0.5, 1.0):
        for deg in range(0, 5):
            a, b, q, al = projection_pairs(shifts, h, deg)
            tag = f"pp_h{h}_d{deg}"
            out[tag + "_a"], out[tag + "_b"], out[tag + "_q"], out[tag + "_alpha"] = a, b, q, al
    out["pp_shifts"] = shifts
    for n in (4, 5, 16, 48, 128, 288):
        mult, denom, z, sden = pk._factors(n)
        out[f"fac{n}"] = np.concatenate([mult, denom, z, [sden]])
    # dg line sweeps
    for p in (1, 2, 3, 4):
        for C in (4, 9, 16):
            n = C * p
            lines = rng.standard_normal((64, n))
            tab = rng.uniform(-3.0, 3.0, 6) * 0.4
            tab[0] = 0.0
            tab[1] = 2 * 0.4  # whole-cell shift -> alpha == 0 branch
            a, b, q, al = projection_pairs(tab, 0.4, p - 1)
            idx = rng.integers(0, 6, 64).astype(np.int64)
            res = ck.dg_sweep_contig(lines, idx, a, b, q, al, C, p, 2)
            tag = f"dg_p{p}_c{C}"
            out[tag + "_lines"], out[tag + "_idx"], out[tag + "_table"] = lines, idx, tab
            out[tag + "_out"] = res
    for n in (4, 16, 48, 128):
        lines = rng.standard_normal((48, n))
        tab = np.concatenate([[0.0, 3 * 0.25, -0.25, 40.0], rng.uniform(-20.0, 20.0, 4)])
        idx = rng.integers(0, tab.size, 48).astype(np.int64)
        res = ck.spline_sweep_contig(np.ascontiguousarray(lines), idx, tab, 0.25, 2)
        tag = f"sp_n{n}"
        out[tag + "_lines"], out[tag + "_idx"], out[tag + "_table"], out[tag + "_out"] = (
            lines, idx, tab, res)
    return out


def steps_fixture(slvp) -> dict:
    out = {}
    cases = [
        ("landau4d_dg3", "landau4d", "dg", 12, 3, 0.1, 3, None),
        ("landau4d_dg4", "landau4d", "dg", 16, 4, 0.1, 2, None),
        ("landau4d_spline", "landau4d", "spline", 12, 0, 0.1, 3, None),
        ("twostream_dg2", "twostream4d", "dg", 12, 2, 0.1, 3, "baseline"),
        ("twostream_ref_dg3", "twostream4d", "dg", 12, 3, 0.1, 2, None),
        ("landau2d_dg4", "landau2d", "dg", 32, 4, 0.1, 3, None),
        ("landau2d_spline", "landau2d", "spline", 32, 0, 0.1, 3, None),
    ]
    for tag, prob, method, dofs, order, tau, nsteps, ic in cases:
        problem = slvp.problem_spec(prob)
        grid = slvp.make_grid(problem, method, dofs, dg_order=order)
        if ic == "baseline":
            field = slvp.DistributionField.from_values(grid, baseline_twostream_values(grid))
        else:
            field = slvp.initialize(problem, grid)
        recs = [slvp.diagnostics(field, 0.0)]
        states = [field.array.copy()]
        for m in range(1, nsteps + 1):
            field = slvp.strang_step(field, tau, workers=2, consume=True)
            recs.append(slvp.diagnostics(field, m * tau))
            states.append(field.array.copy())
        out[tag + "_f"] = np.stack(states)
        out[tag + "_rec"] = records_array(recs)
    return out


def series_fixture(slvp) -> dict:
    out = {}
    cases = [
        # tag, problem, method, dofs, order, tau, nsteps, ic
        ("cfg1", "landau4d", "dg", 48, 3, 0.1, 20, None),
        ("cfg3_small", "twostream4d", "dg", 32, 2, 0.1, 200, "baseline"),
        ("cfg4_small", "landau4d", "spline", 32, 0, 0.1, 50, None),
    ]
    workers = len(os.sched_getaffinity(0))
    for tag, prob, method, dofs, order, tau, nsteps, ic in cases:
        problem = slvp.problem_spec(prob)
        grid = slvp.make_grid(problem, method, dofs, dg_order=order)
        if ic == "baseline":
            field = slvp.DistributionField.from_values(grid, baseline_twostream_values(grid))
        else:
            field = slvp.initialize(problem, grid)
        recs = [slvp.diagnostics(field, 0.0)]
        sums = []
        for m in range(1, nsteps + 1):
            field = slvp.strang_step(field, tau, workers=workers, consume=True)
            recs.append(slvp.diagnostics(field, m * tau))
            a = field.array
            sums.append([float(np.sum(a)), float(np.sum(a * a)), float(np.max(np.abs(a)))])
        out[tag + "_rec"] = records_array(recs)
        out[tag + "_sums"] = np.array(sums)
    return out


def snapshot_fixture(slvp) -> dict:
    """VLF1 files written by the reference's write_snapshot (field.py:260-271),
    raw bytes, plus the logical array each one holds."""
    from slvp.grid import SPACE, VELOCITY, Axis, GridSpec

    out = {}
    tmp = Path(tempfile.mkdtemp(prefix="vlf_"))
    cases = [
        # tag, problem, method, dofs, order, steps
        ("landau4d_dg3", "landau4d", "dg", 12, 3, 1),
        ("landau4d_spline", "landau4d", "spline", 8, 0, 1),
        ("landau2d_dg2", "landau2d", "dg", 16, 2, 2),
    ]
    for tag, prob, method, dofs, order, nsteps in cases:
        problem = slvp.problem_spec(prob)
        grid = slvp.make_grid(problem, method, dofs, dg_order=order)
        field = slvp.initialize(problem, grid)
        for _ in range(nsteps):
            field = slvp.strang_step(field, 0.1, workers=2, consume=True)
        path = tmp / f"{tag}.vlf"
        slvp.write_snapshot(field, path)
        out[tag + "_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
        out[tag + "_array"] = np.ascontiguousarray(field.array)
        out[tag + "_steps"] = np.array(nsteps)
    # the frozen 4x4 spline header case of tests/test_grid.py:309-320
    grid = GridSpec((Axis(0.0, 2.0, 4, SPACE), Axis(-1.0, 1.0, 4, VELOCITY)), "spline")
    field = slvp.DistributionField.from_values(grid, np.arange(16.0).reshape(4, 4))
    path = tmp / "h4x4.vlf"
    slvp.write_snapshot(field, path)
    out["h4x4_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
    shutil.rmtree(tmp, ignore_errors=True)
    return out


def main() -> None:
    slvp = load_reference()
    if "--snapshots-only" in sys.argv:
        np.savez_compressed(HERE / "snapshots.npz", **snapshot_fixture(slvp))
        return
    np.savez_compressed(HERE / "snapshots.npz", **snapshot_fixture(slvp))
    np.savez_compressed(HERE / "kernels.npz", **kernels_fixture(slvp))
    np.savez_compressed(HERE / "steps.npz", **steps_fixture(slvp))
    np.savez_compressed(HERE / "series.npz", **series_fixture(slvp))
    for f in ("kernels.npz", "steps.npz", "series.npz", "snapshots.npz"):
        print(f, (HERE / f).stat().st_size)


if __name__ == "__main__":
    main()
