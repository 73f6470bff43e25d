"""ORACLE -- TEST INFRASTRUCTURE ONLY.  The UNMODIFIED reference, driven
through its own public API, on the GPU box's host cores.

``slvp`` is the reference package installed into ``oracle/_ref/site`` by
``oracle/build.py`` (pip install of /root/reference/pkg, compiled backend).
This module

* builds a BASELINE configuration with the reference's own ``make_grid`` /
  ``initialize`` (config 3: BASELINE's two-stream IC through
  ``DistributionField.from_values``), and
* times ``strang_step(field, tau, workers=T, consume=True)`` with the
  reference's ``bench_step`` protocol (/root/reference/pkg/src/slvp/
  bench.py:54-68: warm-up steps, then per-step ``perf_counter`` samples,
  median), timing as many FULL steps as fit in a wall-clock budget.

It is used by bench.py's ``--impl reference`` arm and ``cpu_baseline`` leg
and by the full-size GPU parity tests (reference trajectories at BASELINE
sizes).  Nothing here is on the product path.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import build


def load():
    slvp = build.load_ref_pkg()
    if slvp is None:
        raise RuntimeError("reference package not built (python -m oracle.build)")
    if slvp.backend_name() != "compiled":
        slvp.set_backend("compiled")
    return slvp


def host_threads() -> int:
    return len(os.sched_getaffinity(0))


def baseline_twostream_values(slvp, grid) -> np.ndarray:
    """BASELINE.json config 3 initial data in logical order (the same numpy
    expression as tests/golden/make_golden.py and the product's
    ``twostream4d_baseline`` problem)."""
    eps, k, d = 1e-3, 0.2, 2.4
    pts = [grid.axis_points(a) for a in range(4)]
    root = math.sqrt(2.0 * math.pi)
    space = 1.0 + eps * (np.cos(k * pts[1])[:, None] + np.cos(k * pts[0])[None, :])
    g1 = 0.5 * (np.exp(-0.5 * (pts[2] - d) ** 2) + np.exp(-0.5 * (pts[2] + d) ** 2)) / root
    g2 = np.exp(-0.5 * pts[3] ** 2) / root
    phys = (g2[:, None] * g1[None, :])[:, :, None, None] * space[None, None, :, :]
    return np.ascontiguousarray(phys.transpose(3, 2, 1, 0))


def make_field(slvp, problem: str, method: str, dofs, order: int):
    """(grid, field) of a BASELINE configuration, reference default strategy."""
    if problem == "twostream4d_baseline":
        # the reference's twostream4d geometry (x in [0, 10 pi]^2, v in [-6, 6]^2)
        # with BASELINE's initial data (tests/golden/make_golden.py does the same)
        grid = slvp.make_grid(slvp.problem_spec("twostream4d"), method, dofs, dg_order=order)
        field = slvp.DistributionField.from_values(grid, baseline_twostream_values(slvp, grid))
        return grid, field
    prob = slvp.problem_spec(problem)
    grid = slvp.make_grid(prob, method, dofs, dg_order=order)
    return grid, slvp.initialize(prob, grid)


def time_steps(problem: str, method: str, dofs, order: int, tau: float, *,
               threads: int | None = None, warmup: int = 1, max_steps: int = 3,
               budget_s: float = 240.0) -> dict:
    """Reference ``strang_step`` wall times: ``warmup`` untimed steps, then up
    to ``max_steps`` timed steps while the elapsed timed time stays inside
    ``budget_s`` (at least one).  Returns the median like ``bench_step``."""
    slvp = load()
    threads = threads or host_threads()
    t0 = time.perf_counter()
    grid, field = make_field(slvp, problem, method, dofs, order)
    init_s = time.perf_counter() - t0
    n = int(np.prod([grid.dof(a) for a in range(grid.ndim)]))
    for _ in range(warmup):
        field = slvp.strang_step(field, tau, workers=threads, consume=True)
    samples = []
    spent = 0.0
    while len(samples) < max(1, max_steps):
        t0 = time.perf_counter()
        field = slvp.strang_step(field, tau, workers=threads, consume=True)
        dt = time.perf_counter() - t0
        samples.append(dt)
        spent += dt
        if spent + dt > budget_s:
            break
    step = float(np.median(samples))
    return {
        "dof_per_s": n / step,
        "step_s": step,
        "samples_s": samples,
        "steps_timed": len(samples),
        "warmup": warmup,
        "threads": threads,
        "dofs": n,
        "init_s": init_s,
        "kind": "reference",
        "sample": (f"reference slvp.strang_step(consume=True, workers={threads}) on the full "
                   f"{problem} {method}{order if method == 'dg' else ''} {dofs}^4 grid "
                   f"({n:,} dofs): {warmup} warm-up + {len(samples)} timed full steps, median "
                   "(bench_step protocol, slvp/bench.py:54-68)"),
    }
