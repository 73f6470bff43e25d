"""ORACLE -- TEST INFRASTRUCTURE ONLY.  CPU reference arm for bench.py.

Times the reference's own CPU implementation of one Strang step
(/root/reference/pkg/src/slvp/driver.py:245-265) on a BOUNDED, scaled
sample of a BASELINE configuration, with every host thread:

* line sweeps use the reference's compiled kernels (``oracle/_ref``, built
  from _kernels.pyx) with the reference's default strategies: dG sweeps
  ``dg_sweep_strided`` in place on the canonical array with cache_block=8,
  spline sweeps transposed to contiguous lines + ``spline_sweep_contig``
  (field.py:35, 176-202).  When _ref is absent the oracle's C restatement
  is used instead and the result is labelled "port".
* the sample: x1/x2/v1 sweeps, the per-sub-step finite checks and the
  density run on a slab of the full grid that keeps every axis whole except
  v2 (``slab`` rows); the v2 sweep runs on a slab that keeps v2 whole and
  cuts x2.  Per-dof times are scaled to the full grid.  The v-sweep
  projection tables and the Poisson solve are timed at full size.

Returns DOF-updates/s for the full configuration.
"""

from __future__ import annotations

import time

import numpy as np

from . import core, ref_kernels


def _kernels():
    mod = ref_kernels.load()
    return mod, ("reference" if mod is not None else "port")


def _slab_values(og: core.OGrid, prob: str, keep_axis_slab: dict) -> np.ndarray:
    """Initial values on a sub-box (logical order), canonical storage."""
    full = core.OGrid(og.lowers, og.uppers, og.counts, og.method, og.degree)
    pts = [full.points(a) for a in range(4)]
    for a, n in keep_axis_slab.items():
        pts[a] = pts[a][:n]
    _, _, eps, k, d, _ = core.PROBLEMS[prob]
    space = 1.0 + eps * (np.cos(k * pts[1])[:, None] + np.cos(k * pts[0])[None, :])
    g1 = np.exp(-0.5 * (pts[2] - d) ** 2)
    g2 = np.exp(-0.5 * pts[3] ** 2)
    phys = (g2[:, None] * g1[None, :])[:, :, None, None] * space[None, None, :, :]
    return np.ascontiguousarray(phys).transpose(3, 2, 1, 0)


def _sweep_inplace(mod, kind, arr, og, axis, shifts, table_axes, h, threads, block=8):
    """One reference sweep on (a slab of) the field; returns seconds."""
    t0 = time.perf_counter()
    idx = _table_index(arr.shape, axis, table_axes)
    if og.method == "dg":
        a, b, q, al = core.projection_pairs(shifts, h, og.degree)
        view = np.moveaxis(arr, axis, -1)
        if kind == "reference":
            mod.dg_sweep_strided(view, idx, a, b, q, al, view.shape[-1] // og.p, og.p, block,
                                 threads)
        else:
            lines = np.ascontiguousarray(view).reshape(-1, view.shape[-1])
            view[...] = core.dg_lines(lines, idx, a, b, q, al, view.shape[-1] // og.p, og.p,
                                      threads).reshape(view.shape)
    else:
        view = np.moveaxis(arr, axis, -1)
        lines = np.ascontiguousarray(view).reshape(-1, view.shape[-1])
        if kind == "reference":
            out = mod.spline_sweep_contig(lines, idx, np.ascontiguousarray(shifts), float(h),
                                          threads)
        else:
            out = core.spline_lines(lines, idx, shifts, h, threads)
        view[...] = out.reshape(view.shape)
    return time.perf_counter() - t0


def _table_index(shape, axis, table_axes):
    other = tuple(a for a in range(4) if a != axis)
    lead = tuple(shape[a] for a in other)
    idx = np.zeros(lead, dtype=np.int64)
    mult = 1
    for a in reversed(table_axes):
        pos = other.index(a)
        shp = [1] * 3
        shp[pos] = lead[pos]
        idx += (mult * np.arange(lead[pos], dtype=np.int64)).reshape(shp)
        mult *= shape[a]
    return idx.reshape(-1)


def _warmup(mod, kind, og, prob, tau, threads):
    """Spin up the OpenMP pool and caches on a tiny slab (untimed)."""
    W = _slab_values(og, prob, {2: og.p, 3: og.p})
    _sweep_inplace(mod, kind, W, og, 0, og.points(2)[:og.p] * tau, (2,), og.h(0), threads)
    _sweep_inplace(mod, kind, W, og, 2, np.zeros(og.shape[0] * og.shape[1]), (0, 1), og.h(2),
                   threads)


def reference_step_rate(prob: str, method: str, dofs: int, order: int, tau: float,
                        threads: int | None = None, slab: int = 0,
                        target_dofs: float = 4.0e7) -> dict:
    """Estimated reference DOF-updates/s of one full Strang step."""
    threads = threads or core.host_threads()
    mod, kind = _kernels()
    og = core.make_grid(prob, method, dofs, order)
    n1, n2, nv1, nv2 = og.shape
    N = n1 * n2 * nv1 * nv2
    if slab <= 0:  # size the sample to ~target_dofs, whole cells
        slab = -(-int(target_dofs) // (n1 * n2 * nv1))
    slab = min(nv2, max(og.p, -(-slab // og.p) * og.p) if method == "dg" else max(1, slab))
    _warmup(mod, kind, og, prob, tau, threads)
    A = _slab_values(og, prob, {3: slab})          # v2 cut
    B = _slab_values(og, prob, {1: slab})          # x2 cut
    nA, nB = A.size, B.size
    rng = np.random.default_rng(0)
    hx = [og.h(0), og.h(1)]
    hv = [og.h(2), og.h(3)]
    t = {}
    # x sweeps (tables over the matching velocity axis; x2's over the slab rows)
    t["x1"] = _sweep_inplace(mod, kind, A, og, 0, og.points(2) * (0.5 * tau), (2,), hx[0],
                             threads) * N / nA
    t["x2"] = _sweep_inplace(mod, kind, A, og, 1, og.points(3)[:slab] * (0.5 * tau), (3,),
                             hx[1], threads) * N / nA
    # v sweeps: E-like shifts of realistic size (|E| ~ 1)
    e1 = rng.uniform(-1.0, 1.0, n1 * n2) * tau
    t["v1"] = _sweep_inplace(mod, kind, A, og, 2, e1, (0, 1), hv[0], threads) * N / nA
    e2 = rng.uniform(-1.0, 1.0, n1 * slab) * tau
    t["v2"] = _sweep_inplace(mod, kind, B, og, 3, e2, (0, 1), hv[1], threads) * N / nB
    # per-sub-step finite checks (driver.py:209-211)
    t0 = time.perf_counter()
    np.isfinite(np.sum(A.transpose(3, 2, 1, 0).reshape(-1)))  # field.data is the flat storage
    t["checks"] = 6 * (time.perf_counter() - t0) * N / nA
    # density (poisson.py:85-95) on the slab, scaled
    t0 = time.perf_counter()
    rho = np.einsum("abcd,c,d->ab", A, og.weights(2), og.weights(3)[:slab], optimize=False)
    t["density"] = (time.perf_counter() - t0) * N / nA
    # Poisson at full size, and the two full-size v-sweep table builds
    t0 = time.perf_counter()
    core.solve_poisson(rho * (nv2 / slab), og)
    t["field_solve"] = time.perf_counter() - t0
    if method == "dg":
        t0 = time.perf_counter()
        core.projection_pairs(e1, hv[0], og.degree)
        core.projection_pairs(e1, hv[1], og.degree)
        t["v_tables"] = time.perf_counter() - t0
    step = 2 * t["x1"] + 2 * t["x2"] + sum(v for k, v in t.items() if k not in ("x1", "x2"))
    return {
        "dof_per_s": N / step,
        "step_s": step,
        "kind": kind,
        "threads": threads,
        "sample": (f"{prob} {method}{order if method == 'dg' else ''} {dofs}^4 step scaled from "
                   f"sweeps on slabs of {nA:,} (v2 cut to {slab}) and {nB:,} (x2 cut) dofs, "
                   "full-size Poisson and tables"),
        "parts_s": t,
    }
