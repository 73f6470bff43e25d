"""Multi-GPU layer: x-sharded distribution function, halo exchange, ρ gather.

SURVEY.md §8e / BASELINE north star.  The 4-D field is split along x1 (and x2
on 8 GPUs, a 4 x 2 process grid) into whole cells; every rank owns the
canonical-layout box f[v2][v1][x2 local][x1 local].  One Strang step:

* x half sweeps: each sharded x axis needs the source cells c-q-1, c-q of
  its neighbours: one-sided halo slabs whose widths come from the sweep's
  q range (wl = max(q)+1 cells on the left, wr = -min(q) on the right) are
  packed on device (``vpb_halo_pack``), exchanged with the two neighbours
  (grouped NCCL send/recv over NVLink), and the sweep reads them in place
  (``vpb_dg_sweep_axis_halo``).  An unsharded x axis is swept locally
  (periodic).  When neither x axis is sharded the fused x-plane kernel runs.
* density: the local ρ slab is all-gathered and every rank solves the
  Poisson problem redundantly (a few hundred kB, microseconds).
* v sweeps: fully local, tables from the local slice of E.
* non-finite flags are max-reduced so every rank raises the same
  ``SubstepError``; diagnostics are sum-reduced.

Communication is pluggable: :class:`TorchComm` wraps ``torch.distributed``
(NCCL on GPUs, gloo in the CPU tests); :class:`VirtualComm` runs several
shards inside one process (halo "messages" are device copies), which lets a
single GPU check the sharded kernels bitwise against the unsharded step.
The local compute is pluggable too (:class:`CudaOps` is the product; the
CPU tests substitute an oracle-backed implementation).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from .grid import DG, SPLINE, GridSpec


# ---------------------------------------------------------------------------
# Decomposition
# ---------------------------------------------------------------------------
def process_grid(world: int) -> tuple[int, int]:
    """(p1, p2) for x1 x x2 sharding: x1 only up to 4 ranks, 4 x 2 at 8
    (the north-star layout); other counts split x1 as evenly as possible."""
    if world == 8:
        return 4, 2
    if world <= 4:
        return world, 1
    for p2 in (2, 3, 4):
        if world % p2 == 0 and world // p2 <= 8:
            return world // p2, p2
    return world, 1


def split_cells(ncells: int, parts: int, r: int) -> tuple[int, int]:
    """Cell range [c0, c1) of part r (near-equal contiguous split)."""
    base, extra = divmod(ncells, parts)
    c0 = r * base + min(r, extra)
    return c0, c0 + base + (1 if r < extra else 0)


@dataclass(frozen=True)
class Decomposition:
    grid: GridSpec
    p1: int
    p2: int

    def __post_init__(self) -> None:
        if self.grid.ndim != 4:
            raise ValueError("sharding needs a 2x2v grid")
        for p, ax in ((self.p1, 0), (self.p2, 1)):
            if p < 1 or p > self.grid.axes[ax].count:
                raise ValueError(f"cannot split {self.grid.axes[ax].count} cells into {p} shards")

    @property
    def world(self) -> int:
        return self.p1 * self.p2

    def coords(self, rank: int) -> tuple[int, int]:
        return divmod(rank, self.p2)

    def rank_of(self, r1: int, r2: int) -> int:
        return (r1 % self.p1) * self.p2 + (r2 % self.p2)

    def cells(self, rank: int, axis: int) -> tuple[int, int]:
        r = self.coords(rank)[axis]
        return split_cells(self.grid.axes[axis].count, (self.p1, self.p2)[axis], r)

    def local_dims(self, rank: int) -> tuple[int, int, int, int]:
        p = self.grid.order
        a0, b0 = self.cells(rank, 0)
        a1, b1 = self.cells(rank, 1)
        return ((b0 - a0) * p, (b1 - a1) * p, self.grid.dof(2), self.grid.dof(3))

    def neighbours(self, rank: int, axis: int) -> tuple[int, int]:
        """(left, right) ranks along a sharded x axis (periodic)."""
        r1, r2 = self.coords(rank)
        if axis == 0:
            return self.rank_of(r1 - 1, r2), self.rank_of(r1 + 1, r2)
        return self.rank_of(r1, r2 - 1), self.rank_of(r1, r2 + 1)

    def sharded(self, axis: int) -> bool:
        return (self.p1, self.p2)[axis] > 1

    # host-side views for tests and I/O
    def local_slice(self, rank: int, logical: np.ndarray) -> np.ndarray:
        p = self.grid.order
        a0, b0 = self.cells(rank, 0)
        a1, b1 = self.cells(rank, 1)
        return logical[a0 * p:b0 * p, a1 * p:b1 * p]


def halo_widths(q: np.ndarray) -> tuple[int, int]:
    """Cells needed left / right of a shard for cell offsets q (dg.py:116-124)."""
    q = np.asarray(q)
    if q.size == 0:
        return 0, 0
    return max(0, int(q.max()) + 1), max(0, -int(q.min()))


# ---------------------------------------------------------------------------
# Communication
# ---------------------------------------------------------------------------
# message kinds of a halo exchange: "L" becomes the receiver's LEFT halo (the
# sender's last cells, sent to its right neighbour); "R" its RIGHT halo.
KIND_L, KIND_R = 0, 1
KIND_A2A = 2  # all-to-all reshard chunks (one per peer pair)
# x2 halos of the x1 x x2 stencil pass: receiver's left / right x2 halo, parts
# 0 (x1 dofs), 1 (their left x1 halo cells), 2 (their right x1 halo cells)
KIND_X2L = (10, 11, 12)
KIND_X2R = (13, 14, 15)


class TorchComm:
    """torch.distributed: one shard per process (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, msgs: dict) -> None:
        """msgs: {local_rank: [(kind, send_peer, send_buf, recv_peer, recv_buf), ...]}.
        Every rank posts, per kind in order, its send and its receive."""
        ops = []
        for _, items in msgs.items():
            for kind, sp, sbuf, rp, rbuf in items:
                if sbuf is not None and sbuf.numel():
                    ops.append(self.dist.P2POp(self.dist.isend, sbuf, sp, self.group, tag=kind))
                if rbuf is not None and rbuf.numel():
                    ops.append(self.dist.P2POp(self.dist.irecv, rbuf, rp, self.group, tag=kind))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def exchange_async(self, msgs: dict) -> list:
        """Post the exchange and return its requests: ``wait(reqs)`` later
        orders the current stream after it (NCCL) / blocks until done (gloo),
        so device work queued in between overlaps the transfer."""
        ops = []
        for _, items in msgs.items():
            for kind, sp, sbuf, rp, rbuf in items:
                if sbuf is not None and sbuf.numel():
                    ops.append(self.dist.P2POp(self.dist.isend, sbuf, sp, self.group, tag=kind))
                if rbuf is not None and rbuf.numel():
                    ops.append(self.dist.P2POp(self.dist.irecv, rbuf, rp, self.group, tag=kind))
        return list(self.dist.batch_isend_irecv(ops)) if ops else []

    @staticmethod
    def wait(reqs: list) -> None:
        for req in reqs:
            req.wait()

    def allgather_object(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier_device(self) -> None:
        """Order every rank's stream after every other rank's queued work
        (a one-element all-reduce on the stream; no host synchronisation)."""
        t = torch.zeros(1, dtype=torch.int32,
                        device=torch.device("cuda", torch.cuda.current_device())
                        if torch.cuda.is_available() else "cpu")
        self.dist.all_reduce(t, group=self.group)

    def allgather(self, local: dict) -> list:
        (t,) = local.values()
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def allreduce(self, local: dict, op: str) -> torch.Tensor:
        (t,) = local.values()
        t = t.clone()
        red = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX}[op]
        self.dist.all_reduce(t, op=red, group=self.group)
        return t


class VirtualComm:
    """All shards live in this process; messages are tensor copies."""

    def __init__(self, world: int):
        self.world = world

    def exchange(self, msgs: dict) -> None:
        # index sends by (receiver, kind, sender)
        sent = {}
        for rank, items in msgs.items():
            for kind, sp, sbuf, _, _ in items:
                if sbuf is not None:
                    sent[(sp, kind, rank)] = sbuf
        for rank, items in msgs.items():
            for kind, _, _, rp, rbuf in items:
                if rbuf is not None and rbuf.numel():
                    rbuf.copy_(sent[(rank, kind, rp)])

    def exchange_async(self, msgs: dict) -> list:
        self.exchange(msgs)
        return []

    @staticmethod
    def wait(reqs: list) -> None:
        return None

    def barrier_device(self) -> None:
        return None  # one process, one stream: already ordered

    def allgather(self, local: dict) -> list:
        return [local[r] for r in range(self.world)]

    def allreduce(self, local: dict, op: str) -> torch.Tensor:
        ts = [local[r] for r in sorted(local)]
        out = ts[0].clone()
        for t in ts[1:]:
            out = out + t if op == "sum" else torch.maximum(out, t)
        return out


# ---------------------------------------------------------------------------
# Local compute (product: the CUDA kernels)
# ---------------------------------------------------------------------------
class CudaOps:
    """Local kernels of a shard, through the C ABI."""

    def __init__(self):
        from . import _device, _lib

        self.lib = _lib.load()
        self._lib = _lib
        self._device = _device

    def tables(self, values, scale, h, degree):
        from .dg import DeviceTables

        return DeviceTables(values, scale, h, degree)

    def tables_q(self, tab) -> np.ndarray:
        return tab.q.cpu().numpy()

    def sweep(self, axis, src, dst, dims, order, tab, flag):
        L = self._lib
        L.check(self.lib.vpb_dg_sweep_axis(axis, src.data_ptr(), dst.data_ptr(), L.dims(dims), order,
                                           tab.a.data_ptr(), tab.b.data_ptr(), tab.q.data_ptr(),
                                           tab.alpha.data_ptr(), flag.data_ptr(),
                                           self._device.stream()), "vpb_dg_sweep_axis")

    def xplane(self, src, dst, dims, order, t1, t2, f1, f2):
        L = self._lib
        L.check(self.lib.vpb_dg_sweep_xplane(src.data_ptr(), dst.data_ptr(), L.dims(dims), order,
                                             t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(),
                                             t1.alpha.data_ptr(), t2.a.data_ptr(), t2.b.data_ptr(),
                                             t2.q.data_ptr(), t2.alpha.data_ptr(), f1.data_ptr(),
                                             f2.data_ptr(), self._device.stream()),
                "vpb_dg_sweep_xplane")

    def spline_sweep(self, axis, src, dst, dims, values, scale, h, flag):
        L = self._lib
        L.check(self.lib.vpb_spline_sweep_axis(axis, src.data_ptr(), dst.data_ptr(), L.dims(dims),
                                               values.data_ptr(), float(scale), float(h),
                                               flag.data_ptr(), self._device.stream()),
                "vpb_spline_sweep_axis")

    def slab_copy(self, src, src_stride, dst, dst_stride, outer, run):
        L = self._lib
        L.check(self.lib.vpb_slab_copy(src.data_ptr(), src_stride, dst.data_ptr(), dst_stride,
                                       outer, run, self._device.stream()), "vpb_slab_copy")

    def vplane(self, src, dst, dims, order, t1, t2, f1, f2):
        """Both v sweeps of a shard in one pass (they are local in x)."""
        L = self._lib
        L.check(self.lib.vpb_dg_sweep_vplane(src.data_ptr(), dst.data_ptr(), L.dims(dims), order,
                                             t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(),
                                             t1.alpha.data_ptr(), t2.a.data_ptr(), t2.b.data_ptr(),
                                             t2.q.data_ptr(), t2.alpha.data_ptr(), f1.data_ptr(),
                                             f2.data_ptr(), self._device.stream()),
                "vpb_dg_sweep_vplane")

    # -- three-cell x-plane stencil with x1 halos (merged / single x half steps)
    def stencil_tables(self, tab, single: bool) -> torch.Tensor:
        """[n][3][p][p]: {AA, AB+BA, BB} (merged pair) or {0, A, B} (one sweep)."""
        L = self._lib
        p = tab.order
        out = torch.empty((tab.n, 3, p, p), dtype=torch.float64, device=tab.a.device)
        fn = self.lib.vpb_dg_single_tables if single else self.lib.vpb_dg_compose_tables
        L.check(fn(tab.a.data_ptr(), tab.b.data_ptr(), tab.n, p, out.data_ptr(),
                   self._device.stream()), "vpb_dg_compose_tables")
        return out

    def xstencil_work(self, dims, order, wl, wr) -> int:
        return int(self.lib.vpb_dg_xstencil_density_work_len(self._lib.dims(dims), order, wl,
                                                             wr))

    def xstencil(self, src, dst, dims, order, k1, t1, k2, t2, qmul, hl, wl, hr, wr, flag,
                 dens=None):
        """dens: (wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats) or None."""
        L = self._lib
        head = (src.data_ptr(), dst.data_ptr(), L.dims(dims), order, k1.data_ptr(),
                t1.q.data_ptr(), t1.alpha.data_ptr(), k2.data_ptr(), t2.q.data_ptr(),
                t2.alpha.data_ptr(), qmul, hl.data_ptr() if wl else None, wl,
                hr.data_ptr() if wr else None, wr, flag.data_ptr())
        if dens is None:
            L.check(self.lib.vpb_dg_sweep_xstencil(*head, self._device.stream()),
                    "vpb_dg_sweep_xstencil")
            return
        wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
        L.check(self.lib.vpb_dg_sweep_xstencil_density(
            *head, wv1.data_ptr(), wv2.data_ptr(), mid.ctypes.data, wc1.ctypes.data,
            wc2.ctypes.data, volume, work.data_ptr(), rc_out.data_ptr(), stats.data_ptr(),
            self._device.stream()), "vpb_dg_sweep_xstencil_density")

    def xcomp_rows(self, src, dst, dims, order, v2_0, v2_rows, t1, t2, flag, dens, phase):
        """Merged x pass with the density epilogue on v2 rows [v2_0, v2_0 +
        v2_rows) of a shard (vpb_dg_sweep_xcomp_rows; t2 rows = the shard's
        rows); the density accumulates over the calls of one pass (phase bit
        1: first call, bit 2: last call, which reduces into rc / stats)."""
        L = self._lib
        wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
        L.check(self.lib.vpb_dg_sweep_xcomp_rows(
            src.data_ptr(), dst.data_ptr(), L.dims(dims), order, int(v2_0), int(v2_rows),
            t1.composed().data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(),
            t2.composed().data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(), flag.data_ptr(),
            wv1.data_ptr(), wv2.data_ptr(), mid.ctypes.data, wc1.ctypes.data, wc2.ctypes.data,
            volume, work.data_ptr(), rc_out.data_ptr(), stats.data_ptr(), int(phase),
            self._device.stream()), "vpb_dg_sweep_xcomp_rows")

    def xstencil2(self, src, dst, dims, order, k1, t1, k2, t2, qmul, hl, wl, hr, wr, wl2, x2l,
                  wr2, x2r, flag, dens=None):
        """The stencil pass of an x1 x x2 shard (vpb_dg_sweep_xstencil2): x2l /
        x2r = (x1 dofs, left x1 halo, right x1 halo) of the x2 halo cells."""
        import ctypes

        L = self._lib
        ptrs = lambda parts, w: (ctypes.c_void_p * 3)(*[  # noqa: E731
            t.data_ptr() if (w and t is not None and t.numel()) else None for t in parts])
        if dens is not None:
            wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
            tail = (wv1.data_ptr(), wv2.data_ptr(), mid.ctypes.data, wc1.ctypes.data,
                    wc2.ctypes.data, volume, work.data_ptr(), rc_out.data_ptr(),
                    stats.data_ptr())
        else:
            tail = (None,) * 5 + (0.0,) + (None,) * 3
        L.check(self.lib.vpb_dg_sweep_xstencil2(
            src.data_ptr(), dst.data_ptr(), L.dims(dims), order, k1.data_ptr(), t1.q.data_ptr(),
            t1.alpha.data_ptr(), k2.data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(), qmul,
            hl.data_ptr() if wl else None, wl, hr.data_ptr() if wr else None, wr,
            wl2, ptrs(x2l, wl2), wr2, ptrs(x2r, wr2), flag.data_ptr(), *tail,
            self._device.stream()), "vpb_dg_sweep_xstencil2")

    def xstencil_rows(self, src, dst, dims, order, v2_0, v2_rows, k1, t1, k2, t2, qmul, hl, wl,
                      hr, wr, flag, dens=None, phase=3):
        """The stencil pass on v2 rows [v2_0, v2_0 + v2_rows) (one block of the
        pipelined pass); dens as in :meth:`xstencil`, accumulated over the
        blocks of one pass (phase bit 1: first block, bit 2: last)."""
        L = self._lib
        head = (src.data_ptr(), dst.data_ptr(), L.dims(dims), order, int(v2_0), int(v2_rows),
                k1.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(), k2.data_ptr(),
                t2.q.data_ptr(), t2.alpha.data_ptr(), qmul, hl.data_ptr() if wl else None, wl,
                hr.data_ptr() if wr else None, wr, flag.data_ptr())
        if dens is None:
            tail = (None,) * 5 + (0.0,) + (None,) * 3
        else:
            wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
            tail = (wv1.data_ptr(), wv2.data_ptr(), mid.ctypes.data, wc1.ctypes.data,
                    wc2.ctypes.data, volume, work.data_ptr(), rc_out.data_ptr(), stats.data_ptr())
        L.check(self.lib.vpb_dg_sweep_xstencil_rows(*head, *tail, int(phase),
                                                     self._device.stream()),
                "vpb_dg_sweep_xstencil_rows")

    # -- velocity-sharded field (VShardedSolver) ------------------------------------
    def xpass_work(self, dims, order, qmul) -> int:
        fn = (self.lib.vpb_dg_xplane_density_work_len if qmul == 1
              else self.lib.vpb_dg_xcomp_density_work_len)
        return int(fn(self._lib.dims(dims), order))

    def xpass_rows(self, src, dst, dims, order, t1, t2, r0, qmul, f1, f2, dens=None):
        """x half step (qmul 1: vpb_dg_sweep_xplane[_density]) or the merged
        closing + opening pair (qmul 2: vpb_dg_sweep_xcomp_density) of a v2
        slab whose first dof row is global row r0 (x2 tables offset by r0);
        dens = (wv1, wv2 of the slab, mid, wc1, wc2, volume, work, rc, stats)."""
        L = self._lib
        st = self._device.stream()
        nv2 = dims[3]
        a2, b2, q2, al2 = (t2.a[r0:r0 + nv2], t2.b[r0:r0 + nv2], t2.q[r0:r0 + nv2],
                           t2.alpha[r0:r0 + nv2])
        tail = ()
        if dens is not None:
            wv1, wv2, mid, wc1, wc2, volume, work, rc, stats = dens
            tail = (wv1.data_ptr(), wv2.data_ptr(), mid.ctypes.data, wc1.ctypes.data,
                    wc2.ctypes.data, volume, work.data_ptr(), rc.data_ptr(), stats.data_ptr())
        if qmul == 2:
            k2 = t2.composed()[r0:r0 + nv2]
            L.check(self.lib.vpb_dg_sweep_xcomp_density(
                src.data_ptr(), dst.data_ptr(), L.dims(dims), order, t1.composed().data_ptr(),
                t1.q.data_ptr(), t1.alpha.data_ptr(), k2.data_ptr(), q2.data_ptr(),
                al2.data_ptr(), f1.data_ptr(), *tail, st), "vpb_dg_sweep_xcomp_density")
            return
        head = (src.data_ptr(), dst.data_ptr(), L.dims(dims), order, t1.a.data_ptr(),
                t1.b.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(), a2.data_ptr(),
                b2.data_ptr(), q2.data_ptr(), al2.data_ptr(), f1.data_ptr(), f2.data_ptr())
        if dens is None:
            L.check(self.lib.vpb_dg_sweep_xplane(*head, st), "vpb_dg_sweep_xplane")
        else:
            L.check(self.lib.vpb_dg_sweep_xplane_density(*head, *tail, st),
                    "vpb_dg_sweep_xplane_density")

    def vplane_v2halo(self, src_ext, dst, dims, order, c2e, off, t1, t2, f1, f2, hflag):
        L = self._lib
        L.check(self.lib.vpb_dg_sweep_vplane_v2halo(
            src_ext.data_ptr(), dst.data_ptr(), L.dims(dims), order, int(c2e), int(off),
            t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(),
            t2.a.data_ptr(), t2.b.data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(),
            f1.data_ptr(), f2.data_ptr(), hflag.data_ptr(), self._device.stream()),
            "vpb_dg_sweep_vplane_v2halo")

    def vplane_v2peer(self, src_l, l_cells, l0, src, c_cells, c0, src_r, r_cells, r0, H, dst,
                      dims, order, t1, t2, f1, f2, hflag):
        L = self._lib
        L.check(self.lib.vpb_dg_sweep_vplane_v2peer(
            src_l.data_ptr(), int(l_cells), int(l0), src.data_ptr(), int(c_cells), int(c0),
            src_r.data_ptr(), int(r_cells), int(r0), int(H), dst.data_ptr(), L.dims(dims), order,
            t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(),
            t2.a.data_ptr(), t2.b.data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(),
            f1.data_ptr(), f2.data_ptr(), hflag.data_ptr(), self._device.stream()),
            "vpb_dg_sweep_vplane_v2peer")

    def pack(self, axis, f, dims, order, cell0, width, buf):
        L = self._lib
        L.check(self.lib.vpb_halo_pack(axis, f.data_ptr(), L.dims(dims), order, cell0, width,
                                       buf.data_ptr(), self._device.stream()), "vpb_halo_pack")

    def halo_sweep(self, axis, src, dst, dims, order, left, wl, right, wr, tab, flag):
        L = self._lib
        L.check(self.lib.vpb_dg_sweep_axis_halo(
            axis, src.data_ptr(), dst.data_ptr(), L.dims(dims), order,
            left.data_ptr() if wl else None, wl, right.data_ptr() if wr else None, wr,
            tab.a.data_ptr(), tab.b.data_ptr(), tab.q.data_ptr(), tab.alpha.data_ptr(),
            flag.data_ptr(), self._device.stream()), "vpb_dg_sweep_axis_halo")

    def density(self, f, dims, wv1, wv2, rho, work):
        L = self._lib
        L.check(self.lib.vpb_density(f.data_ptr(), L.dims(dims), wv1.data_ptr(), wv2.data_ptr(),
                                     rho.data_ptr(), work.data_ptr(), self._device.stream()),
                "vpb_density")

    def density_work(self, dims) -> int:
        return int(self.lib.vpb_density_work_len(self._lib.dims(dims)))

    def field_solve(self, grid, rho, e, stats, flag):
        from .poisson import solve_into

        solve_into(rho, grid, e, stats, flag)

    def field_solve_centred(self, grid, rc, e, flag):
        """E from the cell-centre density of the fused x passes."""
        from .poisson import solve_into

        solve_into(rc, grid, e, None, flag, centred=True)

    def diag_work(self, dims) -> int:
        return int(self.lib.vpb_diag_work_len(self._lib.dims(dims)))

    def diag_sums(self, f, dims, wx, wv1, wv2, v1sq, v2sq, out, work):
        """out[0..3] = local mass, l1, l2^2, kinetic (EE excluded)."""
        L = self._lib
        L.check(self.lib.vpb_diagnostics(f.data_ptr(), L.dims(dims), wx.data_ptr(),
                                         wv1.data_ptr(), wv2.data_ptr(), v1sq.data_ptr(),
                                         v2sq.data_ptr(), None, 2, out.data_ptr(),
                                         work.data_ptr(), self._device.stream()),
                "vpb_diagnostics")

    def electric_energy(self, e, nx, wx, out):
        L = self._lib
        L.check(self.lib.vpb_electric_energy(e.data_ptr(), 2, nx, wx.data_ptr(), out.data_ptr(),
                                             self._device.stream()), "vpb_electric_energy")


# ---------------------------------------------------------------------------
# Sharded solver
# ---------------------------------------------------------------------------
class Shard:
    """One rank's box of f plus its scratch buffers."""

    def __init__(self, dec: Decomposition, rank: int, device, dtype=torch.float64):
        self.rank = rank
        self.dims = dec.local_dims(rank)
        n = int(np.prod(self.dims))
        self.f = torch.empty(n, dtype=dtype, device=device)
        self.buf = torch.empty(n, dtype=dtype, device=device)
        self.flags = torch.zeros(8, dtype=torch.int32, device=device)
        self.cells = (dec.cells(rank, 0), dec.cells(rank, 1))

    def swap(self) -> None:
        self.f, self.buf = self.buf, self.f


class ShardedSolver:
    """Strang steps of a sharded 2x2v dG field (driver.py:245-265)."""

    def __init__(self, grid: GridSpec, dec: Decomposition, comm, ranks, ops=None, device=None):
        if grid.method != DG:
            raise NotImplementedError("the sharded step covers the SLDG path")
        self.grid = grid
        self.dec = dec
        self.comm = comm
        self.ops = ops or CudaOps()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.shards = {r: Shard(dec, r, self.device) for r in ranks}
        self.order = grid.order
        self._xtab = {}
        self._geom = None
        # v2 row blocks of the pipelined halo exchange + stencil pass (1: off)
        self.halo_blocks = int(os.environ.get("VPB_HALO_BLOCKS", "4"))
        n1, n2 = grid.dof(0), grid.dof(1)
        self.n1, self.n2 = n1, n2
        dev = self.device
        w = [torch.as_tensor(grid.axis_weights(a), dtype=torch.float64).to(dev) for a in range(4)]
        self.wv1, self.wv2 = w[2], w[3]
        self.v1sq = torch.as_tensor(grid.axis_points(2) ** 2, dtype=torch.float64).to(dev)
        self.v2sq = torch.as_tensor(grid.axis_points(3) ** 2, dtype=torch.float64).to(dev)
        self.wx_full = (w[1][:, None] * w[0][None, :]).reshape(-1).contiguous()
        self.vpoints = [torch.as_tensor(grid.axis_points(a), dtype=torch.float64).to(dev)
                        for a in (2, 3)]
        self.rho = torch.empty(n1 * n2, dtype=torch.float64, device=dev)
        self.e = torch.empty(2 * n1 * n2, dtype=torch.float64, device=dev)
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)
        self.solve_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.names = ["x1 half (open)", "x2 half (open)", "field solve", "v1 full", "v2 full",
                      "x1 half (close)", "x2 half (close)"]
        self.fused = (not dec.sharded(0) and not dec.sharded(1)
                      and (n1 * self.order) % 2 == 0 and hasattr(self.ops, "xplane"))

    # -- data movement helpers (tests / I/O) ----------------------------------
    def initialize(self, problem) -> None:
        """Initial data of every local shard, built on the device from the
        separable factors (driver.py:182-198) restricted to the shard's x box."""
        from . import _device, _lib
        from .driver import separable_factors

        g1, g2, space = separable_factors(problem, self.grid)
        space = np.asarray(space).reshape(self.n2, self.n1)
        p = self.order
        lib = _lib.load()
        dg1 = torch.as_tensor(g1, dtype=torch.float64).to(self.device)
        dg2 = torch.as_tensor(g2, dtype=torch.float64).to(self.device)
        for sh in self.shards.values():
            (a0, b0), (a1, b1) = sh.cells
            sp = torch.as_tensor(np.ascontiguousarray(space[a1 * p:b1 * p, a0 * p:b0 * p]),
                                 dtype=torch.float64).to(self.device).reshape(-1)
            _lib.check(lib.vpb_fill_separable(sh.f.data_ptr(), _lib.dims(sh.dims),
                                              dg1.data_ptr(), dg2.data_ptr(), sp.data_ptr(),
                                              _device.stream()), "vpb_fill_separable")

    def scatter(self, logical: np.ndarray) -> None:
        for r, sh in self.shards.items():
            box = np.ascontiguousarray(self.dec.local_slice(r, logical).transpose(3, 2, 1, 0))
            sh.f.copy_(torch.from_numpy(box.reshape(-1)).to(sh.f.device))

    def local_logical(self, rank: int) -> np.ndarray:
        sh = self.shards[rank]
        d = sh.dims
        return sh.f.view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0).cpu().numpy()

    def gather(self) -> np.ndarray:
        """Full logical f (only valid when this process holds every shard)."""
        g = self.grid
        out = np.empty(g.dofs)
        for r in self.shards:
            p = self.order
            a0, b0 = self.dec.cells(r, 0)
            a1, b1 = self.dec.cells(r, 1)
            out[a0 * p:b0 * p, a1 * p:b1 * p] = self.local_logical(r)
        return out

    # -- tables -----------------------------------------------------------------
    def x_tables(self, d: int, tau: float):
        key = (d, float(tau))
        if key not in self._xtab:
            tab = self.ops.tables(self.vpoints[d], 0.5 * tau, self.grid.axes[d].h,
                                  self.grid.dg_degree)
            self._xtab[key] = (tab, halo_widths(self.ops.tables_q(tab)))
        return self._xtab[key]

    # -- sweeps -------------------------------------------------------------------
    def _x_sweep(self, axis: int, tau: float, slot: int) -> None:
        tab, (wl, wr) = self.x_tables(axis, tau)
        p = self.order
        if not self.dec.sharded(axis):
            for sh in self.shards.values():
                self.ops.sweep(axis, sh.f, sh.buf, sh.dims, p, tab, sh.flags[slot:slot + 1])
                sh.swap()
            return
        cells_min = min(c1 - c0 for sh in self.shards.values() for (c0, c1) in [sh.cells[axis]])
        if max(wl, wr) > cells_min:
            raise NotImplementedError(
                f"halo of {max(wl, wr)} cells exceeds a shard of {cells_min} cells")
        msgs = {}
        bufs = {}
        for r, sh in self.shards.items():
            left, right = self.dec.neighbours(r, axis)
            d = sh.dims
            cl = d[axis] // p
            hd = list(d)
            hd[axis] = wl * p
            send_l = torch.empty(int(np.prod(hd)), dtype=sh.f.dtype, device=sh.f.device)
            recv_l = torch.empty_like(send_l)
            hd[axis] = wr * p
            send_r = torch.empty(int(np.prod(hd)), dtype=sh.f.dtype, device=sh.f.device)
            recv_r = torch.empty_like(send_r)
            if wl:
                self.ops.pack(axis, sh.f, d, p, cl - wl, wl, send_l)
            if wr:
                self.ops.pack(axis, sh.f, d, p, 0, wr, send_r)
            msgs[r] = [(KIND_L, right, send_l, left, recv_l),
                       (KIND_R, left, send_r, right, recv_r)]
            bufs[r] = (recv_l, recv_r)
        self.comm.exchange(msgs)
        for r, sh in self.shards.items():
            recv_l, recv_r = bufs[r]
            self.ops.halo_sweep(axis, sh.f, sh.buf, sh.dims, p, recv_l, wl, recv_r, wr, tab,
                                sh.flags[slot:slot + 1])
            sh.swap()

    def _advect_space(self, tau: float, slot: int) -> None:
        if self.fused:
            t1, _ = self.x_tables(0, tau)
            t2, _ = self.x_tables(1, tau)
            for sh in self.shards.values():
                self.ops.xplane(sh.f, sh.buf, sh.dims, self.order, t1, t2,
                                sh.flags[slot:slot + 1], sh.flags[slot + 1:slot + 2])
                sh.swap()
            return
        self._x_sweep(0, tau, slot)
        self._x_sweep(1, tau, slot + 1)

    def _gather_rho(self) -> None:
        """Local density slabs -> full ρ on every rank."""
        locs = {}
        for r, sh in self.shards.items():
            d = sh.dims
            rl = torch.empty(d[0] * d[1], dtype=torch.float64, device=sh.f.device)
            work = torch.empty(self.ops.density_work(d), dtype=torch.float64, device=sh.f.device)
            self.ops.density(sh.f, d, self.wv1, self.wv2, rl, work)
            # pad to the largest slab so all_gather sees equal sizes
            pad = torch.zeros(self._max_slab(), dtype=torch.float64, device=sh.f.device)
            pad[: rl.numel()] = rl
            locs[r] = pad
        parts = self.comm.allgather(locs)
        full = self.rho.view(self.n2, self.n1)
        p = self.order
        for r, part in enumerate(parts):
            a0, b0 = self.dec.cells(r, 0)
            a1, b1 = self.dec.cells(r, 1)
            n1l, n2l = (b0 - a0) * p, (b1 - a1) * p
            full[a1 * p:b1 * p, a0 * p:b0 * p] = part[: n1l * n2l].view(n2l, n1l)

    def _max_slab(self) -> int:
        p = self.order
        m = 0
        for r in range(self.dec.world):
            a0, b0 = self.dec.cells(r, 0)
            a1, b1 = self.dec.cells(r, 1)
            m = max(m, (b0 - a0) * (b1 - a1) * p * p)
        return m

    def _local_e(self, sh: Shard, d: int) -> torch.Tensor:
        p = self.order
        (a0, b0), (a1, b1) = sh.cells
        full = self.e[d * self.n1 * self.n2:(d + 1) * self.n1 * self.n2].view(self.n2, self.n1)
        return full[a1 * p:b1 * p, a0 * p:b0 * p].contiguous().view(-1)

    def step(self, tau: float, time_label: float | None = None) -> None:
        from .driver import SubstepError

        for sh in self.shards.values():
            sh.flags.zero_()
        self.solve_flag.zero_()
        self._advect_space(tau, 0)  # x half (open); the x tables carry the tau/2
        self._gather_rho()
        self.ops.field_solve(self.grid, self.rho, self.e, self.stats, self.solve_flag)
        for sh in self.shards.values():
            tabs = [self.ops.tables(self._local_e(sh, d), tau, self.grid.axes[2 + d].h,
                                    self.grid.dg_degree) for d in range(2)]
            if hasattr(self.ops, "vplane"):  # v1 + v2 in one pass (local in x)
                self.ops.vplane(sh.f, sh.buf, sh.dims, self.order, tabs[0], tabs[1],
                                sh.flags[3:4], sh.flags[4:5])
                sh.swap()
                continue
            for d in range(2):
                self.ops.sweep(2 + d, sh.f, sh.buf, sh.dims, self.order, tabs[d],
                               sh.flags[3 + d:4 + d])
                sh.swap()
        self._advect_space(tau, 5)
        # flags: max over shards and ranks, field solve is redundant (slot 2)
        for sh in self.shards.values():
            sh.flags[2:3] = torch.maximum(sh.flags[2:3], self.solve_flag)
        flags = self.comm.allreduce({r: sh.flags for r, sh in self.shards.items()}, "max")
        host = flags.cpu().numpy()
        for k, name in enumerate(self.names):
            if host[k]:
                raise SubstepError(name, time_label)

    # -- K steps with merged x half steps on the x1-sharded field -------------
    def _stencil_ready(self, tau: float | None = None) -> bool:
        """Whether advance() can run the three-cell stencil passes: an
        x1-only decomposition of a 2x2v field, every shard meeting the
        stencil kernel's preconditions (``xplane_args_ok`` in fused.cu: a
        cell row of x1 dofs is a 16-byte multiple; ``plan_xcomp`` in
        xcomp.cu: at most 128 local x1 cells), and -- given tau -- the
        single half step's x1 halo fitting every shard.  Otherwise advance()
        runs step() (the halo sweeps) in a loop."""
        if not (self.dec.sharded(0) and hasattr(self.ops, "xstencil") and self.grid.ndim == 4):
            return False
        if self.dec.sharded(1) and not hasattr(self.ops, "xstencil2"):
            return False
        p = self.order
        for r in range(self.dec.world):
            c0, c1 = self.dec.cells(r, 0)
            if ((c1 - c0) * p * p) % 2 or c1 - c0 > 128:
                return False
        if tau is not None:
            _, _, tabs = self._stencil_setup(tau)
            _, _, wl, wr = tabs[1]
            cells_min = min(c1 - c0 for r in range(self.dec.world)
                            for (c0, c1) in [self.dec.cells(r, 0)])
            if max(wl, wr) > cells_min:
                return False
            if self.dec.sharded(1) and max(self._x2_widths(tau, 1)) > self._x2_cells_min():
                return False
        return True

    def _x2_cells_min(self) -> int:
        return min(c1 - c0 for r in range(self.dec.world) for (c0, c1) in [self.dec.cells(r, 1)])

    def _x2_widths(self, tau: float, qmul: int) -> tuple[int, int]:
        """x2 halo cells of a stencil pass on an x2-sharded field: source x2
        cells c - Q - 2 .. c - Q, Q = qmul q2, over every v2 row."""
        t2, _ = self.x_tables(1, tau)
        q = qmul * np.asarray(self.ops.tables_q(t2))
        return (max(0, int(q.max()) + 2) if q.size else 0, max(0, -int(q.min())) if q.size else 0)

    def _stencil_setup(self, tau: float):
        """Tables of the three-cell x passes and their x1 halo widths."""
        key = ("stencil", float(tau))
        if key not in self._xtab:
            t1, _ = self.x_tables(0, tau)
            t2, _ = self.x_tables(1, tau)
            q1 = self.ops.tables_q(t1)
            out = {}
            for qmul, single in ((1, True), (2, False)):
                q = qmul * np.asarray(q1)
                wl = max(0, int(q.max()) + 2) if q.size else 0
                wr = max(0, -int(q.min())) if q.size else 0
                if self.order % 2:  # halo blocks staged by bulk copies: 16-byte multiples
                    wl += wl % 2
                    wr += wr % 2
                out[qmul] = (self.ops.stencil_tables(t1, single),
                             self.ops.stencil_tables(t2, single), wl, wr)
            self._xtab[key] = (t1, t2, out)
        return self._xtab[key]

    def _merged_halo_fits(self, tau: float) -> bool:
        _, _, tabs = self._stencil_setup(tau)
        _, _, wl, wr = tabs[2]
        cells_min = min(c1 - c0 for r in range(self.dec.world)
                        for (c0, c1) in [self.dec.cells(r, 0)])
        if self.dec.sharded(1) and max(self._x2_widths(tau, 2)) > self._x2_cells_min():
            return False
        return max(wl, wr) <= cells_min

    def _density_consts(self):
        if getattr(self, "_dens", None) is None:
            from .grid import gauss_nodes
            from .poisson import _lagrange_row

            p = self.order
            nodes, _ = gauss_nodes(p)
            mid = np.ascontiguousarray(_lagrange_row(nodes, 0.5))
            cells = [np.ascontiguousarray(np.asarray(self.grid.axis_weights(a))[:p])
                     for a in (0, 1)]
            ax = self.grid.axes
            volume = (ax[0].upper - ax[0].lower) * (ax[1].upper - ax[1].lower)
            self._dens = (mid, cells[0], cells[1], float(volume))
        return self._dens

    def _x_stencil_pass(self, tau: float, qmul: int, flag_slot, with_density: bool,
                        flags_row: dict, stats_row: dict, rc_parts: dict) -> None:
        """One x pass (qmul 1: an x half step; 2: the merged closing + opening
        half steps) on every local shard: x1 halo exchange, then the
        three-cell stencil kernel; the density epilogue fills rc_parts."""
        t1, t2, tabs = self._stencil_setup(tau)
        k1, k2, wl, wr = tabs[qmul]
        p = self.order
        mark = getattr(self, "_mark", None) or (lambda label: None)
        mark("halo_x1")
        cells_min = min(c1 - c0 for sh in self.shards.values() for (c0, c1) in [sh.cells[0]])
        if max(wl, wr) > cells_min:
            raise NotImplementedError(
                f"halo of {max(wl, wr)} cells exceeds a shard of {cells_min} cells")
        msgs, bufs = {}, {}
        for r, sh in self.shards.items():
            left, right = self.dec.neighbours(r, 0)
            d = sh.dims
            cl = d[0] // p
            hd = list(d)
            hd[0] = wl * p
            send_l = torch.empty(int(np.prod(hd)), dtype=sh.f.dtype, device=sh.f.device)
            recv_l = torch.empty_like(send_l)
            hd[0] = wr * p
            send_r = torch.empty(int(np.prod(hd)), dtype=sh.f.dtype, device=sh.f.device)
            recv_r = torch.empty_like(send_r)
            if wl:
                self.ops.pack(0, sh.f, d, p, cl - wl, wl, send_l)
            if wr:
                self.ops.pack(0, sh.f, d, p, 0, wr, send_r)
            msgs[r] = [(KIND_L, right, send_l, left, recv_l),
                       (KIND_R, left, send_r, right, recv_r)]
            bufs[r] = (recv_l, recv_r)
        self._halo_bytes = getattr(self, "_halo_bytes", 0) + sum(
            8 * (m[0][2].numel() * (wl > 0) + m[1][2].numel() * (wr > 0)) for m in msgs.values())
        mid, wc1, wc2, volume = self._density_consts()
        if self.dec.sharded(1):
            self._x2_stencil_pass(tau, qmul, msgs, bufs, k1, t1, k2, t2, wl, wr, flag_slot,
                                  with_density, flags_row, stats_row, rc_parts, mark)
            return
        blocks = self._row_blocks()
        if blocks is not None:
            self._pipelined_pass(msgs, bufs, blocks, k1, t1, k2, t2, qmul, wl, wr, flag_slot,
                                 with_density, flags_row, stats_row, rc_parts, mark)
            return
        self.comm.exchange(msgs)
        mark(("sweep_x12x12" if qmul == 2 else "sweep_x12") + ("_rho" if with_density else ""))
        for r, sh in self.shards.items():
            recv_l, recv_r = bufs[r]
            fl = flags_row[r][flag_slot:flag_slot + 1]
            dens = None
            if with_density:
                d = sh.dims
                work = torch.empty(self.ops.xstencil_work(d, p, wl, wr), dtype=torch.float64,
                                   device=sh.f.device)
                rc = torch.empty((d[1] // p) * (d[0] // p), dtype=torch.float64,
                                 device=sh.f.device)
                dens = (self.wv1, self.wv2, mid, wc1, wc2, volume, work, rc, stats_row[r])
                rc_parts[r] = rc
            self.ops.xstencil(sh.f, sh.buf, sh.dims, p, k1, t1, k2, t2, qmul, recv_l, wl,
                              recv_r, wr, fl, dens)
            sh.swap()

    def _x2_stencil_pass(self, tau, qmul, msgs, bufs, k1, t1, k2, t2, wl, wr, flag_slot,
                         with_density, flags_row, stats_row, rc_parts, mark):
        """The stencil pass of an x1 x x2 decomposition (the 4 x 2 grid at 8
        GPUs): the x1 halo exchange, then the x2 halo exchange of the
        boundary cells' x1 dofs and of their x1 halo rows (the corners, from
        the x1 halos just received), then vpb_dg_sweep_xstencil2 per shard."""
        p = self.order
        wl2, wr2 = self._x2_widths(tau, qmul)
        self.comm.exchange(msgs)
        mark("halo_x2")
        msgs2, bufs2 = {}, {}
        for r, sh in self.shards.items():
            left2, right2 = self.dec.neighbours(r, 1)
            d = sh.dims
            n1, nx2 = d[0], d[1]
            c2l = nx2 // p
            planes = d[2] * d[3]
            recv_l, recv_r = bufs[r]
            send = {}
            recv = {}
            # my last wl2 cells -> right2's left halo; my first wr2 cells -> left2's right halo
            for side, w, cell0 in (("L", wl2, c2l - wl2), ("R", wr2, 0)):
                parts_s, parts_r = [], []
                for k, (h, hw) in enumerate(((None, n1), (recv_l, wl * p), (recv_r, wr * p))):
                    n = planes * w * p * hw if (w and hw) else 0
                    sb = torch.empty(n, dtype=sh.f.dtype, device=sh.f.device)
                    rb = torch.empty(n, dtype=sh.f.dtype, device=sh.f.device)
                    if n:
                        if k == 0:
                            self.ops.pack(1, sh.f, d, p, cell0, w, sb)
                        else:  # rows of the boundary cells in the x1 halo buffer
                            run = w * p * hw
                            self.ops.slab_copy(h[cell0 * p * hw:], c2l * p * hw, sb, run,
                                               planes, run)
                    parts_s.append(sb)
                    parts_r.append(rb)
                send[side], recv[side] = parts_s, parts_r
            items = []
            for k in range(3):
                items.append((KIND_X2L[k], right2, send["L"][k], left2, recv["L"][k]))
                items.append((KIND_X2R[k], left2, send["R"][k], right2, recv["R"][k]))
            msgs2[r] = items
            bufs2[r] = (recv["L"], recv["R"])
        self._halo_bytes = getattr(self, "_halo_bytes", 0) + sum(
            8 * it[2].numel() for m in msgs2.values() for it in m)
        self.comm.exchange(msgs2)
        mark(("sweep_x12x12" if qmul == 2 else "sweep_x12") + ("_rho" if with_density else ""))
        mid, wc1, wc2, volume = self._density_consts()
        for r, sh in self.shards.items():
            recv_l, recv_r = bufs[r]
            x2l, x2r = bufs2[r]
            fl = flags_row[r][flag_slot:flag_slot + 1]
            dens = None
            if with_density:
                d = sh.dims
                work = torch.empty(self.ops.xstencil_work(d, p, wl, wr), dtype=torch.float64,
                                   device=sh.f.device)
                rc = torch.empty((d[1] // p) * (d[0] // p), dtype=torch.float64,
                                 device=sh.f.device)
                dens = (self.wv1, self.wv2, mid, wc1, wc2, volume, work, rc, stats_row[r])
                rc_parts[r] = rc
            self.ops.xstencil2(sh.f, sh.buf, sh.dims, p, k1, t1, k2, t2, qmul, recv_l, wl,
                               recv_r, wr, wl2, x2l, wr2, x2r, fl, dens)
            sh.swap()

    def _row_blocks(self):
        """v2 row blocks of the pipelined stencil pass (``halo_blocks`` > 1 and
        ops that run a block of rows), else None (one exchange, one pass)."""
        nb = int(getattr(self, "halo_blocks", 1))
        if nb <= 1 or not hasattr(self.ops, "xstencil_rows"):
            return None
        nv2 = self.shards[next(iter(self.shards))].dims[3]
        nb = min(nb, nv2)
        edges = [round(i * nv2 / nb) for i in range(nb + 1)]
        return [(edges[i], edges[i + 1] - edges[i]) for i in range(nb) if edges[i + 1] > edges[i]]

    def _pipelined_pass(self, msgs, bufs, blocks, k1, t1, k2, t2, qmul, wl, wr, flag_slot,
                        with_density, flags_row, stats_row, rc_parts, mark):
        """Halo exchange and stencil pass in blocks of v2 rows:
        the exchanges of all blocks are posted first (NCCL runs them in order
        on its own stream), then the pass of block b waits only for block b's
        messages, so it overlaps the transfer of blocks b+1, ...  The halo
        buffers are [plane][x2 row][w P], so a block of v2 rows is one
        contiguous slice of every message."""
        p = self.order
        reqs = []
        for v0, nv in blocks:
            sub = {}
            for r, items in msgs.items():
                d = self.shards[r].dims
                per = d[1] * d[2]  # halo rows of one v2 row, per halo dof column
                sub[r] = []
                for kind, sp, sbuf, rp, rbuf in items:
                    w = sbuf.numel() // (per * d[3]) if d[3] else 0
                    a, b = v0 * per * w, (v0 + nv) * per * w
                    sub[r].append((kind, sp, sbuf[a:b], rp, rbuf[a:b]))
            reqs.append(self.comm.exchange_async(sub))
        mark(("sweep_x12x12" if qmul == 2 else "sweep_x12") + ("_rho" if with_density else ""))
        work = {}
        for i, (v0, nv) in enumerate(blocks):
            self.comm.wait(reqs[i])
            phase = (1 if i == 0 else 0) | (2 if i + 1 == len(blocks) else 0)
            for r, sh in self.shards.items():
                recv_l, recv_r = bufs[r]
                fl = flags_row[r][flag_slot:flag_slot + 1]
                dens = None
                if with_density:
                    d = sh.dims
                    if r not in work:
                        work[r] = torch.empty(self.ops.xstencil_work(d, p, wl, wr),
                                              dtype=torch.float64, device=sh.f.device)
                        rc_parts[r] = torch.empty((d[1] // p) * (d[0] // p),
                                                  dtype=torch.float64, device=sh.f.device)
                    dens = (self.wv1, self.wv2, *self._density_consts()[:3],
                            self._density_consts()[3], work[r], rc_parts[r], stats_row[r])
                self.ops.xstencil_rows(sh.f, sh.buf, sh.dims, p, v0, nv, k1, t1, k2, t2, qmul,
                                       recv_l, wl, recv_r, wr, fl, dens, phase)
        for sh in self.shards.values():
            sh.swap()

    def _gather_rc(self, rc_parts: dict) -> torch.Tensor:
        """Shard cell-centre density slabs [C2 local][C1 local] -> full [C2][C1]."""
        p = self.order
        C1, C2 = self.n1 // p, self.n2 // p
        m = max((b0 - a0) * (b1 - a1) for r in range(self.dec.world)
                for (a0, b0), (a1, b1) in [(self.dec.cells(r, 0), self.dec.cells(r, 1))])
        locs = {}
        for r, rc in rc_parts.items():
            pad = torch.zeros(m, dtype=torch.float64, device=rc.device)
            pad[: rc.numel()] = rc
            locs[r] = pad
        parts = self.comm.allgather(locs)
        full = torch.empty((C2, C1), dtype=torch.float64, device=self.device)
        for r, part in enumerate(parts):
            a0, b0 = self.dec.cells(r, 0)
            a1, b1 = self.dec.cells(r, 1)
            full[a1:b1, a0:b0] = part[: (b0 - a0) * (b1 - a1)].view(b1 - a1, b0 - a0)
        return full.view(-1)

    def advance(self, tau: float, nsteps: int, first_step: int | None = None,
                timer=None) -> None:
        """``nsteps`` Strang steps (driver.advance on the sharded field).

        x1-sharded fields run the single-GPU pass structure: one x pass per
        step boundary (the closing x half step of step m and the opening one
        of step m+1 as composed three-cell stencils, "fast" arithmetic), each
        after one x1 halo exchange, with the density as its epilogue; the v
        passes are local.  Other decompositions run ``step`` in a loop."""
        from .driver import ARITH, SubstepError
        from .poisson import _warn_if_not_neutral

        if nsteps <= 0:
            return
        self._mark = timer
        try:
            self._advance(tau, nsteps, first_step, ARITH, SubstepError, _warn_if_not_neutral)
        finally:
            self._mark = None
            if timer is not None:
                timer(None)

    def _advance(self, tau, nsteps, first_step, ARITH, SubstepError, _warn_if_not_neutral):
        mark = self._mark or (lambda label: None)
        if ARITH != "fast" or not self._stencil_ready(tau):
            for m in range(nsteps):
                self.step(tau, None if first_step is None else (first_step + m) * tau)
            return
        dev = self.device
        flags = {r: torch.zeros((nsteps, 8), dtype=torch.int32, device=dev) for r in self.shards}
        stats = {r: torch.zeros((nsteps, 4), dtype=torch.float64, device=dev)
                 for r in self.shards}
        solve_flags = torch.zeros((nsteps, 1), dtype=torch.int32, device=dev)
        rc_parts = {}
        self._x_stencil_pass(tau, 1, 0, True, {r: flags[r][0] for r in self.shards},
                             {r: stats[r][0] for r in self.shards}, rc_parts)
        for m in range(nsteps):
            mark("rho_allgather")
            rc = self._gather_rc(rc_parts)
            mark("field_solve")
            self.ops.field_solve_centred(self.grid, rc, self.e, solve_flags[m])
            for r, sh in self.shards.items():
                mark("tables_v12")
                tabs = [self.ops.tables(self._local_e(sh, d), tau, self.grid.axes[2 + d].h,
                                        self.grid.dg_degree) for d in range(2)]
                mark("sweep_v12")
                self.ops.vplane(sh.f, sh.buf, sh.dims, self.order, tabs[0], tabs[1],
                                flags[r][m][3:4], flags[r][m][4:5])
                sh.swap()
            if m + 1 < nsteps and self._merged_halo_fits(tau):
                # closing of step m + opening of step m+1, one pass
                rc_parts = {}
                self._x_stencil_pass(tau, 2, 5, True, {r: flags[r][m] for r in self.shards},
                                     {r: stats[r][m + 1] for r in self.shards}, rc_parts)
            elif m + 1 < nsteps:  # the doubled reach needs more halo than a shard holds
                self._x_stencil_pass(tau, 1, 5, False, {r: flags[r][m] for r in self.shards},
                                     {}, {})
                rc_parts = {}
                self._x_stencil_pass(tau, 1, 0, True, {r: flags[r][m + 1] for r in self.shards},
                                     {r: stats[r][m + 1] for r in self.shards}, rc_parts)
            else:
                self._x_stencil_pass(tau, 1, 5, False, {r: flags[r][m] for r in self.shards},
                                     {}, {})
        mark("flags")
        for r in self.shards:
            flags[r][:, 2:3] = torch.maximum(flags[r][:, 2:3], solve_flags)
        fl = self.comm.allreduce(flags, "max").cpu().numpy()
        st = self.comm.allreduce(stats, "sum").cpu().numpy()
        for m in range(nsteps):
            _warn_if_not_neutral(float(st[m, 0]))
            for k, name in enumerate(self.names):
                if fl[m, k]:
                    raise SubstepError(name, None if first_step is None
                                       else (first_step + m) * tau)

    def diagnostics(self, time: float = 0.0) -> dict:
        """Global conserved quantities (driver.py:279-316)."""
        self._gather_rho()
        self.ops.field_solve(self.grid, self.rho, self.e, None, self.solve_flag)
        sums = {}
        p = self.order
        for r, sh in self.shards.items():
            d = sh.dims
            (a0, b0), (a1, b1) = sh.cells
            wx = self.wx_full.view(self.n2, self.n1)[a1 * p:b1 * p, a0 * p:b0 * p].contiguous()
            out = torch.zeros(8, dtype=torch.float64, device=sh.f.device)
            work = torch.empty(self.ops.diag_work(d), dtype=torch.float64, device=sh.f.device)
            self.ops.diag_sums(sh.f, d, wx.view(-1), self.wv1, self.wv2, self.v1sq, self.v2sq,
                               out, work)
            sums[r] = out
        tot = self.comm.allreduce(sums, "sum").cpu().numpy()
        ee_t = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.ops.electric_energy(self.e, self.n1 * self.n2, self.wx_full, ee_t)
        ee = float(ee_t.cpu()[0])
        mass, l1, l2sq, kin = (float(x) for x in tot[:4])
        return {"time": float(time), "electric_energy": ee, "mass": mass, "l1_norm": l1,
                "l2_norm": math.sqrt(max(l2sq, 0.0)), "kinetic_energy": kin,
                "total_energy": kin + ee}


# ---------------------------------------------------------------------------
# Sharded spline solver: all-to-all reshards (SURVEY §8e "Spline")
# ---------------------------------------------------------------------------
class SplineShardedSolver:
    """Strang steps of a cubic-spline 2x2v field on W ranks.

    The spline solve needs whole lines, so the field moves between two
    layouts with an all-to-all (grouped send/recv; NCCL over NVLink) twice
    per step:

    * home layout A, split along v2: rank r holds f[v2 in V_r][v1][x2][x1],
      a contiguous slab of the canonical buffer.  Both x sweeps are local
      (x1 and x2 lines are whole) and so is the density partial
      sum_{v in V_r} w f, which an all-reduce completes (every rank then
      solves the Poisson problem redundantly).
    * layout B, split along x2: rank s holds f[v2][v1][x2 in X_s][x1]; both
      v sweeps are local, with tables from the local rows of E.

    A -> B: rank r sends rank s the x2 rows X_s of its slab (packed with
    vpb_slab_copy); they land as the contiguous v2 block V_r of B_s.  B -> A
    is the reverse (received into a contiguous buffer, unpacked with
    vpb_slab_copy).  Every line sweep is the single-GPU kernel on whole
    lines, so f matches the single-GPU step up to the summation order of the
    density all-reduce.
    """

    def __init__(self, grid: GridSpec, comm, ranks, world: int, ops=None, device=None):
        if grid.method != SPLINE or grid.ndim != 4:
            raise ValueError("the spline sharded step needs a 2x2v spline grid")
        n1, n2, nv1, nv2 = grid.dims4
        if world > nv2 or world > n2:
            raise ValueError(f"cannot split {nv2} v2 / {n2} x2 points over {world} ranks")
        self.grid = grid
        self.comm = comm
        self.world = world
        self.ops = ops or CudaOps()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.n1, self.n2, self.nv1, self.nv2 = n1, n2, nv1, nv2
        self.vr = [split_cells(nv2, world, r) for r in range(world)]
        self.xr = [split_cells(n2, world, r) for r in range(world)]
        dev = self.device
        self.ranks = list(ranks)
        self.a = {}
        self.b = {}
        self.flags = {}
        for r in self.ranks:
            v0, v1 = self.vr[r]
            x0, x1 = self.xr[r]
            na = n1 * n2 * nv1 * (v1 - v0)
            nb = n1 * (x1 - x0) * nv1 * nv2
            self.a[r] = [torch.empty(na, dtype=torch.float64, device=dev),
                         torch.empty(na, dtype=torch.float64, device=dev)]
            self.b[r] = [torch.empty(nb, dtype=torch.float64, device=dev),
                         torch.empty(nb, dtype=torch.float64, device=dev)]
            self.flags[r] = torch.zeros(8, dtype=torch.int32, device=dev)
        w = [torch.as_tensor(grid.axis_weights(a), dtype=torch.float64).to(dev) for a in range(4)]
        self.wv1, self.wv2 = w[2], w[3]
        self.wx_full = (w[1][:, None] * w[0][None, :]).reshape(-1).contiguous()
        self.vpoints = [torch.as_tensor(grid.axis_points(a), dtype=torch.float64).to(dev)
                        for a in (2, 3)]
        self.v1sq = self.vpoints[0] ** 2
        self.v2sq = self.vpoints[1] ** 2
        self.rho = torch.empty(n1 * n2, dtype=torch.float64, device=dev)
        self.e = torch.empty(2 * n1 * n2, dtype=torch.float64, device=dev)
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)
        self.solve_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.names = ["x1 half (open)", "x2 half (open)", "field solve", "v1 full", "v2 full",
                      "x1 half (close)", "x2 half (close)"]

    # -- geometry ------------------------------------------------------------------
    def dims_a(self, r: int):
        v0, v1 = self.vr[r]
        return (self.n1, self.n2, self.nv1, v1 - v0)

    def dims_b(self, r: int):
        x0, x1 = self.xr[r]
        return (self.n1, x1 - x0, self.nv1, self.nv2)

    # -- data movement helpers (tests / I/O) ----------------------------------------
    def initialize(self, problem) -> None:
        from . import _device, _lib
        from .driver import separable_factors

        g1, g2, space = separable_factors(problem, self.grid)
        lib = _lib.load()
        dg1 = torch.as_tensor(np.asarray(g1), dtype=torch.float64).to(self.device)
        sp = torch.as_tensor(np.asarray(space).reshape(-1), dtype=torch.float64).to(self.device)
        for r in self.ranks:
            v0, v1 = self.vr[r]
            dg2 = torch.as_tensor(np.asarray(g2)[v0:v1], dtype=torch.float64).to(self.device)
            _lib.check(lib.vpb_fill_separable(self.a[r][0].data_ptr(), _lib.dims(self.dims_a(r)),
                                              dg1.data_ptr(), dg2.data_ptr(), sp.data_ptr(),
                                              _device.stream()), "vpb_fill_separable")

    def scatter(self, logical: np.ndarray) -> None:
        for r in self.ranks:
            v0, v1 = self.vr[r]
            box = np.ascontiguousarray(logical[:, :, :, v0:v1].transpose(3, 2, 1, 0))
            self.a[r][0].copy_(torch.from_numpy(box.reshape(-1)).to(self.device))

    def gather(self) -> np.ndarray:
        out = np.empty(self.grid.dofs)
        for r in self.ranks:
            v0, v1 = self.vr[r]
            d = self.dims_a(r)
            out[:, :, :, v0:v1] = (self.a[r][0].view(d[3], d[2], d[1], d[0])
                                   .permute(3, 2, 1, 0).cpu().numpy())
        return out

    # -- reshards ----------------------------------------------------------------------
    def _a_to_b(self) -> None:
        n1, nv1 = self.n1, self.nv1
        msgs = {}
        for r in self.ranks:
            src = self.a[r][0]
            v0, v1 = self.vr[r]
            items = []
            for s in range(self.world):
                x0, x1 = self.xr[s]
                run = (x1 - x0) * n1
                outer = (v1 - v0) * nv1
                b_off = v0 * nv1 * run  # v2 block V_r of B_s
                if s in self.b and s == r:  # own chunk: copy straight into B
                    dst = self.b[s][0][b_off:b_off + outer * run]
                    self.ops.slab_copy(src[x0 * n1:], self.n2 * n1, dst, run, outer, run)
                    continue
                send = torch.empty(outer * run, dtype=torch.float64, device=self.device)
                self.ops.slab_copy(src[x0 * n1:], self.n2 * n1, send, run, outer, run)
                items.append((KIND_A2A, s, send, s, None))
            msgs[r] = items
        # receives: B_s gets the V_r block from every rank r != s
        for s in self.ranks:
            x0, x1 = self.xr[s]
            run = (x1 - x0) * n1
            for r in range(self.world):
                if r == s:
                    continue
                v0, v1 = self.vr[r]
                off = v0 * nv1 * run
                recv = self.b[s][0][off:off + (v1 - v0) * nv1 * run]
                msgs.setdefault(s, []).append((KIND_A2A, None, None, r, recv))
        self.comm.exchange(msgs)

    def _b_to_a(self) -> None:
        n1, nv1 = self.n1, self.nv1
        msgs = {}
        for s in self.ranks:
            x0, x1 = self.xr[s]
            run = (x1 - x0) * n1
            items = []
            for r in range(self.world):
                v0, v1 = self.vr[r]
                off = v0 * nv1 * run
                chunk = self.b[s][0][off:off + (v1 - v0) * nv1 * run]
                if r == s:
                    self.ops.slab_copy(chunk, run, self.a[r][0][x0 * n1:], self.n2 * n1,
                                       (v1 - v0) * nv1, run)
                    continue
                items.append((KIND_A2A, r, chunk, r, None))
            msgs[s] = items
        recvs = {}
        for r in self.ranks:
            v0, v1 = self.vr[r]
            for s in range(self.world):
                if s == r:
                    continue
                x0, x1 = self.xr[s]
                buf = torch.empty((v1 - v0) * nv1 * (x1 - x0) * n1, dtype=torch.float64,
                                  device=self.device)
                recvs[(r, s)] = buf
                msgs.setdefault(r, []).append((KIND_A2A, None, None, s, buf))
        self.comm.exchange(msgs)
        for (r, s), buf in recvs.items():
            v0, v1 = self.vr[r]
            x0, x1 = self.xr[s]
            run = (x1 - x0) * n1
            self.ops.slab_copy(buf, run, self.a[r][0][x0 * n1:], self.n2 * n1, (v1 - v0) * nv1,
                               run)

    # -- sub-steps ---------------------------------------------------------------------
    def _x_half(self, tau: float, slot: int) -> None:
        """_advect_space(tau/2) on layout A (driver.py:220-228)."""
        g = self.grid
        for r in self.ranks:
            v0, v1 = self.vr[r]
            vals = (self.vpoints[0], self.vpoints[1][v0:v1].contiguous())
            for d in range(2):
                src, dst = self.a[r]
                self.ops.spline_sweep(d, src, dst, self.dims_a(r), vals[d], 0.5 * tau,
                                      g.axes[d].h, self.flags[r][slot + d:slot + d + 1])
                self.a[r].reverse()

    def _density(self) -> None:
        parts = {}
        for r in self.ranks:
            d = self.dims_a(r)
            v0, v1 = self.vr[r]
            rl = torch.empty(self.n1 * self.n2, dtype=torch.float64, device=self.device)
            work = torch.empty(self.ops.density_work(d), dtype=torch.float64, device=self.device)
            self.ops.density(self.a[r][0], d, self.wv1, self.wv2[v0:v1].contiguous(), rl, work)
            parts[r] = rl
        self.rho.copy_(self.comm.allreduce(parts, "sum"))

    def _local_e(self, s: int, d: int) -> torch.Tensor:
        x0, x1 = self.xr[s]
        full = self.e[d * self.n1 * self.n2:(d + 1) * self.n1 * self.n2].view(self.n2, self.n1)
        return full[x0:x1].contiguous().view(-1)

    def step(self, tau: float, time_label: float | None = None) -> None:
        from .driver import SubstepError

        g = self.grid
        for r in self.ranks:
            self.flags[r].zero_()
        self.solve_flag.zero_()
        self._x_half(tau, 0)
        self._density()
        self.ops.field_solve(g, self.rho, self.e, self.stats, self.solve_flag)
        self._a_to_b()
        for s in self.ranks:
            for d in range(2):
                src, dst = self.b[s]
                self.ops.spline_sweep(2 + d, src, dst, self.dims_b(s), self._local_e(s, d), tau,
                                      g.axes[2 + d].h, self.flags[s][3 + d:4 + d])
                self.b[s].reverse()
        self._b_to_a()
        self._x_half(tau, 5)
        for r in self.ranks:
            self.flags[r][2:3] = torch.maximum(self.flags[r][2:3], self.solve_flag)
        flags = self.comm.allreduce({r: self.flags[r] for r in self.ranks}, "max")
        host = flags.cpu().numpy()
        for k, name in enumerate(self.names):
            if host[k]:
                raise SubstepError(name, time_label)

    def diagnostics(self, time: float = 0.0) -> dict:
        """Global conserved quantities (driver.py:279-316) from layout A."""
        self._density()
        self.ops.field_solve(self.grid, self.rho, self.e, None, self.solve_flag)
        sums = {}
        for r in self.ranks:
            d = self.dims_a(r)
            v0, v1 = self.vr[r]
            out = torch.zeros(8, dtype=torch.float64, device=self.device)
            work = torch.empty(self.ops.diag_work(d), dtype=torch.float64, device=self.device)
            self.ops.diag_sums(self.a[r][0], d, self.wx_full, self.wv1,
                               self.wv2[v0:v1].contiguous(), self.v1sq,
                               self.v2sq[v0:v1].contiguous(), out, work)
            sums[r] = out
        tot = self.comm.allreduce(sums, "sum").cpu().numpy()
        ee_t = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.ops.electric_energy(self.e, self.n1 * self.n2, self.wx_full, ee_t)
        ee = float(ee_t.cpu()[0])
        mass, l1, l2sq, kin = (float(x) for x in tot[:4])
        return {"time": float(time), "electric_energy": ee, "mass": mass, "l1_norm": l1,
                "l2_norm": math.sqrt(max(l2sq, 0.0)), "kinetic_energy": kin,
                "total_energy": kin + ee}


# ---------------------------------------------------------------------------
# Velocity-sharded dG solver (the paper's decomposition)
# ---------------------------------------------------------------------------
KIND_VL, KIND_VR = 3, 4  # v2 halo messages: receiver's left / right halo


class _RowsTab:
    """Rows [r0, r1) of x2 tables, composed form included (views, no copy)."""

    def __init__(self, t, r0: int, r1: int):
        self.t, self.r0, self.r1 = t, r0, r1
        self.q, self.alpha = t.q[r0:r1], t.alpha[r0:r1]

    def composed(self):
        return self.t.composed()[self.r0:self.r1]


class VShardedSolver:
    """Strang steps of a 2x2v dG field split along v2 over W ranks.

    The paper parallelises over velocity; SURVEY §8f.3
    asks for that alternative to the x sharding of :class:`ShardedSolver`.
    Rank r owns the v2 cells V_r = [c0, c1) as a contiguous slab of the
    canonical buffer, stored between H halo cells of each neighbour
    (v2 is the outermost axis, so every halo is one contiguous block of
    rows and travels zero-copy: NCCL sends straight from the field).

    * x half steps (and the merged closing + opening pair, "fast"
      arithmetic) are LOCAL: whole (x1, x2) planes, the single-GPU kernels
      on the slab with the x2 tables offset to the slab's rows; their
      density epilogue gives the slab's partial cell-centre density.
    * density: the partials are all-gathered and summed in rank order on
      every rank (deterministic), every rank solves the Poisson problem.
    * v pass: one halo exchange of H v2 cells per side, then the fused
      v1 v2 kernel streams [halo | slab | halo] non-periodically
      (``vpb_dg_sweep_vplane_v2halo``).  H bounds the E shift: the v2 cell
      offset q2 = floor(E2 tau / h_v2) must lie in [-H, H-1] (H = 1: a
      shift of less than one cell either way, true for the BASELINE
      configurations); the kernel raises a flag beyond that and the solver
      raises ``RuntimeError``.
    * overlap: the x pass that precedes a v pass runs its two H-cell
      boundary blocks of v2 rows first, posts the halo exchange of their
      output, and runs the interior rows while it is in flight.

    Per step and rank: 2 x H x P rows of n1 n2 nv1 doubles of halo (vs the x
    sharding's x1 halos of the doubled reach on every plane) and a
    C1 C2-double allgather of the density partials.
    """

    def __init__(self, grid: GridSpec, comm, ranks, world: int, ops=None, device=None,
                 halo_cells: int = 1, peer_halos: bool = False):
        if grid.method != DG or grid.ndim != 4:
            raise NotImplementedError("the velocity-sharded step covers the 2x2v SLDG path")
        p = grid.order
        n1, n2, nv1, nv2 = grid.dims4
        C2v = nv2 // p
        self.H = int(halo_cells)
        self.cr = [split_cells(C2v, world, r) for r in range(world)]
        if min(c1 - c0 for c0, c1 in self.cr) < self.H:
            raise ValueError(f"{C2v} v2 cells over {world} ranks leave a shard narrower than "
                             f"the {self.H}-cell halo")
        self.grid = grid
        self.comm = comm
        self.world = world
        self.ops = ops or CudaOps()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.order = p
        self.n1, self.n2, self.nv1, self.nv2 = n1, n2, nv1, nv2
        self.row = n1 * n2 * nv1  # doubles per v2 dof row
        self.ranks = list(ranks)
        dev = self.device
        self.f, self.buf, self.flags = {}, {}, {}
        for r in self.ranks:
            c0, c1 = self.cr[r]
            n = (c1 - c0 + 2 * self.H) * p * self.row
            self.f[r] = torch.empty(n, dtype=torch.float64, device=dev)
            self.buf[r] = torch.empty(n, dtype=torch.float64, device=dev)
        w = [torch.as_tensor(grid.axis_weights(a), dtype=torch.float64).to(dev) for a in range(4)]
        self.wv1, self.wv2 = w[2], w[3]
        self.wx_full = (w[1][:, None] * w[0][None, :]).reshape(-1).contiguous()
        self.vpoints = [torch.as_tensor(grid.axis_points(a), dtype=torch.float64).to(dev)
                        for a in (2, 3)]
        self.v1sq = self.vpoints[0] ** 2
        self.v2sq = self.vpoints[1] ** 2
        self.rho = torch.empty(n1 * n2, dtype=torch.float64, device=dev)
        self.e = torch.empty(2 * n1 * n2, dtype=torch.float64, device=dev)
        self.solve_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.names = ["x1 half (open)", "x2 half (open)", "field solve", "v1 full", "v2 full",
                      "x1 half (close)", "x2 half (close)"]
        self._xtab = {}
        self._dens = None
        self._halo_bytes = 0
        # peer_halos: the v pass reads the neighbours' boundary rows in place
        # (vpb_dg_sweep_vplane_v2peer) instead of receiving them into halo rows
        self.peer_halos = bool(peer_halos)
        self._nswap = 0  # passes so far: every shard's f is its buffer pair[_nswap % 2]
        self._peer_pair = {}
        if self.peer_halos:
            self._map_peers()

    def _map_peers(self) -> None:
        """Buffer pairs of the v2 neighbours: this process's own tensors when
        they are local (VirtualComm), else CUDA IPC mappings of the remote
        ones (peer memory over NVLink), exchanged once with the communicator."""
        need = set()
        for r in self.ranks:
            need.update({(r - 1) % self.world, (r + 1) % self.world})
        remote = sorted(need - set(self.ranks))
        for nb in need & set(self.ranks):
            self._peer_pair[nb] = (self.f[nb], self.buf[nb])
        if remote:
            from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor

            (r,) = self.ranks
            mine = tuple(reduce_tensor(t)[1] for t in (self.f[r], self.buf[r]))
            allargs = self.comm.allgather_object(mine)
            for nb in remote:
                self._peer_pair[nb] = tuple(rebuild_cuda_tensor(*a) for a in allargs[nb])

    def _peer_f(self, nb: int) -> torch.Tensor:
        """Neighbour nb's current f (its buffers swap in lockstep with ours)."""
        return self._peer_pair[nb][self._nswap % 2]

    # -- geometry ----------------------------------------------------------------
    def dims(self, r: int):
        c0, c1 = self.cr[r]
        return (self.n1, self.n2, self.nv1, (c1 - c0) * self.order)

    def local(self, t: torch.Tensor, r: int) -> torch.Tensor:
        """The shard's own rows of an extended buffer."""
        c0, c1 = self.cr[r]
        a = self.H * self.order * self.row
        return t[a:a + (c1 - c0) * self.order * self.row]

    # -- data movement helpers (tests / I/O) -------------------------------------
    def initialize(self, problem) -> None:
        from . import _device, _lib
        from .driver import separable_factors

        g1, g2, space = separable_factors(problem, self.grid)
        lib = _lib.load()
        dg1 = torch.as_tensor(np.asarray(g1), dtype=torch.float64).to(self.device)
        sp = torch.as_tensor(np.asarray(space).reshape(-1), dtype=torch.float64).to(self.device)
        p = self.order
        for r in self.ranks:
            c0, c1 = self.cr[r]
            dg2 = torch.as_tensor(np.asarray(g2)[c0 * p:c1 * p], dtype=torch.float64).to(self.device)
            _lib.check(lib.vpb_fill_separable(self.local(self.f[r], r).data_ptr(),
                                              _lib.dims(self.dims(r)), dg1.data_ptr(),
                                              dg2.data_ptr(), sp.data_ptr(), _device.stream()),
                       "vpb_fill_separable")

    def scatter(self, logical: np.ndarray) -> None:
        p = self.order
        for r in self.ranks:
            c0, c1 = self.cr[r]
            box = np.ascontiguousarray(logical[:, :, :, c0 * p:c1 * p].transpose(3, 2, 1, 0))
            self.local(self.f[r], r).copy_(torch.from_numpy(box.reshape(-1)).to(self.device))

    def local_logical(self, r: int) -> np.ndarray:
        d = self.dims(r)
        return (self.local(self.f[r], r).view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)
                .cpu().numpy())

    def gather(self) -> np.ndarray:
        out = np.empty(self.grid.dofs)
        p = self.order
        for r in self.ranks:
            c0, c1 = self.cr[r]
            out[:, :, :, c0 * p:c1 * p] = self.local_logical(r)
        return out

    # -- pieces of the step --------------------------------------------------------
    def x_tables(self, tau: float):
        key = float(tau)
        if key not in self._xtab:
            g = self.grid
            self._xtab = {key: [self.ops.tables(self.vpoints[d], 0.5 * tau, g.axes[d].h,
                                                g.dg_degree) for d in range(2)]}
        return self._xtab[key]

    def _density_consts(self):
        if self._dens is None:
            from .grid import gauss_nodes
            from .poisson import _lagrange_row

            p = self.order
            nodes, _ = gauss_nodes(p)
            mid = np.ascontiguousarray(_lagrange_row(nodes, 0.5))
            cells = [np.ascontiguousarray(np.asarray(self.grid.axis_weights(a))[:p])
                     for a in (0, 1)]
            ax = self.grid.axes
            volume = (ax[0].upper - ax[0].lower) * (ax[1].upper - ax[1].lower)
            self._dens = (mid, cells[0], cells[1], float(volume))
        return self._dens

    def _x_pass(self, tau, qmul, fl, stats_row, rc_parts, mark):
        """One local x pass on every shard (qmul 1: a half step; 2: the merged
        pair); with rc_parts the density epilogue fills the partials and the
        pass feeds a v pass: its H-cell boundary blocks of v2 rows run first,
        the v2 halo exchange of their output is posted, and the interior rows
        run while it is in flight (comm/compute overlap).
        Returns the pending exchange requests (wait before the v pass)."""
        t1, t2 = self.x_tables(tau)
        p, H = self.order, self.H
        mid, wc1, wc2, volume = self._density_consts()
        mark(("sweep_x12x12" if qmul == 2 else "sweep_x12") + ("_rho" if rc_parts is not None
                                                               else ""))
        feeds_v = rc_parts is not None

        def run_block(r, a, b, with_dens, parts):
            """x pass on the shard's v2 cells [a, b) (local numbering), its own
            density partial appended to parts."""
            c0, _ = self.cr[r]
            d = (self.n1, self.n2, self.nv1, (b - a) * p)
            off = a * p * self.row
            src = self.local(self.f[r], r)[off:off + d[3] * self.row]
            dst = self.local(self.buf[r], r)[off:off + d[3] * self.row]
            dens = None
            if with_dens:
                work = torch.empty(self.ops.xpass_work(d, p, qmul), dtype=torch.float64,
                                   device=self.device)
                rc = torch.empty((self.n1 // p) * (self.n2 // p), dtype=torch.float64,
                                 device=self.device)
                st = torch.zeros(4, dtype=torch.float64, device=self.device)
                wv2 = self.wv2[(c0 + a) * p:(c0 + b) * p].contiguous()
                dens = (self.wv1, wv2, mid, wc1, wc2, volume, work, rc, st)
                parts.append((rc, st))
            f1, f2 = fl[r]
            self.ops.xpass_rows(src, dst, d, p, t1, t2, (c0 + a) * p, qmul, f1, f2, dens)

        parts = {r: [] for r in self.ranks}
        # split every shard (decided on the global decomposition, so every
        # rank sums its density blocks in the same pattern) when all have an
        # interior beyond the two boundary blocks
        split = (feeds_v and not self.peer_halos
                 and all(c1 - c0 >= 2 * H + 1 for c0, c1 in self.cr))
        blocks = {}
        for r in self.ranks:
            c0, c1 = self.cr[r]
            nl = c1 - c0
            blocks[r] = [(0, H), (nl - H, nl), (H, nl - H)] if split else [(0, nl)]
        # the merged pass with the density: the blocks of a shard accumulate
        # into one set of CTA slabs (vpb_dg_sweep_xcomp_rows), one reduction
        acc = {}
        if feeds_v and qmul == 2 and hasattr(self.ops, "xcomp_rows"):
            for r in self.ranks:
                c0, c1 = self.cr[r]
                work = torch.empty(self.ops.xpass_work(self.dims(r), p, 2),
                                   dtype=torch.float64, device=self.device)
                rc = torch.empty((self.n1 // p) * (self.n2 // p), dtype=torch.float64,
                                 device=self.device)
                st = torch.zeros(4, dtype=torch.float64, device=self.device)
                wv2 = self.wv2[c0 * p:c1 * p].contiguous()
                acc[r] = ((self.wv1, wv2, mid, wc1, wc2, volume, work, rc, st),
                          _RowsTab(t2, c0 * p, c1 * p), [0, len(blocks[r])])
                parts[r].append((rc, st))

        def run_block_acc(r, a, b):
            dens, t2r, count = acc[r]
            count[0] += 1
            phase = (1 if count[0] == 1 else 0) | (2 if count[0] == count[1] else 0)
            self.ops.xcomp_rows(self.local(self.f[r], r), self.local(self.buf[r], r),
                                self.dims(r), p, a * p, (b - a) * p, t1, t2r, fl[r][0], dens,
                                phase)

        def run(r, a, b, with_dens):
            if acc:
                run_block_acc(r, a, b)
            else:
                run_block(r, a, b, with_dens, parts[r])

        for r in self.ranks:
            for a, b in (blocks[r][:2] if split else blocks[r]):
                run(r, a, b, feeds_v)
        reqs = []
        if feeds_v and not self.peer_halos:
            # the boundary cells of the new state are in buf: send them now
            # (NCCL runs on its own stream; the pass's timer label spans it)
            reqs = self._post_halos(self.buf)
        if split:
            for r in self.ranks:
                a, b = blocks[r][2]
                run(r, a, b, True)
        if feeds_v:
            for r in self.ranks:  # fixed order: left block, right block, interior
                rc = parts[r][0][0].clone()
                mean = parts[r][0][1][0].clone()
                for rc_k, st_k in parts[r][1:]:
                    rc += rc_k
                    mean += st_k[0]
                rc_parts[r] = rc
                stats_row[r][0] = mean
        for r in self.ranks:
            self.f[r], self.buf[r] = self.buf[r], self.f[r]
        self._nswap += 1
        return reqs

    def _sum_parts(self, parts: dict) -> torch.Tensor:
        """Rank-order sum of per-rank partials, identical on every rank."""
        full = self.comm.allgather(parts)
        out = full[0].clone()
        for t in full[1:]:
            out += t
        return out

    def _post_halos(self, bufs: dict) -> list:
        """Post the v2 halo exchange of the extended buffers ``bufs``: my
        first H cells go to the left neighbour's right halo, my last H cells
        to the right neighbour's left halo; contiguous rows, sent and
        received in place (no packing)."""
        H, p = self.H, self.order
        hrows = H * p * self.row
        msgs = {}
        for r in self.ranks:
            c0, c1 = self.cr[r]
            nl = (c1 - c0) * p * self.row
            f = bufs[r]
            left, right = (r - 1) % self.world, (r + 1) % self.world
            first = f[hrows:2 * hrows]              # my first H cells -> left's right halo
            last = f[nl:nl + hrows]                 # my last H cells -> right's left halo
            msgs[r] = [(KIND_VR, left, first, right, f[hrows + nl:2 * hrows + nl]),
                       (KIND_VL, right, last, left, f[0:hrows])]
        self._halo_bytes += 8 * 2 * hrows * len(self.ranks)
        return self.comm.exchange_async(msgs)

    def _v_pass(self, tau, fl, hflag, mark, reqs=None) -> None:
        """Fused v pass of every shard; ``reqs``: the pending halo exchange of
        the preceding x pass (None: exchange here)."""
        g = self.grid
        mark("tables_v12")
        nx = self.n1 * self.n2
        tv = [self.ops.tables(self.e[d * nx:(d + 1) * nx], tau, g.axes[2 + d].h, g.dg_degree)
              for d in range(2)]
        p, H = self.order, self.H
        if self.peer_halos:
            # the neighbours' x passes are complete: the rho gather that the
            # field solve waited for ordered every rank after them
            mark("sweep_v12")
            for r in self.ranks:
                c0, c1 = self.cr[r]
                left, right = (r - 1) % self.world, (r + 1) % self.world
                nl_l = self.cr[left][1] - self.cr[left][0]
                nl_r = self.cr[right][1] - self.cr[right][0]
                f1, f2 = fl[r]
                self.ops.vplane_v2peer(self._peer_f(left), nl_l + 2 * H, nl_l, self.f[r],
                                       c1 - c0 + 2 * H, H, self._peer_f(right), nl_r + 2 * H, H,
                                       H, self.local(self.buf[r], r), self.dims(r), p, tv[0],
                                       tv[1], f1, f2, hflag)
            self._halo_bytes += sum(8 * 2 * H * p * self.row for _ in self.ranks)
            for r in self.ranks:
                self.f[r], self.buf[r] = self.buf[r], self.f[r]
            self._nswap += 1
            # a neighbour's next x pass overwrites the buffer just read here
            self.comm.barrier_device()
            return
        if reqs is None:
            mark("halo_v2")
            reqs = self._post_halos(self.f)
        self.comm.wait(reqs)
        mark("sweep_v12")
        for r in self.ranks:
            c0, c1 = self.cr[r]
            f1, f2 = fl[r]
            self.ops.vplane_v2halo(self.f[r], self.local(self.buf[r], r), self.dims(r), p,
                                   c1 - c0 + 2 * H, H, tv[0], tv[1], f1, f2, hflag)
            self.f[r], self.buf[r] = self.buf[r], self.f[r]
        self._nswap += 1

    def advance(self, tau: float, nsteps: int, first_step: int | None = None,
                timer=None) -> None:
        """``nsteps`` Strang steps (driver.py:245-265 each) with the merged x
        passes of the "fast" arithmetic between them (driver.advance)."""
        from .driver import SubstepError
        from .poisson import _warn_if_not_neutral

        if nsteps <= 0:
            return
        mark = timer or (lambda label: None)
        dev = self.device
        flags = {r: torch.zeros((nsteps, 8), dtype=torch.int32, device=dev) for r in self.ranks}
        stats = {r: torch.zeros((nsteps, 4), dtype=torch.float64, device=dev)
                 for r in self.ranks}
        solve_flags = torch.zeros((nsteps, 1), dtype=torch.int32, device=dev)
        hflag = torch.zeros(1, dtype=torch.int32, device=dev)

        def fl(m, k):
            return {r: (flags[r][m][k:k + 1], flags[r][m][k + 1:k + 2]) for r in self.ranks}

        rc_parts = {}
        reqs = self._x_pass(tau, 1, fl(0, 0), {r: stats[r][0] for r in self.ranks}, rc_parts,
                            mark)
        for m in range(nsteps):
            mark("rho_allgather")
            rc = self._sum_parts(rc_parts)
            mark("field_solve")
            self.ops.field_solve_centred(self.grid, rc, self.e, solve_flags[m])
            self._v_pass(tau, fl(m, 3), hflag, mark, reqs)
            if m + 1 < nsteps:  # closing of step m + opening of step m+1, one pass
                rc_parts = {}
                reqs = self._x_pass(tau, 2, fl(m, 5), {r: stats[r][m + 1] for r in self.ranks},
                                    rc_parts, mark)
            else:
                self._x_pass(tau, 1, fl(m, 5), None, None, mark)
        mark("flags")
        for r in self.ranks:
            flags[r][:, 2:3] = torch.maximum(flags[r][:, 2:3], solve_flags)
        fh = self.comm.allreduce(flags, "max").cpu().numpy()
        sh = self._sum_parts(stats).cpu().numpy()
        hmax = self.comm.allreduce({r: hflag for r in self.ranks}, "max").cpu().numpy()
        mark(None)
        if hmax.any():
            raise RuntimeError(f"an E shift exceeded the {self.H}-cell v2 halo; "
                               "construct VShardedSolver with a wider halo_cells")
        for m in range(nsteps):
            _warn_if_not_neutral(float(sh[m, 0]))
            for k, name in enumerate(self.names):
                if fh[m, k]:
                    raise SubstepError(name, None if first_step is None
                                       else (first_step + m) * tau)

    def diagnostics(self, time: float = 0.0) -> dict:
        """Global conserved quantities (driver.py:279-316)."""
        p = self.order
        parts, sums = {}, {}
        for r in self.ranks:
            c0, _ = self.cr[r]
            d = self.dims(r)
            wv2 = self.wv2[c0 * p:c0 * p + d[3]].contiguous()
            v2sq = self.v2sq[c0 * p:c0 * p + d[3]].contiguous()
            rl = torch.empty(self.n1 * self.n2, dtype=torch.float64, device=self.device)
            work = torch.empty(self.ops.density_work(d), dtype=torch.float64, device=self.device)
            f = self.local(self.f[r], r)
            self.ops.density(f, d, self.wv1, wv2, rl, work)
            parts[r] = rl
            out = torch.zeros(8, dtype=torch.float64, device=self.device)
            dwork = torch.empty(self.ops.diag_work(d), dtype=torch.float64, device=self.device)
            self.ops.diag_sums(f, d, self.wx_full, self.wv1, wv2, self.v1sq, v2sq, out, dwork)
            sums[r] = out
        self.rho.copy_(self._sum_parts(parts))
        self.ops.field_solve(self.grid, self.rho, self.e, None, self.solve_flag)
        tot = self._sum_parts(sums).cpu().numpy()
        ee_t = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.ops.electric_energy(self.e, self.n1 * self.n2, self.wx_full, ee_t)
        ee = float(ee_t.cpu()[0])
        mass, l1, l2sq, kin = (float(x) for x in tot[:4])
        return {"time": float(time), "electric_energy": ee, "mass": mass, "l1_norm": l1,
                "l2_norm": math.sqrt(max(l2sq, 0.0)), "kinetic_energy": kin,
                "total_energy": kin + ee}
