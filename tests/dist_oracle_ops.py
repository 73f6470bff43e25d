"""TEST INFRASTRUCTURE: oracle-backed local compute for the sharded solver.

Implements the ``CudaOps`` interface of ``paper_1803_02143_b200.dist`` on CPU
tensors with the oracle's restatement of the reference arithmetic, so the
multi-GPU layer's decomposition, halo packing, message pattern and ρ
assembly can be exercised with the gloo backend (or in-process) on CPU.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import core


class _Tab:
    def __init__(self, a, b, q, alpha):
        self.a, self.b, self.q, self.alpha = a, b, q, alpha


def _box(t: torch.Tensor, dims) -> np.ndarray:
    """flat canonical box -> logical (x1, x2, v1, v2) numpy view."""
    n1, n2, nv1, nv2 = dims
    return t.numpy().reshape(nv2, nv1, n2, n1).transpose(3, 2, 1, 0)


def _line_table_index(dims, axis) -> np.ndarray:
    """Device table row of every line of a sweep (lines in C order over the
    other logical axes), matching the CUDA kernels' indexing."""
    n1, n2, nv1, nv2 = dims
    other = [a for a in range(4) if a != axis]
    shape = [dims[a] for a in other]
    idx = np.indices(shape)
    coord = {a: idx[i] for i, a in enumerate(other)}
    if axis == 0:
        row = coord[2]
    elif axis == 1:
        row = coord[3]
    else:
        row = coord[1] * n1 + coord[0]
    return row.reshape(-1).astype(np.int64)


class NumpyOps:
    def tables(self, values, scale, h, degree):
        shifts = values.cpu().numpy() * scale
        return _Tab(*core.projection_pairs(shifts, h, degree))

    def tables_q(self, tab):
        return tab.q

    def _sweep_lines(self, arr, axis, dims, order, tab, ext=None):
        moved = np.moveaxis(arr if ext is None else ext, axis, -1)
        lead = moved.shape[:-1]
        n = moved.shape[-1]
        lines = np.ascontiguousarray(moved).reshape(-1, n)
        idx = _line_table_index(dims, axis)
        out = core.dg_lines(lines, idx, tab.a, tab.b, tab.q, tab.alpha, n // order, order)
        return np.moveaxis(out.reshape(lead + (n,)), -1, axis)

    def _store(self, dst, dims, logical, flag):
        n1, n2, nv1, nv2 = dims
        dst.copy_(torch.from_numpy(np.ascontiguousarray(logical.transpose(3, 2, 1, 0)).reshape(-1)))
        if not np.all(np.isfinite(logical)):
            flag.fill_(1)

    def sweep(self, axis, src, dst, dims, order, tab, flag):
        out = self._sweep_lines(_box(src, dims), axis, dims, order, tab)
        self._store(dst, dims, out, flag)

    def spline_sweep(self, axis, src, dst, dims, values, scale, h, flag):
        arr = _box(src, dims)
        moved = np.moveaxis(arr, axis, -1)
        lead = moved.shape[:-1]
        n = moved.shape[-1]
        lines = np.ascontiguousarray(moved).reshape(-1, n)
        idx = _line_table_index(dims, axis)
        out = core.spline_lines(lines, idx, values.cpu().numpy() * scale, h)
        self._store(dst, dims, np.moveaxis(out.reshape(lead + (n,)), -1, axis), flag)

    def slab_copy(self, src, src_stride, dst, dst_stride, outer, run):
        for k in range(outer):
            dst[k * dst_stride:k * dst_stride + run] = src[k * src_stride:k * src_stride + run]

    def pack(self, axis, f, dims, order, cell0, width, buf):
        arr = _box(f, dims)
        sl = [slice(None)] * 4
        sl[axis] = slice(cell0 * order, (cell0 + width) * order)
        part = arr[tuple(sl)]
        buf.copy_(torch.from_numpy(np.ascontiguousarray(part.transpose(3, 2, 1, 0)).reshape(-1)))

    def halo_sweep(self, axis, src, dst, dims, order, left, wl, right, wr, tab, flag):
        arr = _box(src, dims)
        pieces = []
        for buf, w in ((left, wl), (right, wr)):
            d = list(dims)
            d[axis] = w * order
            pieces.append(_box(buf, d) if w else None)
        ext = np.concatenate([p for p in (pieces[0], arr, pieces[1]) if p is not None], axis=axis)
        out = self._sweep_lines(None, axis, dims, order, tab, ext=ext)
        sl = [slice(None)] * 4
        sl[axis] = slice(wl * order, wl * order + dims[axis])
        self._store(dst, dims, out[tuple(sl)], flag)

    # -- velocity-sharded field (VShardedSolver) -------------------------------
    def xpass_work(self, dims, order, qmul):
        return 1

    def xpass_rows(self, src, dst, dims, order, t1, t2, r0, qmul, f1, f2, dens=None):
        """x half step (qmul 1) or the two consecutive half steps (qmul 2) of
        a v2 slab (x2 table rows from r0), periodic x, sweep by sweep; density
        partial of the result as the kernels' epilogue defines it."""
        nv2 = dims[3]
        t2s = _Tab(t2.a[r0:r0 + nv2], t2.b[r0:r0 + nv2], t2.q[r0:r0 + nv2],
                   t2.alpha[r0:r0 + nv2])
        arr = _box(src, dims)
        for _ in range(qmul):
            arr = self._sweep_lines(arr, 0, dims, order, t1)
            arr = self._sweep_lines(arr, 1, dims, order, t2s)
        self._store(dst, dims, arr, f1)
        if dens is not None:
            wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
            p = order
            n1, n2, nv1, _ = dims
            o = arr.reshape(n1 // p, p, n2 // p, p, nv1, nv2)
            wa, wb = wv1.numpy(), wv2.numpy()
            rc = np.einsum("aibjvw,i,j,v,w->ba", o, mid, mid, wa, wb, optimize=False)
            rc_out.copy_(torch.from_numpy(np.ascontiguousarray(rc).reshape(-1)))
            mean = np.einsum("aibjvw,i,j,v,w->", o, wc1, wc2, wa, wb, optimize=False)
            stats[0] = float(mean) / volume

    def xcomp_rows(self, src, dst, dims, order, v2_0, v2_rows, t1, t2r, flag, dens, phase):
        """Merged pass on v2 rows [v2_0, v2_0 + v2_rows) of a shard (t2r: the
        shard's rows of the global tables) with the density accumulated over
        the calls of one pass (phase bit 1: reset, bit 2: last)."""
        wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
        n1, n2, nv1, _ = dims
        plane = n1 * n2 * nv1
        sub = (n1, n2, nv1, v2_rows)
        a, b = v2_0 * plane, (v2_0 + v2_rows) * plane
        rc_b = torch.empty_like(rc_out)
        st_b = torch.zeros_like(stats)
        self.xpass_rows(src[a:b], dst[a:b], sub, order, t1, t2r.t, t2r.r0 + v2_0, 2, flag, None,
                        (wv1, wv2[v2_0:v2_0 + v2_rows], mid, wc1, wc2, volume, work, rc_b, st_b))
        if phase & 1:
            rc_out.zero_()
            stats[0] = 0.0
        rc_out += rc_b
        stats[0] += st_b[0]

    def vplane_v2halo(self, src_ext, dst, dims, order, c2e, off, t1, t2, f1, f2, hflag):
        """v1 then v2 sweep of [halo | slab | halo]: swept periodically over
        the extended rows (whose wrap-around only reaches discarded cells when
        the halos are wide enough), the slab's cells kept."""
        n1, n2, nv1, nv2 = dims
        ed = (n1, n2, nv1, c2e * order)
        ext = _box(src_ext, ed)
        q = np.asarray(t2.q)
        if q.size and (off - q.max() - 1 < 0 or off - q.min() + nv2 // order - 1 > c2e - 1):
            hflag.fill_(1)
        ext = self._sweep_lines(ext, 2, ed, order, t1)
        ext = self._sweep_lines(ext, 3, ed, order, t2)
        self._store(dst, dims, ext[:, :, :, off * order:off * order + nv2], f2)

    def vplane_v2peer(self, src_l, l_cells, l0, src, c_cells, c0, src_r, r_cells, r0, H, dst,
                      dims, order, t1, t2, f1, f2, hflag):
        """The halo regions read from the neighbours' buffers: assemble the
        stream [left H cells | own cells | right H cells] and run the
        extended-buffer pass."""
        n1, n2, nv1, nv2 = dims
        row = n1 * n2 * nv1 * order  # doubles per v2 cell
        nc = nv2 // order
        ext = torch.cat([src_l[l0 * row:(l0 + H) * row], src[c0 * row:(c0 + nc) * row],
                         src_r[r0 * row:(r0 + H) * row]])
        self.vplane_v2halo(ext, dst, dims, order, nc + 2 * H, H, t1, t2, f1, f2, hflag)

    # -- three-cell x-plane stencil passes (ShardedSolver.advance) ------------
    def stencil_tables(self, tab, single: bool):
        a, b = tab.a, tab.b
        if single:
            return np.stack([np.zeros_like(a), a, b], axis=1)
        return np.stack([a @ a, a @ b + b @ a, b @ b], axis=1)

    def xstencil_work(self, dims, order, wl, wr):
        return 1

    def xstencil(self, src, dst, dims, order, k1, t1, k2, t2, qmul, hl, wl, hr, wr, flag,
                 dens=None):
        """x1 stencil with halos (cells c-Q-2 .. c-Q, Q = qmul q), then the
        periodic x2 stencil, on the logical box; optional density epilogue."""
        p = order
        n1, n2, nv1, nv2 = dims
        c1n, c2n = n1 // p, n2 // p
        pieces = []
        if wl:
            pieces.append(_box(hl, (wl * p, n2, nv1, nv2)))
        pieces.append(_box(src, dims))
        if wr:
            pieces.append(_box(hr, (wr * p, n2, nv1, nv2)))
        ext = np.concatenate(pieces, axis=0).reshape(wl + c1n + wr, p, n2, nv1, nv2)
        g = np.zeros((c1n, p, n2, nv1, nv2))
        for iv1 in range(nv1):
            qq = qmul * int(t1.q[iv1])
            for k in range(3):
                j = np.arange(c1n) - qq - 2 + k + wl
                g[:, :, :, iv1, :] += np.einsum("jm,cmxv->cjxv", k1[iv1, k],
                                                ext[:, :, :, iv1, :][j], optimize=False)
        g2 = g.reshape(c1n, p, c2n, p, nv1, nv2)
        o = np.zeros_like(g2)
        for iv2 in range(nv2):
            qq = qmul * int(t2.q[iv2])
            for k in range(3):
                j = (np.arange(c2n) - qq - 2 + k) % c2n
                o[..., iv2] += np.einsum("jm,aibmv->aibjv", k2[iv2, k],
                                         g2[..., iv2][:, :, j], optimize=False)
        out = o.reshape(n1, n2, nv1, nv2)
        self._store(dst, dims, out, flag)
        if dens is not None:
            wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
            wa, wb = wv1.numpy(), wv2.numpy()
            rc = np.einsum("aibjvw,i,j,v,w->ba", o, mid, mid, wa, wb, optimize=False)
            rc_out.copy_(torch.from_numpy(np.ascontiguousarray(rc).reshape(-1)))
            mean = np.einsum("aibjvw,i,j,v,w->", o, wc1, wc2, wa, wb, optimize=False)
            stats[0] = float(mean) / volume

    def xstencil2(self, src, dst, dims, order, k1, t1, k2, t2, qmul, hl, wl, hr, wr, wl2, x2l,
                  wr2, x2r, flag, dens=None):
        """x1 x x2 shard: the extended box [x2 halo | rows | x2 halo] x [x1
        halo | x1 | x1 halo] (corners from the x2 halos' x1 parts), x1
        stencil on every row of it, then the x2 stencil without wrap."""
        p = order
        n1, n2, nv1, nv2 = dims
        c1n, c2n = n1 // p, n2 // p

        def row_block(own, l, r, rows):
            parts = []
            if wl:
                parts.append(_box(l, (wl * p, rows, nv1, nv2)))
            parts.append(_box(own, (n1, rows, nv1, nv2)))
            if wr:
                parts.append(_box(r, (wr * p, rows, nv1, nv2)))
            return np.concatenate(parts, axis=0)

        blocks = []
        if wl2:
            blocks.append(row_block(x2l[0], x2l[1], x2l[2], wl2 * p))
        blocks.append(row_block(src, hl, hr, n2))
        if wr2:
            blocks.append(row_block(x2r[0], x2r[1], x2r[2], wr2 * p))
        ext = np.concatenate(blocks, axis=1)  # (x1 ext, x2 ext, v1, v2)
        c2e = wl2 + c2n + wr2
        ext = ext.reshape(wl + c1n + wr, p, c2e * p, nv1, nv2)
        g = np.zeros((c1n, p, c2e * p, nv1, nv2))
        for iv1 in range(nv1):
            qq = qmul * int(t1.q[iv1])
            for k in range(3):
                j = np.arange(c1n) - qq - 2 + k + wl
                g[:, :, :, iv1, :] += np.einsum("jm,cmxv->cjxv", k1[iv1, k],
                                                ext[:, :, :, iv1, :][j], optimize=False)
        g2 = g.reshape(c1n, p, c2e, p, nv1, nv2)
        o = np.zeros((c1n, p, c2n, p, nv1, nv2))
        for iv2 in range(nv2):
            qq = qmul * int(t2.q[iv2])
            for k in range(3):
                j = np.arange(c2n) - qq - 2 + k + wl2
                assert j.min() >= 0 and j.max() < c2e, "x2 halo too narrow"
                o[..., iv2] += np.einsum("jm,aibmv->aibjv", k2[iv2, k],
                                         g2[..., iv2][:, :, j], optimize=False)
        out = o.reshape(n1, n2, nv1, nv2)
        self._store(dst, dims, out, flag)
        if dens is not None:
            wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
            wa, wb = wv1.numpy(), wv2.numpy()
            rc = np.einsum("aibjvw,i,j,v,w->ba", o, mid, mid, wa, wb, optimize=False)
            rc_out.copy_(torch.from_numpy(np.ascontiguousarray(rc).reshape(-1)))
            mean = np.einsum("aibjvw,i,j,v,w->", o, wc1, wc2, wa, wb, optimize=False)
            stats[0] = float(mean) / volume

    def xstencil_rows(self, src, dst, dims, order, v2_0, v2_rows, k1, t1, k2, t2, qmul, hl, wl,
                      hr, wr, flag, dens=None, phase=3):
        """One block of v2 rows of the pipelined pass: the whole-shard pass
        on the rows' slices (tables of the rows' v2 indices), the density
        partials accumulated over the blocks of the pass."""
        n1, n2, nv1, nv2 = dims
        plane = n1 * n2 * nv1
        a, b = v2_0 * plane, (v2_0 + v2_rows) * plane
        sub = (n1, n2, nv1, v2_rows)
        hw = n2 * nv1
        hl_s = hl[v2_0 * hw * wl * order:(v2_0 + v2_rows) * hw * wl * order] if wl else hl
        hr_s = hr[v2_0 * hw * wr * order:(v2_0 + v2_rows) * hw * wr * order] if wr else hr
        t2s = _Tab(None, None, np.asarray(t2.q)[v2_0:v2_0 + v2_rows], None)
        k2s = k2[v2_0:v2_0 + v2_rows]
        out = dst[a:b]
        sub_dens = None
        if dens is not None:
            wv1, wv2, mid, wc1, wc2, volume, work, rc_out, stats = dens
            rc_tmp = torch.empty_like(rc_out)
            st_tmp = torch.zeros_like(stats)
            sub_dens = (wv1, wv2[v2_0:v2_0 + v2_rows], mid, wc1, wc2, volume, work, rc_tmp,
                        st_tmp)
        self.xstencil(src[a:b], out, sub, order, k1, t1, k2s, t2s, qmul, hl_s, wl, hr_s, wr, flag,
                      sub_dens)
        if dens is not None:
            if phase & 1:
                rc_out.zero_()
                stats[0] = 0.0
            rc_out += rc_tmp
            stats[0] += st_tmp[0]

    def vplane(self, src, dst, dims, order, t1, t2, f1, f2):
        tmp = torch.empty_like(src)
        self.sweep(2, src, tmp, dims, order, t1, f1)
        self.sweep(3, tmp, dst, dims, order, t2, f2)

    def field_solve_centred(self, grid, rc, e, flag):
        og = core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                        tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)
        c1n, c2n = grid.axes[0].count, grid.axes[1].count
        logical = rc.numpy().reshape(c2n, c1n).T
        comps = core.solve_poisson_centred(logical, og)
        e.copy_(torch.from_numpy(np.concatenate([c.T.reshape(-1) for c in comps])))

    def density_work(self, dims):
        return 1

    def density(self, f, dims, wv1, wv2, rho, work):
        arr = _box(f, dims)
        r = np.einsum("abcd,c,d->ab", arr, wv1.numpy(), wv2.numpy(), optimize=False)
        rho.copy_(torch.from_numpy(np.ascontiguousarray(r.T).reshape(-1)))

    def field_solve(self, grid, rho, e, stats, flag):
        og = core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                        tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)
        n1, n2 = grid.dof(0), grid.dof(1)
        logical = rho.numpy().reshape(n2, n1).T
        comps, mean = core.solve_poisson(logical, og)
        e.copy_(torch.from_numpy(np.concatenate([c.T.reshape(-1) for c in comps])))
        if stats is not None:
            stats[0] = mean

    def diag_work(self, dims):
        return 1

    def diag_sums(self, f, dims, wx, wv1, wv2, v1sq, v2sq, out, work):
        arr = _box(f, dims)
        n1, n2 = dims[0], dims[1]
        wxl = wx.numpy().reshape(n2, n1).T
        w = wxl[:, :, None, None] * (wv1.numpy()[:, None] * wv2.numpy()[None, :])[None, None]
        out[0] = float(np.sum(arr * w))
        out[1] = float(np.sum(np.abs(arr) * w))
        out[2] = float(np.sum(arr * arr * w))
        vsq = v1sq.numpy()[:, None] + v2sq.numpy()[None, :]
        out[3] = 0.5 * float(np.sum(arr * w * vsq[None, None]))

    def electric_energy(self, e, nx, wx, out):
        ev = e.numpy()
        out[0] = 0.5 * float(np.sum(ev * ev * np.tile(wx.numpy(), 2)))
