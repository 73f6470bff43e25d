// Merged x half steps with composed stencils (the "fast" arithmetic mode).
//
// Between two Strang steps the reference applies x1(τ/2) x2(τ/2) (closing
// half step of step m, driver.py:262-265) and then x1(τ/2) x2(τ/2) again
// (opening half step of step m+1, driver.py:257-258), with the same tables
// (run loop driver.py:371-377).  Each sweep is the projection
//     out[c] = A u[c-q-1] + B u[c-q]              (_kernels.pyx:113-123)
// so two sweeps along one axis are the three-cell stencil
//     out[c] = AA u[c-2q-2] + (AB+BA) u[c-2q-1] + BB u[c-2q]
// -- both projections are kept (this is (P T)(P T), not the P T_τ merge
// SURVEY.md §8f rules out), only the matrix products are formed once per
// table row.  x1 and x2 act on different indices of a (v1, v2) plane, so
// x1 x2 x1 x2 = (x1 x1)(x2 x2) exactly in real arithmetic; the pass applies
// the composed x1 stencil and then the composed x2 stencil while the plane
// streams through shared memory.  Per dof that is 2 x 3P fused multiply-adds
// instead of 4 x (4P-1) separately rounded operations of the bitwise chain
// (fused2.cu), so the pass is HBM-bound instead of fp64-issue bound.  The
// result differs from the bitwise chain by round-off only (≈1e-16 relative
// per step; tests hold it to the 1e-12 per-step bar against the oracle).
//
// alpha == 0 rows (exact shifts, dg.py:130-132: A = 0, B = I) stay exact
// copies: out[c] = u[c-2q].
//
// Streaming along x2 (per plane, source order from s0 = -2(q2+1) mod C2):
// C2+2 source cells t = 0, 1, ..., C2+1 arrive in chunks of G cells through an
// mbarrier ring of 1-D bulk copies; thread c = x1 cell c applies the composed
// x1 stencil to source cell t (3 x1 cells of each of its P rows), folds the
// result into the running x2 sums of output cells t-2, t-1 and t (registers),
// and from t = 2 on emits output x2 cell t-2 (streaming stores), optionally
// with the density epilogue of xplane.cuh.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "async_copy.cuh"
#include "common.cuh"
#include "tensormap.cuh"
#include "xplane.cuh"

namespace vpb {

// out[t][0] = A A, out[t][1] = A B + B A, out[t][2] = B B  (row-major P x P);
// single != 0: out[t] = {0, A, B}, one sweep as the same three-cell stencil
// with offset q instead of 2q (the sharded step's single x half steps)
__global__ void compose_tables_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                      int64_t T, int P, double* __restrict__ out, int single) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t pp = (int64_t)P * P;
  if (e >= T * pp) return;
  const int64_t t = e / pp;
  const int j = (int)((e / P) % P), m = (int)(e % P);
  const double* A = a + t * pp;
  const double* B = b + t * pp;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  if (single) {
    c1 = A[j * P + m];
    c2 = B[j * P + m];
  } else
  for (int k = 0; k < P; ++k) {
    c0 = fma(A[j * P + k], A[k * P + m], c0);
    c1 = fma(A[j * P + k], B[k * P + m], c1);
    c1 = fma(B[j * P + k], A[k * P + m], c1);
    c2 = fma(B[j * P + k], B[k * P + m], c2);
  }
  double* o = out + t * 3 * pp + j * P + m;
  o[0] = c0;
  o[pp] = c1;
  o[2 * pp] = c2;
}

template <int P>
__device__ __forceinline__ void load_cell_row(const double* p, double (&u)[P]) {
  lds_row_cell<P>(p, u);
}

// Which planes a launch covers: source plane l (contiguous in src) is the
// global (iv2, iv1) = (iv2_0 + l / nv1, iv1_0 + l % nv1) and lands at dst
// plane iv2 * nv1_glob + iv1.  The whole field is the identity map (nv1 =
// nv1_glob, offsets 0).  Each plane may be split into nseg x2 segments of SL
// output cells (work items = planes x segments) when a launch covers few
// planes.  (A blocked v -> x variant that fed blocks of planes through an
// L2-resident scratch buffer used this; it measured slower.)
struct XcMap {
  int64_t nv1, iv1_0, iv2_0, nv1_glob;
  int nseg, SL;
};

// Stencil offset and x1 halos.  Source cells of output cell c are
// c - Q - 2, c - Q - 1, c - Q with Q = qmul * q (qmul = 2: the composed merged
// pass; 1: a single sweep with tables {0, A, B}).  HALO (x1-sharded field):
// the row is the shard's cells 0..C1-1, not periodic; cells -wl..-1 come from
// hl and C1..C1+wr-1 from hr, laid out [plane][x2 row][w*P] (vpb_halo_pack).
// x2-sharded fields (x2 != 0, x1 x x2 process grids): the plane's x2 rows
// are not periodic either; source x2 cells -wl2..-1 and C2..C2+wr2-1 come
// from the x2 halo buffers x2l / x2r, each three parts in the layouts of the
// shard's own data: [0] the x1 dofs [plane][w2 cells][P rows][n1]
// (vpb_halo_pack axis 1), [1] / [2] their left / right x1 halo cells
// [plane][w2 cells][P rows][wl*P] / [wr*P] (the x1 halo rows of the
// neighbour's boundary cells: the corners).
struct XcStencil {
  int qmul;
  const double* hl;
  const double* hr;
  int wl, wr;
  int x2 = 0, wl2 = 0, wr2 = 0;
  const double* x2l[3] = {nullptr, nullptr, nullptr};
  const double* x2r[3] = {nullptr, nullptr, nullptr};
};

// Register budget.  A sub-partition holds 16K registers: at 224 per thread
// two warps fit (8 per SM; config 5's 3-warp CTAs: only 2 CTAs = 6 warps),
// at 168 three (12 per SM).  The T2S instances keep the composed x2 tables
// in shared memory (broadcast loads the compiler may not hoist), which frees
// the 27 doubles per thread that make 168 reachable at P = 3 without spills.
// Measured (tune_xcomp.py, one B200): config 5 (3-warp CTAs) 22.8 -> 21.8
// ms with T2S; config 2 (2-warp CTAs, 4 CTAs at 224) 3.59 -> 4.09 ms, so
// T2S is used only where the 224-register plan strands warp slots (P = 3,
// 3-warp CTAs; VPB_XCOMP_T2S=0/1 forces it off / on).
#ifndef VPB_XCOMP_MAXNREG
#define VPB_XCOMP_MAXNREG 224
#endif

// broadcast shared-memory load that stays in the loop (not hoisted to a register)
__device__ __forceinline__ double lds_keep(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
template <int P, bool DENS, bool HALO = false, bool T2S = false, bool BST = false>
__global__ void __launch_bounds__(128) __maxnreg__(P >= 3 ? (T2S ? 168 : VPB_XCOMP_MAXNREG) : 168)
    dg_xcomp_kernel(const double* __restrict__ src, double* __restrict__ dst, int n1, int C2,
                    int G, int nst, int64_t nitems, int64_t items_per_block, const XcMap mp,
                    const double* __restrict__ k1, const int64_t* __restrict__ q1,
                    const double* __restrict__ al1, const double* __restrict__ k2,
                    const int64_t* __restrict__ q2, const double* __restrict__ al2,
                    int32_t* __restrict__ flag, const XDensity dn, int dacc,
                    const XcStencil sx) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int cell = P * n1;  // one x2 cell: P rows of n1 dofs
  const int rl = n1, cells = cell;
  const int slot = G * cell;
  double* inb = reinterpret_cast<double*>(smem_raw);
  // HALO: the chunk's left / right x1 halo cells arrive by their own bulk
  // copies (contiguous per chunk in the vpb_halo_pack layout) into
  // [nst][G cells][P rows][w*P] regions next to the ring
  const int hls = HALO ? G * P * sx.wl * P : 0, hrs = HALO ? G * P * sx.wr * P : 0;
  double* hlb = inb + nst * slot;
  double* hrb = hlb + nst * hls;
  // BST: output cells are staged in shared memory ([2][G cells], one buffer
  // per ring chunk parity) and leave by one bulk copy per chunk (the chunk's
  // output cells are consecutive x2 cells of one plane: contiguous in HBM)
  double* obuf = hrb + nst * hrs;
  uint64_t* bars = reinterpret_cast<uint64_t*>(obuf + (BST ? 2 * slot : 0));
  int ob = 0;  // BST: staging buffer of the current chunk

  const int tid = threadIdx.x;
  const int it_begin = (int)(blockIdx.x * items_per_block);
  const int it_end = (int)min(nitems, (int64_t)it_begin + items_per_block);
  if (it_begin >= it_end) return;
  const int64_t plane_elems = (int64_t)C2 * cell;
  const uint64_t pol_stream = l2_evict_first();
  const uint64_t pol_keep = l2_evict_last();

  // item -> (source plane, first output cell, source cells to stream, chunks)
  struct Item {
    int l, oa, L, nch;
  };
  auto item_of = [&](int it) {
    Item r;
    r.l = it / mp.nseg;
    r.oa = (int)(it - r.l * mp.nseg) * mp.SL;
    r.L = min(mp.SL, C2 - r.oa) + 2;
    r.nch = (r.L + G - 1) / G;
    return r;
  };
  const int nv1l = (int)mp.nv1;
  auto iv2_of = [&](int l) { return (int)mp.iv2_0 + l / nv1l; };
  // first source cell of an item: -(qmul q2 + 2) + oa (mod C2)
  auto s0_of = [&](const Item& r) {
    const int64_t s = -((int64_t)sx.qmul * q2[iv2_of(r.l)] + 2) + r.oa;
    return HALO && sx.x2 ? (int)s : (int)wrap_mod(s, C2);  // x2-sharded: halo cells
  };
  // producer (thread 0)
  int p_it = it_begin;
  Item p_r{};
  int p_k = 0, p_s0 = 0, p_st = 0;
  auto issue_next = [&]() {
    const int t0 = p_k * G;
    const int ns = min(G, p_r.L - t0);
    int sb = p_s0 + t0;
    if constexpr (HALO) {
      if (sx.x2) {
        // x2-sharded: the chunk's cells [sb, sb + ns) lie in [-wl2, C2 + wr2)
        // (host-sized halos); runs by region, each region in the shard's
        // own layouts (rows, x1 halo rows)
        const int hcl = P * sx.wl * P, hcr = P * sx.wr * P;
        mbar_arrive_expect_tx(bars + p_st, (uint32_t)ns * (cell + hcl + hcr) * 8u);
        int c = sb, k = 0;
        while (k < ns) {
          const double *own, *xl, *xr;
          int run;
          if (c < 0) {
            const int64_t b = (int64_t)p_r.l * sx.wl2 + (c + sx.wl2);
            own = sx.x2l[0] + b * cell;
            xl = sx.x2l[1] + b * hcl;
            xr = sx.x2l[2] + b * hcr;
            run = min(ns - k, -c);
          } else if (c < C2) {
            const int64_t b = (int64_t)p_r.l * C2 + c;
            own = src + (int64_t)p_r.l * plane_elems + (int64_t)c * cell;
            xl = sx.hl + b * hcl;
            xr = sx.hr + b * hcr;
            run = min(ns - k, C2 - c);
          } else {
            const int64_t b = (int64_t)p_r.l * sx.wr2 + (c - C2);
            own = sx.x2r[0] + b * cell;
            xl = sx.x2r[1] + b * hcl;
            xr = sx.x2r[2] + b * hcr;
            run = ns - k;
          }
          bulk_g2s(inb + p_st * slot + k * cell, own, (uint32_t)run * cell * 8u, bars + p_st);
          if (hcl)
            bulk_g2s(hlb + p_st * hls + k * hcl, xl, (uint32_t)run * hcl * 8u, bars + p_st);
          if (hcr)
            bulk_g2s(hrb + p_st * hrs + k * hcr, xr, (uint32_t)run * hcr * 8u, bars + p_st);
          k += run;
          c += run;
        }
        if (++p_st == nst) p_st = 0;
        if (++p_k == p_r.nch) {
          p_k = 0;
          if (++p_it < it_end) {
            p_r = item_of(p_it);
            p_s0 = s0_of(p_r);
          }
        }
        return;
      }
    }
    while (sb >= C2) sb -= C2;
    const double* base = src + (int64_t)p_r.l * plane_elems;
    double* d = inb + p_st * slot;
    const int run1 = min(ns, C2 - sb);
    if constexpr (HALO) {
      const int hcl = P * sx.wl * P, hcr = P * sx.wr * P;  // halo doubles per x2 cell
      mbar_arrive_expect_tx(bars + p_st, (uint32_t)ns * (cell + hcl + hcr) * 8u);
      const int64_t hb = (int64_t)p_r.l * C2;
      if (hcl) {
        double* hd = hlb + p_st * hls;
        bulk_g2s(hd, sx.hl + (hb + sb) * hcl, (uint32_t)run1 * hcl * 8u, bars + p_st);
        if (run1 < ns)
          bulk_g2s(hd + run1 * hcl, sx.hl + hb * hcl, (uint32_t)(ns - run1) * hcl * 8u,
                   bars + p_st);
      }
      if (hcr) {
        double* hd = hrb + p_st * hrs;
        bulk_g2s(hd, sx.hr + (hb + sb) * hcr, (uint32_t)run1 * hcr * 8u, bars + p_st);
        if (run1 < ns)
          bulk_g2s(hd + run1 * hcr, sx.hr + hb * hcr, (uint32_t)(ns - run1) * hcr * 8u,
                   bars + p_st);
      }
    } else {
      mbar_arrive_expect_tx(bars + p_st, (uint32_t)ns * cell * 8u);
    }
    {
    if (DENS)
      bulk_g2s_hint(d, base + (int64_t)sb * cell, (uint32_t)run1 * cell * 8u, bars + p_st,
                    pol_stream);
    else
      bulk_g2s(d, base + (int64_t)sb * cell, (uint32_t)run1 * cell * 8u, bars + p_st);
    if (run1 < ns) {  // wrapped: the rest starts at source cell 0
      if (DENS)
        bulk_g2s_hint(d + run1 * cell, base, (uint32_t)(ns - run1) * cell * 8u, bars + p_st,
                      pol_stream);
      else
        bulk_g2s(d + run1 * cell, base, (uint32_t)(ns - run1) * cell * 8u, bars + p_st);
    }
    }
    if (++p_st == nst) p_st = 0;
    if (++p_k == p_r.nch) {
      p_k = 0;
      if (++p_it < it_end) {
        p_r = item_of(p_it);
        p_s0 = s0_of(p_r);
      }
    }
  };

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
    p_r = item_of(it_begin);
    p_s0 = s0_of(p_r);
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < nst && p_it < it_end; ++s) issue_next();

  const int C1 = n1 / P;
  const bool active = tid < C1;
  double T1[3][P][P];
  double T2[3][P][P];                // !T2S: this item's composed x2 table {AA, AB+BA, BB}
  __shared__ double t2s[3 * P * P];  // T2S: the same table in shared memory
  auto t2c = [&](int s_, int j_, int m_) -> double {
    if constexpr (T2S)
      return lds_keep(t2s + (s_ * P + j_) * P + m_);
    else
      return T2[s_][j_][m_];
  };
#define VPB_T2(s, j, m) t2c(s, j, m)
  bool ex1 = true, ex2 = true;
  int off0 = 0, off1 = 0, off2 = 0;  // element offsets of the three x1 source cells
  int hrs0 = 0, hrs1 = 0, hrs2 = 0;  // HALO: row strides of their regions

  // running x2 partial sums: a1 = output t-2 after the AA and AB+BA terms of
  // source cells t-2, t-1; a2 = output t-1 after the AA term of cell t-1.
  // Each output's fma chain runs in the same order as a one-shot sum over
  // (t-2, t-1, t) -- bitwise the same -- but every x1 result is consumed
  // when it is formed, so no register window shifts between cells.
  // (P <= 2: a1 / a2 are the x1 results of cells t-2 / t-1 instead; measured
  // in the bench loop, the running sums win at P = 3 (config 2: 4.02 -> 3.83
  // ms) and lose at P = 2 (config 3: 0.766 -> 0.788 ms))
  constexpr bool kRunningSums = P >= 3;
  double a1[P][P], a2[P][P];
  bool bad = false;
  int st = 0;
  uint32_t phase = 0;
  double wplane = 0.0, meanacc = 0.0;
  double* mypart = DENS ? dn.rc_part + (int64_t)blockIdx.x * C2 * C1 : nullptr;
  if (DENS && active && !dacc)
    for (int c2 = 0; c2 < C2; ++c2) mypart[c2 * C1 + tid] = 0.0;

  for (int it = it_begin; it < it_end; ++it) {
    const Item r = item_of(it);
    const int l2 = r.l / nv1l;
    const int iv2 = (int)mp.iv2_0 + l2, iv1 = (int)mp.iv1_0 + (r.l - l2 * nv1l);
    if (active) {
      if (DENS) wplane = dn.wv1[iv1] * dn.wv2[iv2];
      ex1 = (al1[iv1] == 0.0);
      ex2 = (al2[iv2] == 0.0);
#pragma unroll
      for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int jj = 0; jj < P; ++jj)
#pragma unroll
          for (int m = 0; m < P; ++m) {
            T1[s][jj][m] = __ldg(k1 + (iv1 * 3 + s) * P * P + jj * P + m);
            if constexpr (!T2S) T2[s][jj][m] = __ldg(k2 + (iv2 * 3 + s) * P * P + jj * P + m);
          }
      if constexpr (HALO) {
        // source cell j = tid - Q - 2 + k lives in the rows (0 <= j < C1) or in a
        // halo region; its row m2 of ring cell sc of slot st starts at
        // hbase_k + ((st G + sc) P + m2) * hrs_k  (branch-free in the loop)
        const int lo = tid - sx.qmul * (int)q1[iv1] - 2;
        auto place = [&](int j, int& base, int& rs) {
          if (j < 0) {
            base = (int)(hlb - inb) + (j + sx.wl) * P;
            rs = sx.wl * P;
          } else if (j >= C1) {
            base = (int)(hrb - inb) + (j - C1) * P;
            rs = sx.wr * P;
          } else {
            base = j * P;
            rs = n1;
          }
        };
        place(lo, off0, hrs0);
        place(lo + 1, off1, hrs1);
        place(lo + 2, off2, hrs2);
      } else {
        const int qq = (int)wrap_mod((int64_t)sx.qmul * q1[iv1], C1);
        int lo = tid - qq - 2;
        while (lo < 0) lo += C1;
        const int mid = lo + 1 == C1 ? 0 : lo + 1;
        const int up = mid + 1 == C1 ? 0 : mid + 1;
        off0 = lo * P;
        off1 = mid * P;
        off2 = up * P;
      }
    }
    if constexpr (T2S) {
      // every thread finished the previous item (barrier after its last chunk)
      for (int e = tid; e < 3 * P * P; e += blockDim.x) t2s[e] = __ldg(k2 + iv2 * 3 * P * P + e);
      __syncthreads();
    }
    double* outp = dst + ((int64_t)iv2 * mp.nv1_glob + iv1) * plane_elems;
    for (int k = 0; k < r.nch; ++k) {
      const int t0 = k * G;
      const int ns = min(G, r.L - t0);
      mbar_wait(bars + st, phase);
      const double* in = inb + st * slot;

      auto run = [&](auto ex1c, auto ex2c) {
        constexpr bool E1 = decltype(ex1c)::value, E2 = decltype(ex2c)::value;
        for (int sc = 0; sc < ns; ++sc) {
          const int t = t0 + sc;
          const double* rows = in + sc * cells;
          double g[P][P];
          // HALO: (st G + sc) P = first row index of this ring cell in every region
          const int hrow0 = HALO ? (st * G + sc) * P : 0;
          auto src_row = [&](const double* row, int m2, int off, int rs) -> const double* {
            if constexpr (HALO)
              return inb + off + (hrow0 + m2) * rs;
            else
              return row + off;
          };
          // composed x1 stencil on this source x2 cell: g[m2][jj]
#pragma unroll
          for (int m2 = 0; m2 < P; ++m2) {
            const double* row = rows + m2 * rl;
            double u2[P];
            load_cell_row<P>(src_row(row, m2, off2, hrs2), u2);
            if constexpr (E1) {
#pragma unroll
              for (int jj = 0; jj < P; ++jj) g[m2][jj] = u2[jj];
            } else {
              double u0[P], u1[P];
              load_cell_row<P>(src_row(row, m2, off0, hrs0), u0);
              load_cell_row<P>(src_row(row, m2, off1, hrs1), u1);
#pragma unroll
              for (int jj = 0; jj < P; ++jj) {
                double acc = T1[0][jj][0] * u0[0];
#pragma unroll
                for (int m = 1; m < P; ++m) acc = fma(T1[0][jj][m], u0[m], acc);
#pragma unroll
                for (int m = 0; m < P; ++m) acc = fma(T1[1][jj][m], u1[m], acc);
#pragma unroll
                for (int m = 0; m < P; ++m) acc = fma(T1[2][jj][m], u2[m], acc);
                g[m2][jj] = acc;
              }
            }
          }
          // output x2 cell t-2 (streaming stores, optional density epilogue)
          auto emit = [&](const double (&o)[P][P]) {
            ExpMax eo;
            const int oc = r.oa + t - 2;
            double* ot = BST ? obuf + ob * slot + (t - t0) * cell + tid * P
                             : outp + (int64_t)oc * cell + tid * P;
#pragma unroll
            for (int j2 = 0; j2 < P; ++j2) {
#pragma unroll
              for (int jj = 0; jj < P; ++jj) eo.add(o[j2][jj]);
              if constexpr (BST) {
#pragma unroll
                for (int jj = 0; jj < P; ++jj) ot[j2 * n1 + jj] = o[j2][jj];
              } else if constexpr (P % 2 == 0) {
#pragma unroll
                for (int jj = 0; jj < P; jj += 2)
                  __stcs(reinterpret_cast<double2*>(ot + j2 * n1 + jj),
                         make_double2(o[j2][jj], o[j2][jj + 1]));
              } else {
#pragma unroll
                for (int jj = 0; jj < P; ++jj) __stcs(ot + j2 * n1 + jj, o[j2][jj]);
              }
            }
            bad |= eo.bad();
            if constexpr (DENS) {
              double rcv, mv = 0.0;
              if constexpr (P % 2 == 1) {
                rcv = o[P / 2][P / 2];  // mid = e_centre exactly (checked on the host)
              } else {
                rcv = 0.0;
#pragma unroll
                for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                  for (int jj = 0; jj < P; ++jj) rcv = fma(dn.mm[j2 * P + jj], o[j2][jj], rcv);
              }
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int jj = 0; jj < P; ++jj) mv = fma(dn.ww[j2 * P + jj], o[j2][jj], mv);
              red_add_hint(mypart + oc * C1 + tid, dmul(wplane, rcv), pol_keep);
              meanacc = fma(wplane, mv, meanacc);
            }
          };
          if constexpr (E2) {
            if (t >= 2) emit(g);
          } else if constexpr (!kRunningSums) {
            // P <= 2: a1 / a2 hold the x1 results of source cells t-2 / t-1
            // (a few register moves per cell; the AA and AB+BA products of an
            // output do not wait for cell t)
            if (t >= 2) {
              double o[P][P];
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2) {
                double acc[P];
                {
                  const double c = VPB_T2(0, j2, 0);
#pragma unroll
                  for (int jj = 0; jj < P; ++jj) acc[jj] = c * a1[0][jj];
                }
#pragma unroll
                for (int m = 1; m < P; ++m) {
                  const double c = VPB_T2(0, j2, m);
#pragma unroll
                  for (int jj = 0; jj < P; ++jj) acc[jj] = fma(c, a1[m][jj], acc[jj]);
                }
#pragma unroll
                for (int m = 0; m < P; ++m) {
                  const double c = VPB_T2(1, j2, m);
#pragma unroll
                  for (int jj = 0; jj < P; ++jj) acc[jj] = fma(c, a2[m][jj], acc[jj]);
                }
#pragma unroll
                for (int m = 0; m < P; ++m) {
                  const double c = VPB_T2(2, j2, m);
#pragma unroll
                  for (int jj = 0; jj < P; ++jj) acc[jj] = fma(c, g[m][jj], acc[jj]);
                }
#pragma unroll
                for (int jj = 0; jj < P; ++jj) o[j2][jj] = acc[jj];
              }
              emit(o);
            }
#pragma unroll
            for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) {
                a1[m2][jj] = a2[m2][jj];
                a2[m2][jj] = g[m2][jj];
              }
          } else {
            // each table coefficient is loaded once and applied to the P x1
            // nodes (same per-output operation order as a jj-outer loop)
            if (t >= 2) {
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int m = 0; m < P; ++m) {
                  const double c = VPB_T2(2, j2, m);
#pragma unroll
                  for (int jj = 0; jj < P; ++jj) a1[j2][jj] = fma(c, g[m][jj], a1[j2][jj]);
                }
              emit(a1);
            }
            if (t >= 1) {
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int m = 0; m < P; ++m) {
                  const double c = VPB_T2(1, j2, m);
#pragma unroll
                  for (int jj = 0; jj < P; ++jj)
                    a1[j2][jj] = fma(c, g[m][jj], m == 0 ? a2[j2][jj] : a1[j2][jj]);
                }
            }
#pragma unroll
            for (int j2 = 0; j2 < P; ++j2) {
              {
                const double c = VPB_T2(0, j2, 0);
#pragma unroll
                for (int jj = 0; jj < P; ++jj) a2[j2][jj] = c * g[0][jj];
              }
#pragma unroll
              for (int m = 1; m < P; ++m) {
                const double c = VPB_T2(0, j2, m);
#pragma unroll
                for (int jj = 0; jj < P; ++jj) a2[j2][jj] = fma(c, g[m][jj], a2[j2][jj]);
              }
            }
          }
        }
      };
      if (active) {
        using F = std::false_type;
        using T = std::true_type;
        if (!ex1 && !ex2) run(F{}, F{});
        else if (!ex1) run(F{}, T{});
        else if (!ex2) run(T{}, F{});
        else run(T{}, T{});
      }
      if constexpr (BST) {
        fence_proxy_async_smem();            // staged outputs -> async proxy
        if (tid == 0) bulk_wait_read<0>();   // chunk k-1's store released the other buffer
      }
      __syncthreads();  // every thread is done with ring slot st
      if constexpr (BST) {
        // outputs of this chunk: source cells t >= 2, i.e. output cells
        // oa + max(t0, 2) - 2 .. oa + t0 + ns - 3
        const int tb = max(t0, 2), nout = t0 + ns - tb;
        if (tid == 0 && nout > 0) {
          const double* sb = obuf + ob * slot + (tb - t0) * cell;
          double* gd = outp + (int64_t)(r.oa + tb - 2) * cell;
          if (DENS)
            bulk_s2g_hint(gd, sb, (uint32_t)nout * cell * 8u, pol_stream);
          else
            bulk_s2g(gd, sb, (uint32_t)nout * cell * 8u);
          bulk_commit();
        }
        ob ^= 1;
      }
      if (tid == 0 && p_it < it_end) issue_next();
      if (++st == nst) {
        st = 0;
        phase ^= 1u;
      }
    }
  }
  if constexpr (BST) {
    if (tid == 0) bulk_wait<0>();  // staged stores complete before the CTA retires
  }
  report_flag(bad, flag);
  if (DENS) {
    __shared__ double red[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) meanacc += __shfl_down_sync(0xffffffffu, meanacc, o);
    if ((tid & 31) == 0) red[tid >> 5] = meanacc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      if (dacc)
        dn.mean_part[blockIdx.x] += s;
      else
        dn.mean_part[blockIdx.x] = s;
    }
  }
}

struct XcLaunch {
  int threads, G, nst;
  bool bst;  // output cells leave through shared memory by bulk copies
  size_t smem;
  int64_t ppb, blocks, max_blocks;
};

// T2S instances only where the 224-register plan strands warp slots: P = 3
// with 3-warp CTAs (65..96 local x1 cells).  VPB_XCOMP_T2S=0/1 overrides.
template <int P>
static bool xcomp_t2s(const int64_t dims[4]) {
  if constexpr (P != 3) {
    return false;
  } else {
    static const int env = getenv("VPB_XCOMP_T2S") ? atoi(getenv("VPB_XCOMP_T2S")) : -1;
    if (env >= 0) return env != 0;
    const int C1 = (int)(dims[0] / P);
    return (C1 + 31) / 32 == 3;
  }
}

template <int P, bool DENS, bool HALO, bool T2S, bool BST>
static void xcomp_occupancy(int threads, size_t smem, int* occ) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dg_xcomp_kernel<P, DENS, HALO, T2S, BST>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, dg_xcomp_kernel<P, DENS, HALO, T2S, BST>,
                                                threads, smem);
}

// Launch an instance: T2S per xcomp_t2s, BST (halo-free passes only) per the plan.
#define VPB_XCOMP_DISPATCH(T2S_, BST_, ...)                                           \
  do {                                                                                \
    if (T2S_) {                                                                       \
      if (BST_) { constexpr bool T2 = (P == 3), BS = !HALO; __VA_ARGS__; }            \
      else { constexpr bool T2 = (P == 3), BS = false; __VA_ARGS__; }                 \
    } else {                                                                          \
      if (BST_) { constexpr bool T2 = false, BS = !HALO; __VA_ARGS__; }               \
      else { constexpr bool T2 = false, BS = false; __VA_ARGS__; }                    \
    }                                                                                 \
  } while (0)

template <int P, bool DENS, bool HALO = false>
static int plan_xcomp(const int64_t dims[4], int64_t nitems, XcLaunch* L, int hcells = 0) {
  const int n1 = (int)dims[0];
  const int C1 = n1 / P;
  const int C2 = (int)(dims[1] / P);
  if (C1 > 128) {
    set_error("x1 lines of %d cells exceed one CTA", C1);
    return VPB_ERR_UNSUPPORTED;
  }
  static const int env_chunk =
      getenv("VPB_XCOMP_CHUNK") ? atoi(getenv("VPB_XCOMP_CHUNK")) : 9216;
  // measured on B200 (scripts/tune_xcomp.py): 3 stages x 2 cells at P = 3
  // (config 2: 91 %, config 5: 80 % of HBM), 6 stages x 4 cells at P = 2
  // (config 3: 91 %); G = 1 costs config 5 12 %
  static const int env_st =
      getenv("VPB_XCOMP_STAGES") ? atoi(getenv("VPB_XCOMP_STAGES")) : (P >= 3 ? 3 : 6);
  static const int env_smem =
      getenv("VPB_XCOMP_SMEM") ? atoi(getenv("VPB_XCOMP_SMEM")) : 56 * 1024;
  L->threads = ((C1 + 31) / 32) * 32;
  L->nst = std::max(2, std::min(8, env_st));
  const size_t cell_bytes = (size_t)P * n1 * 8;
  // hcells: x1 halo cells (left + right) staged with every x2 cell
  auto smem_for = [&](int g) {
    return (size_t)L->nst * g * (cell_bytes + (size_t)hcells * P * P * 8) + L->nst * 8;
  };
  int G = std::max<int>(2, (int)(env_chunk / cell_bytes));
  G = std::min(G, C2);
  while (G > 1 && (int)smem_for(G) > env_smem) --G;
  L->G = G;
  L->smem = smem_for(G);
  if (L->smem > 220 * 1024) {
    set_error("x plane chunk of %d dofs does not fit shared memory", P * n1);
    return VPB_ERR_UNSUPPORTED;
  }
  // BST: two chunks of output cells staged in shared memory (coalesced bulk
  // stores instead of 24-byte-strided lane stores), when they fit the same
  // budget without shrinking the chunk; VPB_XCOMP_BST=0/1 forces it off / on
  static const int env_bst = getenv("VPB_XCOMP_BST") ? atoi(getenv("VPB_XCOMP_BST")) : -1;
  const size_t obytes = 2 * (size_t)G * cell_bytes;
  L->bst = !HALO && env_bst != 0 &&
           (env_bst == 1 ? L->smem + obytes <= 220 * 1024 : L->smem + obytes <= (size_t)env_smem);
  if (L->bst) L->smem += obytes;
  int occ = 0;
  VPB_XCOMP_DISPATCH(xcomp_t2s<P>(dims), L->bst,
                     (xcomp_occupancy<P, DENS, HALO, T2, BS>(L->threads, L->smem, &occ)));
  if (occ < 1) occ = 1;
  L->max_blocks = (int64_t)occ * xplane_sm_count();
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(nitems, L->max_blocks));
  L->ppb = (nitems + grid - 1) / grid;
  L->blocks = (nitems + L->ppb - 1) / L->ppb;
  return VPB_OK;
}

template <int P, bool DENS, bool HALO = false>
static int launch_xcomp(const double* src, double* dst, const int64_t dims[4], int64_t nitems,
                        const XcMap& mp, const double* k1, const int64_t* q1, const double* al1,
                        const double* k2, const int64_t* q2, const double* al2, int32_t* flag,
                        const XDensity& dn, int dacc, cudaStream_t st, int64_t* nblocks_out,
                        const XcStencil& sx = XcStencil{2, nullptr, nullptr, 0, 0}) {
  if (nitems == 0) return VPB_OK;
  XcLaunch L;
  int rc = plan_xcomp<P, DENS, HALO>(dims, nitems, &L, HALO ? sx.wl + sx.wr : 0);
  if (rc) return rc;
  VPB_XCOMP_DISPATCH(xcomp_t2s<P>(dims), L.bst,
                     (dg_xcomp_kernel<P, DENS, HALO, T2, BS>
                      <<<(unsigned)L.blocks, L.threads, L.smem, st>>>(
                          src, dst, (int)dims[0], (int)(dims[1] / P), L.G, L.nst, nitems, L.ppb,
                          mp, k1, q1, al1, k2, q2, al2, flag, dn, dacc, sx)));
  if (nblocks_out) *nblocks_out = L.blocks;
  return launched("dg_xcomp_kernel");
}

inline XcMap xcomp_whole_field(const int64_t dims[4], int P) {
  const int C2 = (int)(dims[1] / P);
  return XcMap{dims[2], 0, 0, dims[2], 1, C2};
}

template <int P, bool HALO = false>
static int xcomp_density_len(const int64_t dims[4], int64_t* len, int hcells = 0) {
  XcLaunch L;
  int rc = plan_xcomp<P, true, HALO>(dims, dims[2] * dims[3], &L, hcells);
  if (rc) return rc;
  const int64_t cc = (dims[0] / P) * (dims[1] / P);
  *len = L.blocks * (cc + 1);
  return VPB_OK;
}

}  // namespace vpb

using namespace vpb;

static int compose_tables(const double* a, const double* b, int64_t n, int32_t order,
                          double* out, int single, void* stream);

extern "C" int vpb_dg_compose_tables(const double* a, const double* b, int64_t n, int32_t order,
                                     double* out, void* stream) {
  return compose_tables(a, b, n, order, out, 0, stream);
}

extern "C" int vpb_dg_single_tables(const double* a, const double* b, int64_t n, int32_t order,
                                    double* out, void* stream) {
  return compose_tables(a, b, n, order, out, 1, stream);
}

static int compose_tables(const double* a, const double* b, int64_t n, int32_t order,
                          double* out, int single, void* stream) {
  VPB_REQUIRE(order >= 1 && order <= kMaxOrder, "order %d outside 1..9", order);
  VPB_REQUIRE(n >= 0, "negative table length");
  if (n == 0) return VPB_OK;
  VPB_REQUIRE(a && b && out, "null pointer");
  const int64_t total = n * order * order;
  compose_tables_kernel<<<(unsigned)((total + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      a, b, n, order, out, single);
  return launched("compose_tables_kernel");
}

extern "C" int vpb_dg_sweep_xcomp(const double* src, double* dst, const int64_t dims[4],
                                  int32_t order, const double* k1, const int64_t* q1,
                                  const double* alpha1, const double* k2, const int64_t* q2,
                                  const double* alpha2, int32_t* flag, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(k1 && q1 && alpha1 && k2 && q2 && alpha2, "null pointer");
  const XDensity none{nullptr, nullptr, nullptr, nullptr, {}, {}};
  VPB_XPLANE_SWITCH(order, rc = launch_xcomp<PP, false>(
                               src, dst, dims, dims[2] * dims[3], xcomp_whole_field(dims, PP), k1,
                               q1, alpha1, k2, q2, alpha2, flag, none, 0, (cudaStream_t)stream,
                               nullptr));
  return rc;
}

extern "C" int64_t vpb_dg_xcomp_density_work_len(const int64_t dims[4], int32_t order) {
  if (order < 1 || order > kMaxOrder || dims[0] % order || dims[1] % order) return -1;
  int64_t len = -1;
  int rc = VPB_OK;
  VPB_XPLANE_SWITCH(order, rc = xcomp_density_len<PP>(dims, &len));
  return rc == VPB_OK ? len : -1;
}

extern "C" int vpb_dg_sweep_xcomp_density(
    const double* src, double* dst, const int64_t dims[4], int32_t order, const double* k1,
    const int64_t* q1, const double* alpha1, const double* k2, const int64_t* q2,
    const double* alpha2, int32_t* flag, const double* wv1, const double* wv2,
    const double* mid_host, const double* wcell1_host, const double* wcell2_host, double volume,
    double* work, double* rc_out, double* stats, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(k1 && q1 && alpha1 && k2 && q2 && alpha2 && rc_out, "null pointer");
  const int64_t cc = (dims[0] / order) * (dims[1] / order);
  const int64_t len = vpb_dg_xcomp_density_work_len(dims, order);
  VPB_REQUIRE(len > 0, "cannot plan the x-plane launch");
  const int64_t nblk = len / (cc + 1);
  XDensity dn;
  rc = xdensity_setup(&dn, order, wv1, wv2, mid_host, wcell1_host, wcell2_host, work, nblk, cc);
  if (rc) return rc;
  int64_t used = 0;
  cudaStream_t st = (cudaStream_t)stream;
  VPB_XPLANE_SWITCH(order, rc = launch_xcomp<PP, true>(
                               src, dst, dims, dims[2] * dims[3], xcomp_whole_field(dims, PP), k1,
                               q1, alpha1, k2, q2, alpha2, flag, dn, 0, st, &used));
  if (rc) return rc;
  VPB_REQUIRE(used == nblk, "x-plane launch plan changed (%lld vs %lld CTAs)", (long long)used,
              (long long)nblk);
  return launch_xdens_reduce(work, nblk, cc, volume, rc_out, stats, st);
}

// ---------------------------------------------------------------------------
// Three-cell x-plane stencil on an x1-sharded field (dist.py ShardedSolver):
// qmul = 2 with composed tables is the merged pair of x half steps, qmul = 1
// with {0, A, B} tables (vpb_dg_single_tables) one x half step; x1 source
// cells outside the shard come from the halo buffers (vpb_halo_pack layout).
// ---------------------------------------------------------------------------
static int xstencil_args(const double* src, const double* dst, const int64_t dims[4],
                         int32_t order, int32_t qmul, const double* hl, int32_t wl,
                         const double* hr, int32_t wr) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(qmul == 1 || qmul == 2, "qmul must be 1 or 2");
  VPB_REQUIRE(wl >= 0 && wr >= 0 && (wl == 0 || hl) && (wr == 0 || hr), "bad halo");
  VPB_REQUIRE((order * order * wl) % 2 == 0 && (order * order * wr) % 2 == 0,
              "halo cells of %d x %d dofs per x2 cell must be 16-byte multiples (even widths "
              "for odd orders)", order, order);
  VPB_REQUIRE((reinterpret_cast<uintptr_t>(hl) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(hr) & 15) == 0,
              "halo buffers must be 16-byte aligned");
  VPB_REQUIRE(wl <= dims[0] / order && wr <= dims[0] / order, "halo wider than the shard");
  return VPB_OK;
}

extern "C" int vpb_dg_sweep_xstencil(const double* src, double* dst, const int64_t dims[4],
                                     int32_t order, const double* k1, const int64_t* q1,
                                     const double* alpha1, const double* k2, const int64_t* q2,
                                     const double* alpha2, int32_t qmul, const double* hl,
                                     int32_t wl, const double* hr, int32_t wr, int32_t* flag,
                                     void* stream) {
  int rc = xstencil_args(src, dst, dims, order, qmul, hl, wl, hr, wr);
  if (rc) return rc;
  const XDensity none{nullptr, nullptr, nullptr, nullptr, {}, {}};
  const XcStencil sx{qmul, hl, hr, wl, wr};
  VPB_XPLANE_SWITCH(order, rc = launch_xcomp<PP, false, true>(
                               src, dst, dims, dims[2] * dims[3], xcomp_whole_field(dims, PP), k1,
                               q1, alpha1, k2, q2, alpha2, flag, none, 0, (cudaStream_t)stream,
                               nullptr, sx));
  return rc;
}

extern "C" int64_t vpb_dg_xstencil_density_work_len(const int64_t dims[4], int32_t order,
                                                    int32_t wl, int32_t wr) {
  if (order < 1 || order > kMaxOrder || dims[0] % order || dims[1] % order) return -1;
  int64_t len = -1;
  int rc = VPB_OK;
  VPB_XPLANE_SWITCH(order, rc = (xcomp_density_len<PP, true>(dims, &len, wl + wr)));
  return rc == VPB_OK ? len : -1;
}

extern "C" int vpb_dg_sweep_xstencil_density(
    const double* src, double* dst, const int64_t dims[4], int32_t order, const double* k1,
    const int64_t* q1, const double* alpha1, const double* k2, const int64_t* q2,
    const double* alpha2, int32_t qmul, const double* hl, int32_t wl, const double* hr,
    int32_t wr, int32_t* flag, const double* wv1, const double* wv2, const double* mid_host,
    const double* wcell1_host, const double* wcell2_host, double volume, double* work,
    double* rc_out, double* stats, void* stream) {
  int rc = xstencil_args(src, dst, dims, order, qmul, hl, wl, hr, wr);
  if (rc) return rc;
  VPB_REQUIRE(rc_out != nullptr, "null pointer");
  const int64_t cc = (dims[0] / order) * (dims[1] / order);
  const int64_t len = vpb_dg_xstencil_density_work_len(dims, order, wl, wr);
  VPB_REQUIRE(len > 0, "cannot plan the x-plane launch");
  const int64_t nblk = len / (cc + 1);
  XDensity dn;
  rc = xdensity_setup(&dn, order, wv1, wv2, mid_host, wcell1_host, wcell2_host, work, nblk, cc);
  if (rc) return rc;
  int64_t used = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const XcStencil sx{qmul, hl, hr, wl, wr};
  VPB_XPLANE_SWITCH(order, rc = (launch_xcomp<PP, true, true>(
                               src, dst, dims, dims[2] * dims[3], xcomp_whole_field(dims, PP), k1,
                               q1, alpha1, k2, q2, alpha2, flag, dn, 0, st, &used, sx)));
  if (rc) return rc;
  VPB_REQUIRE(used == nblk, "x-plane launch plan changed (%lld vs %lld CTAs)", (long long)used,
              (long long)nblk);
  return launch_xdens_reduce(work, nblk, cc, volume, rc_out, stats, st);
}

// The merged x pass (composed stencils, density epilogue) on v2 rows
// [v2_0, v2_0 + v2_rows) of an unsharded-in-x field (a velocity shard,
// dist.VShardedSolver): the rows of one call are contiguous in src / dst;
// k2 / q2 / alpha2 are indexed by the field's v2 row.  The CTA slabs of the
// work buffer accumulate over the calls of one pass: phase bit 1 (first
// call) zeroes them, bit 2 (last call) reduces them to rc_out / stats --
// one reduction for the boundary-first blocks of the velocity-sharded step.
extern "C" int vpb_dg_sweep_xcomp_rows(
    const double* src, double* dst, const int64_t dims[4], int32_t order, int64_t v2_0,
    int64_t v2_rows, const double* k1, const int64_t* q1, const double* alpha1, const double* k2,
    const int64_t* q2, const double* alpha2, int32_t* flag, const double* wv1, const double* wv2,
    const double* mid_host, const double* wcell1_host, const double* wcell2_host, double volume,
    double* work, double* rc_out, double* stats, int32_t phase, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(k1 && q1 && alpha1 && k2 && q2 && alpha2 && rc_out && stats, "null pointer");
  VPB_REQUIRE(v2_0 >= 0 && v2_rows >= 0 && v2_0 + v2_rows <= dims[3], "v2 rows outside the field");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t plane = dims[0] * dims[1];
  const int64_t C2 = dims[1] / order;
  const int64_t cc = (dims[0] / order) * C2;
  const int64_t len = vpb_dg_xcomp_density_work_len(dims, order);
  VPB_REQUIRE(len > 0, "cannot plan the composed x pass");
  const int64_t nblk = len / (cc + 1);
  XDensity dn;
  rc = xdensity_setup(&dn, order, wv1, wv2, mid_host, wcell1_host, wcell2_host, work, nblk, cc);
  if (rc) return rc;
  if (phase & 1) {
    if (cudaMemsetAsync(work, 0, (size_t)len * sizeof(double), st) != cudaSuccess)
      return check_launch("cudaMemsetAsync");
  }
  const int64_t nitems = v2_rows * dims[2];
  if (nitems) {
    const XcMap mp{dims[2], 0, v2_0, dims[2], 1, (int)C2};
    int64_t used = 0;
    VPB_XPLANE_SWITCH(order, rc = (launch_xcomp<PP, true, false>(
                                 src + v2_0 * dims[2] * plane, dst, dims, nitems, mp, k1, q1,
                                 alpha1, k2, q2, alpha2, flag, dn, 1, st, &used)));
    if (rc) return rc;
    VPB_REQUIRE(used <= nblk, "x-plane launch plan exceeds the work buffer (%lld > %lld CTAs)",
                (long long)used, (long long)nblk);
  }
  if (phase & 2) return launch_xdens_reduce(work, nblk, cc, volume, rc_out, stats, st);
  return VPB_OK;
}

// The stencil pass on an x1 x x2 sharded field: x1 halos as above and x2
// halos (x2l / x2r, three parts each, see XcStencil) of wl2 / wr2 cells; the
// plane is not periodic in x2.  wv1 == nullptr: no density epilogue.
extern "C" int vpb_dg_sweep_xstencil2(
    const double* src, double* dst, const int64_t dims[4], int32_t order, const double* k1,
    const int64_t* q1, const double* alpha1, const double* k2, const int64_t* q2,
    const double* alpha2, int32_t qmul, const double* hl, int32_t wl, const double* hr,
    int32_t wr, int32_t wl2, const double* const x2l[3], int32_t wr2,
    const double* const x2r[3], int32_t* flag, const double* wv1, const double* wv2,
    const double* mid_host, const double* wcell1_host, const double* wcell2_host, double volume,
    double* work, double* rc_out, double* stats, void* stream) {
  int rc = xstencil_args(src, dst, dims, order, qmul, hl, wl, hr, wr);
  if (rc) return rc;
  VPB_REQUIRE(k1 && q1 && alpha1 && k2 && q2 && alpha2, "null pointer");
  VPB_REQUIRE(wl2 >= 0 && wr2 >= 0 && wl2 <= dims[1] / order && wr2 <= dims[1] / order,
              "x2 halo wider than the shard");
  XcStencil sx{qmul, hl, hr, wl, wr};
  sx.x2 = 1;
  sx.wl2 = wl2;
  sx.wr2 = wr2;
  for (int k = 0; k < 3; ++k) {
    sx.x2l[k] = wl2 ? x2l[k] : nullptr;
    sx.x2r[k] = wr2 ? x2r[k] : nullptr;
    const bool need_l = wl2 && (k == 0 || (k == 1 ? wl : wr));
    const bool need_r = wr2 && (k == 0 || (k == 1 ? wl : wr));
    VPB_REQUIRE(!need_l || (x2l[k] && (reinterpret_cast<uintptr_t>(x2l[k]) & 15) == 0),
                "x2 left halo part %d missing or not 16-byte aligned", k);
    VPB_REQUIRE(!need_r || (x2r[k] && (reinterpret_cast<uintptr_t>(x2r[k]) & 15) == 0),
                "x2 right halo part %d missing or not 16-byte aligned", k);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (wv1 == nullptr) {
    const XDensity none{nullptr, nullptr, nullptr, nullptr, {}, {}};
    VPB_XPLANE_SWITCH(order, rc = (launch_xcomp<PP, false, true>(
                                 src, dst, dims, dims[2] * dims[3], xcomp_whole_field(dims, PP),
                                 k1, q1, alpha1, k2, q2, alpha2, flag, none, 0, st, nullptr, sx)));
    return rc;
  }
  VPB_REQUIRE(rc_out != nullptr && stats != nullptr, "null pointer");
  const int64_t cc = (dims[0] / order) * (dims[1] / order);
  const int64_t len = vpb_dg_xstencil_density_work_len(dims, order, wl, wr);
  VPB_REQUIRE(len > 0, "cannot plan the x-plane launch");
  const int64_t nblk = len / (cc + 1);
  XDensity dn;
  rc = xdensity_setup(&dn, order, wv1, wv2, mid_host, wcell1_host, wcell2_host, work, nblk, cc);
  if (rc) return rc;
  int64_t used = 0;
  VPB_XPLANE_SWITCH(order, rc = (launch_xcomp<PP, true, true>(
                               src, dst, dims, dims[2] * dims[3], xcomp_whole_field(dims, PP), k1,
                               q1, alpha1, k2, q2, alpha2, flag, dn, 0, st, &used, sx)));
  if (rc) return rc;
  VPB_REQUIRE(used == nblk, "x-plane launch plan changed (%lld vs %lld CTAs)", (long long)used,
              (long long)nblk);
  return launch_xdens_reduce(work, nblk, cc, volume, rc_out, stats, st);
}

// The halo stencil pass on v2 rows [v2_0, v2_0 + v2_rows) of the shard only
// (the sharded advance pipelines the x1 halo exchange of the next block of
// rows against this block's pass).  src / dst / hl / hr are the whole-shard
// buffers; the rows of one call are contiguous in each.  With the density
// epilogue (wv1 != nullptr) the CTA slabs accumulate over the calls of one
// pass: phase bit 1 (first call) zeroes the work buffer, bit 2 (last call)
// reduces it to rc_out / stats.  The launch plan of a block of rows uses at
// most the whole-shard CTA count (the work buffer's slab count), so every
// block adds into the same fixed slabs in program order: deterministic for a
// fixed blocking (and equal to the one-call pass up to summation order).
extern "C" int vpb_dg_sweep_xstencil_rows(
    const double* src, double* dst, const int64_t dims[4], int32_t order, int64_t v2_0,
    int64_t v2_rows, const double* k1, const int64_t* q1, const double* alpha1, const double* k2,
    const int64_t* q2, const double* alpha2, int32_t qmul, const double* hl, int32_t wl,
    const double* hr, int32_t wr, int32_t* flag, const double* wv1, const double* wv2,
    const double* mid_host, const double* wcell1_host, const double* wcell2_host, double volume,
    double* work, double* rc_out, double* stats, int32_t phase, void* stream) {
  int rc = xstencil_args(src, dst, dims, order, qmul, hl, wl, hr, wr);
  if (rc) return rc;
  VPB_REQUIRE(v2_0 >= 0 && v2_rows >= 0 && v2_0 + v2_rows <= dims[3], "v2 rows outside the shard");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t plane = dims[0] * dims[1];
  const int64_t row0 = v2_0 * dims[2];  // first (v1, v2) plane of the block
  const int64_t C2 = dims[1] / order;
  const double* s = src + row0 * plane;
  const double* h_l = wl ? hl + row0 * C2 * order * wl * order : nullptr;
  const double* h_r = wr ? hr + row0 * C2 * order * wr * order : nullptr;
  const XcMap mp{dims[2], 0, v2_0, dims[2], 1, (int)C2};
  const XcStencil sx{qmul, h_l, h_r, wl, wr};
  const int64_t nitems = v2_rows * dims[2];
  if (wv1 == nullptr) {
    if (nitems == 0) return VPB_OK;
    const XDensity none{nullptr, nullptr, nullptr, nullptr, {}, {}};
    VPB_XPLANE_SWITCH(order, rc = launch_xcomp<PP, false, true>(
                                 s, dst, dims, nitems, mp, k1, q1, alpha1, k2, q2, alpha2, flag,
                                 none, 0, st, nullptr, sx));
    return rc;
  }
  VPB_REQUIRE(rc_out != nullptr && stats != nullptr, "null pointer");
  const int64_t cc = (dims[0] / order) * C2;
  const int64_t len = vpb_dg_xstencil_density_work_len(dims, order, wl, wr);
  VPB_REQUIRE(len > 0, "cannot plan the x-plane launch");
  const int64_t nblk = len / (cc + 1);
  XDensity dn;
  rc = xdensity_setup(&dn, order, wv1, wv2, mid_host, wcell1_host, wcell2_host, work, nblk, cc);
  if (rc) return rc;
  if (phase & 1) {
    if (cudaMemsetAsync(work, 0, (size_t)len * sizeof(double), st) != cudaSuccess)
      return check_launch("cudaMemsetAsync");
  }
  if (nitems) {
    int64_t used = 0;
    VPB_XPLANE_SWITCH(order, rc = (launch_xcomp<PP, true, true>(
                                 s, dst, dims, nitems, mp, k1, q1, alpha1, k2, q2, alpha2, flag,
                                 dn, 1, st, &used, sx)));
    if (rc) return rc;
    VPB_REQUIRE(used <= nblk, "x-plane launch plan exceeds the work buffer (%lld > %lld CTAs)",
                (long long)used, (long long)nblk);
  }
  if (phase & 2) return launch_xdens_reduce(work, nblk, cc, volume, rc_out, stats, st);
  return VPB_OK;
}
