// Two consecutive Strang x half steps in one HBM pass.
//
// A run of K Strang steps (driver.py:245-265, run() at driver.py:371-377)
// applies the closing x half step of step m and the opening x half step of
// step m+1 back to back: x1(τ/2) x2(τ/2) x1(τ/2) x2(τ/2), with nothing in
// between.  Both half steps use the same tables, so inside one (iv2, iv1)
// plane this pass chains the four sweeps while the plane streams through
// shared memory, writing only the result of the second half step.  Every
// element goes through exactly the operations of the four separate sweeps
// (same order, no contraction): the output is bitwise the unfused sequence.
// (This is not the P∘T_τ merge SURVEY.md §8f rules out: both projections are
// kept.)
//
// Per plane the pass runs two x2-streaming stages one chunk apart:
//
//   stage 1 (as fused.cu): source chunks from an mbarrier ring (1-D bulk
//     copies); thread c = x1 cell c sweeps the P rows of a source x2 cell
//     along x1, then applies the x2 pair -> first-half output cells h, in
//     the order h0, h0+1, ... with h0 = (-q2-1) mod C2 (the order stage 2
//     consumes them in), written to a shared-memory row buffer;
//   stage 2: the same two sweeps on the first-half cells of the previous
//     chunk (read from that buffer; the x1 stencil needs the neighbours'
//     values) -> output cells 0, 1, ..., C2-1 in order, staged and written
//     with one bulk store per chunk.  First-half cell h0 is needed again at
//     the end of the plane; a copy is kept.
//
// One __syncthreads per chunk separates the stages (double-buffered row
// buffer), plus one drain iteration per plane for the last chunk and h0.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "async_copy.cuh"
#include "common.cuh"
#include "xplane.cuh"

// VPB_X2_DIRECT (default): second-half outputs go straight to HBM with
// streaming stores (each warp row is one contiguous 32*P*8-byte span; L2
// merges the partial sectors) instead of a shared-memory staging tile + bulk
// store, which frees the staging smem for a deeper load ring: 4% faster at
// config 2, 14% at config 3 (profiles/r01_ncu_summary.md).
#ifndef VPB_X2_DIRECT
#define VPB_X2_DIRECT 1
#endif

namespace vpb {

// (st.global.cs already marks the line evict-first; an explicit L2 policy
// operand measured 1.5 % slower here)
template <bool HINT>
__device__ __forceinline__ void st_out(double* p, double v, uint64_t) {
#if VPB_X2_DIRECT
  __stcs(p, v);
#else
  *p = v;
#endif
}

template <int P, bool DENS>
__global__ void __launch_bounds__(128)
    dg_xplane2_kernel(const double* __restrict__ src, double* __restrict__ dst, int n1, int C2,
                      int G, int nst, int64_t nv1, int64_t nplanes, int64_t planes_per_block,
                      const double* __restrict__ a1, const double* __restrict__ b1,
                      const int64_t* __restrict__ q1, const double* __restrict__ al1,
                      const double* __restrict__ a2, const double* __restrict__ b2,
                      const int64_t* __restrict__ q2, const double* __restrict__ al2,
                      int32_t* __restrict__ f1a, int32_t* __restrict__ f2a,
                      int32_t* __restrict__ f1b, int32_t* __restrict__ f2b, const XDensity dn) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int cell = P * n1;    // one x2 cell: P rows of n1 dofs
  const int slot = G * cell;  // ring slot / row-buffer half
  double* inb = reinterpret_cast<double*>(smem_raw);  // [nst][slot] source ring
  double* hb = inb + nst * slot;                      // [2][slot] first-half cells
  double* h0b = hb + 2 * slot;                        // [cell] first-half cell h0
  double* outb = h0b + cell;                          // [2][(G+1)*cell] output staging
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(outb + (VPB_X2_DIRECT ? 0 : 2 * (G + 1) * cell));

  const int tid = threadIdx.x;
  const int64_t pl_begin = blockIdx.x * planes_per_block;
  const int64_t pl_end = min(nplanes, pl_begin + planes_per_block);
  if (pl_begin >= pl_end) return;
  const int per_plane = 1 + (C2 + G - 1) / G;  // ring chunks per plane (prologue + outputs)
  const int iters_plane = per_plane + 1;       // + the drain iteration
  const int64_t nloads = (pl_end - pl_begin) * per_plane;
  const int64_t niters = (pl_end - pl_begin) * iters_plane;
  const int64_t plane_elems = (int64_t)C2 * cell;

  // L2 policies: f streams through (evict first); the density slabs stay
  const uint64_t pol_stream = l2_evict_first();
  const uint64_t pol_keep = l2_evict_last();
  // producer (thread 0): stage 1 needs source cell -2(q2+1) mod C2 first
  XCursor prod;
  prod.lead = 2;
  prod.start(pl_begin, C2, q2, nv1);
  int64_t prod_j = 0;
  int prod_st = 0;
  auto issue_next = [&]() {
    const XChunk c = prod.chunk(G, C2);
    const double* base = src + prod.plane * plane_elems;
    double* dstp = inb + prod_st * slot;
    mbar_arrive_expect_tx(bars + prod_st, (uint32_t)c.nsrc * cell * 8u);
    const int run1 = min(c.nsrc, C2 - c.s_begin);
    // with a density epilogue, keep its slabs in L2: f streams evict-first
    if (DENS)
      bulk_g2s_hint(dstp, base + (int64_t)c.s_begin * cell, (uint32_t)run1 * cell * 8u,
                    bars + prod_st, pol_stream);
    else
      bulk_g2s(dstp, base + (int64_t)c.s_begin * cell, (uint32_t)run1 * cell * 8u, bars + prod_st);
    if (run1 < c.nsrc)
      if (DENS)
        bulk_g2s_hint(dstp + run1 * cell, base, (uint32_t)(c.nsrc - run1) * cell * 8u,
                      bars + prod_st, pol_stream);
      else
        bulk_g2s(dstp + run1 * cell, base, (uint32_t)(c.nsrc - run1) * cell * 8u,
                 bars + prod_st);
    ++prod_j;
    if (++prod_st == nst) prod_st = 0;
    prod.advance(per_plane, C2, q2, nv1, pl_end);
  };

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    while (prod_j < nst && prod_j < nloads) issue_next();

  const int C1 = n1 / P;
  const bool active = tid < C1;
  double A1[P][P], B1[P][P], A2[P][P], B2[P][P];
  bool ex1 = true, ex2 = true;
  int lo_off = 0, up_off = 0;
  double gp[P][P];  // stage 1: x1 result of the previous source cell
  double gq[P][P];  // stage 2: x1 result of the previous first-half cell
  bool bad1a = false, bad2a = false, bad1b = false, bad2b = false;
  XCursor cur;
  cur.lead = 2;
  cur.start(pl_begin, C2, q2, nv1);
  int st = 0;
  uint32_t phase = 0;
  int ipl = 0;  // iteration inside the plane: 0..per_plane-1 chunks, per_plane = drain
  int64_t plane = pl_begin;
  int nout_prev = 0;  // first-half cells produced by the previous iteration
  int o_next = 0;     // next output cell of the plane
  double wplane = 0.0, meanacc = 0.0;
  double* mypart = DENS ? dn.rc_part + (int64_t)blockIdx.x * C2 * C1 : nullptr;
  if (DENS && active)
    for (int c2 = 0; c2 < C2; ++c2) mypart[c2 * C1 + tid] = 0.0;

  for (int64_t it = 0; it < niters; ++it) {
    const bool drain = ipl == per_plane;
    if (ipl == 0) {
      o_next = 0;
      nout_prev = 0;
      if (active) {
        const int64_t iv2 = plane / nv1, iv1 = plane - iv2 * nv1;
        if (DENS) wplane = dn.wv1[iv1] * dn.wv2[iv2];
        ex1 = (al1[iv1] == 0.0);
        ex2 = (al2[iv2] == 0.0);
#pragma unroll
        for (int jj = 0; jj < P; ++jj)
#pragma unroll
          for (int m = 0; m < P; ++m) {
            A1[jj][m] = __ldg(a1 + iv1 * P * P + jj * P + m);
            B1[jj][m] = __ldg(b1 + iv1 * P * P + jj * P + m);
            A2[jj][m] = __ldg(a2 + iv2 * P * P + jj * P + m);
            B2[jj][m] = __ldg(b2 + iv2 * P * P + jj * P + m);
          }
        const int qm1 = (int)wrap_mod(q1[iv1], C1);
        int lo = tid - qm1 - 1;
        if (lo < 0) lo += C1;
        const int up = lo + 1 == C1 ? 0 : lo + 1;
        lo_off = lo * P;
        up_off = up * P;
      }
    }
    const XChunk c = drain ? XChunk{0, 0, 0, 0} : cur.chunk(G, C2);
    const int o_begin = o_next;
#if VPB_X2_DIRECT
    double* out = dst + plane * plane_elems + (int64_t)o_begin * cell;
#else
    double* out = outb + (it & 1) * ((G + 1) * cell);
#endif

    // Both stages for one (ex1, ex2) combination (uniform over the plane).
    auto run = [&](auto ex1c, auto ex2c) {
      constexpr bool E1 = decltype(ex1c)::value, E2 = decltype(ex2c)::value;
      // second half step on the previous chunk's first-half cells
      auto second = [&](const double* hrow) {
        double g[P][P];
        xplane_x1_cell<P, E1>(hrow, n1, lo_off, up_off, A1, B1, g);
        if (o_next < 0) {  // first-half cell h0: prologue of stage 2
          o_next = 0;
        } else {
          double o[P][P];
          xplane_x2_cell<P, E2>(A2, B2, gq, g, o);
          ExpMax eo;
#pragma unroll
          for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
            for (int jj = 0; jj < P; ++jj) eo.add(o[j2][jj]);
          if (eo.bad()) {
            bad2b = true;
            ExpMax eg;
#pragma unroll
            for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) eg.add(g[m2][jj]);
            bad1b |= eg.bad();
          }
          double* ot = out + (o_next - o_begin) * cell + tid * P;
#pragma unroll
          for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
            for (int jj = 0; jj < P; ++jj) st_out<DENS>(ot + j2 * n1 + jj, o[j2][jj], pol_stream);
          if constexpr (DENS) {
            double rcv, mv = 0.0;
            if constexpr (P % 2 == 1) {
              rcv = o[P / 2][P / 2];
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
            red_add_hint(mypart + o_next * C1 + tid, dmul(wplane, rcv), pol_keep);
            meanacc = fma(wplane, mv, meanacc);
          }
          ++o_next;
        }
#pragma unroll
        for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
          for (int jj = 0; jj < P; ++jj) gq[m2][jj] = g[m2][jj];
      };
      // Steady state (all but the first three chunks and the drain of a
      // plane): both stages on one cell each per step, in one basic block so
      // the scheduler interleaves their independent dependency chains.
      if (ipl >= 3 && !drain && nout_prev == c.nsrc && c.nout == c.nsrc) {
        mbar_wait(bars + st, phase);
        const double* in = inb + st * slot;
        const double* hprev = hb + ((ipl - 1) & 1) * slot;
        double* hcur = hb + (ipl & 1) * slot;
        for (int sc = 0; sc < c.nsrc; ++sc) {
          double g2[P][P], g1[P][P], o2[P][P], o1[P][P];
          xplane_x1_cell<P, E1>(hprev + sc * cell, n1, lo_off, up_off, A1, B1, g2);
          xplane_x1_cell<P, E1>(in + sc * cell, n1, lo_off, up_off, A1, B1, g1);
          xplane_x2_cell<P, E2>(A2, B2, gq, g2, o2);
          xplane_x2_cell<P, E2>(A2, B2, gp, g1, o1);
          ExpMax e2, e1;
          double* ot = out + (o_next - o_begin) * cell + tid * P;
          double* ht = hcur + sc * cell + tid * P;
#pragma unroll
          for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
            for (int jj = 0; jj < P; ++jj) {
              e2.add(o2[j2][jj]);
              e1.add(o1[j2][jj]);
              st_out<DENS>(ot + j2 * n1 + jj, o2[j2][jj], pol_stream);
              ht[j2 * n1 + jj] = o1[j2][jj];
            }
          if constexpr (DENS) {
            double rcv, mv = 0.0;
            if constexpr (P % 2 == 1) {
              rcv = o2[P / 2][P / 2];
            } else {
              rcv = 0.0;
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int jj = 0; jj < P; ++jj) rcv = fma(dn.mm[j2 * P + jj], o2[j2][jj], rcv);
            }
#pragma unroll
            for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) mv = fma(dn.ww[j2 * P + jj], o2[j2][jj], mv);
            red_add_hint(mypart + o_next * C1 + tid, dmul(wplane, rcv), pol_keep);
            meanacc = fma(wplane, mv, meanacc);
          }
          if (e2.bad()) {
            bad2b = true;
            ExpMax eg;
#pragma unroll
            for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) eg.add(g2[m2][jj]);
            bad1b |= eg.bad();
          }
          if (e1.bad()) {
            bad2a = true;
            ExpMax eg;
#pragma unroll
            for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) eg.add(g1[m2][jj]);
            bad1a |= eg.bad();
          }
          ++o_next;
#pragma unroll
          for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
            for (int jj = 0; jj < P; ++jj) {
              gq[m2][jj] = g2[m2][jj];
              gp[m2][jj] = g1[m2][jj];
            }
        }
        return;
      }
      if (ipl >= 2) {
        if (ipl == 2) o_next = -1;  // the first cell of chunk 1 is h0 (stage-2 prologue)
        const double* hprev = hb + ((ipl - 1) & 1) * slot;
        for (int sc = 0; sc < nout_prev; ++sc) second(hprev + sc * cell);
        if (drain) second(h0b);
      }
      if (!drain) {
        mbar_wait(bars + st, phase);
        const double* in = inb + st * slot;
        double* hcur = hb + (ipl & 1) * slot;
        for (int sc = 0; sc < c.nsrc; ++sc) {
          double g[P][P];
          xplane_x1_cell<P, E1>(in + sc * cell, n1, lo_off, up_off, A1, B1, g);
          if (c.nout > 0) {
            double o[P][P];
            xplane_x2_cell<P, E2>(A2, B2, gp, g, o);
            ExpMax eo;
#pragma unroll
            for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) eo.add(o[j2][jj]);
            if (eo.bad()) {
              bad2a = true;
              ExpMax eg;
#pragma unroll
              for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
                for (int jj = 0; jj < P; ++jj) eg.add(g[m2][jj]);
              bad1a |= eg.bad();
            }
            double* ht = hcur + sc * cell + tid * P;
            double* h0t = h0b + tid * P;
            const bool keep = ipl == 1 && sc == 0;
#pragma unroll
            for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) {
                ht[j2 * n1 + jj] = o[j2][jj];
                if (keep) h0t[j2 * n1 + jj] = o[j2][jj];
              }
          }
#pragma unroll
          for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
            for (int jj = 0; jj < P; ++jj) gp[m2][jj] = g[m2][jj];
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
#if VPB_X2_DIRECT
    __syncthreads();
    if (tid == 0 && !drain && prod_j < nloads) issue_next();
#else
    fence_proxy_async_smem();
    if (tid == 0) bulk_wait_read<0>();  // the store issued last iteration left the other tile
    __syncthreads();
    if (tid == 0) {
      if (o_next > o_begin) {
        bulk_s2g(dst + plane * plane_elems + (int64_t)o_begin * cell, out,
                 (uint32_t)(o_next - o_begin) * cell * 8u);
        bulk_commit();
      }
      if (!drain && prod_j < nloads) issue_next();
    }
#endif
    if (!drain) {
      nout_prev = c.nout;
      cur.advance(per_plane, C2, q2, nv1, pl_end);
      if (++st == nst) {
        st = 0;
        phase ^= 1u;
      }
    }
    if (++ipl == iters_plane) {
      ipl = 0;
      ++plane;
    }
  }
  if (tid == 0) bulk_wait<0>();
  report_flag(bad1a, f1a);
  report_flag(bad2a, f2a);
  report_flag(bad1b, f1b);
  report_flag(bad2b, f2b);
  if (DENS) {
    __shared__ double red[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) meanacc += __shfl_down_sync(0xffffffffu, meanacc, o);
    if ((tid & 31) == 0) red[tid >> 5] = meanacc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      dn.mean_part[blockIdx.x] = s;
    }
  }
}

struct X2Launch {
  int threads, G, nst;
  size_t smem;
  int64_t ppb, blocks;
};

template <int P, bool DENS>
static int plan_xplane2(const int64_t dims[4], X2Launch* L) {
  const int n1 = (int)dims[0];
  const int C1 = n1 / P;
  const int C2 = (int)(dims[1] / P);
  const int64_t nplanes = dims[2] * dims[3];
  if (C1 > 128) {
    set_error("x1 lines of %d cells exceed one CTA", C1);
    return VPB_ERR_UNSUPPORTED;
  }
  static const int env_chunk =
      getenv("VPB_XPLANE2_CHUNK") ? atoi(getenv("VPB_XPLANE2_CHUNK")) : (VPB_X2_DIRECT ? 9216 : 4608);
  // measured best ring depths (A/B on B200): 4 x 2 cells at P = 3 (config 2),
  // 2 x 4 cells at P = 2 (config 3)
  static const int env_st =
      getenv("VPB_XPLANE2_STAGES") ? atoi(getenv("VPB_XPLANE2_STAGES")) : (P >= 3 ? 4 : 2);
  static const int env_smem =
      getenv("VPB_XPLANE2_SMEM") ? atoi(getenv("VPB_XPLANE2_SMEM")) : 56 * 1024;
  L->threads = ((C1 + 31) / 32) * 32;
  L->nst = std::max(2, std::min(8, env_st));
  const size_t cell_bytes = (size_t)P * n1 * 8;
  auto smem_for = [&](int g) {
    return (size_t)(L->nst + 2) * g * cell_bytes + cell_bytes +
           (VPB_X2_DIRECT ? 0 : 2 * (size_t)(g + 1) * cell_bytes) + L->nst * 8;
  };
  int G = std::max<int>(1, (int)(env_chunk / cell_bytes));
  G = std::min(G, C2);
  while (G > 1 && (int)smem_for(G) > env_smem) --G;
  L->G = G;
  L->smem = smem_for(G);
  if (L->smem > 220 * 1024) {
    set_error("x plane chunk of %d dofs does not fit shared memory", P * n1);
    return VPB_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dg_xplane2_kernel<P, DENS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dg_xplane2_kernel<P, DENS>, L->threads,
                                                L->smem);
  if (occ < 1) occ = 1;
  const int64_t grid =
      std::max<int64_t>(1, std::min<int64_t>(nplanes, (int64_t)occ * xplane_sm_count()));
  L->ppb = (nplanes + grid - 1) / grid;
  L->blocks = (nplanes + L->ppb - 1) / L->ppb;
  return VPB_OK;
}

template <int P, bool DENS>
static int launch_xplane2(const double* src, double* dst, const int64_t dims[4],
                          const double* a1, const double* b1, const int64_t* q1,
                          const double* al1, const double* a2, const double* b2,
                          const int64_t* q2, const double* al2, int32_t* const flags[4],
                          const XDensity& dn, cudaStream_t st, int64_t* nblocks_out) {
  const int64_t nplanes = dims[2] * dims[3];
  if (nplanes == 0) return VPB_OK;
  X2Launch L;
  int rc = plan_xplane2<P, DENS>(dims, &L);
  if (rc) return rc;
  dg_xplane2_kernel<P, DENS><<<(unsigned)L.blocks, L.threads, L.smem, st>>>(
      src, dst, (int)dims[0], (int)(dims[1] / P), L.G, L.nst, dims[2], nplanes, L.ppb, a1, b1,
      q1, al1, a2, b2, q2, al2, flags[0], flags[1], flags[2], flags[3], dn);
  if (nblocks_out) *nblocks_out = L.blocks;
  return launched("dg_xplane2_kernel");
}

template <int P>
static int xplane2_density_len(const int64_t dims[4], int64_t* len) {
  X2Launch L;
  int rc = plan_xplane2<P, true>(dims, &L);
  if (rc) return rc;
  const int64_t cc = (dims[0] / P) * (dims[1] / P);
  *len = L.blocks * (cc + 1);
  return VPB_OK;
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_dg_sweep_xplane2(const double* src, double* dst, const int64_t dims[4],
                                    int32_t order, const double* a1, const double* b1,
                                    const int64_t* q1, const double* alpha1, const double* a2,
                                    const double* b2, const int64_t* q2, const double* alpha2,
                                    int32_t* flag1a, int32_t* flag2a, int32_t* flag1b,
                                    int32_t* flag2b, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  int32_t* const flags[4] = {flag1a, flag2a, flag1b, flag2b};
  const XDensity none{nullptr, nullptr, nullptr, nullptr, {}, {}};
  VPB_XPLANE_SWITCH(order, rc = launch_xplane2<PP, false>(src, dst, dims, a1, b1, q1, alpha1, a2,
                                                   b2, q2, alpha2, flags, none,
                                                   (cudaStream_t)stream, nullptr));
  return rc;
}

extern "C" int64_t vpb_dg_xplane2_density_work_len(const int64_t dims[4], int32_t order) {
  if (order < 1 || order > kMaxOrder || dims[0] % order || dims[1] % order) return -1;
  int64_t len = -1;
  int rc = VPB_OK;
  VPB_XPLANE_SWITCH(order, rc = xplane2_density_len<PP>(dims, &len));
  return rc == VPB_OK ? len : -1;
}

extern "C" int vpb_dg_sweep_xplane2_density(
    const double* src, double* dst, const int64_t dims[4], int32_t order, const double* a1,
    const double* b1, const int64_t* q1, const double* alpha1, const double* a2,
    const double* b2, const int64_t* q2, const double* alpha2, int32_t* flag1a, int32_t* flag2a,
    int32_t* flag1b, int32_t* flag2b, const double* wv1, const double* wv2,
    const double* mid_host, const double* wcell1_host, const double* wcell2_host, double volume,
    double* work, double* rc_out, double* stats, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(rc_out != nullptr, "null pointer");
  const int64_t cc = (dims[0] / order) * (dims[1] / order);
  const int64_t len = vpb_dg_xplane2_density_work_len(dims, order);
  VPB_REQUIRE(len > 0, "cannot plan the x-plane launch");
  const int64_t nblk = len / (cc + 1);
  XDensity dn;
  rc = xdensity_setup(&dn, order, wv1, wv2, mid_host, wcell1_host, wcell2_host, work, nblk, cc);
  if (rc) return rc;
  int32_t* const flags[4] = {flag1a, flag2a, flag1b, flag2b};
  int64_t used = 0;
  cudaStream_t st = (cudaStream_t)stream;
  VPB_XPLANE_SWITCH(order, rc = launch_xplane2<PP, true>(src, dst, dims, a1, b1, q1, alpha1, a2,
                                                   b2, q2, alpha2, flags, dn, st, &used));
  if (rc) return rc;
  VPB_REQUIRE(used == nblk, "x-plane launch plan changed (%lld vs %lld CTAs)", (long long)used,
              (long long)nblk);
  return launch_xdens_reduce(work, nblk, cc, volume, rc_out, stats, st);
}
