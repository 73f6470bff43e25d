// Fused dG sweeps: both space sweeps of a Strang half step in one HBM pass.
//
// In the reference, _advect_space (driver.py:220-228) sweeps x1 and then x2,
// each a full read+write of f.  Inside one (iv2, iv1) plane both shifts are
// constant (x1 shift from v1, x2 shift from v2), so the plane can be swept
// along x1 and then x2 while it streams through shared memory.  Output x2
// cell c reads the x1-swept values g of source x2 cells c-q2-1 and c-q2, so
// the plane is consumed in source order starting at s0 = (-q2-1) mod C2:
//
//   chunk 0 of a plane:  source cell s0 only (prologue, no output)
//   chunk i > 0:         source cells s0+1+(i-1)G ...  -> output cells (i-1)G ...
//
// Per chunk (G x2 cells = G*P rows of n1 dofs):
//   * TMA 1-D bulk copies (one or two pieces when the source range wraps)
//     land the rows in a kXStages-deep shared-memory ring (mbarriers);
//   * thread c owns x1 cell c: for each source x2 cell it sweeps the cell's
//     P rows along x1 (2P smem loads per row, P outputs), keeping the P x P
//     block g in registers, then applies the x2 pair to g(s-1), g(s) and
//     writes the P x P output block to a staging tile;
//   * the tile leaves by a bulk store (double buffered).
// Every element goes through the exact operations of the separate x1 and
// x2 sweeps (same order, no contraction), so the result is bitwise the
// unfused sequence, for 16 B/dof of HBM traffic instead of 32.
//
// CTAs are small (one warp per 32 x1 cells) and persistent over a
// contiguous run of planes; the load ring runs ahead across planes.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "async_copy.cuh"
#include "common.cuh"
#include "tensormap.cuh"
#include "xplane.cuh"

namespace vpb {

constexpr int kXStages = 6;

// DM: 0 = sweeps only, 1 = + density epilogue, 2 = + diagnostics moments
// (mass, l1, l2^2, kinetic of the output, driver.py:279-316) as well.
template <int P, int DM>
__global__ void __launch_bounds__(128)
    dg_xplane_kernel(const double* __restrict__ src, double* __restrict__ dst, int n1, int C2,
                     int G, int64_t nv1, int64_t nplanes, int64_t planes_per_block,
                     const double* __restrict__ a1, const double* __restrict__ b1,
                     const int64_t* __restrict__ q1, const double* __restrict__ al1,
                     const double* __restrict__ a2, const double* __restrict__ b2,
                     const int64_t* __restrict__ q2, const double* __restrict__ al2,
                     int32_t* __restrict__ flag1, int32_t* __restrict__ flag2,
                     const XDensity dn, const XMoments mo) {
  constexpr bool DENS = DM >= 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int cell = P * n1;          // one x2 cell: P rows of n1 dofs
  const int slot = G * cell;        // ring slot
  double* inb = reinterpret_cast<double*>(smem_raw);
  double* outb = inb + kXStages * slot;  // [2][G*cell] staging tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(outb + 2 * G * cell);

  const int tid = threadIdx.x;
  const int64_t pl_begin = blockIdx.x * planes_per_block;
  const int64_t pl_end = min(nplanes, pl_begin + planes_per_block);
  if (pl_begin >= pl_end) return;
  const int per_plane = 1 + (C2 + G - 1) / G;
  const int64_t nchunks = (pl_end - pl_begin) * per_plane;
  const int64_t plane_elems = (int64_t)C2 * cell;

  // L2 policies: f streams through (evict first); the density slabs stay
  const uint64_t pol_stream = l2_evict_first();
  const uint64_t pol_keep = l2_evict_last();
  // producer cursor (thread 0 only)
  XCursor prod;
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
    if (run1 < c.nsrc)  // wrapped: the rest starts at source cell 0
      if (DENS)
        bulk_g2s_hint(dstp + run1 * cell, base, (uint32_t)(c.nsrc - run1) * cell * 8u,
                      bars + prod_st, pol_stream);
      else
        bulk_g2s(dstp + run1 * cell, base, (uint32_t)(c.nsrc - run1) * cell * 8u,
                 bars + prod_st);
    ++prod_j;
    if (++prod_st == kXStages) prod_st = 0;
    prod.advance(per_plane, C2, q2, nv1, pl_end);
  };

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kXStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    while (prod_j < kXStages && prod_j < nchunks) issue_next();

  const int C1 = n1 / P;
  const bool active = tid < C1;
  double A1[P][P], B1[P][P], A2[P][P], B2[P][P];
  bool ex1 = true, ex2 = true;
  int lo_off = 0, up_off = 0;  // element offsets of the two x1 source cells in a row
  double gp[P][P];             // g of the previous source x2 cell: [row m2][dof j]
  bool bad1 = false, bad2 = false;
  XCursor cur;
  cur.start(pl_begin, C2, q2, nv1);
  int st = 0;
  uint32_t phase = 0;
  // density epilogue state
  constexpr bool dens = DENS;
  double wplane = 0.0, meanacc = 0.0;
  double kplane = 0.0, l1acc = 0.0, l2acc = 0.0, kinacc = 0.0;  // DM == 2
  double* mypart = dens ? dn.rc_part + (int64_t)blockIdx.x * C2 * C1 : nullptr;
  if (dens && active)
    for (int c2 = 0; c2 < C2; ++c2) mypart[c2 * C1 + tid] = 0.0;

  for (int64_t j = 0; j < nchunks; ++j) {
    const XChunk c = cur.chunk(G, C2);
    const int64_t plane = cur.plane;
    if (active && cur.i == 0) {
      const int64_t iv2 = plane / nv1, iv1 = plane - iv2 * nv1;
      if (dens) wplane = dn.wv1[iv1] * dn.wv2[iv2];
      if (DM == 2) kplane = 0.5 * (mo.vsq1[iv1] + mo.vsq2[iv2]);
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
    mbar_wait(bars + st, phase);
    const double* in = inb + st * slot;
    double* out = outb + (j & 1) * (G * cell);
    // One body per (ex1, ex2) combination: the alpha == 0 exact-shift cases
    // are uniform over a plane, so the branch is hoisted out of the cell loop.
    auto run_cells = [&](auto ex1c, auto ex2c) {
      constexpr bool E1 = decltype(ex1c)::value, E2 = decltype(ex2c)::value;
      for (int sc = 0; sc < c.nsrc; ++sc) {
        double g[P][P];
        xplane_x1_cell<P, E1>(in + sc * cell, n1, lo_off, up_off, A1, B1, g);
        if (c.nout > 0) {
          // x2 sweep for output x2 cell c.first + sc
          double o[P][P];
          xplane_x2_cell<P, E2>(A2, B2, gp, g, o);
          ExpMax eo;
#pragma unroll
          for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
            for (int jj = 0; jj < P; ++jj) eo.add(o[j2][jj]);
          if (eo.bad()) {
            // Every x1 value enters the output cell it is the B-side source
            // of through a product, so a non-finite x1 result always shows up
            // here: only then look at g to name the sub-step (x1 vs x2).
            bad2 = true;
            ExpMax eg;
#pragma unroll
            for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
              for (int jj = 0; jj < P; ++jj) eg.add(g[m2][jj]);
            bad1 |= eg.bad();
          }
          double* otile = out + sc * cell + tid * P;
#pragma unroll
          for (int j2 = 0; j2 < P; ++j2) {
            if constexpr (P % 2 == 0) {
#pragma unroll
              for (int jj = 0; jj < P; jj += 2)
                *reinterpret_cast<double2*>(otile + j2 * n1 + jj) =
                    make_double2(o[j2][jj], o[j2][jj + 1]);
            } else {
#pragma unroll
              for (int jj = 0; jj < P; ++jj) otile[j2 * n1 + jj] = o[j2][jj];
            }
          }
          if constexpr (DENS) {
            double rcv, mv = 0.0;
            if constexpr (P % 2 == 1) {
              rcv = o[P / 2][P / 2];  // mid = e_centre exactly (checked on the host)
            } else {
              // the density feeds a spectral solve that is not bitwise anyway:
              // contracted arithmetic is fine here
              rcv = 0.0;
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int jj = 0; jj < P; ++jj) rcv = fma(dn.mm[j2 * P + jj], o[j2][jj], rcv);
            }
            if constexpr (DM == 2) {
              double l1 = 0.0, l2 = 0.0;
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int jj = 0; jj < P; ++jj) {
                  const double t = dn.ww[j2 * P + jj] * o[j2][jj];
                  mv += t;
                  l1 += fabs(t);
                  l2 = fma(t, o[j2][jj], l2);
                }
              l1acc = fma(wplane, l1, l1acc);
              l2acc = fma(wplane, l2, l2acc);
              kinacc = fma(wplane * kplane, mv, kinacc);
            } else {
#pragma unroll
              for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
                for (int jj = 0; jj < P; ++jj) mv = fma(dn.ww[j2 * P + jj], o[j2][jj], mv);
            }
            red_add_hint(mypart + (c.first + sc) * C1 + tid, dmul(wplane, rcv), pol_keep);
            meanacc = fma(wplane, mv, meanacc);
          }
        }
#pragma unroll
        for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
          for (int jj = 0; jj < P; ++jj) gp[m2][jj] = g[m2][jj];
      }
    };
    if (active) {
      using F = std::false_type;
      using T = std::true_type;
      if (!ex1 && !ex2) run_cells(F{}, F{});
      else if (!ex1) run_cells(F{}, T{});
      else if (!ex2) run_cells(T{}, F{});
      else run_cells(T{}, T{});
    }
    fence_proxy_async_smem();
    if (tid == 0) bulk_wait_read<0>();  // store of chunk j-1 released the other tile
    __syncthreads();
    if (tid == 0) {
      if (c.nout > 0) {
        if (DENS)
          bulk_s2g_hint(dst + plane * plane_elems + (int64_t)c.first * cell, out,
                        (uint32_t)c.nout * cell * 8u, pol_stream);
        else
          bulk_s2g(dst + plane * plane_elems + (int64_t)c.first * cell, out,
                   (uint32_t)c.nout * cell * 8u);
        bulk_commit();
      }
      if (prod_j < nchunks) issue_next();
    }
    cur.advance(per_plane, C2, q2, nv1, pl_end);
    if (++st == kXStages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (tid == 0) bulk_wait<0>();
  report_flag(bad1, flag1);
  report_flag(bad2, flag2);
  if (dens) {  // fixed-order block sums of the mean (and moment) partials
    __shared__ double red[4][4];
    double v[4] = {meanacc, l1acc, l2acc, kinacc};
    constexpr int nv = DM == 2 ? 4 : 1;
#pragma unroll
    for (int k = 0; k < nv; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
      if ((tid & 31) == 0) red[k][tid >> 5] = v[k];
    }
    __syncthreads();
    if (tid < nv) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[tid][w];
      if (tid == 0)
        dn.mean_part[blockIdx.x] = s;
      else
        mo.mom_part[blockIdx.x * 3 + tid - 1] = s;
    }
  }
}

// rc[c2][c1] = sum over CTAs (in order) of the partial slabs; stats[0] =
// weighted density mean / volume.
// Block = 16 warps over 32 consecutive cells (lane = cell): warp w sums the
// slabs b = w, w+16, ... in order, then the 16 warp partials are added in warp
// order -- a fixed order, independent of timing.
constexpr int kRedWarps = 16;

__global__ void __launch_bounds__(32 * kRedWarps)
    xdens_reduce_kernel(const double* __restrict__ part, const double* __restrict__ mean_part,
                        int64_t nblocks, int64_t cc, double volume, double* __restrict__ rc,
                        double* __restrict__ stats, const double* __restrict__ mom_part,
                        double* __restrict__ diag_out) {
  __shared__ double ws[kRedWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < cc)
    for (int64_t b = w; b < nblocks; b += kRedWarps) s += part[b * cc + e];
  ws[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < cc) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kRedWarps; ++k) t += ws[k][lane];
    rc[e] = t;
  }
  // the scalar partials (density mean; l1, l2^2, kinetic) of block 0: one
  // warp each, lane-strided partial sums then a fixed butterfly (the same
  // order every run)
  if (blockIdx.x == 0 && w < 4) {
    const double* src = nullptr;
    int64_t stride = 1;
    if (w == 0) {
      src = mean_part;
    } else if (diag_out != nullptr && mom_part != nullptr) {
      src = mom_part + (w - 1);
      stride = 3;
    }
    if (src != nullptr) {
      double m = 0.0;
      for (int64_t b = lane; b < nblocks; b += 32) m += src[b * stride];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
      if (lane == 0) {
        if (w == 0) {
          if (stats != nullptr) stats[0] = m / volume;
          if (diag_out != nullptr) diag_out[0] = m;  // mass
        } else {
          diag_out[w] = m;  // l1, l2^2, kinetic
        }
      }
    }
  }
}

int xplane_sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached = v > 0 ? v : 148;
  }
  return cached;
}

struct XLaunch {
  int threads, G;
  size_t smem;
  int64_t ppb, blocks;
};

template <int P, int DM>
static int plan_xplane(const int64_t dims[4], XLaunch* L) {
  const int n1 = (int)dims[0];
  const int C1 = n1 / P;
  const int C2 = (int)(dims[1] / P);
  const int64_t nplanes = dims[2] * dims[3];
  if (C1 > 128) {
    set_error("x1 lines of %d cells exceed one CTA", C1);
    return VPB_ERR_UNSUPPORTED;
  }
  static const int env_chunk =
      getenv("VPB_XPLANE_CHUNK") ? atoi(getenv("VPB_XPLANE_CHUNK")) : 4608;
  static const int env_smem =
      getenv("VPB_XPLANE_SMEM") ? atoi(getenv("VPB_XPLANE_SMEM")) : 56 * 1024;
  L->threads = ((C1 + 31) / 32) * 32;
  const size_t cell_bytes = (size_t)P * n1 * 8;
  auto smem_for = [&](int g) {
    return (size_t)kXStages * g * cell_bytes + 2 * (size_t)g * cell_bytes + kXStages * 8;
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
    cudaFuncSetAttribute(dg_xplane_kernel<P, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dg_xplane_kernel<P, DM>, L->threads,
                                                L->smem);
  if (occ < 1) occ = 1;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(nplanes, (int64_t)occ * xplane_sm_count()));
  L->ppb = (nplanes + grid - 1) / grid;
  L->blocks = (nplanes + L->ppb - 1) / L->ppb;
  return VPB_OK;
}

template <int P, int DM>
static int launch_xplane(const double* src, double* dst, const int64_t dims[4], const double* a1,
                         const double* b1, const int64_t* q1, const double* al1,
                         const double* a2, const double* b2, const int64_t* q2,
                         const double* al2, int32_t* f1, int32_t* f2, const XDensity& dn,
                         cudaStream_t st, int64_t* nblocks_out) {
  const int64_t nplanes = dims[2] * dims[3];
  if (nplanes == 0) return VPB_OK;
  XLaunch L;
  int rc = plan_xplane<P, DM>(dims, &L);
  if (rc) return rc;
  dg_xplane_kernel<P, DM><<<(unsigned)L.blocks, L.threads, L.smem, st>>>(
      src, dst, (int)dims[0], (int)(dims[1] / P), L.G, dims[2], nplanes, L.ppb, a1, b1, q1, al1,
      a2, b2, q2, al2, f1, f2, dn, XMoments{nullptr, nullptr, nullptr});
  if (nblocks_out) *nblocks_out = L.blocks;
  return launched("dg_xplane_kernel");
}

// Work of the density / moments epilogues: [blocks][cc] slabs, [blocks] mean
// partials, [blocks][3] moment partials; sized for the larger of the two plans.
template <int P>
static int xplane_density_len(const int64_t dims[4], int64_t* len) {
  XLaunch L1, L2;
  int rc = plan_xplane<P, 1>(dims, &L1);
  if (rc == VPB_OK) rc = plan_xplane<P, 2>(dims, &L2);
  if (rc) return rc;
  const int64_t cc = (dims[0] / P) * (dims[1] / P);
  *len = std::max(L1.blocks, L2.blocks) * (cc + 4);
  return VPB_OK;
}

// Density (DM 1) or density + diagnostics moments (DM 2) pass, then the
// fixed-order reduction of the CTA partials.
template <int P, int DM>
static int xplane_epilogue_pass(const double* src, double* dst, const int64_t dims[4],
                                const double* a1, const double* b1, const int64_t* q1,
                                const double* al1, const double* a2, const double* b2,
                                const int64_t* q2, const double* al2, int32_t* f1, int32_t* f2,
                                const double* wv1, const double* wv2, const double* mid_host,
                                const double* wc1, const double* wc2, const double* vsq1,
                                const double* vsq2, double volume, double* work, double* rc_out,
                                double* stats, double* diag_out, cudaStream_t st) {
  const int64_t nplanes = dims[2] * dims[3];
  if (nplanes == 0) return VPB_OK;
  XLaunch L;
  int rc = plan_xplane<P, DM>(dims, &L);
  if (rc) return rc;
  const int64_t cc = (dims[0] / P) * (dims[1] / P);
  XDensity dn;
  rc = xdensity_setup(&dn, P, wv1, wv2, mid_host, wc1, wc2, work, L.blocks, cc);
  if (rc) return rc;
  const XMoments mo{dn.mean_part + L.blocks, vsq1, vsq2};
  dg_xplane_kernel<P, DM><<<(unsigned)L.blocks, L.threads, L.smem, st>>>(
      src, dst, (int)dims[0], (int)(dims[1] / P), L.G, dims[2], nplanes, L.ppb, a1, b1, q1, al1,
      a2, b2, q2, al2, f1, f2, dn, mo);
  rc = launched("dg_xplane_kernel");
  if (rc) return rc;
  return launch_xdens_reduce(work, L.blocks, cc, volume, rc_out, stats, st,
                             DM == 2 ? mo.mom_part : nullptr, DM == 2 ? diag_out : nullptr);
}

int xplane_args_ok(const double* src, const double* dst, const int64_t dims[4], int32_t order) {
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1 && order <= kMaxOrder, "order %d outside 1..9", order);
  VPB_REQUIRE(dims[0] % order == 0 && dims[1] % order == 0, "x axes not whole cells");
  VPB_REQUIRE(dims[1] > 1, "fused x sweep needs a 2x2v field");
  VPB_REQUIRE((dims[0] * order) % 2 == 0, "a cell row block must be a multiple of 16 bytes");
  VPB_REQUIRE((reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
              "field buffers must be 16-byte aligned");
  return VPB_OK;
}

int xdensity_setup(XDensity* dn, int order, const double* wv1, const double* wv2,
                   const double* mid_host, const double* wcell1_host, const double* wcell2_host,
                   double* work, int64_t nblk, int64_t cc) {
  VPB_REQUIRE(wv1 && wv2 && mid_host && wcell1_host && wcell2_host && work, "null pointer");
  if (order % 2 == 1)
    for (int j = 0; j < order; ++j)
      VPB_REQUIRE(mid_host[j] == (j == order / 2 ? 1.0 : 0.0),
                  "odd-order centre weights must select the middle node");
  *dn = XDensity{wv1, wv2, work, work + nblk * cc, {}, {}};
  for (int j2 = 0; j2 < order; ++j2)
    for (int jj = 0; jj < order; ++jj) {
      dn->mm[j2 * order + jj] = mid_host[j2] * mid_host[jj];
      dn->ww[j2 * order + jj] = wcell2_host[j2] * wcell1_host[jj];
    }
  return VPB_OK;
}

int launch_xdens_reduce(const double* work, int64_t nblk, int64_t cc, double volume,
                        double* rc_out, double* stats, cudaStream_t st, const double* mom_part,
                        double* diag_out) {
  xdens_reduce_kernel<<<(unsigned)((cc + 31) / 32), 32 * kRedWarps, 0, st>>>(
      work, work + nblk * cc, nblk, cc, volume, rc_out, stats, mom_part, diag_out);
  return launched("xdens_reduce_kernel");
}

}  // namespace vpb

using namespace vpb;


extern "C" int vpb_dg_sweep_xplane(const double* src, double* dst, const int64_t dims[4],
                                   int32_t order, const double* a1, const double* b1,
                                   const int64_t* q1, const double* alpha1, const double* a2,
                                   const double* b2, const int64_t* q2, const double* alpha2,
                                   int32_t* flag1, int32_t* flag2, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  const XDensity none{nullptr, nullptr, nullptr, nullptr, {}, {}};
  VPB_XPLANE_SWITCH(order, rc = launch_xplane<PP, 0>(src, dst, dims, a1, b1, q1, alpha1, a2,
                                                  b2, q2, alpha2, flag1, flag2, none,
                                                  (cudaStream_t)stream, nullptr));
  return rc;
}

extern "C" int64_t vpb_dg_xplane_density_work_len(const int64_t dims[4], int32_t order) {
  if (order < 1 || order > kMaxOrder || dims[0] % order || dims[1] % order) return -1;
  int64_t len = -1;
  int rc = VPB_OK;
  VPB_XPLANE_SWITCH(order, rc = xplane_density_len<PP>(dims, &len));
  return rc == VPB_OK ? len : -1;
}

extern "C" int vpb_dg_sweep_xplane_density(
    const double* src, double* dst, const int64_t dims[4], int32_t order, const double* a1,
    const double* b1, const int64_t* q1, const double* alpha1, const double* a2,
    const double* b2, const int64_t* q2, const double* alpha2, int32_t* flag1, int32_t* flag2,
    const double* wv1, const double* wv2, const double* mid_host, const double* wcell1_host,
    const double* wcell2_host, double volume, double* work, double* rc_out, double* stats,
    void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(rc_out != nullptr, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  VPB_XPLANE_SWITCH(order, rc = xplane_epilogue_pass<PP, 1>(
                               src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1,
                               flag2, wv1, wv2, mid_host, wcell1_host, wcell2_host, nullptr,
                               nullptr, volume, work, rc_out, stats, nullptr, st));
  return rc;
}

extern "C" int vpb_dg_sweep_xplane_moments(
    const double* src, double* dst, const int64_t dims[4], int32_t order, const double* a1,
    const double* b1, const int64_t* q1, const double* alpha1, const double* a2,
    const double* b2, const int64_t* q2, const double* alpha2, int32_t* flag1, int32_t* flag2,
    const double* wv1, const double* wv2, const double* mid_host, const double* wcell1_host,
    const double* wcell2_host, const double* v1sq, const double* v2sq, double volume,
    double* work, double* rc_out, double* stats, double* diag_out, void* stream) {
  int rc = xplane_args_ok(src, dst, dims, order);
  if (rc) return rc;
  VPB_REQUIRE(rc_out != nullptr && v1sq != nullptr && v2sq != nullptr && diag_out != nullptr,
              "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  VPB_XPLANE_SWITCH(order, rc = xplane_epilogue_pass<PP, 2>(
                               src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1,
                               flag2, wv1, wv2, mid_host, wcell1_host, wcell2_host, v1sq, v2sq,
                               volume, work, rc_out, stats, diag_out, st));
  return rc;
}

namespace vpb {

// ---------------------------------------------------------------------------
// Fused velocity sweeps: v1 then v2 (driver.py:231-242 _advect_velocity) in
// one HBM pass.  Both shifts are constant over the (v1, v2) plane of one x
// position (E1(x) tau, E2(x) tau), so thread (x, v1 cell c1) streams the
// plane along v2: for every source v2 cell s it loads the two v1 cells it
// needs (coalesced across the 32 consecutive x of a warp), sweeps them along
// v1 into the P x P block g(s) (v2 rows x v1 dofs of cell c1), and applies
// the v2 pair to g(s-1), g(s), producing output v2 cell s + q2(x).  The
// source order starts at (-q2-1) mod C2 and visits C2+1 cells.  Identical
// operations to the two separate sweeps, so bitwise equal to them.
// Grid: x-fastest is the v1-cell group so the blocks sharing source cells
// (neighbouring c1) run together and hit L1/L2.
// ---------------------------------------------------------------------------
#ifndef VPB_VCELLS
#define VPB_VCELLS 4
#endif
constexpr int kVCells = VPB_VCELLS;  // v1 cells (warps) per CTA

template <int P>
__global__ void __launch_bounds__(32 * kVCells)
    dg_vplane_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nx, int C1,
                     int C2, const double* __restrict__ a1, const double* __restrict__ b1,
                     const int64_t* __restrict__ q1, const double* __restrict__ al1,
                     const double* __restrict__ a2, const double* __restrict__ b2,
                     const int64_t* __restrict__ q2, const double* __restrict__ al2,
                     int32_t* __restrict__ flag1, int32_t* __restrict__ flag2) {
  const int lane = threadIdx.x & 31;
  const int c1 = blockIdx.x * kVCells + (threadIdx.x >> 5);
  const int64_t x = (int64_t)blockIdx.y * 32 + lane;
  if (c1 >= C1 || x >= nx) return;
  const int64_t nv1 = (int64_t)C1 * P;
  const int64_t row_stride = nv1 * nx;  // one v2 dof row
  double A1[P][P], B1[P][P], A2[P][P], B2[P][P];
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int m = 0; m < P; ++m) {
      A1[j][m] = __ldg(a1 + x * P * P + j * P + m);
      B1[j][m] = __ldg(b1 + x * P * P + j * P + m);
      A2[j][m] = __ldg(a2 + x * P * P + j * P + m);
      B2[j][m] = __ldg(b2 + x * P * P + j * P + m);
    }
  const bool ex1 = (al1[x] == 0.0), ex2 = (al2[x] == 0.0);
  const int qm1 = (int)wrap_mod(q1[x], C1);
  const int qm2 = (int)wrap_mod(q2[x], C2);
  int lo1 = c1 - qm1 - 1;
  if (lo1 < 0) lo1 += C1;
  const int up1 = lo1 + 1 == C1 ? 0 : lo1 + 1;
  const double* lo_base = src + (int64_t)lo1 * P * nx + x;
  const double* up_base = src + (int64_t)up1 * P * nx + x;
  ExpMax e1, e2;  // integer-pipe non-finite tracking

  // v1 sweep of source v2 cell s: g[m2][j1] for the P v2 rows of the cell
  auto v1_cell = [&](int s, double (&g)[P][P]) {
    double ul[P][P], uu[P][P];
#pragma unroll
    for (int m2 = 0; m2 < P; ++m2) {
      const int64_t r = ((int64_t)s * P + m2) * row_stride;
#pragma unroll
      for (int m = 0; m < P; ++m) {
        uu[m2][m] = __ldcs(up_base + r + m * nx);
        if (!ex1) ul[m2][m] = __ldcs(lo_base + r + m * nx);
      }
    }
#pragma unroll
    for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        double v;
        if (ex1) {
          v = uu[m2][j];
        } else {
          double acc_a = dmul(A1[j][0], ul[m2][0]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_a = step_madd(acc_a, A1[j][m], ul[m2][m]);
          double acc_b = dmul(B1[j][0], uu[m2][0]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_b = step_madd(acc_b, B1[j][m], uu[m2][m]);
          v = dadd(acc_a, acc_b);
        }
        g[m2][j] = v;
        e1.add(v);
      }
  };

  int s = C2 - qm2 - 1;  // (-q2-1) mod C2
  double gp[P][P];
  v1_cell(s, gp);
  int c2 = s + qm2;  // output cell of the first step: s+1+q2 (mod C2), kept incrementally
  if (c2 >= C2) c2 -= C2;
  for (int k = 0; k < C2; ++k) {
    if (++s == C2) s = 0;
    if (++c2 == C2) c2 = 0;
    double g[P][P];
    v1_cell(s, g);
    double* out = dst + ((int64_t)c2 * P) * row_stride + (int64_t)c1 * P * nx + x;
#pragma unroll
    for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        double o;
        if (ex2) {
          o = g[j2][j];
        } else {
          double acc_a = dmul(A2[j2][0], gp[0][j]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_a = step_madd(acc_a, A2[j2][m], gp[m][j]);
          double acc_b = dmul(B2[j2][0], g[0][j]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_b = step_madd(acc_b, B2[j2][m], g[m][j]);
          o = dadd(acc_a, acc_b);
        }
        e2.add(o);
        __stcs(out + j2 * row_stride + j * nx, o);
      }
#pragma unroll
    for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
      for (int j = 0; j < P; ++j) gp[m2][j] = g[m2][j];
  }
  report_flag(e1.bad(), flag1);
  report_flag(e2.bad(), flag2);
}

// TMA-staged variant.  A CTA owns 32 consecutive x (one per lane) and kVCells
// v1 cells (one per warp).  All lanes stream the same source v2 cells s =
// 0..C2 (each lane's output cell is s + q2(x)); for every s a TMA 3-D tensor
// copy brings the P v2 rows x the block's v1 source window (kVCells+kVSpan
// cells starting at c1a - max(q1) - 1) x 32 x into a kVStages-deep ring.
// Lanes read their own two source cells from the tile: [row][v1 dof][lane]
// keeps every warp access conflict-free whatever the per-lane q1.  Blocks
// whose q1 spread exceeds the window fall back to direct global loads.
constexpr int kVSpan = 3;    // window = kVCells + kVSpan cells (q1 spread <= 2)
#ifndef VPB_VSTAGES
#define VPB_VSTAGES 4
#endif
constexpr int kVStages = VPB_VSTAGES;

// VH (v2-sharded fields, dist.VShardedSolver): the source stream has C2
// v2 cells, the shard's own cells at [v2off, v2off + C2out) with v2off halo
// cells of each neighbouring rank before and after them, and dst holds the
// C2out output cells.  The three regions may live in three buffers: `VHalo`
// gives, per region, the buffer (its own tensor map for the TMA ring and
// its base pointer for direct loads) and the buffer cell of the region's
// first stream cell -- the halos are either rows of this shard's extended
// buffer filled by NCCL, or the neighbours' own boundary rows read in place
// over NVLink (IPC-mapped peer memory: the exchange fused into the pass).
// The stream is not periodic: source cells k = 0 .. C2-1, the pair (k-1, k)
// produces output cell k - v2off + q2(x), stored when inside [0, C2out).  A
// lane whose shift would need a source cell outside the halos raises
// vh_flag (the host's halo width bounds |E tau / h_v|; the solver raises).
struct VHalo {
  const double* src_l;  // left halo region: buffer and the cell of stream cell 0
  const double* src_r;  // right halo region: buffer and the cell of stream cell v2off + C2out
  int cl0, cc0, cr0;    // own region: `src` at cell cc0 for stream cell v2off
};

template <int P, bool VH = false>
__global__ void __launch_bounds__(32 * kVCells)
    dg_vplane_tma_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nx,
                         int C1, int C2, const double* __restrict__ a1,
                         const double* __restrict__ b1, const int64_t* __restrict__ q1,
                         const double* __restrict__ al1, const double* __restrict__ a2,
                         const double* __restrict__ b2, const int64_t* __restrict__ q2,
                         const double* __restrict__ al2, int32_t* __restrict__ flag1,
                         int32_t* __restrict__ flag2, const __grid_constant__ CUtensorMap tmap,
                         int v2off = 0, int C2out = 0, int32_t* __restrict__ vh_flag = nullptr,
                         const __grid_constant__ CUtensorMap tmap_l = CUtensorMap{},
                         const __grid_constant__ CUtensorMap tmap_r = CUtensorMap{},
                         const VHalo vhs = VHalo{}) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int W = kVCells + kVSpan;       // window cells
  constexpr int WP = W * P;                 // window v1 dofs
  constexpr int stage = P * WP * 32;        // doubles per stage
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kVStages * stage);
  __shared__ int s_qmax, s_qmin;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c1a = blockIdx.x * kVCells;
  const int c1 = c1a + warp;
  const int64_t x0 = (int64_t)blockIdx.y * 32;
  const int64_t x = x0 + lane;
  const int64_t nv1 = (int64_t)C1 * P;
  const int64_t row_stride = nv1 * nx;
  const bool active = c1 < C1;

  const int qm1 = (int)wrap_mod(q1[x], C1);
  const int qm2 = VH ? (int)q2[x] : (int)wrap_mod(q2[x], C2);
  // VH: the lane's outputs 0 .. C2out-1 need source cells v2off - q2 - 1 ..
  // v2off - q2 + C2out - 1 of the stream
  const bool vh_bad = VH && (v2off - qm2 - 1 < 0 || v2off - qm2 + C2out - 1 > C2 - 1);
  const int klast = VH ? C2 - 1 : C2;  // last source step (periodic: C2 wraps to cell 0)
  // block-wide window of source v1 cells (q1 in [qmin, qmax], taken mod C1
  // relative to the warp-0 lane-0 value so the spread is the true spread)
  if (threadIdx.x == 0) {
    s_qmax = -(1 << 30);
    s_qmin = 1 << 30;
  }
  __syncthreads();
  {
    const int q0 = (int)wrap_mod(q1[x0], C1);
    int d = qm1 - q0;  // relative offset in (-C1, C1); fold to the nearest
    if (d > C1 / 2) d -= C1;
    if (d < -C1 / 2) d += C1;
    if (warp == 0) {
      int mx = d, mn = d;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      if (lane == 0) {
        s_qmax = q0 + mx;
        s_qmin = q0 + mn;
      }
    }
  }
  __syncthreads();
  const int qmax = s_qmax;
  const bool use_tma = (qmax - s_qmin) <= kVSpan - 1;
  // source v1 cells the block needs: kVCells + 1 + (q1 spread) <= W
  const int wcells = min(W, kVCells + 1 + (qmax - s_qmin));
  int wstart = c1a - qmax - 1;  // first window cell (mod C1)
  wstart %= C1;
  if (wstart < 0) wstart += C1;

  double A1[P][P], B1[P][P], A2[P][P], B2[P][P];
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int m = 0; m < P; ++m) {
      A1[j][m] = __ldg(a1 + x * P * P + j * P + m);
      B1[j][m] = __ldg(b1 + x * P * P + j * P + m);
      A2[j][m] = __ldg(a2 + x * P * P + j * P + m);
      B2[j][m] = __ldg(b2 + x * P * P + j * P + m);
    }
  const bool ex1 = (al1[x] == 0.0), ex2 = (al2[x] == 0.0);
  int lo1 = c1 - qm1 - 1;
  lo1 %= C1;
  if (lo1 < 0) lo1 += C1;
  const int up1 = lo1 + 1 == C1 ? 0 : lo1 + 1;
  // window-relative cell indices (valid when use_tma)
  int wlo = lo1 - wstart;
  if (wlo < 0) wlo += C1;
  int wup = wlo + 1;
  const double* lo_base = src + (int64_t)lo1 * P * nx + x;
  const double* up_base = src + (int64_t)up1 * P * nx + x;
  bool bad1 = false, bad2 = false;

  // VH: stream cell k -> (region tensor map / base pointer, buffer cell)
  auto region = [&](int k, const CUtensorMap*& map, const double*& base, int& bc) {
    if (!VH) {
      map = &tmap;
      base = src;
      bc = k == C2 ? 0 : k;
    } else if (k < v2off) {
      map = &tmap_l;
      base = vhs.src_l;
      bc = vhs.cl0 + k;
    } else if (k < v2off + C2out) {
      map = &tmap;
      base = src;
      bc = vhs.cc0 + k - v2off;
    } else {
      map = &tmap_r;
      base = vhs.src_r;
      bc = vhs.cr0 + k - v2off - C2out;
    }
  };
  auto issue = [&](int k) {  // source v2 cell k (0..klast) into slot k % kVStages
    const CUtensorMap* map;
    const double* base;
    int s;
    region(k, map, base, s);
    const int sl = k % kVStages;
    double* dstp = ring + sl * stage;
    mbar_arrive_expect_tx(bars + sl, (uint32_t)(wcells * P * P * 32) * 8u);
    int cell = wstart;
    for (int w = 0; w < wcells; ++w) {  // one {32 x, P dofs, P rows} box per needed cell
      tma_load_3d(dstp + w * (P * P * 32), map, (int)x0, cell * P, s * P, bars + sl);
      if (++cell == C1) cell = 0;
    }
  };
  if (use_tma && threadIdx.x == 0) {
#pragma unroll
    for (int sl = 0; sl < kVStages; ++sl) mbar_init(bars + sl, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (use_tma && threadIdx.x == 0)
    for (int k = 0; k < kVStages && k <= klast; ++k) issue(k);

  // GEN: per-lane alpha == 0 exact-shift branches; otherwise the common
  // all-lanes-interpolate body without them.
  auto v1_cell = [&](int k, double (&g)[P][P], auto genc) {
    constexpr bool GEN = decltype(genc)::value;
    double ul[P][P], uu[P][P];
    if (use_tma) {
      const int sl = k % kVStages;
      const double* t = ring + sl * stage + lane;
#pragma unroll
      for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
        for (int m = 0; m < P; ++m) {
          uu[m2][m] = t[((wup * P + m2) * P + m) * 32];  // [cell][row][dof][lane]
          ul[m2][m] = t[((wlo * P + m2) * P + m) * 32];
        }
    } else {
      const CUtensorMap* map;
      const double* base;
      int s;
      region(k, map, base, s);
      const int64_t rb = (base - src);  // same x / v1 layout in every region's buffer
#pragma unroll
      for (int m2 = 0; m2 < P; ++m2) {
        const int64_t r = rb + ((int64_t)s * P + m2) * row_stride;
#pragma unroll
        for (int m = 0; m < P; ++m) {
          uu[m2][m] = __ldcs(up_base + r + m * nx);
          ul[m2][m] = __ldcs(lo_base + r + m * nx);
        }
      }
    }
#pragma unroll
    for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        double v;
        if (GEN && ex1) {
          v = uu[m2][j];
        } else {
          double acc_a = dmul(A1[j][0], ul[m2][0]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_a = step_madd(acc_a, A1[j][m], ul[m2][m]);
          double acc_b = dmul(B1[j][0], uu[m2][0]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_b = step_madd(acc_b, B1[j][m], uu[m2][m]);
          v = dadd(acc_a, acc_b);
        }
        g[m2][j] = v;
      }
  };
  auto release = [&](int k) {  // every thread is done with slot k % kVStages
    __syncthreads();
    if (use_tma && threadIdx.x == 0 && k + kVStages <= klast) issue(k + kVStages);
  };

  // Non-finite values: only the outputs are tested in the common path; an
  // x1 (v1) result always reaches the output cell it is the B-side source of
  // through a product, so g is examined (to name the sub-step) only when that
  // output cell is bad.
  auto step = [&](int k, double (&gp)[P][P], int c2, auto genc) {
    constexpr bool GEN = decltype(genc)::value;
    double g[P][P];
    v1_cell(k, g, genc);
    // VH: pairs outside the shard's output cells only advance the chain
    const bool store = !VH || (c2 >= 0 && c2 < C2out);
    double* out = dst + ((int64_t)(store ? c2 : 0) * P) * row_stride + (int64_t)c1 * P * nx + x;
    ExpMax eo;
#pragma unroll
    for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        double o;
        if (GEN && ex2) {
          o = g[j2][j];
        } else {
          double acc_a = dmul(A2[j2][0], gp[0][j]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_a = step_madd(acc_a, A2[j2][m], gp[m][j]);
          double acc_b = dmul(B2[j2][0], g[0][j]);
#pragma unroll
          for (int m = 1; m < P; ++m) acc_b = step_madd(acc_b, B2[j2][m], g[m][j]);
          o = dadd(acc_a, acc_b);
        }
        if (store) {
          eo.add(o);
          __stcs(out + j2 * row_stride + j * nx, o);
        }
      }
    if (eo.bad()) {
      bad2 = true;
      ExpMax eg;
#pragma unroll
      for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
        for (int j = 0; j < P; ++j) eg.add(g[m2][j]);
      bad1 |= eg.bad();
    }
#pragma unroll
    for (int m2 = 0; m2 < P; ++m2)
#pragma unroll
      for (int j = 0; j < P; ++j) gp[m2][j] = g[m2][j];
  };
  // the exact-shift branches are needed only if some lane of the block has them
  const bool gen = __syncthreads_or(active && (ex1 || ex2)) != 0;

  double gp[P][P];
  uint32_t phase = 0;
  if (use_tma) mbar_wait(bars + 0, 0);
  if (active) {
    if (gen)
      v1_cell(0, gp, std::true_type{});
    else
      v1_cell(0, gp, std::false_type{});
  }
  release(0);
  // output cell of source cell s: s + q2 (mod C2), s = 1 first; VH: s - v2off + q2
  int c2 = VH ? qm2 - v2off : qm2;
  for (int k = 1; k <= klast; ++k) {
    const int sl = k % kVStages;
    if (sl == 0) phase ^= 1u;
    if (use_tma) mbar_wait(bars + sl, phase);
    if (++c2 == C2 && !VH) c2 = 0;
    if (active) {
      if (gen)
        step(k, gp, c2, std::true_type{});
      else
        step(k, gp, c2, std::false_type{});
    }
    release(k);
  }
  report_flag(bad1, flag1);
  report_flag(bad2, flag2);
  if (VH) report_flag(active && vh_bad, vh_flag);
}

template <int P>
static int launch_vplane(const double* src, double* dst, const int64_t dims[4], const double* a1,
                         const double* b1, const int64_t* q1, const double* al1,
                         const double* a2, const double* b2, const int64_t* q2,
                         const double* al2, int32_t* f1, int32_t* f2, cudaStream_t st) {
  const int64_t nx = dims[0] * dims[1];
  const int C1 = (int)(dims[2] / P);
  const int C2 = (int)(dims[3] / P);
  if (nx == 0 || C1 == 0 || C2 == 0) return VPB_OK;
  dim3 grid((unsigned)((C1 + kVCells - 1) / kVCells), (unsigned)((nx + 31) / 32));
  static const bool no_tma = getenv("VPB_VPLANE_DIRECT") != nullptr;
  if (!no_tma && nx % 32 == 0 && C1 >= kVCells + kVSpan && P * P * 32 * 8 <= 65536 &&
      (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (nx * 8) % 16 == 0) {
    CUtensorMap tmap;
    const uint64_t nv1 = (uint64_t)C1 * P, nv2 = (uint64_t)C2 * P;
    if (encode_tmap_3d(&tmap, src, (uint64_t)nx, nv1, nv2, (uint64_t)nx * 8,
                       (uint64_t)nx * nv1 * 8, 32, P, P)) {
      const size_t smem = (size_t)kVStages * P * (kVCells + kVSpan) * P * 32 * 8 + kVStages * 8;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(dg_vplane_tma_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
      }
      if (smem <= 200 * 1024) {
        dg_vplane_tma_kernel<P><<<grid, 32 * kVCells, smem, st>>>(
            src, dst, nx, C1, C2, a1, b1, q1, al1, a2, b2, q2, al2, f1, f2, tmap);
        return launched("dg_vplane_tma_kernel");
      }
    }
  }
  dg_vplane_kernel<P><<<grid, 32 * kVCells, 0, st>>>(src, dst, nx, C1, C2, a1, b1, q1, al1, a2,
                                                     b2, q2, al2, f1, f2);
  return launched("dg_vplane_kernel");
}

// v2-sharded shard: the stream [left halo (H cells) | own cells | right
// halo (H cells)], each region in its own buffer (bl / bc / br with nl_cells
// / nc_cells / nr_cells v2 cells; the region starts at buffer cell l0 / c0 /
// r0), dst = the shard's own cells.  TMA ring only (the halo stream has no
// separate direct-load kernel); needs nx % 32 == 0 and at least kVCells +
// kVSpan v1 cells.
template <int P>
static int launch_vplane_vh(const double* bl, int nl_cells, int l0, const double* bc,
                            int nc_cells, int c0, const double* br, int nr_cells, int r0,
                            double* dst, const int64_t dims[4], int H, const double* a1,
                            const double* b1, const int64_t* q1, const double* al1,
                            const double* a2, const double* b2, const int64_t* q2,
                            const double* al2, int32_t* f1, int32_t* f2, int32_t* vh_flag,
                            cudaStream_t st) {
  const int64_t nx = dims[0] * dims[1];
  const int C1 = (int)(dims[2] / P);
  const int C2out = (int)(dims[3] / P);
  if (nx == 0 || C1 == 0 || C2out == 0) return VPB_OK;
  VPB_REQUIRE(nx % 32 == 0 && C1 >= kVCells + kVSpan,
              "v2-halo v pass needs nx %% 32 == 0 and >= %d v1 cells", kVCells + kVSpan);
  VPB_REQUIRE(H >= 1 && l0 >= 0 && l0 + H <= nl_cells && c0 >= 0 && c0 + C2out <= nc_cells &&
                  r0 >= 0 && r0 + H <= nr_cells,
              "v2 halo regions outside their buffers");
  for (const double* b : {bl, bc, br})
    VPB_REQUIRE(b && (reinterpret_cast<uintptr_t>(b) & 15) == 0,
                "field buffers must be 16-byte aligned");
  const uint64_t nv1 = (uint64_t)C1 * P;
  CUtensorMap tl, tc, tr;
  if (!encode_tmap_3d(&tl, bl, (uint64_t)nx, nv1, (uint64_t)nl_cells * P, (uint64_t)nx * 8,
                      (uint64_t)nx * nv1 * 8, 32, P, P) ||
      !encode_tmap_3d(&tc, bc, (uint64_t)nx, nv1, (uint64_t)nc_cells * P, (uint64_t)nx * 8,
                      (uint64_t)nx * nv1 * 8, 32, P, P) ||
      !encode_tmap_3d(&tr, br, (uint64_t)nx, nv1, (uint64_t)nr_cells * P, (uint64_t)nx * 8,
                      (uint64_t)nx * nv1 * 8, 32, P, P)) {
    set_error("cannot encode the v-plane tensor maps");
    return VPB_ERR_UNSUPPORTED;
  }
  const size_t smem = (size_t)kVStages * P * (kVCells + kVSpan) * P * 32 * 8 + kVStages * 8;
  VPB_REQUIRE(smem <= 200 * 1024, "v-plane ring does not fit shared memory");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dg_vplane_tma_kernel<P, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const VHalo vhs{bl, br, l0, c0, r0};
  dim3 grid((unsigned)((C1 + kVCells - 1) / kVCells), (unsigned)((nx + 31) / 32));
  dg_vplane_tma_kernel<P, true><<<grid, 32 * kVCells, smem, st>>>(
      bc, dst, nx, C1, C2out + 2 * H, a1, b1, q1, al1, a2, b2, q2, al2, f1, f2, tc, H, C2out,
      vh_flag, tl, tr, vhs);
  return launched("dg_vplane_tma_kernel");
}

}  // namespace vpb

using namespace vpb;

// Fused v1 v2 pass of one v2 shard (dist.VShardedSolver): `src` holds
// src_v2_cells source v2 cells (the shard's dims[3] / order cells start at
// cell v2_offset, halo cells of the neighbouring shards before and after),
// `dst` the shard's own cells; the v2 tables index the shard's x columns as
// usual.  halo_flag is raised when a shift needs a cell beyond the halos.
extern "C" int vpb_dg_sweep_vplane_v2halo(const double* src, double* dst, const int64_t dims[4],
                                          int32_t order, int32_t src_v2_cells, int32_t v2_offset,
                                          const double* a1, const double* b1, const int64_t* q1,
                                          const double* alpha1, const double* a2, const double* b2,
                                          const int64_t* q2, const double* alpha2, int32_t* flag1,
                                          int32_t* flag2, int32_t* halo_flag, void* stream) {
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1 && order <= kMaxOrder, "order %d outside 1..9", order);
  VPB_REQUIRE(dims[2] % order == 0 && dims[3] % order == 0, "v axes not whole cells");
  const int nc = (int)(dims[3] / order);
  VPB_REQUIRE(v2_offset >= 1 && v2_offset + nc + v2_offset <= src_v2_cells,
              "shard cells and halos outside the source stream");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = VPB_OK;
  const int H = v2_offset;
  VPB_XPLANE_SWITCH(order, rc = launch_vplane_vh<PP>(src, src_v2_cells, 0, src, src_v2_cells, H,
                                                     src, src_v2_cells, H + nc, dst, dims, H, a1,
                                                     b1, q1, alpha1, a2, b2, q2, alpha2, flag1,
                                                     flag2, halo_flag, st));
  return rc;
}

// The same pass with the halo regions read IN PLACE from the neighbouring
// shards' buffers (peer memory over NVLink, CUDA IPC-mapped): the left halo
// is cells [l_cell0, l_cell0 + H) of src_l (src_l_cells cells), the own
// cells start at cell c_cell0 of src, the right halo is cells [r_cell0,
// r_cell0 + H) of src_r.  No exchange, no halo rows: the collective is fused
// into the pass (the host orders it after the neighbours' x pass).
extern "C" int vpb_dg_sweep_vplane_v2peer(const double* src_l, int32_t src_l_cells, int32_t l_cell0,
                                          const double* src, int32_t src_cells, int32_t c_cell0,
                                          const double* src_r, int32_t src_r_cells, int32_t r_cell0,
                                          int32_t halo_cells, double* dst, const int64_t dims[4],
                                          int32_t order, const double* a1, const double* b1,
                                          const int64_t* q1, const double* alpha1, const double* a2,
                                          const double* b2, const int64_t* q2, const double* alpha2,
                                          int32_t* flag1, int32_t* flag2, int32_t* halo_flag,
                                          void* stream) {
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1 && order <= kMaxOrder, "order %d outside 1..9", order);
  VPB_REQUIRE(dims[2] % order == 0 && dims[3] % order == 0, "v axes not whole cells");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = VPB_OK;
  VPB_XPLANE_SWITCH(order, rc = launch_vplane_vh<PP>(src_l, src_l_cells, l_cell0, src, src_cells,
                                                     c_cell0, src_r, src_r_cells, r_cell0, dst,
                                                     dims, halo_cells, a1, b1, q1, alpha1, a2, b2,
                                                     q2, alpha2, flag1, flag2, halo_flag, st));
  return rc;
}

extern "C" int vpb_dg_sweep_vplane(const double* src, double* dst, const int64_t dims[4],
                                   int32_t order, const double* a1, const double* b1,
                                   const int64_t* q1, const double* alpha1, const double* a2,
                                   const double* b2, const int64_t* q2, const double* alpha2,
                                   int32_t* flag1, int32_t* flag2, void* stream) {
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1 && order <= kMaxOrder, "order %d outside 1..9", order);
  VPB_REQUIRE(dims[2] % order == 0 && dims[3] % order == 0, "v axes not whole cells");
  VPB_REQUIRE(dims[3] > 1, "fused v sweep needs a 2x2v field");
  cudaStream_t st = (cudaStream_t)stream;
  switch (order) {
    case 1: return launch_vplane<1>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 2: return launch_vplane<2>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 3: return launch_vplane<3>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 4: return launch_vplane<4>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 5: return launch_vplane<5>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 6: return launch_vplane<6>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 7: return launch_vplane<7>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 8: return launch_vplane<8>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    default: return launch_vplane<9>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
  }
}

