// Fused dG sweeps: both space sweeps of a Strang half step in one HBM pass.
//
// In the reference, _advect_space (driver.py:220-228) sweeps x1 and then x2,
// each a full read+write of f.  Inside one (iv2, iv1) plane both shifts are
// constant (x1 shift from v1, x2 shift from v2), so the plane can be swept
// along x1 and then x2 while it streams through shared memory:
//
//   for every source x2-cell s of the plane (in the order the x2 stencil
//   consumes them, starting at (-q2-1) mod C2, one extra to close the wrap):
//     TMA-bulk-load the p rows of cell s into shared memory
//     g(s)   = x1 sweep of those rows                 (registers)
//     out    = A2 g(s-1) + B2 g(s)  -> x2-cell s+q2   (shared -> bulk store)
//
// Every element goes through exactly the operations of the two separate
// sweeps (same order, no contraction), so the result is bitwise the
// unfused x1-then-x2 sequence, with 16 B/dof of traffic instead of 32.
//
// Thread t of a CTA owns x1 dof t (cell t/p, node t%p) of every row.  CTAs
// are persistent: each walks a contiguous run of planes while the bulk-copy
// pipeline (kXStages chunks in flight) runs ahead across plane boundaries.
#include <algorithm>

#include "async_copy.cuh"
#include "common.cuh"

namespace vpb {

constexpr int kXStages = 6;

template <int P>
__global__ void __launch_bounds__(256, 2)
    dg_xplane_kernel(const double* __restrict__ src, double* __restrict__ dst, int n1, int C2,
                     int64_t nv1, int64_t nplanes, int64_t planes_per_block,
                     const double* __restrict__ a1, const double* __restrict__ b1,
                     const int64_t* __restrict__ q1, const double* __restrict__ al1,
                     const double* __restrict__ a2, const double* __restrict__ b2,
                     const int64_t* __restrict__ q2, const double* __restrict__ al2,
                     int32_t* __restrict__ flag1, int32_t* __restrict__ flag2) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int chunk = P * n1;  // one x2 cell: P rows of n1 dofs
  double* inb = reinterpret_cast<double*>(smem_raw);
  double* outb = inb + kXStages * chunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(outb + 2 * chunk);

  const int tid = threadIdx.x;
  const int64_t pl_begin = blockIdx.x * planes_per_block;
  const int64_t pl_end = min(nplanes, pl_begin + planes_per_block);
  if (pl_begin >= pl_end) return;
  const int per_plane = C2 + 1;
  const int64_t nchunks = (pl_end - pl_begin) * per_plane;
  const int64_t plane_elems = (int64_t)C2 * chunk;

  // Producer (thread 0): chunk j = (plane pl_begin + j / per_plane, step j % per_plane)
  auto issue_load = [&](int64_t j) {
    const int64_t pl = pl_begin + j / per_plane;
    const int k = (int)(j % per_plane);
    const int64_t iv2 = pl / nv1;
    const int qm = (int)wrap_mod(q2[iv2], C2);
    int s = C2 - qm - 1 + k;  // source cell (-q2-1+k) mod C2
    while (s >= C2) s -= C2;
    const int st = (int)(j % kXStages);
    mbar_arrive_expect_tx(bars + st, (uint32_t)chunk * 8u);
    bulk_g2s(inb + st * chunk, src + pl * plane_elems + (int64_t)s * chunk, (uint32_t)chunk * 8u,
             bars + st);
  };

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kXStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t j = 0; j < kXStages && j < nchunks; ++j) issue_load(j);

  const bool active = tid < n1;
  const int c1 = tid / P, j1 = tid % P;
  const int C1 = n1 / P;
  double A1[P], B1[P], A2[P][P], B2[P][P];
  bool ex1 = true, ex2 = true;
  int lo1 = 0, up1 = 0;
  double gprev[P], gcur[P];
  bool bad1 = false, bad2 = false;
#pragma unroll
  for (int m = 0; m < P; ++m) gprev[m] = gcur[m] = 0.0;

  int64_t j = 0;
  for (int64_t pl = pl_begin; pl < pl_end; ++pl) {
    const int64_t iv2 = pl / nv1, iv1 = pl - iv2 * nv1;
    const int qm2 = (int)wrap_mod(q2[iv2], C2);
    if (active) {
      // per-plane coefficients: row j1 of the x1 pair, full x2 pair
      ex1 = (al1[iv1] == 0.0);
      ex2 = (al2[iv2] == 0.0);
#pragma unroll
      for (int m = 0; m < P; ++m) {
        A1[m] = __ldg(a1 + iv1 * P * P + j1 * P + m);
        B1[m] = __ldg(b1 + iv1 * P * P + j1 * P + m);
      }
#pragma unroll
      for (int jj = 0; jj < P; ++jj)
#pragma unroll
        for (int m = 0; m < P; ++m) {
          A2[jj][m] = __ldg(a2 + iv2 * P * P + jj * P + m);
          B2[jj][m] = __ldg(b2 + iv2 * P * P + jj * P + m);
        }
      const int qm1 = (int)wrap_mod(q1[iv1], C1);
      lo1 = c1 - qm1 - 1;
      if (lo1 < 0) lo1 += C1;
      up1 = lo1 + 1 == C1 ? 0 : lo1 + 1;
    }
    for (int k = 0; k < per_plane; ++k, ++j) {
      const int st = (int)(j % kXStages);
      mbar_wait(bars + st, (uint32_t)((j / kXStages) & 1));
      const double* in = inb + st * chunk;
      double* out = outb + (j & 1) * chunk;
      if (active) {
        // x1 sweep of the P rows of this x2 cell, dof `tid` (_kernels.pyx:113-123)
#pragma unroll
        for (int m2 = 0; m2 < P; ++m2) {
          const double* row = in + m2 * n1;
          double v;
          if (ex1) {
            v = row[up1 * P + j1];
          } else {
            double acc_a = dmul(A1[0], row[lo1 * P]);
#pragma unroll
            for (int m = 1; m < P; ++m) acc_a = dadd(acc_a, dmul(A1[m], row[lo1 * P + m]));
            double acc_b = dmul(B1[0], row[up1 * P]);
#pragma unroll
            for (int m = 1; m < P; ++m) acc_b = dadd(acc_b, dmul(B1[m], row[up1 * P + m]));
            v = dadd(acc_a, acc_b);
          }
          gcur[m2] = v;
          bad1 |= not_finite(v);
        }
        if (k > 0) {
          // x2 sweep: output cell k-1 from g(s-1), g(s)
#pragma unroll
          for (int jj = 0; jj < P; ++jj) {
            double o;
            if (ex2) {
              o = gcur[jj];
            } else {
              double acc_a = dmul(A2[jj][0], gprev[0]);
#pragma unroll
              for (int m = 1; m < P; ++m) acc_a = dadd(acc_a, dmul(A2[jj][m], gprev[m]));
              double acc_b = dmul(B2[jj][0], gcur[0]);
#pragma unroll
              for (int m = 1; m < P; ++m) acc_b = dadd(acc_b, dmul(B2[jj][m], gcur[m]));
              o = dadd(acc_a, acc_b);
            }
            bad2 |= not_finite(o);
            out[jj * n1 + tid] = o;
          }
        }
#pragma unroll
        for (int m = 0; m < P; ++m) gprev[m] = gcur[m];
      }
      fence_proxy_async_smem();
      if (tid == 0) bulk_wait_read<0>();  // store of chunk j-1 released outb[(j+1)&1]
      __syncthreads();
      if (tid == 0) {
        if (k > 0) {
          // output x2 cell c2 = k-1 (exact: (c2 - q2) mod C2 source pairing)
          bulk_s2g(dst + pl * plane_elems + (int64_t)(k - 1) * chunk, out, (uint32_t)chunk * 8u);
          bulk_commit();
        }
        if (j + kXStages < nchunks) issue_load(j + kXStages);
      }
    }
    (void)qm2;
  }
  if (tid == 0) bulk_wait<0>();
  report_flag(bad1, flag1);
  report_flag(bad2, flag2);
}

static int xplane_sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached = v > 0 ? v : 148;
  }
  return cached;
}

template <int P>
static int launch_xplane(const double* src, double* dst, const int64_t dims[4], const double* a1,
                         const double* b1, const int64_t* q1, const double* al1,
                         const double* a2, const double* b2, const int64_t* q2,
                         const double* al2, int32_t* f1, int32_t* f2, cudaStream_t st) {
  const int n1 = (int)dims[0];
  const int C2 = (int)(dims[1] / P);
  const int64_t nv1 = dims[2];
  const int64_t nplanes = dims[2] * dims[3];
  if (nplanes == 0) return VPB_OK;
  const int threads = ((n1 + 31) / 32) * 32;
  if (threads > 1024) {
    set_error("x rows of %d dofs exceed one CTA", n1);
    return VPB_ERR_UNSUPPORTED;
  }
  const size_t smem = (size_t)(kXStages + 2) * P * n1 * sizeof(double) + kXStages * 8;
  if (smem > 200 * 1024) {
    set_error("x plane chunk of %d dofs does not fit shared memory", P * n1);
    return VPB_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dg_xplane_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dg_xplane_kernel<P>, threads, smem);
  if (occ < 1) occ = 1;
  const int64_t grid = std::min<int64_t>(nplanes, (int64_t)occ * xplane_sm_count());
  const int64_t ppb = (nplanes + grid - 1) / grid;
  const int64_t blocks = (nplanes + ppb - 1) / ppb;
  dg_xplane_kernel<P><<<(unsigned)blocks, threads, smem, st>>>(
      src, dst, n1, C2, nv1, nplanes, ppb, a1, b1, q1, al1, a2, b2, q2, al2, f1, f2);
  return check_launch("dg_xplane_kernel");
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_dg_sweep_xplane(const double* src, double* dst, const int64_t dims[4],
                                   int32_t order, const double* a1, const double* b1,
                                   const int64_t* q1, const double* alpha1, const double* a2,
                                   const double* b2, const int64_t* q2, const double* alpha2,
                                   int32_t* flag1, int32_t* flag2, void* stream) {
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1 && order <= kMaxOrder, "order %d outside 1..9", order);
  VPB_REQUIRE(dims[0] % order == 0 && dims[1] % order == 0, "x axes not whole cells");
  VPB_REQUIRE(dims[1] > 1, "fused x sweep needs a 2x2v field");
  VPB_REQUIRE((dims[0] * order) % 2 == 0, "x1 rows must be a multiple of 16 bytes per cell row");
  VPB_REQUIRE((reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
              "field buffers must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  switch (order) {
    case 1: return launch_xplane<1>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 2: return launch_xplane<2>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 3: return launch_xplane<3>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 4: return launch_xplane<4>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 5: return launch_xplane<5>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 6: return launch_xplane<6>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 7: return launch_xplane<7>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    case 8: return launch_xplane<8>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
    default: return launch_xplane<9>(src, dst, dims, a1, b1, q1, alpha1, a2, b2, q2, alpha2, flag1, flag2, st);
  }
}
