// Velocity moments, spectral field solve, diagnostics and initial data.
//
//   vpb_density       <- poisson.compute_density  (poisson.py:85-95)
//   vpb_field_solve   <- poisson.solve_poisson    (poisson.py:123-196)
//   vpb_diagnostics   <- driver.diagnostics       (driver.py:279-316)
//                        + poisson.electric_energy (poisson.py:199-217)
//   vpb_fill_separable<- driver.initialize broadcast product (driver.py:182-198)
//
// All reductions are two-level with a fixed partition that depends only on
// the grid shape, so results are bitwise reproducible run to run and across
// devices.  The Fourier transforms are dense complex matrix products (the
// spatial grid is at most a few hundred points per axis, so a tiled small
// GEMM is both simpler and faster than an FFT plan at this size).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace vpb {

constexpr int kRedThreads = 256;

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV values per thread (deterministic order).  Result is
// valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i][wid] = v[i];
  }
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (wid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double x = lane < nw ? red[i][lane] : 0.0;
      v[i] = warp_sum(x);
    }
  }
}

// ---------------------------------------------------------------------------
// Density: rho[x] = sum_{iv2, iv1} (f * wv1[iv1]) * wv2[iv2]
// ---------------------------------------------------------------------------
static int64_t density_chunks(const int64_t dims[4]) {
  int64_t nx = dims[0] * dims[1];
  int64_t nplanes = dims[2] * dims[3];
  int64_t lanes = std::max<int64_t>(1, nx / 2);
  int64_t ch = std::max<int64_t>(1, 262144 / lanes);
  return std::min(ch, nplanes);
}

template <int VEC>
__global__ void __launch_bounds__(256)
    density_partial_kernel(const double* __restrict__ f, int64_t nx, int64_t nv1, int64_t nplanes,
                           int64_t per_chunk, const double* __restrict__ wv1,
                           const double* __restrict__ wv2, double* __restrict__ part) {
  const int64_t x = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * VEC;
  if (x >= nx) return;
  const int64_t p0 = blockIdx.y * per_chunk;
  const int64_t p1 = min(nplanes, p0 + per_chunk);
  double acc0 = 0.0, acc1 = 0.0;
  int64_t iv1 = p0 % nv1, iv2 = p0 / nv1;
#pragma unroll 4
  for (int64_t p = p0; p < p1; ++p) {
    const double w1 = wv1[iv1], w2 = wv2[iv2];
    if constexpr (VEC == 2) {
      double2 v = __ldcs(reinterpret_cast<const double2*>(f + p * nx + x));
      acc0 += (v.x * w1) * w2;
      acc1 += (v.y * w1) * w2;
    } else {
      acc0 += (__ldcs(f + p * nx + x) * w1) * w2;
    }
    if (++iv1 == nv1) {
      iv1 = 0;
      ++iv2;
    }
  }
  part[blockIdx.y * nx + x] = acc0;
  if constexpr (VEC == 2) part[blockIdx.y * nx + x + 1] = acc1;
}

__global__ void density_final_kernel(const double* __restrict__ part, int64_t nchunks, int64_t nx,
                                     double* __restrict__ rho) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= nx) return;
  double acc = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) acc += part[c * nx + x];
  rho[x] = acc;
}

// ---------------------------------------------------------------------------
// Small complex GEMM: C[i][j] = sum_k A[i][k] * (S[k][j] * B[k][j]).
// Element (i,k) of an operand lives at p[i*rs + k*cs] (complex: 2 doubles).
// ---------------------------------------------------------------------------
struct ZOp {
  const double* p;
  int64_t rs, cs;
  int cplx;  // 0: real operand
  int64_t zstride;  // per-batch offset (in elements)
};

__device__ __forceinline__ double2 zload(const ZOp& o, int64_t i, int64_t k, int z) {
  int64_t e = i * o.rs + k * o.cs + z * o.zstride;
  if (o.cplx) return *reinterpret_cast<const double2*>(o.p + 2 * e);
  return make_double2(o.p[e], 0.0);
}

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void zgemm_kernel(int64_t M, int64_t N, int64_t K, ZOp A, ZOp B, ZOp S, int has_scale,
                             double* __restrict__ Cp, int64_t crs, int64_t ccs, int64_t czs,
                             int real_out, int32_t* __restrict__ flag) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  if (i >= M || j >= N) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t k = 0; k < K; ++k) {
    double2 b = zload(B, k, j, z);
    if (has_scale) b = zmul(zload(S, k, j, z), b);
    double2 a = zload(A, i, k, z);
    acc.x += a.x * b.x - a.y * b.y;
    acc.y += a.x * b.y + a.y * b.x;
  }
  int64_t e = i * crs + j * ccs + z * czs;
  if (real_out) {
    Cp[e] = acc.x;
    report_flag(not_finite(acc.x), flag);
  } else {
    reinterpret_cast<double2*>(Cp)[e] = acc;
  }
}

// Shared-memory tiled variant: an 8 x 8 output tile per 64-thread CTA (more
// CTAs than the 16 x 16 one-output-per-thread kernel for the <= 288-point
// transforms of the field solve), K in steps of 64 staged through shared
// memory (2 instead of 8 load round trips at K = 128: field solve 0.085 ->
// 0.077 ms at config 4); the k order of every sum is unchanged (ascending).
constexpr int kZT = 8, kZK = 64;
__global__ void __launch_bounds__(kZT * kZT)
    zgemm_tiled_kernel(int64_t M, int64_t N, int64_t K, ZOp A, ZOp B, ZOp S, int has_scale,
                       double* __restrict__ Cp, int64_t crs, int64_t ccs, int64_t czs,
                       int real_out, int32_t* __restrict__ flag) {
  __shared__ double2 as[kZT][kZK + 1];
  __shared__ double2 bs[kZK][kZT + 1];
  const int tx = threadIdx.x % kZT, ty = threadIdx.x / kZT;
  const int64_t j = (int64_t)blockIdx.x * kZT + tx;
  const int64_t i = (int64_t)blockIdx.y * kZT + ty;
  const int z = blockIdx.z;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t k0 = 0; k0 < K; k0 += kZK) {
    // 64 threads stage an 8 x 16 slab of A and a 16 x 8 slab of B
    for (int e = threadIdx.x; e < kZT * kZK; e += kZT * kZT) {
      const int r = e / kZK, c = e % kZK;
      const int64_t ai = (int64_t)blockIdx.y * kZT + r, ak = k0 + c;
      as[r][c] = (ai < M && ak < K) ? zload(A, ai, ak, z) : make_double2(0.0, 0.0);
      const int br = e / kZT, bc = e % kZT;
      const int64_t bk = k0 + br, bj = (int64_t)blockIdx.x * kZT + bc;
      double2 b = make_double2(0.0, 0.0);
      if (bk < K && bj < N) {
        b = zload(B, bk, bj, z);
        if (has_scale) b = zmul(zload(S, bk, bj, z), b);
      }
      bs[br][bc] = b;
    }
    __syncthreads();
    const int kn = (int)min((int64_t)kZK, K - k0);
    for (int k = 0; k < kn; ++k) {
      const double2 a = as[ty][k], b = bs[k][tx];
      acc.x += a.x * b.x - a.y * b.y;
      acc.y += a.x * b.y + a.y * b.x;
    }
    __syncthreads();
  }
  if (i >= M || j >= N) return;
  int64_t e = i * crs + j * ccs + z * czs;
  if (real_out) {
    Cp[e] = acc.x;
    report_flag(not_finite(acc.x), flag);
  } else {
    reinterpret_cast<double2*>(Cp)[e] = acc;
  }
}

static int zgemm(int64_t M, int64_t N, int64_t K, int batch, ZOp A, ZOp B, const ZOp* S,
                 double* C, int64_t crs, int64_t ccs, int64_t czs, int real_out, int32_t* flag,
                 cudaStream_t st) {
  ZOp s0 = S ? *S : ZOp{nullptr, 0, 0, 0, 0};
  static const bool naive = getenv("VPB_ZGEMM_NAIVE") != nullptr;
  if (naive) {
    dim3 blk(16, 16);
    dim3 grd((unsigned)((N + 15) / 16), (unsigned)((M + 15) / 16), (unsigned)batch);
    zgemm_kernel<<<grd, blk, 0, st>>>(M, N, K, A, B, s0, S != nullptr, C, crs, ccs, czs,
                                      real_out, flag);
    return launched("zgemm_kernel");
  }
  dim3 grd((unsigned)((N + kZT - 1) / kZT), (unsigned)((M + kZT - 1) / kZT), (unsigned)batch);
  zgemm_tiled_kernel<<<grd, kZT * kZT, 0, st>>>(M, N, K, A, B, s0, S != nullptr, C, crs, ccs,
                                                czs, real_out, flag);
  return launched("zgemm_tiled_kernel");
}

// Weighted mean of rho for the neutrality warning (poisson.py:143-160).
__global__ void density_mean_kernel(const double* __restrict__ rho, int64_t n1, int64_t n2,
                                    const double* __restrict__ wx1,
                                    const double* __restrict__ wx2, double volume,
                                    double* __restrict__ stats) {
  double v[1] = {0.0};
  for (int64_t x = threadIdx.x; x < n1 * n2; x += blockDim.x) {
    int64_t i2 = x / n1, i1 = x - i2 * n1;
    v[0] += wx2[i2] * (wx1[i1] * rho[x]);
  }
  block_sum<1>(v);
  if (threadIdx.x == 0) stats[0] = v[0] / volume;
}

// ---------------------------------------------------------------------------
// Diagnostics: per-plane sums s0 = sum f wx, s1 = sum |f| wx, s2 = sum f^2 wx,
// then a single-block weighted combination over planes.
// ---------------------------------------------------------------------------
static int64_t diag_blocks(const int64_t dims[4]) {
  int64_t nplanes = dims[2] * dims[3];
  return std::min<int64_t>(nplanes, 4096);
}

__global__ void __launch_bounds__(kRedThreads)
    diag_planes_kernel(const double* __restrict__ f, int64_t nx, int64_t nplanes,
                       const double* __restrict__ wx, double* __restrict__ psum) {
  for (int64_t p = blockIdx.x; p < nplanes; p += gridDim.x) {
    const double* fp = f + p * nx;
    double v[3] = {0.0, 0.0, 0.0};
    for (int64_t x = threadIdx.x; x < nx; x += blockDim.x) {
      double a = __ldcs(fp + x), w = wx[x];
      v[0] += a * w;
      v[1] += fabs(a) * w;
      v[2] += (a * a) * w;
    }
    block_sum<3>(v);
    if (threadIdx.x == 0) {
      psum[3 * p + 0] = v[0];
      psum[3 * p + 1] = v[1];
      psum[3 * p + 2] = v[2];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024)
    diag_final_kernel(const double* __restrict__ psum, int64_t nv1, int64_t nv2,
                      const double* __restrict__ wv1, const double* __restrict__ wv2,
                      const double* __restrict__ v1sq, const double* __restrict__ v2sq,
                      const double* __restrict__ e, int32_t ncomp, int64_t nx,
                      const double* __restrict__ wx, double* __restrict__ out) {
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t np = nv1 * nv2;
  for (int64_t p = threadIdx.x; p < np; p += blockDim.x) {
    int64_t i2 = p / nv1, i1 = p - i2 * nv1;
    double w = wv1[i1] * wv2[i2];
    double s0 = psum[3 * p];
    v[0] += s0 * w;
    v[1] += psum[3 * p + 1] * w;
    v[2] += psum[3 * p + 2] * w;
    v[3] += s0 * ((wv1[i1] * v1sq[i1]) * wv2[i2]) + s0 * (wv1[i1] * (wv2[i2] * v2sq[i2]));
  }
  if (e != nullptr) {
    for (int64_t x = threadIdx.x; x < nx * ncomp; x += blockDim.x) {
      double a = e[x];
      v[4] += (a * a) * wx[x % nx];
    }
  }
  block_sum<5>(v);
  if (threadIdx.x == 0) {
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
    out[3] = 0.5 * v[3];
    out[4] = 0.5 * v[4];
  }
}

// ---------------------------------------------------------------------------
// Separable initial data (driver.py:187-198): (g2[iv2]*g1[iv1]) * space[x].
// ---------------------------------------------------------------------------
__global__ void fill_separable_kernel(double* __restrict__ f, int64_t nx, int64_t nv1,
                                      int64_t total, const double* __restrict__ g1,
                                      const double* __restrict__ g2,
                                      const double* __restrict__ space) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  int64_t p = e / nx, x = e - p * nx;
  int64_t i2 = p / nv1, i1 = p - i2 * nv1;
  f[e] = __dmul_rn(__dmul_rn(g2[i2], g1[i1]), space[x]);
}

}  // namespace vpb

using namespace vpb;

extern "C" int64_t vpb_density_work_len(const int64_t dims[4]) {
  return density_chunks(dims) * dims[0] * dims[1];
}

extern "C" int vpb_density(const double* f, const int64_t dims[4], const double* wv1,
                           const double* wv2, double* rho, double* work, void* stream) {
  VPB_REQUIRE(f && wv1 && wv2 && rho && work, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nx = dims[0] * dims[1];
  const int64_t nplanes = dims[2] * dims[3];
  const int64_t nch = density_chunks(dims);
  const int64_t per = (nplanes + nch - 1) / nch;
  const bool vec2 = (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(f) & 15) == 0);
  const int64_t lanes = vec2 ? nx / 2 : nx;
  dim3 grd((unsigned)((lanes + 255) / 256), (unsigned)nch);
  if (vec2)
    density_partial_kernel<2><<<grd, 256, 0, st>>>(f, nx, dims[2], nplanes, per, wv1, wv2, work);
  else
    density_partial_kernel<1><<<grd, 256, 0, st>>>(f, nx, dims[2], nplanes, per, wv1, wv2, work);
  int rc = launched("density_partial_kernel");
  if (rc) return rc;
  density_final_kernel<<<(unsigned)((nx + 255) / 256), 256, 0, st>>>(work, nch, nx, rho);
  return launched("density_final_kernel");
}

extern "C" int64_t vpb_field_work_len(const vpb_field_geom* g) {
  // T [c1][n2] + Rh [c1][c2] + U [ncomp][n1][c2], complex
  return 2 * (g->c1 * g->n2 + g->c1 * g->c2 + (int64_t)g->ncomp * g->n1 * g->c2);
}

extern "C" int vpb_field_solve(const double* rho, const vpb_field_geom* g, double* e,
                               double* stats, double* work, int32_t* flag, void* stream) {
  VPB_REQUIRE(rho && g && e && work, "null pointer");
  VPB_REQUIRE(g->ncomp == 1 || g->ncomp == 2, "ncomp must be 1 or 2");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n1 = g->n1, n2 = g->n2, c1 = g->c1, c2 = g->c2;
  const int64_t r1 = g->r1 > 0 ? g->r1 : n1, r2 = g->r2 > 0 ? g->r2 : n2;  // input grid
  double* T = work;
  double* Rh = T + 2 * c1 * n2;
  double* U = Rh + 2 * c1 * c2;
  int rc;
  if (stats && r1 == n1 && r2 == n2) {
    density_mean_kernel<<<1, 1024, 0, st>>>(rho, n1, n2, g->wx1, g->wx2, g->volume, stats);
    if ((rc = launched("density_mean_kernel"))) return rc;
  }
  // T[k1][i2] = sum_i1 G1[k1][i1] R[i1][i2],  R[i1][i2] = rho[i2*r1+i1]
  rc = zgemm(c1, r2, r1, 1, ZOp{g->g1, r1, 1, 1, 0}, ZOp{rho, 1, r1, 0, 0}, nullptr, T, r2, 1, 0,
             0, nullptr, st);
  if (rc) return rc;
  // Rh[k1][k2] = sum_i2 T[k1][i2] G2[k2][i2]
  rc = zgemm(c1, c2, r2, 1, ZOp{T, r2, 1, 1, 0}, ZOp{g->g2, 1, r2, 1, 0}, nullptr, Rh, c2, 1, 0,
             0, nullptr, st);
  if (rc) return rc;
  // U_d[i1][k2] = sum_k1 M1[i1][k1] (K_d[k1][k2] Rh[k1][k2])
  ZOp kscale{g->kmul, c2, 1, 1, c1 * c2};
  rc = zgemm(n1, c2, c1, g->ncomp, ZOp{g->m1, c1, 1, 1, 0}, ZOp{Rh, c2, 1, 1, 0}, &kscale, U, c2,
             1, n1 * c2, 0, nullptr, st);
  if (rc) return rc;
  // E_d[i2*n1+i1] = Re sum_k2 U_d[i1][k2] M2[i2][k2]
  rc = zgemm(n1, n2, c2, g->ncomp, ZOp{U, c2, 1, 1, n1 * c2}, ZOp{g->m2, 1, c2, 1, 0}, nullptr, e,
             1, n1, n1 * n2, 1, flag, st);
  return rc;
}

extern "C" int64_t vpb_diag_work_len(const int64_t dims[4]) { return 3 * dims[2] * dims[3]; }

extern "C" int vpb_diagnostics(const double* f, const int64_t dims[4], const double* wx,
                               const double* wv1, const double* wv2, const double* v1sq,
                               const double* v2sq, const double* e, int32_t ncomp, double* out,
                               double* work, void* stream) {
  VPB_REQUIRE(f && wx && wv1 && wv2 && v1sq && v2sq && out && work, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nx = dims[0] * dims[1];
  const int64_t nplanes = dims[2] * dims[3];
  diag_planes_kernel<<<(unsigned)diag_blocks(dims), kRedThreads, 0, st>>>(f, nx, nplanes, wx,
                                                                            work);
  int rc = launched("diag_planes_kernel");
  if (rc) return rc;
  diag_final_kernel<<<1, 1024, 0, st>>>(work, dims[2], dims[3], wv1, wv2, v1sq, v2sq, e, ncomp,
                                        nx, wx, out);
  return launched("diag_final_kernel");
}

__global__ void __launch_bounds__(1024)
    electric_energy_kernel(const double* __restrict__ e, int32_t ncomp, int64_t nx,
                           const double* __restrict__ wx, double* __restrict__ out) {
  double v[1] = {0.0};
  for (int64_t x = threadIdx.x; x < nx * ncomp; x += blockDim.x) {
    double a = e[x];
    v[0] += (a * a) * wx[x % nx];
  }
  block_sum<1>(v);
  if (threadIdx.x == 0) out[0] = 0.5 * v[0];
}

extern "C" int vpb_electric_energy(const double* e, int32_t ncomp, int64_t nx, const double* wx,
                                   double* out, void* stream) {
  VPB_REQUIRE(e && wx && out, "null pointer");
  VPB_REQUIRE(ncomp == 1 || ncomp == 2, "ncomp must be 1 or 2");
  electric_energy_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(e, ncomp, nx, wx, out);
  return launched("electric_energy_kernel");
}

extern "C" int vpb_fill_separable(double* f, const int64_t dims[4], const double* g1,
                                  const double* g2, const double* space, void* stream) {
  VPB_REQUIRE(f && g1 && g2 && space, "null pointer");
  const int64_t nx = dims[0] * dims[1];
  const int64_t total = nx * dims[2] * dims[3];
  if (total == 0) return VPB_OK;
  fill_separable_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      f, nx, dims[2], total, g1, g2, space);
  return launched("fill_separable_kernel");
}
