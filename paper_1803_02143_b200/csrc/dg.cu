// Semi-Lagrangian discontinuous Galerkin sweeps for sm_100a.
//
// Reference arithmetic (pkg/src/slvp/_kernels.pyx:96-123, _dg_line):
//   alpha == 0 : out cell c = u cell (c - q) mod C, exact copy
//   otherwise  : out[c*p+j] = (sum_m A[j,m]*u[lo*p+m]) + (sum_m B[j,m]*u[up*p+m])
//                lo = (c-q-1) mod C, up = (c-q) mod C, sums sequential in m.
// The first product of each sum is taken as the initial accumulator (the
// reference adds it to +0.0, which only differs in the sign of an exact zero).
//
// Two kernel shapes:
//   * dg_rows_kernel   - the sweep axis is contiguous (x1 of the canonical
//                        layout, or the plugin's [lines][n] batch).  Row
//                        chunks are staged in shared memory by the bulk-async
//                        copy engine (cp.async.bulk, 2-deep pipeline) and
//                        written back by bulk stores.
//   * dg_cols_kernel   - the sweep axis is strided (x2, v1, v2).  One thread
//                        owns one line, consecutive threads own consecutive
//                        x1 positions (256-B coalesced rows), and the two-cell
//                        stencil slides through registers so every source
//                        cell is read from HBM once.
#include <cmath>
#include <cstdio>
#include <mutex>
#include <type_traits>
#include <vector>

#include "async_copy.cuh"
#include "common.cuh"

namespace vpb {

// ---------------------------------------------------------------------------
// Gauss-Legendre rules on (0, 1) for orders 1..9 (dg.py:25-39) in constant
// memory, plus Lagrange denominators prod_{k!=j}(xi_j - xi_k).
// ---------------------------------------------------------------------------
__constant__ double c_nodes[kMaxOrder + 1][kMaxOrder];
__constant__ double c_weights[kMaxOrder + 1][kMaxOrder];
__constant__ double c_lagden[kMaxOrder + 1][kMaxOrder];

static void gauss_legendre(int n, double* x01, double* w01) {
  // Newton on P_n with the standard cosine initial guesses.
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = x; p0 = 1.0; }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-17) break;
    }
    // recompute derivative at the converged root
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= n; ++k) {
      double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = (n == 1) ? 1.0 : n * (x * p1 - p0) / (x * x - 1.0);
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    // ascending order on (0,1)
    x01[n - 1 - i] = 0.5 * (x + 1.0);
    w01[n - 1 - i] = 0.5 * w;
  }
}

static int ensure_gauss_tables() {
  static std::mutex mu;
  static std::vector<int> done_devices;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return check_launch("cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  for (int d : done_devices)
    if (d == dev) return VPB_OK;
  double nodes[kMaxOrder + 1][kMaxOrder] = {};
  double weights[kMaxOrder + 1][kMaxOrder] = {};
  double lagden[kMaxOrder + 1][kMaxOrder] = {};
  for (int p = 1; p <= kMaxOrder; ++p) {
    gauss_legendre(p, nodes[p], weights[p]);
    for (int j = 0; j < p; ++j) {
      double d = 1.0;
      for (int k = 0; k < p; ++k)
        if (k != j) d *= nodes[p][j] - nodes[p][k];
      lagden[p][j] = d;
    }
  }
  if (cudaMemcpyToSymbol(c_nodes, nodes, sizeof(nodes)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_weights, weights, sizeof(weights)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_lagden, lagden, sizeof(lagden)) != cudaSuccess)
    return check_launch("upload gauss tables");
  done_devices.push_back(dev);
  return VPB_OK;
}

// ---------------------------------------------------------------------------
// K3: projection matrices (dg.py:99-152) in the Lagrange closed form
//   A[j,m] = (alpha/w_j)     sum_g w_g l_j(alpha xi_g)             l_m(alpha xi_g + 1 - alpha)
//   B[j,m] = ((1-alpha)/w_j) sum_g w_g l_j(alpha + (1-alpha) xi_g) l_m((alpha + (1-alpha) xi_g) - alpha)
// which equals the reference's orthonormal-Legendre reproducing-kernel form
// because the Lagrange basis on Gauss nodes is orthogonal with norms w_j.
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void lagrange_all(double x, double (&l)[P]) {
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double num = 1.0;
#pragma unroll
    for (int k = 0; k < P; ++k)
      if (k != j) num *= (x - c_nodes[P][k]);
    l[j] = num / c_lagden[P][j];
  }
}

template <int P>
__global__ void dg_tables_kernel(const double* __restrict__ values, int64_t T, double scale,
                                 double h, double* __restrict__ a, double* __restrict__ b,
                                 int64_t* __restrict__ q, double* __restrict__ alpha) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  // shifts = values*scale (driver.py:224, 238), s = shifts/h (dg.py:116)
  double shift = dmul(values[t], scale);
  double s = __ddiv_rn(shift, h);
  double qf = floor(s);
  double al = dsub(s, qf);
  if (al >= 1.0) {  // carry (dg.py:121-123)
    qf = dadd(qf, 1.0);
    al = 0.0;
  }
  q[t] = (int64_t)qf;
  alpha[t] = al;
  double* A = a + t * P * P;
  double* B = b + t * P * P;
  if (!(al > 0.0)) {
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int m = 0; m < P; ++m) {
        A[j * P + m] = 0.0;
        B[j * P + m] = (j == m) ? 1.0 : 0.0;
      }
    return;
  }
  double oma = 1.0 - al;
  double sa[P][P], sb[P][P];
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int m = 0; m < P; ++m) sa[j][m] = sb[j][m] = 0.0;
#pragma unroll
  for (int g = 0; g < P; ++g) {
    double wg = c_weights[P][g];
    double lj[P], lm[P];
    double xa = al * c_nodes[P][g];
    lagrange_all<P>(xa, lj);
    lagrange_all<P>(xa + oma, lm);
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int m = 0; m < P; ++m) sa[j][m] += wg * lj[j] * lm[m];
    double xb = al + oma * c_nodes[P][g];
    lagrange_all<P>(xb, lj);
    lagrange_all<P>(xb - al, lm);
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int m = 0; m < P; ++m) sb[j][m] += wg * lj[j] * lm[m];
  }
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double fa = al / c_weights[P][j];
    double fb = oma / c_weights[P][j];
#pragma unroll
    for (int m = 0; m < P; ++m) {
      A[j * P + m] = fa * sa[j][m];
      B[j * P + m] = fb * sb[j][m];
    }
  }
}

// ---------------------------------------------------------------------------
// The per-cell update, shared by both kernel shapes.
// ---------------------------------------------------------------------------
template <int P>
struct Coeffs {
  double A[P][P];
  double B[P][P];
  int64_t q;
  bool exact;
};

template <int P>
__device__ __forceinline__ void load_coeffs(Coeffs<P>& k, int64_t t, const double* __restrict__ ta,
                                            const double* __restrict__ tb,
                                            const int64_t* __restrict__ tq,
                                            const double* __restrict__ tal) {
  k.q = tq[t];
  k.exact = (tal[t] == 0.0);
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int m = 0; m < P; ++m) {
      k.A[j][m] = __ldg(ta + t * P * P + j * P + m);
      k.B[j][m] = __ldg(tb + t * P * P + j * P + m);
    }
}

template <int P>
__device__ __forceinline__ void cell_update(const Coeffs<P>& k, const double (&lo)[P],
                                            const double (&up)[P], double (&out)[P]) {
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double acc_a = dmul(k.A[j][0], lo[0]);
#pragma unroll
    for (int m = 1; m < P; ++m) acc_a = dadd(acc_a, dmul(k.A[j][m], lo[m]));
    double acc_b = dmul(k.B[j][0], up[0]);
#pragma unroll
    for (int m = 1; m < P; ++m) acc_b = dadd(acc_b, dmul(k.B[j][m], up[m]));
    out[j] = dadd(acc_a, acc_b);
  }
}

template <int P>
__device__ __forceinline__ void lds_cell(const double* p, double (&u)[P]) {
  if constexpr (P % 2 == 0) {
#pragma unroll
    for (int m = 0; m < P; m += 2) {
      double2 v = *reinterpret_cast<const double2*>(p + m);
      u[m] = v.x;
      u[m + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int m = 0; m < P; ++m) u[m] = p[m];
  }
}

template <int P>
__device__ __forceinline__ void sts_cell(double* p, const double (&u)[P]) {
  if constexpr (P % 2 == 0) {
#pragma unroll
    for (int m = 0; m < P; m += 2) *reinterpret_cast<double2*>(p + m) = make_double2(u[m], u[m + 1]);
  } else {
#pragma unroll
    for (int m = 0; m < P; ++m) p[m] = u[m];
  }
}

// ---------------------------------------------------------------------------
// K1: contiguous-axis sweep.  A persistent CTA owns `rows_per_block`
// consecutive rows (whole (iv2, iv1) planes in the product layout, so the
// projection coefficients stay in registers) and streams them through
// shared memory in chunks of R rows: kStages bulk-async loads (TMA 1-D
// bulk copies completing on mbarriers) are in flight while one chunk is
// computed, and results leave through double-buffered bulk stores.  One
// __syncthreads per chunk.  Thread layout inside a chunk: cpp cells x rpp
// rows.
// ---------------------------------------------------------------------------
constexpr int kStages = 4;

template <int P>
__global__ void __launch_bounds__(256, 2)
    dg_rows_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nrows, int C,
                   int64_t rows_per_block, int R, int cpp, int rpp,
                   const int64_t* __restrict__ idx, int64_t tdiv, int64_t tmod,
                   const double* __restrict__ ta, const double* __restrict__ tb,
                   const int64_t* __restrict__ tq, const double* __restrict__ tal,
                   int32_t* __restrict__ flag) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n = C * P;
  const int chunk = R * n;
  double* inb = reinterpret_cast<double*>(smem_raw);
  double* outb = inb + kStages * chunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(outb + 2 * chunk);

  const int tid = threadIdx.x;
  const int64_t r_begin = blockIdx.x * rows_per_block;
  const int64_t r_end = min(nrows, r_begin + rows_per_block);
  if (r_begin >= r_end) return;
  const int nchunks = (int)((r_end - r_begin + R - 1) / R);

  auto issue_load = [&](int kc) {
    int64_t r0 = r_begin + (int64_t)kc * R;
    int rows = (int)min((int64_t)R, r_end - r0);
    uint32_t bytes = (uint32_t)rows * n * 8u;
    uint64_t* bar = bars + (kc % kStages);
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(inb + (kc % kStages) * chunk, src + r0 * n, bytes, bar);
  };

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages && s < nchunks; ++s) issue_load(s);
  }

  const bool active = tid < cpp * rpp;
  const int c0 = tid % cpp;
  const int rr0 = tid / cpp;
  int64_t cached = -1;
  Coeffs<P> k;
  k.q = 0;
  k.exact = true;
  int qm = 0;
  bool bad = false;

  for (int kc = 0; kc < nchunks; ++kc) {
    const int s = kc % kStages;
    const int64_t r0 = r_begin + (int64_t)kc * R;
    const int rows = (int)min((int64_t)R, r_end - r0);
    mbar_wait(bars + s, (kc / kStages) & 1);
    const double* in = inb + s * chunk;
    double* out = outb + (kc & 1) * chunk;
    if (active) {
      for (int r = rr0; r < rows; r += rpp) {
        const int64_t grow = r0 + r;
        const int64_t t = idx ? idx[grow] : (grow / tdiv) % tmod;
        if (t != cached) {
          load_coeffs<P>(k, t, ta, tb, tq, tal);
          qm = (int)wrap_mod(k.q, C);
          cached = t;
        }
        const double* rin = in + r * n;
        double* rout = out + r * n;
        for (int c = c0; c < C; c += cpp) {
          int lo = c - qm - 1;
          if (lo < 0) lo += C;
          int up = lo + 1;
          if (up == C) up = 0;
          double uu[P], res[P];
          lds_cell<P>(rin + up * P, uu);
          if (k.exact) {
#pragma unroll
            for (int j = 0; j < P; ++j) res[j] = uu[j];
          } else {
            double ul[P];
            lds_cell<P>(rin + lo * P, ul);
            cell_update<P>(k, ul, uu, res);
          }
#pragma unroll
          for (int j = 0; j < P; ++j) bad |= not_finite(res[j]);
          sts_cell<P>(rout + c * P, res);
        }
      }
    }
    fence_proxy_async_smem();
    // the store of chunk kc-1 must have finished reading outb[(kc+1)&1]
    // before anyone computes chunk kc+1 into it
    if (tid == 0) bulk_wait_read<0>();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(dst + r0 * n, out, (uint32_t)rows * n * 8u);
      bulk_commit();
      if (kc + kStages < nchunks) issue_load(kc + kStages);
    }
  }
  if (tid == 0) bulk_wait<0>();
  report_flag(bad, flag);
}

// Fallback for rows whose byte length is not a multiple of 16 (odd n): one
// thread per output cell straight from global memory.
template <int P>
__global__ void dg_rows_simple_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                      int64_t nrows, int C, const int64_t* __restrict__ idx,
                                      int64_t tdiv, int64_t tmod, const double* __restrict__ ta,
                                      const double* __restrict__ tb,
                                      const int64_t* __restrict__ tq,
                                      const double* __restrict__ tal, int32_t* __restrict__ flag) {
  int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it >= nrows * C) return;
  int64_t row = it / C;
  int c = (int)(it - row * C);
  int64_t t = idx ? idx[row] : (row / tdiv) % tmod;
  Coeffs<P> k;
  load_coeffs<P>(k, t, ta, tb, tq, tal);
  int qm = (int)wrap_mod(k.q, C);
  int lo = c - qm - 1;
  if (lo < 0) lo += C;
  int up = lo + 1;
  if (up == C) up = 0;
  const double* rin = src + row * (int64_t)C * P;
  double uu[P], res[P];
#pragma unroll
  for (int m = 0; m < P; ++m) uu[m] = rin[up * P + m];
  if (k.exact) {
#pragma unroll
    for (int j = 0; j < P; ++j) res[j] = uu[j];
  } else {
    double ul[P];
#pragma unroll
    for (int m = 0; m < P; ++m) ul[m] = rin[lo * P + m];
    cell_update<P>(k, ul, uu, res);
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    dst[row * (int64_t)C * P + c * P + j] = res[j];
    bad |= not_finite(res[j]);
  }
  report_flag(bad, flag);
}

// ---------------------------------------------------------------------------
// K2: strided-axis sweep.  Line id L = outer*S + inner; the line's dofs sit
// at base + (cell*P + m)*S.  VEC=2 processes two adjacent lines with 16-B
// accesses (requires a table row shared by both lines and even S).
// ---------------------------------------------------------------------------
template <int P, int VEC>
__global__ void __launch_bounds__(256)
    dg_cols_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t S, int64_t O,
                   int C, int64_t tdiv, int64_t tmod, const double* __restrict__ ta,
                   const double* __restrict__ tb, const int64_t* __restrict__ tq,
                   const double* __restrict__ tal, int32_t* __restrict__ flag) {
  using vec_t = typename std::conditional<VEC == 2, double2, double>::type;
  const int64_t L = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * VEC;
  if (L >= O * S) return;
  const int64_t outer = L / S;
  const int64_t inner = L - outer * S;
  const int64_t t = (L / tdiv) % tmod;
  const int64_t cs = (int64_t)P * S;  // cell stride
  const double* sp = src + outer * cs * C + inner;
  double* dp = dst + outer * cs * C + inner;

  Coeffs<P> k;
  load_coeffs<P>(k, t, ta, tb, tq, tal);
  const int qm = (int)wrap_mod(k.q, C);
  bool bad = false;

  auto ld = [&](int cell, vec_t (&u)[P]) {
#pragma unroll
    for (int m = 0; m < P; ++m)
      u[m] = *reinterpret_cast<const vec_t*>(sp + cell * cs + m * S);
  };
  auto st = [&](int cell, const vec_t (&u)[P]) {
#pragma unroll
    for (int m = 0; m < P; ++m) *reinterpret_cast<vec_t*>(dp + cell * cs + m * S) = u[m];
  };

  int up = C - qm;  // source cell of output 0: (0 - q) mod C
  if (up == C) up = 0;
  if (k.exact) {
    for (int c = 0; c < C; ++c) {
      vec_t u[P];
      ld(up, u);
      st(c, u);
      if constexpr (VEC == 2) {
#pragma unroll
        for (int m = 0; m < P; ++m) bad |= not_finite(u[m].x) | not_finite(u[m].y);
      } else {
#pragma unroll
        for (int m = 0; m < P; ++m) bad |= not_finite(u[m]);
      }
      if (++up == C) up = 0;
    }
    report_flag(bad, flag);
    return;
  }
  int lo = up - 1;
  if (lo < 0) lo += C;
  vec_t prev[P];
  ld(lo, prev);
  // G source cells are loaded back to back before any of them is used, so
  // each thread keeps G*P independent loads in flight.
  constexpr int G = (VEC == 2 || P > 4) ? 2 : 4;
  auto step = [&](int c, const vec_t (&cur)[P]) {
    vec_t res[P];
    if constexpr (VEC == 2) {
      double l0[P], u0[P], r0[P], l1[P], u1[P], r1[P];
#pragma unroll
      for (int m = 0; m < P; ++m) {
        l0[m] = prev[m].x;
        l1[m] = prev[m].y;
        u0[m] = cur[m].x;
        u1[m] = cur[m].y;
      }
      cell_update<P>(k, l0, u0, r0);
      cell_update<P>(k, l1, u1, r1);
#pragma unroll
      for (int m = 0; m < P; ++m) {
        res[m] = make_double2(r0[m], r1[m]);
        bad |= not_finite(r0[m]) | not_finite(r1[m]);
      }
    } else {
      cell_update<P>(k, prev, cur, res);
#pragma unroll
      for (int m = 0; m < P; ++m) bad |= not_finite(res[m]);
    }
    st(c, res);
#pragma unroll
    for (int m = 0; m < P; ++m) prev[m] = cur[m];
  };
  int c = 0;
  for (; c + G <= C; c += G) {
    vec_t cur[G][P];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      ld(up, cur[g]);
      if (++up == C) up = 0;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) step(c + g, cur[g]);
  }
  for (; c < C; ++c) {
    vec_t cur[P];
    ld(up, cur);
    if (++up == C) up = 0;
    step(c, cur);
  }
  report_flag(bad, flag);
}

// ---------------------------------------------------------------------------
// Gather/scatter between a 4-D strided view and contiguous lines.
// ---------------------------------------------------------------------------
__global__ void gather4d_kernel(const double* __restrict__ view, double* __restrict__ lines,
                                int64_t s0, int64_t s1, int64_t s2, int64_t n, int64_t st0,
                                int64_t st1, int64_t st2, int64_t st3, int scatter,
                                double* __restrict__ view_out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = s0 * s1 * s2 * n;
  if (e >= total) return;
  int64_t r = e / n, kk = e - r * n;
  int64_t i2 = r % s2;
  int64_t r2 = r / s2;
  int64_t i1 = r2 % s1;
  int64_t i0 = r2 / s1;
  int64_t off = i0 * st0 + i1 * st1 + i2 * st2 + kk * st3;
  if (scatter)
    view_out[off] = lines[e];
  else
    lines[e] = view[off];
}

// ---------------------------------------------------------------------------
// Host-side launchers
// ---------------------------------------------------------------------------
static int sm_count() {
  static int cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

struct RowsArgs {
  const double* src;
  double* dst;
  int64_t nrows;
  int C;
  int64_t rows_per_block;  // <= 0: choose
  const int64_t* idx;
  int64_t tdiv, tmod;
  const double *a, *b;
  const int64_t* q;
  const double* alpha;
  int32_t* flag;
};

template <int P>
static int launch_rows(const RowsArgs& g, cudaStream_t st) {
  const int n = g.C * P;
  if (g.nrows == 0) return VPB_OK;
  bool aligned = (n % 2 == 0) && ((reinterpret_cast<uintptr_t>(g.src) & 15) == 0) &&
                 ((reinterpret_cast<uintptr_t>(g.dst) & 15) == 0);
  if (!aligned) {
    int64_t items = g.nrows * g.C;
    int64_t blocks = (items + 255) / 256;
    dg_rows_simple_kernel<P><<<(unsigned)blocks, 256, 0, st>>>(
        g.src, g.dst, g.nrows, g.C, g.idx, g.tdiv, g.tmod, g.a, g.b, g.q, g.alpha, g.flag);
    return launched("dg_rows_simple_kernel");
  }
  const int target_bytes = 12288;
  int R = (int)std::max<int64_t>(1, target_bytes / (n * 8));
  int64_t unit = g.rows_per_block > 0 ? g.rows_per_block : R;  // rows that share coefficients
  int cpp = std::min(g.C, 256);
  int rpp = std::max(1, 256 / g.C);
  if (rpp > R) rpp = R;
  int threads = cpp * rpp;
  threads = ((threads + 31) / 32) * 32;
  size_t smem = (size_t)(kStages + 2) * R * n * sizeof(double) + kStages * sizeof(uint64_t);
  if (smem > 110 * 1024) {
    set_error("dg row of %d dofs does not fit the shared-memory pipeline", n);
    return VPB_ERR_UNSUPPORTED;
  }
  static bool attr_set[kMaxOrder + 1] = {};
  if (!attr_set[P]) {
    cudaFuncSetAttribute(dg_rows_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         110 * 1024);
    attr_set[P] = true;
  }
  // persistent grid: 2 CTAs per SM, each owning a contiguous run of units
  int64_t units = (g.nrows + unit - 1) / unit;
  int64_t grid = std::min<int64_t>(units, 2 * (int64_t)sm_count());
  int64_t rpb = ((units + grid - 1) / grid) * unit;
  int64_t blocks = (g.nrows + rpb - 1) / rpb;
  dg_rows_kernel<P><<<(unsigned)blocks, threads, smem, st>>>(
      g.src, g.dst, g.nrows, g.C, rpb, R, cpp, rpp, g.idx, g.tdiv, g.tmod, g.a, g.b, g.q,
      g.alpha, g.flag);
  return launched("dg_rows_kernel");
}

struct ColsArgs {
  const double* src;
  double* dst;
  int64_t S, O;
  int C;
  int64_t tdiv, tmod;
  bool uniform_pairs;  // table row shared by lines L, L+1 for even L
  const double *a, *b;
  const int64_t* q;
  const double* alpha;
  int32_t* flag;
};

template <int P>
static int launch_cols(const ColsArgs& g, cudaStream_t st) {
  int64_t lines = g.O * g.S;
  if (lines == 0) return VPB_OK;
  bool vec2 = g.uniform_pairs && (g.S % 2 == 0) &&
              ((reinterpret_cast<uintptr_t>(g.src) & 15) == 0) &&
              ((reinterpret_cast<uintptr_t>(g.dst) & 15) == 0);
  if (vec2) {
    int64_t threads = lines / 2;
    int64_t blocks = (threads + 255) / 256;
    dg_cols_kernel<P, 2><<<(unsigned)blocks, 256, 0, st>>>(
        g.src, g.dst, g.S, g.O, g.C, g.tdiv, g.tmod, g.a, g.b, g.q, g.alpha, g.flag);
  } else {
    int64_t blocks = (lines + 255) / 256;
    dg_cols_kernel<P, 1><<<(unsigned)blocks, 256, 0, st>>>(
        g.src, g.dst, g.S, g.O, g.C, g.tdiv, g.tmod, g.a, g.b, g.q, g.alpha, g.flag);
  }
  return launched("dg_cols_kernel");
}

#define VPB_DISPATCH_ORDER(P_, FN, ...)                                \
  switch (P_) {                                                        \
    case 1: return FN<1>(__VA_ARGS__);                                 \
    case 2: return FN<2>(__VA_ARGS__);                                 \
    case 3: return FN<3>(__VA_ARGS__);                                 \
    case 4: return FN<4>(__VA_ARGS__);                                 \
    case 5: return FN<5>(__VA_ARGS__);                                 \
    case 6: return FN<6>(__VA_ARGS__);                                 \
    case 7: return FN<7>(__VA_ARGS__);                                 \
    case 8: return FN<8>(__VA_ARGS__);                                 \
    case 9: return FN<9>(__VA_ARGS__);                                 \
    default:                                                           \
      set_error("dG order %d outside the supported range 1..9", P_);   \
      return VPB_ERR_UNSUPPORTED;                                      \
  }

template <int P>
static int launch_tables(const double* values, int64_t T, double scale, double h, double* a,
                         double* b, int64_t* q, double* alpha, cudaStream_t st) {
  if (T == 0) return VPB_OK;
  int64_t blocks = (T + 127) / 128;
  dg_tables_kernel<P><<<(unsigned)blocks, 128, 0, st>>>(values, T, scale, h, a, b, q, alpha);
  return launched("dg_tables_kernel");
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_dg_tables(const double* values, int64_t ntable, double scale, double h,
                             int32_t order, double* a, double* b, int64_t* q, double* alpha,
                             void* stream) {
  VPB_REQUIRE(h > 0.0, "cell width must be positive, got %g", h);
  VPB_REQUIRE(ntable >= 0, "negative table length");
  VPB_REQUIRE(ntable == 0 || (values && a && b && q && alpha), "null table pointer");
  int rc = ensure_gauss_tables();
  if (rc) return rc;
  VPB_DISPATCH_ORDER(order, launch_tables, values, ntable, scale, h, a, b, q, alpha,
                     (cudaStream_t)stream);
}

extern "C" int vpb_dg_sweep_contig(const double* lines, double* out, int64_t nlines, int64_t n,
                                   const int64_t* idx, const double* a, const double* b,
                                   const int64_t* q, const double* alpha, int64_t ntable,
                                   int32_t ncells, int32_t nloc, void* stream) {
  VPB_REQUIRE(nloc >= 1 && ncells >= 1, "ncells and nloc must be positive");
  VPB_REQUIRE((int64_t)ncells * nloc == n, "line length %lld != ncells*nloc", (long long)n);
  VPB_REQUIRE(lines != out, "out must not alias lines");
  VPB_REQUIRE(idx != nullptr && ntable > 0, "table index required");
  RowsArgs g{lines, out, nlines, ncells, 0, idx, 1, ntable, a, b, q, alpha, nullptr};
  VPB_DISPATCH_ORDER(nloc, launch_rows, g, (cudaStream_t)stream);
}

extern "C" int vpb_dg_sweep_strided(double* view, const int64_t shape[4],
                                    const int64_t strides[4], const int64_t* idx,
                                    const double* a, const double* b, const int64_t* q,
                                    const double* alpha, int64_t ntable, int32_t ncells,
                                    int32_t nloc, void* stream) {
  VPB_REQUIRE(shape[3] == (int64_t)ncells * nloc, "line length != ncells*nloc");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nlines = shape[0] * shape[1] * shape[2];
  int64_t total = nlines * shape[3];
  if (total == 0) return VPB_OK;
  double* tmp = nullptr;
  if (cudaMallocAsync(&tmp, 2 * total * sizeof(double), st) != cudaSuccess)
    return check_launch("cudaMallocAsync");
  int64_t blocks = (total + 255) / 256;
  gather4d_kernel<<<(unsigned)blocks, 256, 0, st>>>(view, tmp, shape[0], shape[1], shape[2],
                                                    shape[3], strides[0], strides[1],
                                                    strides[2], strides[3], 0, nullptr);
  int rc = vpb_dg_sweep_contig(tmp, tmp + total, nlines, shape[3], idx, a, b, q, alpha, ntable,
                               ncells, nloc, stream);
  if (rc == VPB_OK) {
    gather4d_kernel<<<(unsigned)blocks, 256, 0, st>>>(nullptr, tmp + total, shape[0], shape[1],
                                                      shape[2], shape[3], strides[0],
                                                      strides[1], strides[2], strides[3], 1,
                                                      view);
    rc = launched("gather4d_kernel", 2);
  }
  cudaFreeAsync(tmp, st);
  return rc;
}

extern "C" int vpb_dg_sweep_axis(int32_t axis, const double* src, double* dst,
                                 const int64_t dims[4], int32_t order, const double* a,
                                 const double* b, const int64_t* q, const double* alpha,
                                 int32_t* flag, void* stream) {
  VPB_REQUIRE(axis >= 0 && axis < 4, "axis %d out of range", axis);
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1, "order must be positive");
  const int64_t n1 = dims[0], n2 = dims[1], nv1 = dims[2], nv2 = dims[3];
  VPB_REQUIRE(dims[axis] % order == 0, "axis length %lld is not a multiple of %d",
              (long long)dims[axis], order);
  const int C = (int)(dims[axis] / order);
  cudaStream_t st = (cudaStream_t)stream;
  if (axis == 0) {
    // rows = (iv2, iv1, ix2); table row = iv1.  A block spans whole
    // (iv2, iv1) planes so its coefficients stay in registers.
    int64_t nrows = n2 * nv1 * nv2;
    int64_t rpb = n2;  // one (iv2, iv1) plane shares its coefficients
    RowsArgs g{src, dst, nrows, C, rpb, nullptr, n2, nv1, a, b, q, alpha, flag};
    VPB_DISPATCH_ORDER(order, launch_rows, g, st);
  }
  ColsArgs g{src, dst, 0, 0, C, 1, 1, false, a, b, q, alpha, flag};
  if (axis == 1) {
    g.S = n1;
    g.O = nv1 * nv2;
    g.tdiv = n1 * nv1;  // table row = iv2
    g.tmod = nv2;
    g.uniform_pairs = true;
  } else if (axis == 2) {
    g.S = n1 * n2;
    g.O = nv2;
    g.tdiv = 1;  // table row = x index
    g.tmod = n1 * n2;
  } else {
    g.S = n1 * n2 * nv1;
    g.O = 1;
    g.tdiv = 1;
    g.tmod = n1 * n2;
  }
  VPB_DISPATCH_ORDER(order, launch_cols, g, st);
}
