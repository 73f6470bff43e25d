// Periodic cubic-spline sweeps for sm_100a.
//
// Reference arithmetic (pkg/src/slvp/_kernels.pyx:37-93, _kernels_py.py:16-77):
//   solve  y = 6u; y_i -= mult_i*y_{i-1}; y_{n-1} /= denom_{n-1};
//          y_i = (y_i - y_{i+1}) / denom_i; fac = (y_0 - 0.25 y_{n-1}) / sden;
//          w_i = y_i - fac*z_i
//   eval   s = shift/h; off = floor(-s); theta = -s - off (carry theta>=1);
//          out_i = w0 om[j0+i] + w1 om[j0+i+1] + w2 om[j0+i+2] + w3 om[j0+i+3]
//          with j0 = (off-1) mod n, summed left to right.
// Every operation keeps the reference's order and rounding (no contraction).
// The divisions by the constant denominators use the Markstein sequence
//   q = y*r;  e = fma(-q, d, y);  q' = fma(e, r, q)      (r = RN(1/d))
// which returns the correctly rounded y/d for all finite normal operands, so
// the result is bitwise that of the reference's `/`.
//
// Kernel shape: a CTA owns a tile of T lines.  The tile is staged in shared
// memory in [point][line] order, each thread runs the sequential Thomas
// recurrence on its own line (the recurrence is latency bound, so the tile
// is sized to keep several CTAs per SM), then the evaluation is remapped so
// that stores are coalesced along the memory-contiguous direction.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "async_copy.cuh"
#include "common.cuh"
#include "tensormap.cuh"

namespace vpb {
int xplane_sm_count();  // fused.cu

constexpr int kSplineT = 32;   // lines per CTA
constexpr int kPcrLevels = 5;  // cyclic-reduction levels (strides 1..16)

struct SplineFactors {
  int64_t n;
  double* dev;  // [mult n][denom n][rden n][z n][sden, rsden]
};

// _factors(n) restated (pkg/src/slvp/_kernels_py.py:22-46), same operation
// order; compiled with -ffp-contract=off so it rounds exactly like NumPy.
static void host_factors(int64_t n, double* mult, double* denom, double* z, double* sden) {
  const double gamma = -4.0;
  double* diag = new double[n];
  for (int64_t i = 0; i < n; ++i) diag[i] = 4.0;
  diag[0] -= gamma;
  diag[n - 1] -= 1.0 / gamma;
  mult[0] = 0.0;
  denom[0] = diag[0];
  for (int64_t i = 1; i < n; ++i) {
    mult[i] = 1.0 / denom[i - 1];
    denom[i] = diag[i] - mult[i];
  }
  for (int64_t i = 0; i < n; ++i) z[i] = 0.0;
  z[0] = gamma;
  z[n - 1] = 1.0;
  for (int64_t i = 1; i < n; ++i) z[i] -= mult[i] * z[i - 1];
  z[n - 1] /= denom[n - 1];
  for (int64_t i = n - 2; i >= 0; --i) {
    z[i] -= z[i + 1];
    z[i] /= denom[i];
  }
  *sden = 1.0 + z[0] - 0.25 * z[n - 1];
  delete[] diag;
}

static int get_factors(int64_t n, const double** out) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, double*> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return check_launch("cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, n);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return VPB_OK;
  }
  // [mult | denom | rden | z | 8 scalars | PCR k_l, 6/b_L | z1^k, k = 0..n]
  const int64_t len = 5 * n + 9 + kPcrLevels;
  double* h = new double[len];
  double sden;
  host_factors(n, h, h + n, h + 3 * n, &sden);
  for (int64_t i = 0; i < n; ++i) h[2 * n + i] = 1.0 / h[n + i];
  h[4 * n] = sden;
  h[4 * n + 1] = 1.0 / sden;
  // The elimination factors reach an exact floating-point fixed point after a
  // few dozen rows.  kf: mult[i] == mc for all i in [kf, n-1]; kb: denom[i] ==
  // dc (and rden == rc) for all i in [kb, n-2].  Past those rows the kernel
  // keeps the factors in registers instead of loading them per point.
  const double mc = h[n - 1], dc = n >= 2 ? h[n + n - 2] : h[n];
  int64_t kf = n - 1;
  while (kf > 1 && h[kf - 1] == mc) --kf;
  int64_t kb = n - 2 >= 0 ? n - 2 : 0;
  while (kb > 0 && h[n + kb - 1] == dc) --kb;
  h[4 * n + 2] = (double)kf;
  h[4 * n + 3] = (double)kb;
  h[4 * n + 4] = mc;
  h[4 * n + 5] = dc;
  h[4 * n + 6] = 1.0 / dc;
  // Parallel cyclic reduction of w_{i-1} + 4 w_i + w_{i+1} = u_i (constant
  // coefficients, periodic): level l eliminates stride 2^l neighbours with
  // k_l = a_l/b_l, a_{l+1} = -a_l k_l, b_{l+1} = b_l - 2 a_l k_l.  After
  // kPcrLevels the coupling |a/b| is ~5e-19, and the solution is d/b (plus
  // 2a when the final stride wraps onto the row itself).  The 6 of the
  // right-hand side 6u is folded into the final scale.
  {
    double pa = 1.0, pb = 4.0;
    for (int l = 0; l < kPcrLevels; ++l) {
      const double k = pa / pb;
      h[4 * n + 7 + l] = k;
      const double na = -pa * k;
      const double nb = pb - 2.0 * pa * k;
      pa = na;
      pb = nb;
    }
    const bool wraps = ((1LL << kPcrLevels) % n) == 0;
    h[4 * n + 7 + kPcrLevels] = 6.0 / (wraps ? pb + 2.0 * pa : pb);
  }
  {  // powers of the recursive-filter pole z1 = sqrt(3) - 2 (spline_rows_kernel)
    const double z1 = std::sqrt(3.0) - 2.0;
    double pz = 1.0;
    for (int64_t k = 0; k <= n; ++k) {
      h[4 * n + 8 + kPcrLevels + k] = pz;
      pz *= z1;
    }
  }
  double* d = nullptr;
  if (cudaMalloc(&d, len * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(d, h, len * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    delete[] h;
    return check_launch("spline factors upload");
  }
  delete[] h;
  cache[key] = d;
  *out = d;
  return VPB_OK;
}

__device__ __forceinline__ double div_exact(double y, double d, double r) {
  double q = __dmul_rn(y, r);
  double e = __fma_rn(-q, d, y);
  return __fma_rn(e, r, q);
}

// Line geometry of a tile.  Line L's point i sits at
//   CONTIG:  src + L*n + i
//   strided: src + (L / S) * S * n + (L % S) + i*S
// Table row: idx ? idx[L] : (L / tdiv) % tmod.
struct SplineTileArgs {
  const double* src;
  double* dst;
  int64_t nlines;
  int n;
  int64_t S;
  const int64_t* idx;
  int64_t tdiv, tmod;
  const double* values;
  double scale, h;
  const double* fac;
  int32_t* flag;
  int use_tma;  // strided tiles: one TMA tensor copy per tile (tmap valid)
  int iir;      // fast path: recursive filters (n % 8 == 0, n >= 32) instead of PCR
  int dbl;      // two consecutive sweeps with the same shift in one pass (see below)
  // density epilogue of the contiguous (x1) double sweep: a tile's 32 lines
  // are 32 consecutive v1 rows at one (v2, x2) (line = ((iv2 nv1 + iv1) n2 +
  // ix2)), and part[((iv2 (nv1/32) + blk) n2 + ix2) n + k] = sum over the
  // tile's lines of out * w1[iv1] (fixed order); nullptr = no epilogue
  double* part;
  const double* pw1;
  int64_t pn2, pnv1;
};

// Two sweeps by the same shift (the closing and opening x half steps of
// consecutive Strang steps, driver.py:245-265 / 371-377) in one pass.  One
// sweep is out = E w with w = 6 T^-1 u (_kernels.pyx:37-93): T the periodic
// (1, 4, 1) matrix, E the periodic 4-tap evaluation at offset j0.  Both are
// circulant, so they commute and two sweeps are E^2 (6 T^-1)^2 u: the
// recursive-filter solve runs twice and the evaluation is the 7-tap
// self-convolution of the weights at offset 2 j0.  Equal to two separate
// sweeps up to round-off.
__device__ __forceinline__ void spline_weights2(const double (&w)[4], double (&c)[7]) {
#pragma unroll
  for (int m = 0; m < 7; ++m) c[m] = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) c[k + kk] = fma(w[k], w[kk], c[k + kk]);
}

constexpr int kSplineBars = 8;  // row groups with their own mbarrier (strided tiles)

// Row stride of the contiguous-axis tile [line][point]: even (16-B aligned
// bulk destinations) and not a multiple of 16 doubles (few bank conflicts).
__host__ __device__ __forceinline__ int contig_rs(int n) { return n + 2 - (n & 1); }

// One warp per tile of kSplineT lines; each lane runs the Thomas recurrence
// of one line in shared memory.  Strided axes: the tile is [point][lane] and
// every point row (kSplineT consecutive lines, 256 contiguous bytes) arrives
// by its own bulk copy; the forward elimination consumes row groups as their
// mbarriers complete, overlapping the solve with the load.  Contiguous axis:
// [lane][point] rows land by one bulk copy per line.  The evaluation writes
// HBM coalesced: lane-parallel along the line index (strided) or along the
// points of each line (contiguous).
// One level of cyclic reduction with stride S, in place on one line:
//   y_i <- y_i - k (y_{i-S} + y_{i+S})   (indices mod n), all i from OLD values.
// Points go in blocks of B = 16: the block's old values (and the S values
// past it) are loaded before any of its results is stored, so the loads are
// not serialised behind the stores.  Old y_{i-S} of the block's first S
// points comes from a register ring (the previous block's tail); in the last
// block y_{i+S} wrapped onto the first block and comes from `first`.
// Requires n % 16 == 0 and n >= 2S.
template <int S>
__device__ __forceinline__ void pcr_level(double* y, const int YS, const int n, const double k) {
  constexpr int B = 16;
  double first[S], ring[S];
#pragma unroll
  for (int r = 0; r < S; ++r) {
    first[r] = y[r * YS];
    ring[r] = y[(n - S + r) * YS];
  }
  for (int i0 = 0; i0 < n; i0 += B) {
    const bool last = i0 + B == n;
    double c[B], nb[S], o[B];
#pragma unroll
    for (int r = 0; r < B; ++r) c[r] = y[(i0 + r) * YS];
#pragma unroll
    for (int r = 0; r < S; ++r) nb[r] = last ? first[r] : y[(i0 + B + r) * YS];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      const double lo = r < S ? ring[r] : c[r - S];
      const double hi = r + S < B ? c[r + S] : nb[r + S - B];
      o[r] = __fma_rn(-k, lo + hi, c[r]);
    }
#pragma unroll
    for (int r = 0; r < S; ++r) ring[r] = c[B - S + r];
#pragma unroll
    for (int r = 0; r < B; ++r) y[(i0 + r) * YS] = o[r];
  }
}

// The same periodic solve as spline_rows_kernel, one line per lane, serial
// along the line in shared memory: causal then anticausal recursive filter
// (pole z1), each started from its periodic value summed over the 32 points
// that wrap into it (z1^32 ~ 5e-19).  Five shared-memory accesses per point
// instead of the eleven of five PCR levels.  Requires n >= 32.  Leaves
// y = w / g with g = -6 z1.
__device__ __forceinline__ void iir_solve(double* y, const int YS, const int n, const double z1) {
  constexpr int U = 8;
  double p = 0.0;
  for (int k = n - 32; k < n; k += U) {  // y+_{n-1}, periodic
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = 0; r < U; ++r) p = fma(z1, p, u[r]);
  }
  for (int k = 0; k < n; k += U) {  // causal: y+_k = u_k + z1 y+_{k-1}
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      p = fma(z1, p, u[r]);
      u[r] = p;
    }
#pragma unroll
    for (int r = 0; r < U; ++r) y[(k + r) * YS] = u[r];
  }
  double q = 0.0;
  for (int k = 32 - U; k >= 0; k -= U) {  // y_0, periodic
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) q = fma(z1, q, u[r]);
  }
  for (int k = n - U; k >= 0; k -= U) {  // anticausal: y_k = y+_k + z1 y_{k+1}
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) {
      q = fma(z1, q, u[r]);
      u[r] = q;
    }
#pragma unroll
    for (int r = 0; r < U; ++r) y[(k + r) * YS] = u[r];
  }
}

constexpr int kDblWarm = 40;  // warm-up points of the double recursion (multiple of 8)

// Two recursive-filter solves (the double sweep's (6 T^-1)^2 up to the gain)
// in one causal and one anticausal pass: y1 <- u + z1 y1, y2 <- y1 + z1 y2
// advance together, so every point is loaded and stored once per direction
// and the two chains overlap.  The periodic start values come from a
// kDblWarm-point warm-up over the wrapping end: started J points back, the
// pair of recursions computes exactly the truncated sums y1 = sum_{j<J} z1^j
// u_{-j} and y2 = sum_{j<J} (j+1) z1^j u_{-j}, whose tails are below
// (J+1) z1^J / (1-z1)^2 ~ 1e-21 of max|u| at J = 40 (z1^40 = 1.3e-23; the
// round-1 warm-up of 64 points was 24 points longer than needed).
// Requires n >= 64 (else two iir_solve calls).
__device__ __forceinline__ void iir_solve2(double* y, const int YS, const int n, const double z1) {
  constexpr int U = 8;
  double p1 = 0.0, p2 = 0.0;
  for (int k = n - kDblWarm; k < n; k += U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      p1 = fma(z1, p1, u[r]);
      p2 = fma(z1, p2, p1);
    }
  }
  for (int k = 0; k < n; k += U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      p1 = fma(z1, p1, u[r]);
      p2 = fma(z1, p2, p1);
      u[r] = p2;
    }
#pragma unroll
    for (int r = 0; r < U; ++r) y[(k + r) * YS] = u[r];
  }
  double q1 = 0.0, q2 = 0.0;
  for (int k = kDblWarm - U; k >= 0; k -= U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) {
      q1 = fma(z1, q1, u[r]);
      q2 = fma(z1, q2, q1);
    }
  }
  for (int k = n - U; k >= 0; k -= U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = y[(k + r) * YS];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) {
      q1 = fma(z1, q1, u[r]);
      q2 = fma(z1, q2, q1);
      u[r] = q2;
    }
#pragma unroll
    for (int r = 0; r < U; ++r) y[(k + r) * YS] = u[r];
  }
}

// Evaluation weights of one line (_kernels.pyx:62-87), the gain g folded in.
__device__ __forceinline__ void spline_eval_weights(const SplineTileArgs& a, int64_t L, int n,
                                                    double g, double (&w)[4], int& j0) {
  const int64_t trow = a.idx ? a.idx[L] : (L / a.tdiv) % a.tmod;
  const double shift = __dmul_rn(a.values[trow], a.scale);
  const double sh = __ddiv_rn(shift, a.h);
  double off = floor(-sh);
  double th = __dsub_rn(-sh, off);
  if (th >= 1.0) {
    off = __dadd_rn(off, 1.0);
    th = 0.0;
  }
  const double omt = __dsub_rn(1.0, th);
  w[0] = g * __ddiv_rn(__dmul_rn(__dmul_rn(omt, omt), omt), 6.0);
  w[1] = g * __ddiv_rn(__dadd_rn(__dsub_rn(4.0, __dmul_rn(__dmul_rn(6.0, th), th)),
                                 __dmul_rn(__dmul_rn(__dmul_rn(3.0, th), th), th)),
                       6.0);
  w[2] = g * __ddiv_rn(__dadd_rn(__dsub_rn(4.0, __dmul_rn(__dmul_rn(6.0, omt), omt)),
                                 __dmul_rn(__dmul_rn(__dmul_rn(3.0, omt), omt), omt)),
                       6.0);
  w[3] = g * __ddiv_rn(__dmul_rn(__dmul_rn(th, th), th), 6.0);
  j0 = (int)wrap_mod((int64_t)off - 1, n);
}

// Contiguous-axis sweep (single, or the double sweep of merged half steps),
// one line per lane in a [line][RS] tile: the recursive-filter solve
// (iir_solve / iir_solve2) with the evaluation fused into the anticausal
// pass, so the solved values are never re-read from shared memory: walking
// backwards, w_j is ready while w_{j+1} .. w_{j+TAPS-1} are still in
// registers, and out at position j (= sum_m c_m w_{j+m}; single sweep: the
// reference's 4-tap order with separate roundings, _kernels.pyx:88-93) goes
// to in-place slot j + sigma, whose causal value has already been consumed.
// The TAPS-1 positions whose window wraps past the end are emitted last,
// from saved values.  sigma = rotation & 1 makes the row's rotation
// (j0, or 2 j0 for the double sweep) plus sigma even, so the row leaves by
// two 16-byte aligned bulk stores (the caller's write-out).
//
// Bank conflicts: with the row stride RS = n + 2 (even, for 16-byte bulk
// copy destinations) lanes t and t + 8 of a half-warp hit the same bank
// pair at equal point index.  Lanes with bit 3 set therefore walk their line
// starting at point 1 (logical index j lives at physical (j + s) mod n,
// s = (lane >> 3) & 1): the periodic filters may start anywhere (their
// periodic start values are sums over the preceding points), so only the
// rounding of the two half-warps' lines differs.  Requires n >= 64, n % 8 == 0.
// Returns true when an output is not finite.
template <bool DBL>
__device__ __forceinline__ bool iir_eval_fused(double* y, const int n, const double z1,
                                               const double (&c)[DBL ? 7 : 4], const int s,
                                               const int sigma) {
  constexpr int U = 8;
  constexpr int TAPS = DBL ? 7 : 4;
  constexpr int D = TAPS - 1;      // deferred (wrapped) outputs
  constexpr int WARM = DBL ? kDblWarm : 32;
  // logical j lives at y[j + s]: for s = 1 the row's first point is parked in
  // the padding slot y[n] (RS = n + 2) so no access needs a wrap, and moved
  // back at the end (the in-place outputs are position-relative)
  double* yb = y + s;
  if (s) y[n] = y[0];
  auto eval = [&](double w, const double (&win)[D]) -> double {
    if constexpr (DBL) {
      // oldest value first, the value just solved (w) last: only one fma of
      // the 7-term chain waits for the recursion step that produced w, the
      // rest can issue while earlier points' chains are in flight
      double o = c[TAPS - 1] * win[TAPS - 2];
#pragma unroll
      for (int m = TAPS - 2; m >= 1; --m) o = fma(c[m], win[m - 1], o);
      return fma(c[0], w, o);
    } else {  // out = w0 w_j + w1 w_{j+1} + w2 w_{j+2} + w3 w_{j+3}, left to right
      double o = __dmul_rn(c[0], w);
      o = __dadd_rn(o, __dmul_rn(c[1], win[0]));
      o = __dadd_rn(o, __dmul_rn(c[2], win[1]));
      return __dadd_rn(o, __dmul_rn(c[3], win[2]));
    }
  };
  // ---- causal pass, periodic start from the WARM points before 0
  double p1 = 0.0, p2 = 0.0;
  for (int k = n - WARM; k < n; k += U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = yb[k + r];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      p1 = fma(z1, p1, u[r]);
      if constexpr (DBL) p2 = fma(z1, p2, p1);
    }
  }
  for (int k = 0; k < n; k += U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = yb[k + r];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      p1 = fma(z1, p1, u[r]);
      if constexpr (DBL) {
        p2 = fma(z1, p2, p1);
        u[r] = p2;
      } else {
        u[r] = p1;
      }
    }
#pragma unroll
    for (int r = 0; r < U; ++r) yb[k + r] = u[r];
  }
  // ---- anticausal pass, periodic start from the WARM points after n - 1
  double q1 = 0.0, q2 = 0.0;
  for (int k = WARM - U; k >= 0; k -= U) {
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = yb[k + r];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) {
      q1 = fma(z1, q1, u[r]);
      if constexpr (DBL) q2 = fma(z1, q2, q1);
    }
  }
  auto chain = [&](double u) -> double {
    q1 = fma(z1, q1, u);
    if constexpr (DBL) {
      q2 = fma(z1, q2, q1);
      return q2;
    } else {
      return q1;
    }
  };
  ExpMax em;
  double win[D];   // w_{j+1} .. w_{j+D}
  double tail[D];  // w_{n-D} .. w_{n-1} (the wrapped windows' first parts)
  // first block: j = n-8 .. n-1; outputs only for j <= n-TAPS
  {
    const int k = n - U;
    double u[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = yb[k + r];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) u[r] = chain(u[r]);  // w_{k+r}
#pragma unroll
    for (int r = 0; r < D; ++r) tail[r] = u[U - D + r];
    double o[U - D];
#pragma unroll
    for (int r = U - D - 1; r >= 0; --r) {
      double wv[D];
#pragma unroll
      for (int m = 0; m < D; ++m) wv[m] = u[r + 1 + m];
      o[r] = eval(u[r], wv);
      em.add(o[r]);
    }
#pragma unroll
    for (int r = 0; r < U - D; ++r) yb[k + r + sigma] = o[r];
#pragma unroll
    for (int m = 0; m < D; ++m) win[m] = u[m];  // w_{n-8} .. w_{n-8+D-1}
  }
  for (int k = n - 2 * U; k >= 0; k -= U) {
    double u[U], o[U];
#pragma unroll
    for (int r = 0; r < U; ++r) u[r] = yb[k + r];
#pragma unroll
    for (int r = U - 1; r >= 0; --r) {
      const double w = chain(u[r]);  // w_{k+r}; window w_{k+r+1 ..} in win
      o[r] = eval(w, win);
#pragma unroll
      for (int m = D - 1; m > 0; --m) win[m] = win[m - 1];
      win[0] = w;
      em.add(o[r]);
    }
#pragma unroll
    for (int r = 0; r < U; ++r) yb[k + r + sigma] = o[r];
  }
  // win = w_0 .. w_{D-1}: the wrapped outputs j = n-D .. n-1
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double wv[D];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int t = r + 1 + m;  // window index: t < D -> tail[t], else w_{t-D} = win[t-D]
      wv[m] = t < D ? tail[t] : win[t - D];
    }
    const double o = eval(tail[r], wv);
    em.add(o);
    const int slot = n - D + r + sigma;
    yb[slot >= n ? slot - n : slot] = o;
  }
  if (s) y[0] = y[n];
  return em.bad();
}

template <bool CONTIG, bool PCR, bool DBL = false>
__global__ void __launch_bounds__(kSplineT)
    spline_tile_kernel(SplineTileArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int T = kSplineT;
  const int n = a.n;
  const int RS = CONTIG ? contig_rs(n) : T;  // row stride
  const int YS = CONTIG ? 1 : T;             // stride between points of one line
  double* tile = reinterpret_cast<double*>(smem_raw);
  const int tile_elems = CONTIG ? T * RS : n * T;
  double* wts = tile + tile_elems;                                   // [T][4]
  int* j0s = reinterpret_cast<int*>(wts + 4 * T);                    // [T]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + ((tile_elems + 4 * T) * 8 + T * 4 + 7) / 8 * 8);
  const int t = threadIdx.x;
  const int64_t L0 = (int64_t)blockIdx.x * T;
  const int lines = (int)min((int64_t)T, a.nlines - L0);
  // the line of lane t: consecutive lines, or (density epilogue, contiguous
  // axis) the 32 v1 rows of one (v2, x2, v1 block)
  int64_t pbase = 0, Lt = L0 + t;
  int tc1 = (int)L0, tc2 = 0;  // contiguous tiles by TMA: box coordinates {0, tc1, tc2}
  if (CONTIG && DBL && a.part) {
    const int64_t nblk = a.pnv1 / T;
    const int64_t ix2 = blockIdx.x % a.pn2, rest = blockIdx.x / a.pn2;
    const int64_t blk = rest % nblk, iv2 = rest / nblk;
    Lt = (iv2 * a.pnv1 + blk * T + t) * a.pn2 + ix2;
    pbase = ((iv2 * nblk + blk) * a.pn2 + ix2) * (int64_t)n;
    tc1 = (int)ix2;
    tc2 = (int)(iv2 * a.pnv1 + blk * T);
  }
  const int64_t outer0 = CONTIG ? 0 : L0 / a.S;
  const int64_t inner0 = CONTIG ? 0 : L0 - outer0 * a.S;

  // ---- stage the tile -------------------------------------------------------
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.src) & 15) == 0);
  bool bulk;
  int nbars = 1, rows_per_bar = n;
  if (CONTIG) {
    bulk = aligned && (n % 2 == 0);
  } else {
    bulk = aligned && lines == T && (a.S % T == 0);
    if (a.use_tma) {
      nbars = 1;
      rows_per_bar = n;
    } else {
      nbars = min(kSplineBars, n);
      rows_per_bar = (n + nbars - 1) / nbars;
      nbars = (n + rows_per_bar - 1) / rows_per_bar;
    }
  }
  if (bulk) {
    if (t == 0) {
      for (int b = 0; b < nbars; ++b) mbar_init(bars + b, 1);
      fence_mbar_init();
      if (CONTIG) {
        // TMA: the whole box counts, zero-filled padding columns and rows included
        mbar_arrive_expect_tx(bars, a.use_tma ? (uint32_t)T * RS * 8u : (uint32_t)lines * n * 8u);
      } else {
        for (int b = 0; b < nbars; ++b) {
          const int rows = min(rows_per_bar, n - b * rows_per_bar);
          mbar_arrive_expect_tx(bars + b, (uint32_t)rows * T * 8u);
        }
      }
    }
    if (CONTIG && a.use_tma) {
      // one tensor copy for the tile: the box is n + 2 points wide, two more
      // than the tensor, so the rows land RS apart (the padding is zero-filled)
      if (t == 0) tma_load_3d(tile, &tmap, 0, tc1, tc2, bars);
    } else if (CONTIG) {
      __syncwarp();  // lane 0's arrive.expect_tx precedes the copies
      if (t < lines) bulk_g2s(tile + t * RS, a.src + Lt * n, (uint32_t)n * 8u, bars);
    } else if (a.use_tma) {
      // the whole [n][32] tile in one (or two, n > 256) TMA tensor copies
      if (t == 0)
        for (int r0 = 0; r0 < n; r0 += 256)
          tma_load_3d(tile + r0 * T, &tmap, (int)inner0, r0, (int)outer0, bars);
    } else {
      const double* base = a.src + outer0 * a.S * n + inner0;
      for (int i = t; i < n; i += T)
        bulk_g2s(tile + i * T, base + (int64_t)i * a.S, (uint32_t)T * 8u, bars + i / rows_per_bar);
    }
  } else {
    if (CONTIG) {
      const double* base = a.src + L0 * n;
      for (int e = t; e < lines * n; e += T) {
        const int r = e / n, i = e - r * n;
        tile[r * RS + i] = __ldcs(base + e);
      }
    } else if (t < lines) {
      const int64_t L = L0 + t;
      const int64_t outer = L / a.S, inner = L - outer * a.S;
      const double* base = a.src + outer * a.S * n + inner;
#pragma unroll 8
      for (int i = 0; i < n; ++i) tile[i * T + t] = __ldcs(base + (int64_t)i * a.S);
    }
    __syncwarp();
  }

  // ---- per-line solve (Thomas + Sherman-Morrison) and evaluation -----------
  bool bad = false;
  double pw_early = 0.0;  // the line's density weight (epilogue), loaded before the wait
  // contiguous recursive-filter sweeps: evaluated inside the solve
  // (iir_eval_fused); uniform over the warp (template flags and arguments)
  const bool fused_eval = CONTIG && PCR && a.iir && n >= 64 && n % 8 == 0;
  if (t < lines) {
    const double* mult = a.fac;
    const double* denom = a.fac + n;
    const double* rden = a.fac + 2 * n;
    const double* z = a.fac + 3 * n;
    const double sden = a.fac[4 * n], rsden = a.fac[4 * n + 1];
    const int kf = (int)a.fac[4 * n + 2], kb = (int)a.fac[4 * n + 3];
    const double mc = a.fac[4 * n + 4], dc = a.fac[4 * n + 5], rc = a.fac[4 * n + 6];
    double* y = CONTIG ? tile + t * RS : tile + t;
    double wscale = 1.0;
    // The line's evaluation weights first (unscaled; _kernels.pyx:62-87): their
    // ~900 instructions (five fp64 divisions, 64-bit index arithmetic) run
    // while the tile's copies are still in flight instead of after the wait.
    double ew[4];
    int ej0;
    spline_eval_weights(a, Lt, n, 1.0, ew, ej0);
    // likewise the filter pole and the line's density weight: global loads
    // whose latency would otherwise follow the wait
    const double z1_early = PCR ? __ldg(a.fac + 4 * n + 7 + kPcrLevels + 2) : 0.0;
    if constexpr (CONTIG && DBL) {
      if (a.part) pw_early = __ldg(a.pw1 + (Lt / a.pn2) % a.pnv1);
    }
    if constexpr (PCR) {
      // parallel cyclic reduction in shared memory: no serial chain per line
      if (bulk)
        for (int bb = 0; bb < nbars; ++bb) mbar_wait(bars + bb, 0);
      const double* pk = a.fac + 4 * n + 7;
      if (a.iir) {
        const double z1 = z1_early;  // z1^1 of the power table
        if (fused_eval) {
          // solve + evaluation in one pass pair over the row (iir_eval_fused);
          // j0s = the row's (even) rotation for the bulk-store write-out
          const double g = -6.0 * z1;
          const double w4[4] = {g * ew[0], g * ew[1], g * ew[2], g * ew[3]};
          const int j0 = ej0;
          if constexpr (DBL) {
            double c[7];
            spline_weights2(w4, c);
            const int jr = (2 * j0) % n;  // even: n is even
            j0s[t] = jr;
            bad |= iir_eval_fused<true>(y, n, z1, c, (t >> 3) & 1, 0);
          } else {
            const int sigma = j0 & 1;
            j0s[t] = (j0 + sigma) % n;
            bad |= iir_eval_fused<false>(y, n, z1, w4, (t >> 3) & 1, sigma);
          }
        } else if constexpr (DBL) {
          if (n >= 64) {
            iir_solve2(y, YS, n, z1);
          } else {
            iir_solve(y, YS, n, z1);
            iir_solve(y, YS, n, z1);
          }
        } else {
          iir_solve(y, YS, n, z1);
        }
        wscale = -6.0 * z1;
      } else {
        pcr_level<1>(y, YS, n, pk[0]);
        pcr_level<2>(y, YS, n, pk[1]);
        pcr_level<4>(y, YS, n, pk[2]);
        pcr_level<8>(y, YS, n, pk[3]);
        pcr_level<16>(y, YS, n, pk[4]);
        wscale = pk[kPcrLevels];  // 6 / b_L: folded into the evaluation weights
      }
    } else {
    // Forward elimination y_i = 6u_i - mult_i*y_{i-1}, in blocks of U points:
    // the U loads are issued before the dependent chain so only the two
    // fp64 ops per point sit on the critical path; past row kf the factor is
    // the exact fixed point mc.
    constexpr int U = 8;
    int b = 0;
    int next_group = 0;  // first row of the next barrier group
    auto wait_rows = [&](int upto) {  // rows [0, upto) landed
      while (bulk && next_group < upto) {
        mbar_wait(bars + b, 0);
        ++b;
        next_group = CONTIG ? n : next_group + rows_per_bar;
      }
    };
    wait_rows(1);
    double prev = __dmul_rn(6.0, y[0]);
    y[0] = prev;
    int i = 1;
    for (; i + U <= n; i += U) {
      wait_rows(i + U);
      double u[U], m[U];
      const bool cst = i >= kf;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        u[k] = y[(i + k) * YS];
        m[k] = cst ? mc : __ldg(mult + i + k);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        prev = __dsub_rn(__dmul_rn(6.0, u[k]), __dmul_rn(m[k], prev));
        u[k] = prev;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) y[(i + k) * YS] = u[k];
    }
    wait_rows(n);
    for (; i < n; ++i) {
      prev = __dsub_rn(__dmul_rn(6.0, y[i * YS]), __dmul_rn(__ldg(mult + i), prev));
      y[i * YS] = prev;
    }
    // Back substitution y_i = (y_i - y_{i+1}) / denom_i (constant past kb)
    prev = div_exact(prev, __ldg(denom + n - 1), __ldg(rden + n - 1));
    y[(n - 1) * YS] = prev;
    i = n - 2;
    for (; i - U + 1 >= 0; i -= U) {
      double v[U], d[U], r[U];
      const bool cst = i - U + 1 >= kb;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        v[k] = y[(i - k) * YS];
        d[k] = cst ? dc : __ldg(denom + i - k);
        r[k] = cst ? rc : __ldg(rden + i - k);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        prev = div_exact(__dsub_rn(v[k], prev), d[k], r[k]);
        v[k] = prev;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) y[(i - k) * YS] = v[k];
    }
    for (; i >= 0; --i) {
      prev = div_exact(__dsub_rn(y[i * YS], prev), __ldg(denom + i), __ldg(rden + i));
      y[i * YS] = prev;
    }
    const double fac = div_exact(__dsub_rn(prev, __dmul_rn(0.25, y[(n - 1) * YS])), sden, rsden);
#pragma unroll 8
    for (int k = 0; k < n; ++k) y[k * YS] = __dsub_rn(y[k * YS], __dmul_rn(fac, __ldg(z + k)));
    }  // Thomas

    if (!fused_eval) {
    // evaluation weights (computed above, before the tile landed)
    const int64_t L = L0 + t;
    double w0 = ew[0], w1 = ew[1], w2 = ew[2], w3 = ew[3];
    if constexpr (PCR) {
      w0 *= wscale;
      w1 *= wscale;
      w2 *= wscale;
      w3 *= wscale;
    }
    const int j0 = ej0;
    j0s[t] = j0;
    if constexpr (DBL) {
      // out_i = sum_m c_m w2[2 j0 + i + m], m = 0..6: a 7-value sliding window
      // (contiguous axis: out_i overwrites w2[2 j0 + i] in place, rotated)
      const double wv[4] = {w0, w1, w2, w3};
      double c[7];
      spline_weights2(wv, c);
      int jn = (2 * j0) % n;
      if (CONTIG) j0s[t] = jn;
      int pw = jn;  // CONTIG: in-place position of out_k
      auto nxt = [&]() {
        const double v = y[jn * YS];
        if (++jn == n) jn = 0;
        return v;
      };
      double sv[6], win[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) win[r] = sv[r] = nxt();
      const int64_t outer = CONTIG ? 0 : L / a.S, inner = CONTIG ? 0 : L - outer * a.S;
      const int64_t obase = outer * a.S * n + inner;
      auto put = [&](int k, double o) {
        if (CONTIG) {
          y[pw] = o;
          if (++pw == n) pw = 0;
        } else {
          __stcs(a.dst + obase + (int64_t)k * a.S, o);
        }
      };
      auto emit = [&](double v6) {
        double o = c[0] * win[0];
#pragma unroll
        for (int m = 1; m < 6; ++m) o = fma(c[m], win[m], o);
        o = fma(c[6], v6, o);
#pragma unroll
        for (int m = 0; m < 5; ++m) win[m] = win[m + 1];
        win[5] = v6;
        bad |= not_finite(o);
        return o;
      };
      constexpr int E = 16;
      int k = 0;
      for (; k + E <= n - 6; k += E) {
        double v[E], o[E];
#pragma unroll
        for (int r = 0; r < E; ++r) v[r] = nxt();
#pragma unroll
        for (int r = 0; r < E; ++r) o[r] = emit(v[r]);
#pragma unroll
        for (int r = 0; r < E; ++r) put(k + r, o[r]);
      }
      for (; k < n; ++k) {
        const int back = k - (n - 6);
        double v6;
        if (back < 0) {
          v6 = nxt();
        } else {
          v6 = sv[0];
#pragma unroll
          for (int r = 1; r < 6; ++r)
            if (back == r) v6 = sv[r];
        }
        put(k, emit(v6));
      }
    } else {

    // out_i = w0 om[j0+i] + w1 om[j0+i+1] + w2 om[j0+i+2] + w3 om[j0+i+3]
    // with a 4-value sliding window (one smem load per output).  On the
    // contiguous axis out_i overwrites om[j0+i] in place (rotated by j0); the
    // three window values that wrap past the start are saved first.
    // (blocks of E outputs: the window values of a block are loaded before
    //  its in-place stores so loads are not serialised behind them)
    int jn = j0;
    auto nxt = [&]() {
      const double v = y[jn * YS];
      if (++jn == n) jn = 0;
      return v;
    };
    const double s0 = nxt(), s1 = nxt(), s2 = nxt();
    double c0 = s0, c1 = s1, c2 = s2;
    int64_t obase = 0;
    if (!CONTIG) {
      const int64_t outer = L / a.S, inner = L - outer * a.S;
      obase = outer * a.S * n + inner;
    }
    int p = j0;  // position of out_i in the rotated in-place row
    auto emit = [&](int k, double c3) {
      double o = __dmul_rn(w0, c0);
      o = __dadd_rn(o, __dmul_rn(w1, c1));
      o = __dadd_rn(o, __dmul_rn(w2, c2));
      o = __dadd_rn(o, __dmul_rn(w3, c3));
      c0 = c1;
      c1 = c2;
      c2 = c3;
      bad |= not_finite(o);
      return o;
    };
    constexpr int E = 16;
    int k = 0;
    for (; k + E <= n - 3; k += E) {
      double v[E], o[E];
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = nxt();
#pragma unroll
      for (int r = 0; r < E; ++r) o[r] = emit(k + r, v[r]);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (CONTIG) {
          y[p] = o[r];
          if (++p == n) p = 0;
        } else {
          __stcs(a.dst + obase + (int64_t)(k + r) * a.S, o[r]);
        }
      }
    }
    for (; k < n; ++k) {
      const int back = k - (n - 3);
      const double c3 = back < 0 ? nxt() : (back == 0 ? s0 : (back == 1 ? s1 : s2));
      const double o = emit(k, c3);
      if (CONTIG) {
        y[p] = o;
        if (++p == n) p = 0;
      } else {
        __stcs(a.dst + obase + (int64_t)k * a.S, o);
      }
    }
    }  // single sweep
    }  // !fused_eval
  }
  __syncwarp();
  if (CONTIG && fused_eval) {
    // double sweep: the rotation 2 j0 mod n is even, so each row leaves as two
    // 16-byte aligned bulk stores (out[0, n - jr) = row[jr, n), out[n - jr, n) =
    // row[0, jr)) issued by its own lane, instead of a warp loop over points
    if (t < lines) {
      const int jr = j0s[t];
      double* out = a.dst + Lt * n;
      const double* row = tile + t * RS;
      fence_proxy_async_smem();  // the rows were written by generic stores
      bulk_s2g(out, row + jr, (uint32_t)(n - jr) * 8u);
      if (jr) bulk_s2g(out + (n - jr), row, (uint32_t)jr * 8u);
      bulk_commit();
    }
    if constexpr (DBL) {
      if (a.part) {
        // density epilogue (compute_density, poisson.py:85-95, summed over
        // this tile's 32 v1 rows): lane t sums the point pairs k = 2t, 2t + 1
        // (+ 2T i) of every row in row order (out[k] = row[(jr + k) mod n];
        // jr and n are even, so a pair never wraps and is one 16-byte load);
        // consecutive lanes read consecutive words of one row, so the column
        // walk is bank-conflict free and runs while the bulk stores read the
        // same rows.  Measured at config 4: +0.09 ms on this pass against the
        // 0.34 ms density pass it replaces (the tile mapping alone +0.01 ms)
        wts[t] = pw_early;
        __syncwarp();
        for (int k = 2 * t; k < n; k += 2 * T) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
          for (int r = 0; r < T; ++r) {
            int q = j0s[r] + k;
            if (q >= n) q -= n;
            const double2 v = *reinterpret_cast<const double2*>(tile + r * RS + q);
            const double w = wts[r];
            s0 = fma(v.x, w, s0);
            s1 = fma(v.y, w, s1);
          }
          *reinterpret_cast<double2*>(a.part + pbase + k) = make_double2(s0, s1);
        }
      }
    }
    if (t < lines) bulk_wait_read<0>();  // shared memory must outlive the reads
  } else if (CONTIG) {
    // rows hold out rotated by j0: write them out coalesced
    for (int r = 0; r < lines; ++r) {
      double* out = a.dst + (L0 + r) * n;
      const double* row = tile + r * RS;
      const int jr = j0s[r];
      for (int k = t; k < n; k += T) {
        int q = jr + k;
        if (q >= n) q -= n;
        __stcs(out + k, row[q]);
      }
    }
  }
  report_flag(bad, a.flag);
}

// Contiguous-axis spline sweep with the line spread over a warp: lane L
// holds points NPT*L .. NPT*L+NPT-1 in registers (one coalesced load per
// line).  The periodic system w_{i-1} + 4 w_i + w_{i+1} = 6 u_i is solved with
// the cubic-B-spline recursive filters (pole z1 = sqrt(3) - 2):
//   causal      y+_k = u_k + z1 y+_{k-1},   anticausal  y_k = y+_k + z1 y_{k+1},
//   w = -6 z1 y  (6/(z + 4 + 1/z) = -6 z1 / ((1 - z1/z)(1 - z1 z))),
// each as a local recurrence over the lane's points plus a 5-step
// Kogge-Stone scan of the lane carries (multiplier z1^NPT) and the periodic
// wrap term z1^(k+1) y+_{n-1} (exact to z1^n <= 5e-19, below rounding).
// The evaluation (_kernels.pyx:62-93) reads w from a per-warp shared row
// with lanes along consecutive outputs, so loads and stores are coalesced.
// Same system as the Thomas + Sherman-Morrison solve (_kernels.pyx:37-59) to
// round-off; replaces the shared-memory tile (one line per lane), whose
// five PCR passes were shared-memory bound at 6 warps per SM.
constexpr int kRowWarps = 8;

// H = 32 / LPW lanes per line, LPW lines per warp at a time (independent
// scans interleave; shallower scans), NPT = n / H points per lane.
template <int NPT, int LPW, bool DBL = false>
__global__ void __launch_bounds__(32 * kRowWarps)
    spline_rows_kernel(SplineTileArgs a) {
  constexpr int H = 32 / LPW;
  constexpr int LOGH = H == 32 ? 5 : H == 16 ? 4 : 3;
  constexpr int n = H * NPT;
  constexpr int IT = 32 / LPW;  // iterations covered by one batch of weights
  constexpr int NTAP = DBL ? 7 : 4;  // evaluation taps (DBL: two sweeps, spline_weights2)
  // + wrap copies of points 0..NTAP-1 (row length kept even: 16-B stores)
  __shared__ double wrow[kRowWarps][LPW][n + (NTAP + 1) / 2 * 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / H, hl = lane % H;
  const double* zp = a.fac + 4 * n + 8 + kPcrLevels;  // z1^k
  const double z1 = zp[1];
  const double g = -6.0 * z1;
  double mj[LOGH];  // z1^(NPT 2^j)
#pragma unroll
  for (int j = 0; j < LOGH; ++j) mj[j] = zp[NPT << j];
  double zr[NPT + 1];
#pragma unroll
  for (int r = 0; r <= NPT; ++r) zr[r] = zp[r];
  const double zin = zp[NPT * hl];             // z1^(NPT hl): wrap into the carry-in
  const double zout = zp[n - NPT * (hl + 1)];  // z1^(n - NPT(hl+1))
  ExpMax em;
  const int64_t P0 = (int64_t)blockIdx.x * kRowWarps + warp;  // line group of the warp
  const int64_t Pstep = (int64_t)gridDim.x * kRowWarps;
  auto load_line = [&](int64_t L, double (&v)[NPT]) {
    if (L >= a.nlines) return;
    const double* src = a.src + L * n + NPT * hl;
    if constexpr (NPT % 2 == 0) {
#pragma unroll
      for (int r = 0; r < NPT; r += 2) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(src + r));
        v[r] = t.x;
        v[r + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < NPT; ++r) v[r] = __ldcs(src + r);
    }
  };
  // weights of the next IT iterations: lane t holds those of iteration
  // (t / LPW) for sub-line (t % LPW)
  double wl[NTAP];
#pragma unroll
  for (int m = 0; m < NTAP; ++m) wl[m] = 0.0;
  int jl = 0;
  double nxt[NPT];
  load_line(P0 * LPW + sub, nxt);
  int k = 0;
  for (int64_t P = P0; P * LPW < a.nlines; P += Pstep, ++k) {
    const int64_t L = P * LPW + sub;
    if (k % IT == 0) {
      const int64_t Lw = (P + (lane / LPW) * Pstep) * LPW + lane % LPW;
      if (Lw < a.nlines) {
        if constexpr (DBL) {
          double w4[4];
          spline_eval_weights(a, Lw, n, g, w4, jl);
          spline_weights2(w4, wl);
          jl = (2 * jl) % n;
        } else {
          spline_eval_weights(a, Lw, n, g, wl, jl);
        }
      }
    }
    double x[NPT];
#pragma unroll
    for (int r = 0; r < NPT; ++r) x[r] = nxt[r];
    load_line(L + Pstep * LPW, nxt);  // next lines' loads fly while these are solved
#pragma unroll
    for (int pass = 0; pass < (DBL ? 2 : 1); ++pass) {
    // ---- causal filter
#pragma unroll
    for (int r = 1; r < NPT; ++r) x[r] = fma(z1, x[r - 1], x[r]);
    double X = x[NPT - 1];
#pragma unroll
    for (int j = 0; j < LOGH; ++j) {
      const double t = __shfl_up_sync(0xffffffffu, X, 1 << j, H);
      if (hl >= (1 << j)) X = fma(mj[j], t, X);
    }
    const double W = __shfl_sync(0xffffffffu, X, H - 1, H);  // y+_{n-1} (periodic)
    double E = __shfl_up_sync(0xffffffffu, X, 1, H);
    E = hl == 0 ? W : fma(zin, W, E);
#pragma unroll
    for (int r = 0; r < NPT; ++r) x[r] = fma(zr[r + 1], E, x[r]);
    // ---- anticausal filter
#pragma unroll
    for (int r = NPT - 2; r >= 0; --r) x[r] = fma(z1, x[r + 1], x[r]);
    double Y = x[0];
#pragma unroll
    for (int j = 0; j < LOGH; ++j) {
      const double t = __shfl_down_sync(0xffffffffu, Y, 1 << j, H);
      if (hl + (1 << j) < H) Y = fma(mj[j], t, Y);
    }
    const double V = __shfl_sync(0xffffffffu, Y, 0, H);  // y_0 (periodic)
    double F = __shfl_down_sync(0xffffffffu, Y, 1, H);
    F = hl == H - 1 ? V : fma(zout, V, F);
#pragma unroll
    for (int r = 0; r < NPT; ++r) x[r] = fma(zr[NPT - r], F, x[r]);
    }  // pass
    // ---- w (the -6 z1 gain is folded into the evaluation weights)
    double* row = wrow[warp][sub];
    if constexpr (NPT % 2 == 0) {
#pragma unroll
      for (int r = 0; r < NPT; r += 2)
        *reinterpret_cast<double2*>(row + NPT * hl + r) = make_double2(x[r], x[r + 1]);
    } else {
#pragma unroll
      for (int r = 0; r < NPT; ++r) row[NPT * hl + r] = x[r];
    }
    if (hl < (NTAP + NPT - 1) / NPT)  // wrap copies row[n + i] = row[i], i < NTAP
#pragma unroll
      for (int r = 0; r < NPT; ++r)
        if (NPT * hl + r < NTAP) row[n + NPT * hl + r] = x[r];
    __syncwarp();
    // ---- evaluation: out_i = w0 w[j0+i] + w1 w[j0+i+1] + w2 w[j0+i+2] + w3 w[j0+i+3]
    const int src_lane = (k % IT) * LPW + sub;
    const int j0 = __shfl_sync(0xffffffffu, jl, src_lane);
    if constexpr (DBL) {
      double c[7];
#pragma unroll
      for (int m = 0; m < 7; ++m) c[m] = __shfl_sync(0xffffffffu, wl[m], src_lane);
      if (L < a.nlines) {
        double* dst = a.dst + L * n;
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
          const int i = hl + H * r;
          int q = j0 + i;
          if (q >= n) q -= n;
          double o = c[0] * row[q];
#pragma unroll
          for (int m = 1; m < 7; ++m) o = fma(c[m], row[q + m], o);
          em.add(o);
          __stcs(dst + i, o);
        }
      }
      __syncwarp();
      continue;
    }
    const double w0 = __shfl_sync(0xffffffffu, wl[0], src_lane);
    const double w1 = __shfl_sync(0xffffffffu, wl[1], src_lane);
    const double w2 = __shfl_sync(0xffffffffu, wl[2], src_lane);
    const double w3 = __shfl_sync(0xffffffffu, wl[3], src_lane);
    if (L < a.nlines) {
      double* dst = a.dst + L * n;
#pragma unroll
      for (int r = 0; r < NPT; ++r) {
        const int i = hl + H * r;
        int q = j0 + i;
        if (q >= n) q -= n;
        double o = __dmul_rn(w0, row[q]);
        o = __dadd_rn(o, __dmul_rn(w1, row[q + 1]));
        o = __dadd_rn(o, __dmul_rn(w2, row[q + 2]));
        o = __dadd_rn(o, __dmul_rn(w3, row[q + 3]));
        em.add(o);
        __stcs(dst + i, o);
      }
    }
    __syncwarp();  // the rows are rewritten by the next lines
  }
  report_flag(em.bad(), a.flag);
}

static size_t spline_smem(int n, bool contig) {
  const size_t tile = contig ? (size_t)kSplineT * contig_rs(n) : (size_t)n * kSplineT;
  return ((tile + 4 * kSplineT) * 8 + kSplineT * 4 + 7) / 8 * 8 + kSplineBars * 8;
}

// exact: Thomas + Sherman-Morrison, bitwise the reference (plugin API);
// otherwise parallel cyclic reduction when the line length allows it
// (n % 16 == 0, n >= 32), within ~4e-16 relative of the reference.
static int launch_spline(SplineTileArgs a, bool contig, bool exact, cudaStream_t st) {
  if (a.nlines == 0) return VPB_OK;
  size_t smem = spline_smem(a.n, contig);
  if (smem > 220 * 1024) {
    set_error("spline line of %d points does not fit a shared-memory tile", a.n);
    return VPB_ERR_UNSUPPORTED;
  }
  int rc = get_factors(a.n, &a.fac);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(spline_tile_kernel<true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(spline_tile_kernel<false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(spline_tile_kernel<true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(spline_tile_kernel<false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(spline_tile_kernel<false, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(spline_tile_kernel<true, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  static const bool force_exact = getenv("VPB_SPLINE_EXACT") != nullptr;
  static const bool force_pcr = getenv("VPB_SPLINE_PCR") != nullptr;
  const bool pcr = !exact && !force_exact && a.n % 16 == 0 && a.n >= 32;
  a.iir = pcr && !force_pcr ? 1 : 0;
  if (a.dbl && !a.iir) {
    set_error("double spline sweep needs the recursive-filter solve (n %% 16 == 0, n >= 32)");
    return VPB_ERR_UNSUPPORTED;
  }
  int64_t blocks = (a.nlines + kSplineT - 1) / kSplineT;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  a.use_tma = 0;
  if (!contig && a.S % kSplineT == 0 && a.S % 2 == 0 &&
      (reinterpret_cast<uintptr_t>(a.src) & 15) == 0 && a.nlines % a.S == 0) {
    const uint64_t O = (uint64_t)(a.nlines / a.S);
    a.use_tma = encode_tmap_3d(&tmap, a.src, (uint64_t)a.S, (uint64_t)a.n, O,
                               (uint64_t)a.S * 8, (uint64_t)a.S * a.n * 8, kSplineT,
                               (uint32_t)std::min(a.n, 256), 1)
                    ? 1
                    : 0;
  }
  // fused contiguous sweeps: the [32 lines][n + 2] tile in one tensor copy
  // (rows of a 2-D view of the lines, or -- density epilogue -- the 32 v1 rows
  // of one (v2, x2) in the 3-D view {x1, x2, v}); VPB_SPLINE_CONTIG_TMA=0: one
  // bulk copy per line, issued by its lane
  static const bool contig_tma = !(getenv("VPB_SPLINE_CONTIG_TMA") &&
                                   atoi(getenv("VPB_SPLINE_CONTIG_TMA")) == 0);
  if (contig && contig_tma && a.iir && a.n >= 64 && a.n % 8 == 0 && a.n + 2 <= 256 &&
      getenv("VPB_SPLINE_ROWS") == nullptr &&
      (reinterpret_cast<uintptr_t>(a.src) & 15) == 0) {
    const uint64_t nn = (uint64_t)a.n;
    if (a.part)
      a.use_tma = encode_tmap_3d(&tmap, a.src, nn, (uint64_t)a.pn2,
                                 (uint64_t)(a.nlines / a.pn2), nn * 8, nn * a.pn2 * 8,
                                 (uint32_t)a.n + 2, 1, kSplineT)
                      ? 1
                      : 0;
    else
      a.use_tma = encode_tmap_3d(&tmap, a.src, nn, (uint64_t)a.nlines, 1, nn * 8,
                                 nn * a.nlines * 8, (uint32_t)a.n + 2, kSplineT, 1)
                      ? 1
                      : 0;
  }
  static const bool no_rows = getenv("VPB_SPLINE_TILES") != nullptr;
  const int npt = a.n / 32;
  // double sweeps on the contiguous axis: one line per lane in a padded
  // shared-memory tile with the fused double recursion (1.19 ms at config 4)
  // beats the warp-per-line rows kernel (1.30 ms, shuffle-latency bound);
  // VPB_SPLINE_DBL_ROWS=1 selects the rows kernel
  static const bool dbl_rows = getenv("VPB_SPLINE_DBL_ROWS") != nullptr;
  // single contiguous sweeps: the tile kernel with the fused evaluation and
  // bulk-store write-out (n >= 64, n % 8 == 0) beats the warp-per-line rows
  // kernel; VPB_SPLINE_ROWS=1 selects the rows kernel for them
  static const bool force_rows = getenv("VPB_SPLINE_ROWS") != nullptr;
  const bool tile_fused = a.iir && a.n >= 64 && a.n % 8 == 0 && !force_rows;
  if (a.part && !(contig && a.dbl && tile_fused)) {
    set_error("spline density epilogue needs the fused contiguous double sweep "
              "(n %% 8 == 0, n >= 64, recursive filters)");
    return VPB_ERR_UNSUPPORTED;
  }
  const bool rows_ok = contig && pcr && !no_rows && !(a.dbl && !dbl_rows) && !tile_fused &&
                       a.n % 32 == 0 &&
                       (npt == 1 || npt == 2 || npt == 4 || npt == 8) &&
                       (reinterpret_cast<uintptr_t>(a.src) & 15) == 0;
  if (rows_ok) {
    // one line per warp at a time (two half-warp lines with 4-step scans
    // measured 9 % slower at n = 128)
    const int64_t want = (a.nlines + kRowWarps - 1) / kRowWarps;
    const unsigned rblocks = (unsigned)std::min<int64_t>(want, 148 * 8);
    const dim3 thr(32 * kRowWarps);
    // double sweeps: two half-warp lines per warp (half the scan shuffles per
    // line; measured 9 % faster at n = 128, 1.42 -> 1.29 ms at config 4)
    static const bool dbl_one = getenv("VPB_SPLINE_DBL_LPW1") != nullptr;
    if (a.dbl && !dbl_one && (npt == 2 || npt == 4)) {
      const int64_t want2 = (a.nlines / 2 + kRowWarps - 1) / kRowWarps;
      const unsigned rb2 = (unsigned)std::min<int64_t>(want2, 148 * 8);
      if (npt == 2)
        spline_rows_kernel<4, 2, true><<<rb2, thr, 0, st>>>(a);
      else
        spline_rows_kernel<8, 2, true><<<rb2, thr, 0, st>>>(a);
      return launched("spline_rows_kernel");
    }
    if (a.dbl) {
      switch (npt) {
        case 1: spline_rows_kernel<1, 1, true><<<rblocks, thr, 0, st>>>(a); break;
        case 2: spline_rows_kernel<2, 1, true><<<rblocks, thr, 0, st>>>(a); break;
        case 4: spline_rows_kernel<4, 1, true><<<rblocks, thr, 0, st>>>(a); break;
        default: spline_rows_kernel<8, 1, true><<<rblocks, thr, 0, st>>>(a); break;
      }
      return launched("spline_rows_kernel");
    }
    switch (npt) {
      case 1: spline_rows_kernel<1, 1><<<rblocks, thr, 0, st>>>(a); break;
      case 2: spline_rows_kernel<2, 1><<<rblocks, thr, 0, st>>>(a); break;
      case 4: spline_rows_kernel<4, 1><<<rblocks, thr, 0, st>>>(a); break;
      default: spline_rows_kernel<8, 1><<<rblocks, thr, 0, st>>>(a); break;
    }
    return launched("spline_rows_kernel");
  }
  if (a.dbl) {
    if (contig)
      spline_tile_kernel<true, true, true><<<(unsigned)blocks, kSplineT, smem, st>>>(a, tmap);
    else
      spline_tile_kernel<false, true, true><<<(unsigned)blocks, kSplineT, smem, st>>>(a, tmap);
    return launched("spline_tile_kernel");
  }
  if (contig) {
    if (pcr)
      spline_tile_kernel<true, true><<<(unsigned)blocks, kSplineT, smem, st>>>(a, tmap);
    else
      spline_tile_kernel<true, false><<<(unsigned)blocks, kSplineT, smem, st>>>(a, tmap);
  } else {
    if (pcr)
      spline_tile_kernel<false, true><<<(unsigned)blocks, kSplineT, smem, st>>>(a, tmap);
    else
      spline_tile_kernel<false, false><<<(unsigned)blocks, kSplineT, smem, st>>>(a, tmap);
  }
  return launched("spline_tile_kernel");
}

__global__ void spline_gather4d_kernel(const double* __restrict__ view, double* __restrict__ lines,
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

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_spline_sweep_contig(const double* lines, double* out, int64_t nlines, int64_t n,
                                       const int64_t* idx, const double* table, int64_t ntable,
                                       double h, void* stream) {
  VPB_REQUIRE(n >= 2, "need at least 2 samples per line, got %lld", (long long)n);
  VPB_REQUIRE(h > 0.0, "spacing must be positive, got %g", h);
  VPB_REQUIRE(lines != out, "out must not alias lines");
  VPB_REQUIRE(idx != nullptr && table != nullptr && ntable > 0, "table index required");
  SplineTileArgs a{lines, out, nlines, (int)n, 1, idx, 1, ntable, table, 1.0, h, nullptr, nullptr};
  return launch_spline(a, true, true, (cudaStream_t)stream);
}

extern "C" int vpb_spline_sweep_strided(double* view, const int64_t shape[4],
                                        const int64_t strides[4], const int64_t* idx,
                                        const double* table, int64_t ntable, double h,
                                        void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nlines = shape[0] * shape[1] * shape[2];
  int64_t total = nlines * shape[3];
  if (total == 0) return VPB_OK;
  double* tmp = nullptr;
  if (cudaMallocAsync(&tmp, 2 * total * sizeof(double), st) != cudaSuccess)
    return check_launch("cudaMallocAsync");
  int64_t blocks = (total + 255) / 256;
  spline_gather4d_kernel<<<(unsigned)blocks, 256, 0, st>>>(view, tmp, shape[0], shape[1],
                                                           shape[2], shape[3], strides[0],
                                                           strides[1], strides[2], strides[3], 0,
                                                           nullptr);
  int rc = vpb_spline_sweep_contig(tmp, tmp + total, nlines, shape[3], idx, table, ntable, h,
                                   stream);
  if (rc == VPB_OK) {
    spline_gather4d_kernel<<<(unsigned)blocks, 256, 0, st>>>(
        nullptr, tmp + total, shape[0], shape[1], shape[2], shape[3], strides[0], strides[1],
        strides[2], strides[3], 1, view);
    rc = launched("spline_gather4d_kernel", 2);
  }
  cudaFreeAsync(tmp, st);
  return rc;
}

extern "C" int64_t vpb_spline_density_part_len(const int64_t dims[4]) {
  return dims[2] % kSplineT ? 0 : dims[0] * dims[1] * (dims[2] / kSplineT) * dims[3];
}

// The x1 double sweep of the merged x half steps with the density of its
// output as an epilogue: part (vpb_spline_density_part_len doubles) receives
// per (v2, 32-row v1 block) partial sums of out * wv1, which vpb_density
// over dims {n1, n2, nv1 / 32, nv2} with unit v1 weights reduces to rho.
extern "C" int vpb_spline_sweep_x1dbl_density(const double* src, double* dst,
                                              const int64_t dims[4], const double* values,
                                              double scale, double h, int32_t* flag,
                                              const double* wv1, double* part, void* stream) {
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(h > 0.0, "spacing must be positive, got %g", h);
  VPB_REQUIRE(wv1 && part, "null pointer");
  const int64_t n1 = dims[0], n2 = dims[1], nv1 = dims[2], nv2 = dims[3];
  VPB_REQUIRE(nv1 % kSplineT == 0, "density epilogue needs nv1 %% %d == 0, got %lld", kSplineT,
              (long long)nv1);
  VPB_REQUIRE((reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
              "density epilogue needs 16-byte aligned buffers");
  const int64_t total = n1 * n2 * nv1 * nv2;
  SplineTileArgs a{src, dst, total / n1, (int)n1, 1, nullptr, n2, nv1, values, scale, h,
                   nullptr, flag};
  a.dbl = 1;
  a.part = part;
  a.pw1 = wv1;
  a.pn2 = n2;
  a.pnv1 = nv1;
  return launch_spline(a, true, false, (cudaStream_t)stream);
}

static int spline_axis(int32_t axis, const double* src, double* dst, const int64_t dims[4],
                       const double* values, double scale, double h, int32_t* flag, int dbl,
                       void* stream);

extern "C" int vpb_spline_sweep_axis(int32_t axis, const double* src, double* dst,
                                     const int64_t dims[4], const double* values, double scale,
                                     double h, int32_t* flag, void* stream) {
  return spline_axis(axis, src, dst, dims, values, scale, h, flag, 0, stream);
}

extern "C" int vpb_spline_sweep_axis2(int32_t axis, const double* src, double* dst,
                                      const int64_t dims[4], const double* values, double scale,
                                      double h, int32_t* flag, void* stream) {
  return spline_axis(axis, src, dst, dims, values, scale, h, flag, 1, stream);
}

static int spline_axis(int32_t axis, const double* src, double* dst, const int64_t dims[4],
                       const double* values, double scale, double h, int32_t* flag, int dbl,
                       void* stream) {
  VPB_REQUIRE(axis >= 0 && axis < 4, "axis %d out of range", axis);
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(h > 0.0, "spacing must be positive, got %g", h);
  const int64_t n1 = dims[0], n2 = dims[1], nv1 = dims[2], nv2 = dims[3];
  const int64_t total = n1 * n2 * nv1 * nv2;
  const int64_t n = dims[axis];
  VPB_REQUIRE(n >= 2, "need at least 2 samples per line");
  SplineTileArgs a{src, dst, total / n, (int)n, 1, nullptr, 1, 1, values, scale, h, nullptr, flag};
  a.dbl = dbl;
  if (axis == 0) {
    a.tdiv = n2;  // lines = (iv2, iv1, ix2), row = iv1
    a.tmod = nv1;
    return launch_spline(a, true, false, (cudaStream_t)stream);
  }
  if (axis == 1) {
    a.S = n1;
    a.tdiv = n1 * nv1;  // row = iv2
    a.tmod = nv2;
  } else if (axis == 2) {
    a.S = n1 * n2;
    a.tdiv = 1;  // row = x index
    a.tmod = n1 * n2;
  } else {
    a.S = n1 * n2 * nv1;
    a.tdiv = 1;
    a.tmod = n1 * n2;
  }
  return launch_spline(a, false, false, (cudaStream_t)stream);
}
