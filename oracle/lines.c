/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into or called by the
 * product path (paper_1803_02143_b200/); only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs use it.
 *
 * Plain-C restatement of the reference's compiled line kernels
 * (/root/reference/pkg/src/slvp/_kernels.pyx), operation for operation:
 *   oracle_dg_lines      <- _dg_line                 _kernels.pyx:96-123
 *   oracle_spline_lines  <- _solve_line + _eval_line _kernels.pyx:37-93
 * Lines are independent and processed with OpenMP over lines, so results do
 * not depend on the thread count.  Build with
 * -ffp-contract=off (the reference is built without FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline int64_t wrap(int64_t v, int64_t n) {
  v = v % n;
  if (v < 0) v += n;
  return v;
}

/* _kernels.pyx:96-123 */
static void dg_line(const double* u, double* out, const double* am, const double* bm, int64_t q,
                    double alpha, int64_t nc, int64_t p) {
  if (alpha == 0.0) {
    for (int64_t c = 0; c < nc; ++c) memcpy(out + c * p, u + wrap(c - q, nc) * p, p * sizeof(double));
    return;
  }
  for (int64_t c = 0; c < nc; ++c) {
    int64_t lo = wrap(c - q - 1, nc), up = wrap(c - q, nc);
    for (int64_t j = 0; j < p; ++j) {
      double sa = 0.0, sb = 0.0;
      for (int64_t m = 0; m < p; ++m) sa = sa + am[j * p + m] * u[lo * p + m];
      for (int64_t m = 0; m < p; ++m) sb = sb + bm[j * p + m] * u[up * p + m];
      out[c * p + j] = sa + sb;
    }
  }
}

void oracle_dg_lines(const double* lines, double* out, int64_t nlines, int64_t ncells, int64_t p,
                     const int64_t* idx, const double* a, const double* b, const int64_t* q,
                     const double* alpha, int threads) {
  const int64_t n = ncells * p;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t r = 0; r < nlines; ++r) {
    int64_t t = idx[r];
    dg_line(lines + r * n, out + r * n, a + t * p * p, b + t * p * p, q[t], alpha[t], ncells, p);
  }
}

/* _kernels.pyx:37-59 with the factors of _kernels_py.py:22-46 */
static void solve_line(const double* u, double* y, const double* mult, const double* denom,
                       const double* z, double sden, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = 6.0 * u[i];
  for (int64_t i = 1; i < n; ++i) y[i] = y[i] - mult[i] * y[i - 1];
  y[n - 1] = y[n - 1] / denom[n - 1];
  for (int64_t i = n - 2; i >= 0; --i) {
    y[i] = y[i] - y[i + 1];
    y[i] = y[i] / denom[i];
  }
  double fac = (y[0] - 0.25 * y[n - 1]) / sden;
  for (int64_t i = 0; i < n; ++i) y[i] = y[i] - fac * z[i];
}

/* _kernels.pyx:62-93 */
static void eval_line(const double* om, double* out, double shift, double h, int64_t n) {
  double s = shift / h;
  double off = floor(-s);
  double theta = -s - off;
  if (theta >= 1.0) {
    off += 1.0;
    theta = 0.0;
  }
  int64_t o = (int64_t)off;
  double omt = 1.0 - theta;
  double w0 = omt * omt * omt / 6.0;
  double w1 = (4.0 - 6.0 * theta * theta + 3.0 * theta * theta * theta) / 6.0;
  double w2 = (4.0 - 6.0 * omt * omt + 3.0 * omt * omt * omt) / 6.0;
  double w3 = theta * theta * theta / 6.0;
  int64_t j0 = wrap(o - 1, n);
  int64_t j1 = j0 + 1 < n ? j0 + 1 : 0;
  int64_t j2 = j1 + 1 < n ? j1 + 1 : 0;
  int64_t j3 = j2 + 1 < n ? j2 + 1 : 0;
  for (int64_t i = 0; i < n; ++i) {
    out[i] = w0 * om[j0] + w1 * om[j1] + w2 * om[j2] + w3 * om[j3];
    j0 = j0 + 1 < n ? j0 + 1 : 0;
    j1 = j1 + 1 < n ? j1 + 1 : 0;
    j2 = j2 + 1 < n ? j2 + 1 : 0;
    j3 = j3 + 1 < n ? j3 + 1 : 0;
  }
}

void oracle_spline_lines(const double* lines, double* out, int64_t nlines, int64_t n,
                         const int64_t* idx, const double* table, double h, const double* mult,
                         const double* denom, const double* z, double sden, double* scratch,
                         int threads) {
  /* scratch: threads * n doubles */
#pragma omp parallel num_threads(threads)
  {
#ifdef _OPENMP
    extern int omp_get_thread_num(void);
    double* y = scratch + (int64_t)omp_get_thread_num() * n;
#else
    double* y = scratch;
#endif
#pragma omp for schedule(static)
    for (int64_t r = 0; r < nlines; ++r) {
      solve_line(lines + r * n, y, mult, denom, z, sden, n);
      eval_line(y, out + r * n, table[idx[r]], h, n);
    }
  }
}

/* Markstein division identity used by the CUDA spline kernel: for r = RN(1/d),
 * fma(fma(-q, d, y), r, q) with q = RN(y*r) equals RN(y/d).  Returns the
 * number of mismatches over `count` pseudo-random numerators per
 * denominator in `den`. */
int64_t oracle_check_markstein(const double* den, int64_t nden, int64_t count, uint64_t seed) {
  int64_t bad = 0;
  uint64_t s = seed ? seed : 88172645463325252ULL;
  for (int64_t k = 0; k < nden; ++k) {
    double d = den[k], r = 1.0 / d;
    for (int64_t i = 0; i < count; ++i) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      uint64_t m = s & ((1ULL << 52) - 1);
      int e = (int)((s >> 52) % 121) - 60;
      uint64_t bits = ((s >> 63) << 63) | ((uint64_t)(1023 + e) << 52) | m;
      double y;
      memcpy(&y, &bits, 8);
      double qq = y * r;
      double ee = fma(-qq, d, y);
      double q2 = fma(ee, r, qq);
      if (q2 != y / d) ++bad;
    }
  }
  return bad;
}
