// Shared pieces of the fused x-plane passes (fused.cu: one Strang x half
// step per HBM pass; fused2.cu: two consecutive half steps per pass).
#pragma once

#include "common.cuh"

namespace vpb {

struct XChunk {
  int first;    // first output cell
  int nout;     // output cells
  int nsrc;     // source cells loaded (1 for the prologue chunk, else nout)
  int s_begin;  // first source cell (mod C2)
};

// Walks the chunks of a run of planes with 32-bit bookkeeping only.
// lead = number of x2 sweeps chained behind the loads (1: fused.cu, 2:
// fused2.cu): the first output cell of a plane then needs source cell
// s0 = -lead*(q2+1) mod C2 as its prologue.
struct XCursor {
  int64_t plane;
  int i;         // chunk index inside the plane
  int s0;        // -lead*(q2+1) mod C2 of the current plane
  int lead = 1;
  __device__ __forceinline__ void start(int64_t pl, int C2, const int64_t* __restrict__ q2,
                                        int64_t nv1) {
    plane = pl;
    i = 0;
    s0 = (int)wrap_mod(-(int64_t)lead * (q2[pl / nv1] + 1), C2);
  }
  __device__ __forceinline__ XChunk chunk(int G, int C2) const {
    XChunk c;
    if (i == 0) {
      c.first = 0;
      c.nout = 0;
      c.nsrc = 1;
      c.s_begin = s0;
      return c;
    }
    c.first = (i - 1) * G;
    c.nout = min(G, C2 - c.first);
    c.nsrc = c.nout;
    int sb = s0 + 1 + c.first;
    if (sb >= C2) sb -= C2;
    c.s_begin = sb;
    return c;
  }
  // pl_end: one past the CTA's last plane (its tables are never read)
  __device__ __forceinline__ void advance(int per_plane, int C2, const int64_t* __restrict__ q2,
                                          int64_t nv1, int64_t pl_end) {
    if (++i == per_plane) {
      if (plane + 1 < pl_end) {
        start(plane + 1, C2, q2, nv1);
      } else {
        ++plane;
        i = 0;
      }
    }
  }
};

template <int P>
__device__ __forceinline__ void lds_row_cell(const double* p, double (&u)[P]) {
  if constexpr (P % 2 == 0) {
#pragma unroll
    for (int m = 0; m < P; m += 2) {
      const double2 v = *reinterpret_cast<const double2*>(p + m);
      u[m] = v.x;
      u[m + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int m = 0; m < P; ++m) u[m] = p[m];
  }
}

// x1 sweep of one source x2 cell (P rows) for this thread's x1 cell
// (_kernels.pyx:113-123): g[m2][j] = sum_m A1[j][m] u_lo[m] + sum_m B1[j][m] u_up[m].
template <int P, bool EX1>
__device__ __forceinline__ void xplane_x1_cell(const double* rows, int n1, int lo_off,
                                               int up_off, const double (&A1)[P][P],
                                               const double (&B1)[P][P], double (&g)[P][P]) {
#pragma unroll
  for (int m2 = 0; m2 < P; ++m2) {
    const double* row = rows + m2 * n1;
    double uu[P];
    lds_row_cell<P>(row + up_off, uu);
    if constexpr (EX1) {
#pragma unroll
      for (int jj = 0; jj < P; ++jj) g[m2][jj] = uu[jj];
    } else {
      double ul[P];
      lds_row_cell<P>(row + lo_off, ul);
#pragma unroll
      for (int jj = 0; jj < P; ++jj) {
        double acc_a = dmul(A1[jj][0], ul[0]);
#pragma unroll
        for (int m = 1; m < P; ++m) acc_a = step_madd(acc_a, A1[jj][m], ul[m]);
        double acc_b = dmul(B1[jj][0], uu[0]);
#pragma unroll
        for (int m = 1; m < P; ++m) acc_b = step_madd(acc_b, B1[jj][m], uu[m]);
        g[m2][jj] = dadd(acc_a, acc_b);
      }
    }
  }
}

// x2 sweep of one output cell from the x1-swept source cells gp (= s-1) and
// g (= s): o[j2][jj] = sum_m A2[j2][m] gp[m][jj] + sum_m B2[j2][m] g[m][jj].
template <int P, bool EX2>
__device__ __forceinline__ void xplane_x2_cell(const double (&A2)[P][P], const double (&B2)[P][P],
                                               const double (&gp)[P][P], const double (&g)[P][P],
                                               double (&o)[P][P]) {
#pragma unroll
  for (int j2 = 0; j2 < P; ++j2)
#pragma unroll
    for (int jj = 0; jj < P; ++jj) {
      if constexpr (EX2) {
        o[j2][jj] = g[j2][jj];
      } else {
        double acc_a = dmul(A2[j2][0], gp[0][jj]);
#pragma unroll
        for (int m = 1; m < P; ++m) acc_a = step_madd(acc_a, A2[j2][m], gp[m][jj]);
        double acc_b = dmul(B2[j2][0], g[0][jj]);
#pragma unroll
        for (int m = 1; m < P; ++m) acc_b = step_madd(acc_b, B2[j2][m], g[m][jj]);
        o[j2][jj] = dadd(acc_a, acc_b);
      }
    }
}

// Optional density epilogue of the x-plane pass (poisson.py:85-95 followed by
// the cell-centre collapse of poisson.py:129-139): every output P x P cell
// block is collapsed with the Lagrange weights at the cell centre (for odd P
// the centre is the middle Gauss node and the collapse is a selection),
// weighted by the plane's velocity weight, and added into the CTA's own
// partial slab [C2][C1] with a fire-and-forget reduction (RED; only thread c
// touches column c of its CTA's slab, so the order is program order and the
// result deterministic).  The neutrality mean (poisson.py:143-160) rides
// along as a per-thread scalar.  The cell weight tables live in the kernel
// parameters (constant bank operands, no registers).
struct XDensity {
  const double* wv1;   // [nv1] velocity weights
  const double* wv2;   // [nv2]
  double* rc_part;     // [grid][C2][C1] or nullptr (epilogue off)
  double* mean_part;   // [grid]
  double mm[kMaxOrder * kMaxOrder];  // mid[j2] * mid[jj]
  double ww[kMaxOrder * kMaxOrder];  // cell space weights wcell2[j2] * wcell1[jj]
};

// Diagnostics-moment partials of the single x pass (fused.cu, DM == 2).
struct XMoments {
  double* mom_part;    // [grid][3] = l1, l2^2, kinetic
  const double* vsq1;  // [nv1] v1^2
  const double* vsq2;  // [nv2] v2^2
};

int xplane_sm_count();
int xplane_args_ok(const double* src, const double* dst, const int64_t dims[4], int32_t order);
int xdensity_setup(XDensity* dn, int order, const double* wv1, const double* wv2,
                   const double* mid_host, const double* wcell1_host, const double* wcell2_host,
                   double* work, int64_t nblk, int64_t cc);
// rc[c2][c1] = fixed-order sum of the CTA slabs; stats[0] = mean / volume
// With mom_part / diag_out: diag_out[0..3] = mass, l1, l2^2, kinetic as well.
int launch_xdens_reduce(const double* work, int64_t nblk, int64_t cc, double volume,
                        double* rc_out, double* stats, cudaStream_t st,
                        const double* mom_part = nullptr, double* diag_out = nullptr);

}  // namespace vpb

#ifdef VPB_ONLY_P3  // quick ptxas experiments: orders 2 and 3 only
#define VPB_XPLANE_SWITCH(order, ...)                                              \
  switch (order) {                                                                 \
    case 2: { constexpr int PP = 2; __VA_ARGS__; } break;                                 \
    default: { constexpr int PP = 3; __VA_ARGS__; } break;                                \
  }
#else
#define VPB_XPLANE_SWITCH(order, ...)                                              \
  switch (order) {                                                                 \
    case 1: { constexpr int PP = 1; __VA_ARGS__; } break;                                 \
    case 2: { constexpr int PP = 2; __VA_ARGS__; } break;                                 \
    case 3: { constexpr int PP = 3; __VA_ARGS__; } break;                                 \
    case 4: { constexpr int PP = 4; __VA_ARGS__; } break;                                 \
    case 5: { constexpr int PP = 5; __VA_ARGS__; } break;                                 \
    case 6: { constexpr int PP = 6; __VA_ARGS__; } break;                                 \
    case 7: { constexpr int PP = 7; __VA_ARGS__; } break;                                 \
    case 8: { constexpr int PP = 8; __VA_ARGS__; } break;                                 \
    default: { constexpr int PP = 9; __VA_ARGS__; } break;                                \
  }
#endif
