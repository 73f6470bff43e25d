// Sharded-field support for the multi-GPU layer: halo slab
// packing and the halo-aware dG sweep along a sharded x axis.
//
// A shard of a field sharded along x1 (axis 0) or x2 (axis 1) holds a whole
// number of cells of that axis.  Output cell c of a sweep reads source
// cells c-q-1 and c-q (global shift q), which may fall outside the shard;
// those come from halo slabs exchanged with the neighbouring ranks.  A halo
// slab has the canonical layout of the field restricted to `width` cells of
// the sharded axis.
#include <algorithm>

#include "common.cuh"

namespace vpb {

__global__ void halo_pack_kernel(const double* __restrict__ f, double* __restrict__ buf,
                                 int64_t inner, int64_t nax, int64_t outer, int64_t off,
                                 int64_t wdof) {
  // f viewed as [outer][nax][inner]; buf as [outer][wdof][inner]
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = outer * wdof * inner;
  if (e >= total) return;
  int64_t i = e % inner;
  int64_t r = e / inner;
  int64_t k = r % wdof;
  int64_t o = r / wdof;
  buf[e] = f[(o * nax + off + k) * inner + i];
}

// Strided slab copy: run k of `run` doubles from src + k*ss to dst + k*ds.
// blockIdx.x covers a run in 512-double pieces (double2 per thread when both
// sides are 16-byte aligned), blockIdx.y strides over the runs.
__global__ void slab_copy_kernel(const double* __restrict__ src, int64_t ss,
                                 double* __restrict__ dst, int64_t ds, int64_t outer, int64_t run,
                                 bool vec2) {
  const int64_t i0 = (int64_t)blockIdx.x * 512 + threadIdx.x * 2;
  for (int64_t k = blockIdx.y; k < outer; k += gridDim.y) {
    const double* s = src + k * ss;
    double* d = dst + k * ds;
    if (vec2 && i0 + 1 < run) {
      *reinterpret_cast<double2*>(d + i0) = __ldcs(reinterpret_cast<const double2*>(s + i0));
    } else {
      if (i0 < run) d[i0] = s[i0];
      if (i0 + 1 < run) d[i0 + 1] = s[i0 + 1];
    }
  }
}

template <int P>
struct HCoeffs {
  double A[P][P];
  double B[P][P];
  int64_t q;
  bool exact;
};

template <int P>
__device__ __forceinline__ void h_load(HCoeffs<P>& k, int64_t t, const double* ta,
                                       const double* tb, const int64_t* tq, const double* tal) {
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
__device__ __forceinline__ void h_update(const HCoeffs<P>& k, const double (&lo)[P],
                                         const double (&up)[P], double (&out)[P]) {
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double acc_a = __dmul_rn(k.A[j][0], lo[0]);
#pragma unroll
    for (int m = 1; m < P; ++m) acc_a = __dadd_rn(acc_a, __dmul_rn(k.A[j][m], lo[m]));
    double acc_b = __dmul_rn(k.B[j][0], up[0]);
#pragma unroll
    for (int m = 1; m < P; ++m) acc_b = __dadd_rn(acc_b, __dmul_rn(k.B[j][m], up[m]));
    out[j] = __dadd_rn(acc_a, acc_b);
  }
}

// One thread per (line, output cell).  Lines: f viewed as [outer][C*P][inner]
// with the sweep axis in the middle (inner = 1 for axis 0).
template <int P>
__global__ void dg_halo_kernel(const double* __restrict__ src, double* __restrict__ dst,
                               int64_t inner, int64_t outer, int C, const double* __restrict__ left,
                               int64_t wl, const double* __restrict__ right, int64_t wr,
                               int64_t tdiv, int64_t tmod, const double* __restrict__ ta,
                               const double* __restrict__ tb, const int64_t* __restrict__ tq,
                               const double* __restrict__ tal, int32_t* __restrict__ flag) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = outer * C * inner;
  if (e >= total) return;
  int64_t i = e % inner;
  int64_t r = e / inner;
  int c = (int)(r % C);
  int64_t o = r / C;
  int64_t line = o * inner + i;  // canonical line id (outer, inner)
  int64_t t = (line / tdiv) % tmod;
  HCoeffs<P> k;
  h_load<P>(k, t, ta, tb, tq, tal);
  auto cell = [&](int64_t kc, double (&u)[P]) {
    const double* base;
    int64_t nax, kk;
    if (kc < 0) {
      base = left;
      nax = wl * P;
      kk = kc + wl;
    } else if (kc >= C) {
      base = right;
      nax = wr * P;
      kk = kc - C;
    } else {
      base = src;
      nax = (int64_t)C * P;
      kk = kc;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) u[m] = base[(o * nax + kk * P + m) * inner + i];
  };
  double uu[P], res[P];
  cell((int64_t)c - k.q, uu);
  if (k.exact) {
#pragma unroll
    for (int j = 0; j < P; ++j) res[j] = uu[j];
  } else {
    double ul[P];
    cell((int64_t)c - k.q - 1, ul);
    h_update<P>(k, ul, uu, res);
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    dst[(o * (int64_t)C * P + (int64_t)c * P + j) * inner + i] = res[j];
    bad |= not_finite(res[j]);
  }
  report_flag(bad, flag);
}

template <int P>
static int launch_halo(const double* src, double* dst, int64_t inner, int64_t outer, int C,
                       const double* left, int64_t wl, const double* right, int64_t wr,
                       int64_t tdiv, int64_t tmod, const double* a, const double* b,
                       const int64_t* q, const double* alpha, int32_t* flag, cudaStream_t st) {
  int64_t total = outer * C * inner;
  if (total == 0) return VPB_OK;
  dg_halo_kernel<P><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag);
  return launched("dg_halo_kernel");
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_halo_pack(int32_t axis, const double* f, const int64_t dims[4], int32_t order,
                             int64_t cell0, int64_t width, double* buf, void* stream) {
  VPB_REQUIRE(axis == 0 || axis == 1, "halo axis must be 0 or 1");
  VPB_REQUIRE(order >= 1 && dims[axis] % order == 0, "bad order");
  const int64_t C = dims[axis] / order;
  VPB_REQUIRE(cell0 >= 0 && width >= 0 && cell0 + width <= C, "halo range outside the shard");
  int64_t inner = axis == 0 ? 1 : dims[0];
  int64_t nax = dims[axis];
  int64_t outer = axis == 0 ? dims[1] * dims[2] * dims[3] : dims[2] * dims[3];
  int64_t total = outer * width * order * inner;
  if (total == 0) return VPB_OK;
  halo_pack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      f, buf, inner, nax, outer, cell0 * order, width * order);
  return launched("halo_pack_kernel");
}

extern "C" int vpb_dg_sweep_axis_halo(int32_t axis, const double* src, double* dst,
                                      const int64_t dims[4], int32_t order, const double* left,
                                      int64_t wl, const double* right, int64_t wr,
                                      const double* a, const double* b, const int64_t* q,
                                      const double* alpha, int32_t* flag, void* stream) {
  VPB_REQUIRE(axis == 0 || axis == 1, "halo sweep axis must be 0 or 1");
  VPB_REQUIRE(src != dst, "src and dst must be distinct buffers");
  VPB_REQUIRE(order >= 1 && dims[axis] % order == 0, "bad order");
  VPB_REQUIRE(wl >= 0 && wr >= 0, "negative halo width");
  const int C = (int)(dims[axis] / order);
  const int64_t n1 = dims[0], n2 = dims[1], nv1 = dims[2], nv2 = dims[3];
  int64_t inner, outer, tdiv, tmod;
  if (axis == 0) {
    inner = 1;
    outer = n2 * nv1 * nv2;  // line = (iv2, iv1, ix2); table row = iv1
    tdiv = n2;
    tmod = nv1;
  } else {
    inner = n1;
    outer = nv1 * nv2;  // line = (iv2, iv1) * n1 + ix1; table row = iv2
    tdiv = n1 * nv1;
    tmod = nv2;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (order) {
    case 1: return launch_halo<1>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 2: return launch_halo<2>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 3: return launch_halo<3>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 4: return launch_halo<4>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 5: return launch_halo<5>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 6: return launch_halo<6>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 7: return launch_halo<7>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 8: return launch_halo<8>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    case 9: return launch_halo<9>(src, dst, inner, outer, C, left, wl, right, wr, tdiv, tmod, a, b, q, alpha, flag, st);
    default:
      set_error("dG order %d outside the supported range 1..9", order);
      return VPB_ERR_UNSUPPORTED;
  }
}

extern "C" int vpb_slab_copy(const double* src, int64_t src_stride, double* dst,
                             int64_t dst_stride, int64_t outer, int64_t run, void* stream) {
  VPB_REQUIRE(outer >= 0 && run >= 0 && src_stride >= run && dst_stride >= run,
              "bad slab geometry");
  if (outer == 0 || run == 0) return VPB_OK;
  VPB_REQUIRE(src != nullptr && dst != nullptr, "null pointer");
  const bool vec2 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 &&
                    src_stride % 2 == 0 && dst_stride % 2 == 0;
  dim3 grid((unsigned)((run + 511) / 512), (unsigned)std::min<int64_t>(outer, 65535));
  slab_copy_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(src, src_stride, dst, dst_stride,
                                                           outer, run, vec2);
  return launched("slab_copy_kernel");
}
