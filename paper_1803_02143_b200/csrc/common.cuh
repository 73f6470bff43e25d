// Shared helpers for the vpb200 sm_100a kernels.
//
// Arithmetic note: every kernel that restates a reference line kernel
// (/root/reference/pkg/src/slvp/_kernels.pyx) uses explicit __dmul_rn /
// __dadd_rn so ptxas cannot contract a*b+c into an FMA.  The reference's
// compiled backend is built without FMA contraction (gcc -O3, x86-64
// baseline, pkg/setup.py:5-15), so keeping the same operation order and
// rounding makes the CUDA sweeps bitwise equal to it for identical tables.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vpb200.h"

namespace vpb {

constexpr int kMaxOrder = 9;  // dg_order 1..9 (driver.py:95-107)

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// acc + a*b in the fused step passes: two roundings, in the reference's
// order (bitwise reproduction of its compiled kernels) unless the library is
// built with -DVPB_STEP_FMA=1 (one rounding; an A/B experiment, not the
// shipped configuration -- see DESIGN.md).
#ifndef VPB_STEP_FMA
#define VPB_STEP_FMA 0
#endif
__device__ __forceinline__ double step_madd(double acc, double a, double b) {
#if VPB_STEP_FMA
  return __fma_rn(a, b, acc);
#else
  return dadd(acc, dmul(a, b));
#endif
}

// Python-style modulo into [0, n).
__host__ __device__ __forceinline__ int64_t wrap_mod(int64_t v, int64_t n) {
  int64_t r = v % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ bool not_finite(double x) {
  // exponent all ones <=> inf or nan
  return (__double_as_longlong(x) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
}

// Running non-finite test on the integer pipe: the maximum exponent field
// seen.  (ptxas turns the compare form above into one DSETP per value on
// the fp64 pipe, which the hot sweeps need for their arithmetic.)
struct ExpMax {
  uint32_t m = 0;
  __device__ __forceinline__ void add(double x) {
    m = max(m, (uint32_t)__double2hiint(x) & 0x7ff00000u);
  }
  __device__ __forceinline__ bool bad() const { return m == 0x7ff00000u; }
};

// Non-finite report into a device flag word (the per-sub-step finite check
// of driver.py:209-211, moved into the producing kernel's epilogue).
__device__ __forceinline__ void report_flag(bool bad, int32_t* flag) {
  if (bad && flag != nullptr) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// Error plumbing for the C ABI: no exceptions cross the boundary.
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);
// check_launch + count `n` kernel launches (vpb_launch_count, bench.py gpu_launches)
int launched(const char* what, int n = 1);

}  // namespace vpb

#define VPB_REQUIRE(cond, ...)                 \
  do {                                         \
    if (!(cond)) {                             \
      ::vpb::set_error(__VA_ARGS__);           \
      return VPB_ERR_INVALID;                  \
    }                                          \
  } while (0)
