// C-ABI error plumbing and version strings.
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace vpb {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return VPB_ERR_CUDA;
  }
  return VPB_OK;
}

static std::atomic<unsigned long long> g_launches{0};

int launched(const char* what, int n) {
  g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed);
  return check_launch(what);
}

}  // namespace vpb

extern "C" unsigned long long vpb_launch_count(void) { return vpb::g_launches.load(); }

extern "C" const char* vpb_version(void) { return "vpb200 0.1.0 sm_100a"; }

extern "C" const char* vpb_strerror(int code) {
  switch (code) {
    case VPB_OK: return "ok";
    case VPB_ERR_INVALID: return "invalid argument";
    case VPB_ERR_CUDA: return "CUDA error";
    case VPB_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

extern "C" const char* vpb_last_error(void) { return vpb::g_last_error; }
