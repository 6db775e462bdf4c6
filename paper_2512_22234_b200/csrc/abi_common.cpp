// Error reporting shared by every C-ABI entry point.
#include "abi_common.h"

#include <cstdio>
#include <cstdarg>
#include <atomic>
#include <mutex>
#include <map>
#include <utility>

namespace bd {

static thread_local char g_last_error[512] = "";
static std::atomic<long long> g_launches{0};

void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return BD_OK;
  return set_error(BD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int ensure_smem_attr(const void* func, int bytes, const char* what) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (function, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return check_cuda(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({func, dev});
  if (it != done.end() && it->second >= bytes) return BD_OK;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return check_cuda(e, what);
  done[{func, dev}] = bytes;
  return BD_OK;
}

int current_sm_count(int* n_sm) {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return check_cuda(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it == cache.end()) {
    int n = 0;
    e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return check_cuda(e, "cudaDeviceGetAttribute(SM count)");
    it = cache.emplace(dev, n).first;
  }
  *n_sm = it->second;
  return BD_OK;
}

}  // namespace bd

extern "C" const char* bd_error_string(int code) {
  switch (code) {
    case BD_OK: return "BD_OK";
    case BD_ERR_INVALID_ARG: return "BD_ERR_INVALID_ARG";
    case BD_ERR_LAYOUT: return "BD_ERR_LAYOUT";
    case BD_ERR_UNSUPPORTED: return "BD_ERR_UNSUPPORTED";
    case BD_ERR_ALIGNMENT: return "BD_ERR_ALIGNMENT";
    case BD_ERR_WORKSPACE: return "BD_ERR_WORKSPACE";
    case BD_ERR_CUDA: return "BD_ERR_CUDA";
    default: return "BD_ERR_UNKNOWN";
  }
}

extern "C" const char* bd_last_error(void) { return bd::g_last_error; }

extern "C" int64_t bd_launch_count(void) { return bd::g_launches.load(std::memory_order_relaxed); }
