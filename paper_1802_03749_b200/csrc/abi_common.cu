// Library-level entry points: error buffer, version, device queries.
#include <stdarg.h>

#include "mp_common.cuh"

#include <mutex>
#include <vector>

namespace mp {
namespace {
thread_local std::string g_last_error;
}

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }

const char* last_error() { return g_last_error.c_str(); }

cudaError_t raise_smem_limit(const void* kern, size_t smem) {
  struct Limit {
    const void* k;
    int dev;
    size_t smem;
  };
  static std::mutex mu;
  static std::vector<Limit> limits;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& l : limits)
    if (l.k == kern && l.dev == dev) {
      if (l.smem >= smem) return cudaSuccess;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (!e) l.smem = smem;
      return e;
    }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (!e) limits.push_back({kern, dev, smem});
  return e;
}

}  // namespace mp

extern "C" const char* mp_last_error(void) { return mp::last_error(); }

extern "C" const char* mp_version(void) { return "meshplan-b200 0.1 sm_100a"; }

extern "C" int32_t mp_device_sm_count(int32_t device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

extern "C" void mp_free(void* device_ptr) {
  if (device_ptr) cudaFree(device_ptr);
}
