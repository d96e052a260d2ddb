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

namespace {
struct DfChain {
  int dev;
  cudaEvent_t last;
  bool armed;
};
std::mutex g_df_mu;
std::vector<DfChain> g_df;
DfChain* df_chain(int dev) {
  for (auto& c : g_df)
    if (c.dev == dev) return &c;
  g_df.push_back({dev, nullptr, false});
  return &g_df.back();
}
}  // namespace

// The mutex is held from begin to end, so a launch from another host thread
// cannot slip between this launch's wait and its record.
cudaError_t static_dataflow_begin(cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  g_df_mu.lock();
  DfChain* c = df_chain(dev);
  if (!c->last) {
    e = cudaEventCreateWithFlags(&c->last, cudaEventDisableTiming);
    if (e) {
      g_df_mu.unlock();
      return e;
    }
  }
  e = c->armed ? cudaStreamWaitEvent(st, c->last, 0) : cudaSuccess;
  if (e) g_df_mu.unlock();
  return e;
}

cudaError_t static_dataflow_end(cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (!e) {
    DfChain* c = df_chain(dev);
    e = cudaEventRecord(c->last, st);
    if (!e) c->armed = true;
  }
  g_df_mu.unlock();
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
