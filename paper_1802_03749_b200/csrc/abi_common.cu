// Library-level entry points: error buffer, version, device queries.
#include <stdarg.h>

#include "mp_common.cuh"

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
