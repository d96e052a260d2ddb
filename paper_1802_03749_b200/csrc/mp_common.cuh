// Shared helpers of the native library: status/error plumbing, dtype
// dispatch, memory-order primitives.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/meshplan_b200.h"

namespace mp {

// thread-local message of the last failing call (mp_last_error)
void set_error(const char* fmt, ...);
void clear_error();
// Raise a kernel's dynamic shared-memory limit to at least `smem` bytes on the
// current device.  The limit only ever grows (process-wide, under a mutex), so
// threads launching the same kernel with different sizes never lower it
// between another thread's set and launch.
cudaError_t raise_smem_limit(const void* kern, size_t smem);
// Static-claim dataflow grids (fill f of CTA c takes ticket c + f*grid; CTAs
// spin on predecessor flags) are deadlock-free only while all their CTAs are
// resident.  A non-spinning grid sharing the GPU only delays residency; a
// second spinning static-claim grid can hold the SMs the first one's
// unscheduled CTAs need.  Every such launch on a device is therefore chained
// behind the previous one (process-wide event chain): call begin before and
// end after the launch, on the launch stream.
cudaError_t static_dataflow_begin(cudaStream_t st);
cudaError_t static_dataflow_end(cudaStream_t st);

#define MP_CUDA_TRY(expr)                                                                 \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      ::mp::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,       \
                      __LINE__, cudaGetErrorString(_e));                                  \
      return MP_ERR_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

#define MP_CHECK_LAUNCH() MP_CUDA_TRY(cudaGetLastError())

#define MP_FAIL(code, ...)          \
  do {                              \
    ::mp::set_error(__VA_ARGS__);   \
    return (code);                  \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- memory-order primitives -------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// L2-only load/store for data another CTA may have written this launch
template <typename T>
__device__ __forceinline__ T ld_cg(const T* p) { return __ldcg(p); }

}  // namespace mp

// dtype dispatch: calls F.template operator()<T>()
#define MP_DISPATCH_DTYPE(dtype, ...)                           \
  [&]() -> mp_status {                                          \
    switch (dtype) {                                            \
      case MP_F64: { using scalar_t = double; return __VA_ARGS__(); }  \
      case MP_F32: { using scalar_t = float; return __VA_ARGS__(); }   \
      case MP_I64: { using scalar_t = long long; return __VA_ARGS__(); } \
      case MP_I32: { using scalar_t = int; return __VA_ARGS__(); }     \
      default: MP_FAIL(MP_ERR_KERNEL, "unknown element type %d", (int)(dtype)); \
    }                                                           \
  }()
