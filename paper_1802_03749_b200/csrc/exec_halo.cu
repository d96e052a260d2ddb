// X5: halo pack / unpack of the owner-compute decomposition.
//
// Rows are `comps` contiguous elements (AoS).  Pack gathers the rows a peer
// needs into a contiguous send buffer; unpack-add folds a peer's increments
// for our owned points into the increment array.  One warp per row group,
// coalesced over the row's components.
//
// Peer-memory exchange (no NCCL on the data path): `put` packs rows straight
// into the receiving rank's mailbox (P2P stores over NVLink through an IPC
// mapping, or plain stores when the ranks share a device) and publishes the
// step's epoch in the receiver's flag once every CTA's stores are visible
// (system-scope fence, last-CTA-done counter, release store); `get` waits for
// the epoch in its own flag (acquire) and unpacks (set / add).  The epoch is a
// device counter bumped once per step (`mp_epoch_bump`), so the whole step
// -- bump, puts, gets, loop launches -- is a fixed launch sequence that a
// CUDA graph can capture.  Mailboxes are double-buffered by epoch parity;
// with one import and one export round per step, a sender reuses a slot only
// after the receiver has passed the step that read it (the receiver's next
// put to the sender follows that read in its stream order).
#include <string.h>

#include "mp_common.cuh"

namespace mp {
namespace {

template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ rows, int64_t nrows,
                                   int comps, T* __restrict__ dst) {
  const int64_t total = nrows * comps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / comps, c = i - r * comps;
    dst[i] = src[(int64_t)__ldg(rows + r) * comps + c];
  }
}

// mode 0: set, 1: add, 2: zero (src unused).  Rows are distinct within one
// call, so there is no write race.
template <typename T>
__global__ void scatter_rows_kernel(T* dst, const int32_t* __restrict__ rows, int64_t nrows, int comps,
                                    const T* __restrict__ src, int mode) {
  const int64_t total = nrows * comps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / comps, c = i - r * comps;
    T* a = dst + (int64_t)__ldg(rows + r) * comps + c;
    *a = mode == 2 ? T(0) : (mode == 1 ? *a + src[i] : src[i]);
  }
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__global__ void halo_put_kernel(const T* __restrict__ src, const int32_t* __restrict__ rows, int64_t nrows, int comps,
                                T* remote, int64_t slot_elems, uint32_t* remote_flag, const uint32_t* epoch_p,
                                uint32_t* done) {
  const uint32_t epoch = *epoch_p;
  T* dst = remote + (int64_t)(epoch & 1u) * slot_elems;
  const int64_t total = nrows * comps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / comps, c = i - r * comps;
    dst[i] = src[(int64_t)__ldg(rows + r) * comps + c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's stores, before its arrival
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0u;  // the next step's launch follows this one in stream order
      __threadfence_system();
      st_release_sys(remote_flag, epoch);
    }
  }
}

template <typename T>
__global__ void halo_get_kernel(T* dst, const int32_t* __restrict__ rows, int64_t nrows, int comps, const T* mailbox,
                                int64_t slot_elems, const uint32_t* flag, const uint32_t* epoch_p, int mode) {
  const uint32_t epoch = *epoch_p;
  if (threadIdx.x == 0)
    while ((int32_t)(ld_acquire_sys(flag) - epoch) < 0) __nanosleep(64);
  __syncthreads();
  const T* src = mailbox + (int64_t)(epoch & 1u) * slot_elems;
  const int64_t total = nrows * comps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / comps, c = i - r * comps;
    T* a = dst + (int64_t)__ldg(rows + r) * comps + c;
    const T x = __ldcg(src + i);  // written by the peer: from L2, never a stale L1 line
    *a = mode == 1 ? *a + x : x;
  }
}

__global__ void epoch_bump_kernel(uint32_t* epoch) { *epoch += 1u; }

// the previous kernels on this stream have completed (stream order); make
// their P2P stores visible system-wide before the flag
__global__ void halo_signal_kernel(uint32_t* remote_flag, const uint32_t* epoch_p) {
  __threadfence_system();
  st_release_sys(remote_flag, *epoch_p);
}

inline int grid_of(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_halo_pack(int32_t dtype, const void* src, const int32_t* rows, int64_t nrows, int32_t comps,
                                  void* dst, void* stream) {
  mp::clear_error();
  if (nrows == 0) return MP_OK;
  cudaStream_t st = mp::as_stream(stream);
  return MP_DISPATCH_DTYPE(dtype, [&]() -> mp_status {
    mp::gather_rows_kernel<scalar_t><<<mp::grid_of(nrows * comps), 256, 0, st>>>(
        static_cast<const scalar_t*>(src), rows, nrows, comps, static_cast<scalar_t*>(dst));
    MP_CHECK_LAUNCH();
    return (mp_status)MP_OK;
  });
}

extern "C" mp_status mp_halo_unpack(int32_t dtype, void* dst, const int32_t* rows, int64_t nrows, int32_t comps,
                                    const void* src, int32_t mode, void* stream) {
  mp::clear_error();
  if (nrows == 0) return MP_OK;
  if (mode < 0 || mode > 2) MP_FAIL(MP_ERR_KERNEL, "bad unpack mode %d", mode);
  cudaStream_t st = mp::as_stream(stream);
  return MP_DISPATCH_DTYPE(dtype, [&]() -> mp_status {
    mp::scatter_rows_kernel<scalar_t><<<mp::grid_of(nrows * comps), 256, 0, st>>>(
        static_cast<scalar_t*>(dst), rows, nrows, comps, static_cast<const scalar_t*>(src), mode);
    MP_CHECK_LAUNCH();
    return (mp_status)MP_OK;
  });
}

// exchange kernels are small (a halo is thousands of rows): a few CTAs
static int exchange_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 32 ? 32 : g));
}

extern "C" mp_status mp_halo_put(int32_t dtype, const void* src, const int32_t* rows, int64_t nrows, int32_t comps,
                                 void* remote, int64_t slot_elems, uint32_t* remote_flag, const uint32_t* epoch,
                                 uint32_t* done_counter, void* stream) {
  mp::clear_error();
  cudaStream_t st = mp::as_stream(stream);
  return MP_DISPATCH_DTYPE(dtype, [&]() -> mp_status {
    mp::halo_put_kernel<scalar_t><<<exchange_grid(nrows * comps), 256, 0, st>>>(
        static_cast<const scalar_t*>(src), rows, nrows, comps, static_cast<scalar_t*>(remote), slot_elems,
        remote_flag, epoch, done_counter);
    MP_CHECK_LAUNCH();
    return (mp_status)MP_OK;
  });
}

extern "C" mp_status mp_halo_get(int32_t dtype, void* dst, const int32_t* rows, int64_t nrows, int32_t comps,
                                 const void* mailbox, int64_t slot_elems, const uint32_t* flag, const uint32_t* epoch,
                                 int32_t mode, void* stream) {
  mp::clear_error();
  if (mode != 0 && mode != 1) MP_FAIL(MP_ERR_KERNEL, "bad get mode %d", mode);
  cudaStream_t st = mp::as_stream(stream);
  return MP_DISPATCH_DTYPE(dtype, [&]() -> mp_status {
    mp::halo_get_kernel<scalar_t><<<exchange_grid(nrows * comps), 256, 0, st>>>(
        static_cast<scalar_t*>(dst), rows, nrows, comps, static_cast<const scalar_t*>(mailbox), slot_elems, flag,
        epoch, mode);
    MP_CHECK_LAUNCH();
    return (mp_status)MP_OK;
  });
}

extern "C" mp_status mp_epoch_bump(uint32_t* epoch, void* stream) {
  mp::clear_error();
  mp::epoch_bump_kernel<<<1, 1, 0, mp::as_stream(stream)>>>(epoch);
  MP_CHECK_LAUNCH();
  return MP_OK;
}

extern "C" mp_status mp_mailbox_alloc(int64_t bytes, void** ptr) {
  mp::clear_error();
  *ptr = nullptr;
  MP_CUDA_TRY(cudaMalloc(ptr, bytes > 0 ? (size_t)bytes : 256));
  // zeroed before the caller publishes it: a peer's first put may follow at
  // once, on a stream that does not order after the legacy default stream
  cudaStream_t s;
  MP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemsetAsync(*ptr, 0, bytes > 0 ? (size_t)bytes : 256, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  MP_CUDA_TRY(e);
  return MP_OK;
}

extern "C" mp_status mp_ipc_handle(void* ptr, unsigned char* handle /* 64 bytes */) {
  mp::clear_error();
  cudaIpcMemHandle_t h;
  MP_CUDA_TRY(cudaIpcGetMemHandle(&h, ptr));
  memcpy(handle, &h, sizeof(h));
  return MP_OK;
}

extern "C" mp_status mp_ipc_open(const unsigned char* handle, void** ptr) {
  mp::clear_error();
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  MP_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return MP_OK;
}

extern "C" mp_status mp_ipc_close(void* ptr) {
  mp::clear_error();
  MP_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return MP_OK;
}

extern "C" mp_status mp_halo_signal(uint32_t* remote_flag, const uint32_t* epoch, void* stream) {
  mp::clear_error();
  mp::halo_signal_kernel<<<1, 1, 0, mp::as_stream(stream)>>>(remote_flag, epoch);
  MP_CHECK_LAUNCH();
  return MP_OK;
}
