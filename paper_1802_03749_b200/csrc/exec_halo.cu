// X5: halo pack / unpack of the owner-compute decomposition.
//
// Rows are `comps` contiguous elements (AoS).  Pack gathers the rows a peer
// needs into a contiguous send buffer; unpack-add folds a peer's increments
// for our owned points into the increment array.  One warp per row group,
// coalesced over the row's components.
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
