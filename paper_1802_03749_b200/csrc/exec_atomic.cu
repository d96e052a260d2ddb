// Atomics baseline (the paper's first race-avoidance strategy, PAPER.md:325-341;
// sized by the reference cost model's _alt_strategy_costs, simulator.py:331-341):
// one thread per element in plan order, reads gathered straight from HBM,
// increments applied with hardware atomics (RED.ADD).  The order in which a
// point's increments land is unspecified, so results equal the reference only
// up to floating-point reassociation (exactly on the generators' 1/1024-grid
// data).  A measured comparison baseline, not the product.
#include "mp_loop.cuh"

namespace mp {
namespace {

template <typename T>
__device__ __forceinline__ void atomic_add(T* a, T x) {
  if constexpr (sizeof(T) == 8 && !std::is_floating_point<T>::value)
    atomicAdd(reinterpret_cast<unsigned long long*>(a), static_cast<unsigned long long>(x));
  else
    atomicAdd(a, x);
}

template <class Op, typename T, int LAYOUT>
__global__ void __launch_bounds__(256) atomic_kernel(LoopView<T> v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < v.n; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t p[Op::ARITY];
#pragma unroll
    for (int s = 0; s < Op::ARITY; ++s) p[s] = map_at(v, e, s);
    T r[Op::ARITY][RcArr<Op>::N];
    if (Op::RC > 0) {
#pragma unroll
      for (int s = 0; s < Op::ARITY; ++s)
#pragma unroll
        for (int c = 0; c < Op::RC; ++c) r[s][c] = __ldg(v.ind + ind_index<LAYOUT>(p[s], c, v.ind_comps, v.npts));
    }
    T d[Op::DC];
    load_direct<Op, T>(v, e, d);
    T o[Op::ARITY][Op::IC];
    compute<Op, T>(v, r, d, o);
#pragma unroll
    for (int s = 0; s < Op::ARITY; ++s)
#pragma unroll
      for (int c = 0; c < Op::IC; ++c) atomic_add(v.inc + ind_index<LAYOUT>(p[s], c, Op::IC, v.npts), o[s][c]);
  }
}

template <class Op, typename T>
mp_status launch_atomic(const mp_loop& L, cudaStream_t st) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(L, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (L.n_elems == 0) return MP_OK;
    LoopView<T> v = make_view<T>(L);
    int dev = 0, sms = 0;
    MP_CUDA_TRY(cudaGetDevice(&dev));
    MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t want = (L.n_elems + 255) / 256, cap = (int64_t)sms * 16;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    if (L.ind_layout == MP_AOS)
      atomic_kernel<Op, T, MP_AOS><<<grid, 256, 0, st>>>(v);
    else
      atomic_kernel<Op, T, MP_SOA><<<grid, 256, 0, st>>>(v);
    MP_CHECK_LAUNCH();
    return MP_OK;
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_atomic(const mp_loop* loop, void* stream) {
  mp::clear_error();
  if (!loop) MP_FAIL(MP_ERR_KERNEL, "null argument");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() { return mp::launch_atomic<Op, scalar_t>(L, st); });
  });
}
