// Serial-order executor on the device (the oracle semantics of
// execute_serial, simulator.py:215-242, without a CPU).
//
// Pass 1: every element computes its per-slot increments into a temp array
// (the paper's "temporary array" race-avoidance strategy).
// Pass 2: one thread per point folds its references in (element, slot) order
// starting from the initial value -- exactly np.add.at's order -- so the
// result is bit-identical to the serial loop for any data, not just for the
// quantised generator values.
#include "mp_loop.cuh"

namespace mp {
namespace {

template <class Op, typename T, int LAYOUT>
__global__ void serial_elem_kernel(LoopView<T> v, T* __restrict__ temp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < v.n; e += (int64_t)gridDim.x * blockDim.x) {
    T r[Op::ARITY][RcArr<Op>::N];
    if (Op::RC > 0) {
#pragma unroll
      for (int s = 0; s < Op::ARITY; ++s) {
        int p = map_at(v, e, s);
#pragma unroll
        for (int c = 0; c < Op::RC; ++c) r[s][c] = __ldg(v.ind + ind_index<LAYOUT>(p, c, v.ind_comps, v.npts));
      }
    }
    T d[Op::DC];
    load_direct<Op, T>(v, e, d);
    T o[Op::ARITY][Op::IC];
    compute<Op, T>(v, r, d, o);
#pragma unroll
    for (int s = 0; s < Op::ARITY; ++s)
#pragma unroll
      for (int c = 0; c < Op::IC; ++c) temp[(e * Op::ARITY + s) * Op::IC + c] = o[s][c];
  }
}

template <class Op, typename T, int LAYOUT>
__global__ void serial_point_kernel(LoopView<T> v, const int32_t* __restrict__ inv_off,
                                    const int32_t* __restrict__ inv_refs, const T* __restrict__ temp) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < v.npts; p += (int64_t)gridDim.x * blockDim.x) {
    const int a = inv_off[p], z = inv_off[p + 1];
    if (a == z) continue;
#pragma unroll
    for (int c = 0; c < Op::IC; ++c) {
      T* dst = v.inc + ind_index<LAYOUT>(p, c, Op::IC, v.npts);
      T acc = *dst;
      for (int r = a; r < z; ++r) acc = acc + temp[(int64_t)__ldg(inv_refs + r) * Op::IC + c];
      *dst = acc;
    }
  }
}

template <class Op, typename T>
mp_status launch_serial(const mp_loop& L, const int32_t* inv_off, const int32_t* inv_refs, void* temp,
                        cudaStream_t st) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(L, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (L.n_elems == 0) return MP_OK;
    LoopView<T> v = make_view<T>(L);
    int g1 = (int)((L.n_elems + 255) / 256 < 148 * 64 ? (L.n_elems + 255) / 256 : 148 * 64);
    int g2 = (int)((L.n_points + 255) / 256 < 148 * 64 ? (L.n_points + 255) / 256 : 148 * 64);
    if (g2 < 1) g2 = 1;
    T* t = static_cast<T*>(temp);
    if (L.ind_layout == MP_AOS) {
      serial_elem_kernel<Op, T, MP_AOS><<<g1, 256, 0, st>>>(v, t);
      serial_point_kernel<Op, T, MP_AOS><<<g2, 256, 0, st>>>(v, inv_off, inv_refs, t);
    } else {
      serial_elem_kernel<Op, T, MP_SOA><<<g1, 256, 0, st>>>(v, t);
      serial_point_kernel<Op, T, MP_SOA><<<g2, 256, 0, st>>>(v, inv_off, inv_refs, t);
    }
    MP_CHECK_LAUNCH();
    return MP_OK;
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_serial(const mp_loop* loop, const int32_t* inv_offsets, const int32_t* inv_refs,
                                    void* temp, void* stream) {
  mp::clear_error();
  if (!loop) MP_FAIL(MP_ERR_KERNEL, "null argument");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() {
      return mp::launch_serial<Op, scalar_t>(L, inv_offsets, inv_refs, temp, st);
    });
  });
}
