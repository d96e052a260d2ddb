// Per-element gather / compute helpers shared by the executors.
#pragma once

#include <type_traits>

#include "mp_ops.cuh"

namespace mp {

template <typename T>
struct LoopView {
  int64_t n, npts;
  int32_t arity, map_layout, ind_comps, dir_comps, inc_comps, unit;
  const int32_t* __restrict__ map;
  const T* __restrict__ ind;
  const T* __restrict__ dir;
  T* inc;
};

template <typename T>
inline LoopView<T> make_view(const mp_loop& L) {
  LoopView<T> v;
  v.n = L.n_elems;
  v.npts = L.n_points;
  v.arity = L.arity;
  v.map_layout = L.map_layout;
  v.ind_comps = L.ind_read_comps;
  v.dir_comps = L.dir_comps;
  v.inc_comps = L.inc_comps;
  v.unit = L.unit;
  v.map = L.map;
  v.ind = static_cast<const T*>(L.ind_read);
  v.dir = static_cast<const T*>(L.dir_read);
  v.inc = static_cast<T*>(L.inc);
  return v;
}

template <typename T>
__device__ __forceinline__ int32_t map_at(const LoopView<T>& v, int64_t e, int s) {
  return __ldg(v.map_layout == MP_AOS ? v.map + e * v.arity + s : v.map + (int64_t)s * v.n + e);
}

// direct operands (SoA, plan.py:381-398)
template <class Op, typename T>
__device__ __forceinline__ void load_direct(const LoopView<T>& v, int64_t e, T (&d)[Op::DC]) {
#pragma unroll
  for (int c = 0; c < Op::DC; ++c) d[c] = __ldg(v.dir + (int64_t)c * v.n + e);
}

// per-slot increments (unit variant: all ones, bench_kernels.py:172-173)
template <class Op, typename T>
__device__ __forceinline__ void compute(const LoopView<T>& v, const T (&r)[Op::ARITY][RcArr<Op>::N],
                                        const T (&d)[Op::DC], T (&o)[Op::ARITY][Op::IC]) {
  if (v.unit) {
#pragma unroll
    for (int s = 0; s < Op::ARITY; ++s)
#pragma unroll
      for (int c = 0; c < Op::IC; ++c) o[s][c] = T(1);
  } else {
    Op::template apply<T>(r, d, o);
  }
}

template <class Op, typename T>
constexpr bool op_supported() {
  return !(std::is_same<Op, OpFaceFluxHeavy>::value && std::is_integral<T>::value);
}

inline mp_status check_loop_shape(const mp_loop& L, int arity, int rc, int dc, int ic) {
  if (L.arity != arity)
    MP_FAIL(MP_ERR_KERNEL, "op %d needs an arity-%d mapping, got %d", L.op, arity, L.arity);
  if (rc > 0 && (L.ind_read == nullptr || L.ind_read_comps < rc))
    MP_FAIL(MP_ERR_KERNEL, "op %d reads %d indirect components, array has %d", L.op, rc, L.ind_read_comps);
  if (L.dir_comps < dc) MP_FAIL(MP_ERR_KERNEL, "op %d reads %d direct components, array has %d", L.op, dc, L.dir_comps);
  if (L.inc_comps != ic) MP_FAIL(MP_ERR_KERNEL, "op %d increments %d components, array has %d", L.op, ic, L.inc_comps);
  if (L.n_elems > 0 && (L.map == nullptr || L.inc == nullptr || L.dir_read == nullptr))
    MP_FAIL(MP_ERR_KERNEL, "op %d: missing array pointer", L.op);
  return MP_OK;
}

}  // namespace mp
