// X1: global-colouring executor (the paper's baseline).
//
// One launch per colour range; each thread owns one element, gathers its
// indirect reads straight from HBM, computes, and increments the target
// points with plain (non-atomic) read-modify-writes.  Within a colour no two
// elements write a common point (checked by the planner / mp_race_check), so
// the result equals the reference execute_global bit for bit:
// init + sum over colours in colour order (simulator.py:382-418).
#include <stdlib.h>

#include "mp_loop.cuh"

namespace mp {
namespace {

template <class Op, typename T, int LAYOUT>
__global__ void __launch_bounds__(256) global_colour_kernel(LoopView<T> v, int64_t lo, int64_t hi) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int64_t e = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= hi) return;
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
  // the previous colour launch (programmatic dependent launch) must be done
  // before the increment rows are read
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // slot order matters only for repeated points within one row (np.add.at order)
#pragma unroll
  for (int s = 0; s < Op::ARITY; ++s)
#pragma unroll
    for (int c = 0; c < Op::IC; ++c) {
      T* a = v.inc + ind_index<LAYOUT>(p[s], c, Op::IC, v.npts);
      *a = *a + o[s][c];
    }
}

template <class Op, typename T>
mp_status launch_global(const mp_loop& L, const int64_t* offsets, int32_t ncol, int32_t bs, cudaStream_t st) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(L, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    LoopView<T> v = make_view<T>(L);
    static const bool no_pdl = getenv("MESHPLAN_NO_PDL") != nullptr;
    bool first = true;
    for (int c = 0; c < ncol; ++c) {
      int64_t lo = offsets[c], hi = offsets[c + 1];
      if (hi <= lo) continue;
      int64_t nblk = (hi - lo + bs - 1) / bs;
      // PDL between this call's colour launches only (as the hierarchical executors)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)nblk);
      cfg.blockDim = dim3(bs);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = (!first && !no_pdl) ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (L.ind_layout == MP_AOS)
        MP_CUDA_TRY(cudaLaunchKernelEx(&cfg, global_colour_kernel<Op, T, MP_AOS>, v, lo, hi));
      else
        MP_CUDA_TRY(cudaLaunchKernelEx(&cfg, global_colour_kernel<Op, T, MP_SOA>, v, lo, hi));
      first = false;
    }
    return MP_OK;
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_global(const mp_loop* loop, const int64_t* colour_offsets, int32_t num_colours,
                                    int32_t block_size, void* stream) {
  mp::clear_error();
  if (!loop || (num_colours > 0 && !colour_offsets)) MP_FAIL(MP_ERR_KERNEL, "null argument");
  if (block_size < 32 || block_size > 256 || block_size % 32)
    block_size = 128;  // launch width; the plan's block_size is a modelling knob here
  if (num_colours == 0 || loop->n_elems == 0) return MP_OK;
  if (colour_offsets[num_colours] != loop->n_elems)
    MP_FAIL(MP_ERR_VALIDATION, "colour offsets end at %lld, loop has %lld elements",
            (long long)colour_offsets[num_colours], (long long)loop->n_elems);
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() {
      return mp::launch_global<Op, scalar_t>(L, colour_offsets, num_colours, block_size, st);
    });
  });
}
