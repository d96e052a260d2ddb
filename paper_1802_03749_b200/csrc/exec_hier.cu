// X2: hierarchical two-layer-colouring executor.
//
// One CTA per plan block.  The CTA stages the block's indirectly read data
// into shared memory from the deduplicated ascending staged list, computes
// every element in registers (direct data SoA, coalesced), zeroes a shared
// increment region, applies the increments one thread colour at a time
// (one barrier per colour, threads are colour-sorted so each colour is a
// contiguous thread range), and finally read-modify-writes the block's
// written list in HBM once.  The summation order per point is
// init + ((0 + tc0) + tc1 + ...) per block, blocks in block-colour order:
// exactly the reference execute_hierarchical (simulator.py:613-654).
//
// Two schedules run the same block body:
//  * MP_SCHED_COLOUR   one launch per block colour (the paper's scheme);
//  * MP_SCHED_DATAFLOW one launch for the whole loop.  Blocks take tickets in
//    a topological order of the conflict DAG "same written point, lower
//    block colour first" that stays close to block-id order, and a block
//    waits (acquire) for its lower-colour conflicting blocks before its
//    write-back.  Per point the writers are still applied in block-colour
//    order, so the result is bit-identical to MP_SCHED_COLOUR, while blocks
//    that share points run close in time and their duplicated staged and
//    written points are L2 hits instead of HBM traffic.  A ticket is only
//    taken by a resident CTA and only waits on earlier tickets, so the
//    schedule cannot deadlock.
#include "mp_loop.cuh"

namespace mp {
namespace {

struct HierView {
  const int32_t* __restrict__ block_offsets;
  const int32_t* __restrict__ staged_offsets;
  const int32_t* __restrict__ staged_ids;
  const int32_t* __restrict__ written_offsets;
  const int32_t* __restrict__ written_ids;
  const uint16_t* __restrict__ written_slots;
  const uint16_t* __restrict__ local_slots;
  const uint8_t* __restrict__ tcol;
  const int32_t* __restrict__ ncol;
  const int32_t* __restrict__ blocks_by_colour;
  const int32_t* __restrict__ order;
  const int32_t* __restrict__ pred_offsets;
  const int32_t* __restrict__ preds;
  uint32_t* flags;
  uint32_t* tickets;
  int32_t colour_base;
  int32_t stage_reads;
  uint32_t epoch;
};

template <class Op, typename T, int LAYOUT, bool DATAFLOW>
__global__ void __launch_bounds__(1024) hier_block_kernel(LoopView<T> v, HierView H) {
  constexpr int A = Op::ARITY, RC = Op::RC, IC = Op::IC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_block;
  const int tid = threadIdx.x, nt = blockDim.x;

  int b;
  if constexpr (DATAFLOW) {
    if (tid == 0) {
      uint32_t t = atomicAdd(&H.tickets[0], 1u);  // tickets[0]: next block, tickets[1]: blocks done
      s_block = __ldg(H.order + t);
    }
    __syncthreads();
    b = s_block;
  } else {
    b = __ldg(H.blocks_by_colour + H.colour_base + blockIdx.x);
  }

  const int e0 = __ldg(H.block_offsets + b);
  const int k = __ldg(H.block_offsets + b + 1) - e0;
  const int s0 = __ldg(H.staged_offsets + b);
  const int ns = __ldg(H.staged_offsets + b + 1) - s0;
  const bool stage = RC > 0 && H.stage_reads;

  T* sh_r = reinterpret_cast<T*>(smem_raw);  // [ns][RC] staged reads
  T* sh_i = sh_r + (stage ? ns * RC : 0);    // [ns][IC] increments

  // 1. stage indirect reads from the ascending staged list, zero increments
  if (stage) {
    if (LAYOUT == MP_AOS) {
      for (int i = tid; i < ns * RC; i += nt) {
        int j = i / RC, c = i - j * RC;
        int p = __ldg(H.staged_ids + s0 + j);
        sh_r[i] = __ldg(v.ind + (int64_t)p * v.ind_comps + c);
      }
    } else {
      for (int i = tid; i < ns * RC; i += nt) {
        int c = i / ns, j = i - c * ns;
        int p = __ldg(H.staged_ids + s0 + j);
        sh_r[j * RC + c] = __ldg(v.ind + (int64_t)c * v.npts + p);
      }
    }
  }
  for (int i = tid; i < ns * IC; i += nt) sh_i[i] = T(0);
  __syncthreads();

  // 2. compute this thread's element into registers
  T o[A][IC];
  uint16_t ls[A];
  int my_tc = -1;
  if (tid < k) {
    const int64_t e = (int64_t)e0 + tid;
#pragma unroll
    for (int s = 0; s < A; ++s) ls[s] = __ldg(H.local_slots + e * A + s);
    T r[A][RcArr<Op>::N];
    if (RC > 0) {
      if (stage) {
#pragma unroll
        for (int s = 0; s < A; ++s)
#pragma unroll
          for (int c = 0; c < RC; ++c) r[s][c] = sh_r[ls[s] * RC + c];
      } else {  // increment-only staging: reads go through the mapping (simulator.py:605-610)
#pragma unroll
        for (int s = 0; s < A; ++s) {
          int p = map_at(v, e, s);
#pragma unroll
          for (int c = 0; c < RC; ++c) r[s][c] = __ldg(v.ind + ind_index<LAYOUT>(p, c, v.ind_comps, v.npts));
        }
      }
    }
    T d[Op::DC];
    load_direct<Op, T>(v, e, d);
    compute<Op, T>(v, r, d, o);
    my_tc = __ldg(H.tcol + e);
  }

  // 3. thread-colour loop: colour c adds into shared, then a barrier
  const int nc = __ldg(H.ncol + b);
  for (int c = 0; c < nc; ++c) {
    if (my_tc == c) {
#pragma unroll
      for (int s = 0; s < A; ++s)
#pragma unroll
        for (int cc = 0; cc < IC; ++cc) sh_i[ls[s] * IC + cc] += o[s][cc];
    }
    __syncthreads();
  }

  // 4. dataflow: wait for the lower-colour blocks sharing a written point
  if constexpr (DATAFLOW) {
    const int q0 = __ldg(H.pred_offsets + b), nq = __ldg(H.pred_offsets + b + 1) - q0;
    for (int i = tid; i < nq; i += nt) {
      const uint32_t* f = H.flags + __ldg(H.preds + q0 + i);
      while (ld_acquire_gpu(f) != H.epoch) __nanosleep(64);
    }
    __syncthreads();
  }

  // 5. write back the block's written list once
  const int w0 = __ldg(H.written_offsets + b);
  const int nw = __ldg(H.written_offsets + b + 1) - w0;
  if (LAYOUT == MP_AOS) {
    for (int i = tid; i < nw * IC; i += nt) {
      int j = i / IC, c = i - j * IC;
      int p = __ldg(H.written_ids + w0 + j);
      int sl = __ldg(H.written_slots + w0 + j);
      T* a = v.inc + (int64_t)p * IC + c;
      *a = ld_cg(a) + sh_i[sl * IC + c];
    }
  } else {
    for (int i = tid; i < nw * IC; i += nt) {
      int c = i / nw, j = i - c * nw;
      int p = __ldg(H.written_ids + w0 + j);
      int sl = __ldg(H.written_slots + w0 + j);
      T* a = v.inc + (int64_t)c * v.npts + p;
      *a = ld_cg(a) + sh_i[sl * IC + c];
    }
  }

  if constexpr (DATAFLOW) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(H.flags + b, H.epoch);
      // the last block to finish re-arms the counters for the next launch
      // (stream order makes the next launch see the reset)
      if (atomicAdd(&H.tickets[1], 1u) == gridDim.x - 1) {
        H.tickets[0] = 0u;
        H.tickets[1] = 0u;
      }
    }
  }
}

template <class Op, typename T, int LAYOUT>
mp_status launch_layout(const LoopView<T>& v, HierView H, const mp_hier_plan& P, int32_t schedule, cudaStream_t st,
                        size_t smem, int threads) {
  if (schedule == MP_SCHED_DATAFLOW) {
    auto kern = hier_block_kernel<Op, T, LAYOUT, true>;
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<P.num_blocks, threads, smem, st>>>(v, H);
    MP_CHECK_LAUNCH();
    return MP_OK;
  }
  auto kern = hier_block_kernel<Op, T, LAYOUT, false>;
  MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int c = 0; c < P.num_block_colours; ++c) {
    int lo = P.colour_block_offsets_host[c], hi = P.colour_block_offsets_host[c + 1];
    if (hi <= lo) continue;
    H.colour_base = lo;
    kern<<<hi - lo, threads, smem, st>>>(v, H);
    MP_CHECK_LAUNCH();
  }
  return MP_OK;
}

template <class Op, typename T>
mp_status launch_hier(const mp_loop& L, const mp_hier_plan& P, int32_t schedule, uint32_t epoch, cudaStream_t st) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(L, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (P.num_blocks == 0) return MP_OK;
    const bool stage = Op::RC > 0 && P.stage_reads;
    size_t smem = (size_t)P.max_staged * ((stage ? Op::RC : 0) + Op::IC) * sizeof(T);
    int threads = ((P.block_size + 31) / 32) * 32;
    if (threads < 32) threads = 32;
    if (threads > 1024) MP_FAIL(MP_ERR_CAPACITY, "block size %d exceeds the 1024-thread CTA limit", P.block_size);
    if (smem > 227 * 1024)
      MP_FAIL(MP_ERR_CAPACITY, "block needs %zu shared bytes, over the 232448-byte limit", smem);
    HierView H{P.block_offsets, P.staged_offsets, P.staged_ids, P.written_offsets, P.written_ids,
               P.written_slots, P.local_slots,    P.thread_colours, P.colour_counts, P.blocks_by_colour,
               P.order,         P.pred_offsets,   P.preds,      P.flags,        P.tickets,
               0,               P.stage_reads,    epoch};
    if (schedule == MP_SCHED_DATAFLOW && (!P.order || !P.pred_offsets || !P.flags || !P.tickets))
      MP_FAIL(MP_ERR_KERNEL, "dataflow schedule needs order/preds/flags/tickets");
    if (schedule == MP_SCHED_COLOUR && (!P.blocks_by_colour || !P.colour_block_offsets_host))
      MP_FAIL(MP_ERR_KERNEL, "colour schedule needs blocks_by_colour");
    LoopView<T> v = make_view<T>(L);
    if (L.ind_layout == MP_AOS) return launch_layout<Op, T, MP_AOS>(v, H, P, schedule, st, smem, threads);
    return launch_layout<Op, T, MP_SOA>(v, H, P, schedule, st, smem, threads);
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_hier(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule, uint32_t epoch,
                                  void* stream) {
  mp::clear_error();
  if (!loop || !plan) MP_FAIL(MP_ERR_KERNEL, "null argument");
  if (schedule == MP_SCHED_DATAFLOW && epoch == 0) MP_FAIL(MP_ERR_KERNEL, "dataflow epochs start at 1");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  const mp_hier_plan& P = *plan;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() { return mp::launch_hier<Op, scalar_t>(L, P, schedule, epoch, st); });
  });
}
