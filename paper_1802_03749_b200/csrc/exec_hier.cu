// X2: hierarchical two-layer-colouring executor.
//
// One CTA per plan block.  Structure of a block (one CTA):
//   A. one 16-byte load of the block descriptor {e0, k, s0, ns}; every thread
//      then issues, without waiting, its element's shared-slot indices, direct
//      operands and thread colour, and cp.async (LDGSTS) gathers of the
//      block's staged rows -- the indirect reads and, on the colour schedule,
//      the increment rows themselves -- from the ascending deduplicated staged
//      list into shared memory (16-byte transfers where the row allows);
//   B. compute every element in registers from shared memory;
//   C. zero the shared increment region (it reuses the staged-read buffer) and
//      apply the increments one thread colour at a time, a barrier per colour
//      (threads are colour-sorted, so each colour is a contiguous range);
//   D. write the block's rows back once: out = staged row + shared increment.
// Per point this is init + ((0 + tc0) + tc1 + ...) per block, blocks in
// block-colour order: exactly the reference execute_hierarchical
// (simulator.py:613-654), bit for bit.
//
// Two schedules run the same block body:
//  * MP_SCHED_COLOUR   one launch per block colour (the paper's scheme);
//  * MP_SCHED_DATAFLOW one launch per loop.  Blocks take tickets in a
//    topological order of the conflict DAG ("same written point -> lower
//    block colour first") whose keys stay near block-id order with a lag
//    between dependent blocks, and a block waits (acquire) for its
//    lower-colour conflicting blocks just before its write-back.  Per point the
//    writers are still applied in block-colour order -- bit-identical to the
//    colour schedule -- while blocks that share points run close in time, so
//    their duplicated staged / written rows hit L2 instead of HBM.  A ticket is
//    only taken by a resident CTA and only waits on earlier tickets: no
//    deadlock.  The increment rows are read after the wait (L2-only loads).
#include <stdlib.h>

#include "mp_loop.cuh"

namespace mp {
namespace {

struct HierView {
  const int4* __restrict__ meta;             // {e0, k, s0, ns} per block
  const int32_t* __restrict__ staged_ids;
  const int32_t* __restrict__ written_offsets;
  const int32_t* __restrict__ written_ids;
  const uint16_t* __restrict__ written_slots;
  const void* __restrict__ local_slots;      // u8 or u16 per (element, slot)
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

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
  else if constexpr (BYTES == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem_src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr int vec_bytes(int row_bytes) { return row_bytes % 16 == 0 ? 16 : (row_bytes % 8 == 0 ? 8 : 4); }

template <int BYTES>
struct alignas(BYTES) Chunk {
  unsigned char b[BYTES];
};

// Gather `rows` ascending point rows of `comps_used` leading components (AoS
// rows of `comps` components, or SoA planes) into shared [n][comps_used].
template <typename T, int LAYOUT, int USED>
__device__ __forceinline__ void gather_rows(T* sh, const T* g, const int32_t* ids, int n, int comps, int64_t npts,
                                            int tid, int nt) {
  if constexpr (LAYOUT == MP_AOS) {
    constexpr int VB = vec_bytes(USED * (int)sizeof(T));
    constexpr int CH = USED * (int)sizeof(T) / VB;
    if (((comps * (int)sizeof(T)) % VB) == 0) {
      for (int i = tid; i < n * CH; i += nt) {
        const int j = i / CH, ch = i - j * CH;
        const int64_t p = __ldg(ids + j);
        cp_async<VB>(reinterpret_cast<unsigned char*>(sh + j * USED) + ch * VB,
                     reinterpret_cast<const unsigned char*>(g + p * comps) + ch * VB);
      }
    } else {
      for (int i = tid; i < n * USED; i += nt) {
        const int j = i / USED, c = i - j * USED;
        cp_async<(int)sizeof(T)>(sh + i, g + (int64_t)__ldg(ids + j) * comps + c);
      }
    }
  } else {
    for (int i = tid; i < n * USED; i += nt) {
      const int c = i / n, j = i - c * n;
      cp_async<(int)sizeof(T)>(sh + j * USED + c, g + (int64_t)c * npts + __ldg(ids + j));
    }
  }
}

template <class Op, typename T, int LAYOUT, bool DATAFLOW, typename SlotT, bool WSAME>
__global__ void __launch_bounds__(1024) hier_block_kernel(LoopView<T> v, HierView H) {
  constexpr int A = Op::ARITY, RC = Op::RC, IC = Op::IC;
  constexpr int RCN = RcArr<Op>::N;
  constexpr int REG = RC > IC ? RC : IC;  // staged-read / increment region width
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_block;
  const int tid = threadIdx.x, nt = blockDim.x;

  int b;
  if constexpr (DATAFLOW) {
    if (tid == 0) s_block = __ldg(H.order + atomicAdd(&H.tickets[0], 1u));  // [0]: tickets, [1]: finished
    __syncthreads();
    b = s_block;
  } else {
    b = __ldg(H.blocks_by_colour + H.colour_base + blockIdx.x);
  }
  const int4 md = __ldg(H.meta + b);
  const int e0 = md.x, k = md.y, s0 = md.z, ns = md.w;
  const bool stage = RC > 0 && H.stage_reads;
  constexpr bool PREFETCH_INC = !DATAFLOW && WSAME;

  T* sh_a = reinterpret_cast<T*>(smem_raw);  // [ns][REG]: staged reads, then increments
  T* sh_r = sh_a + ns * REG;                 // [ns][IC]: increment rows (colour schedule)

  // A. issue everything that does not depend on another block; then wait for
  //    the previous colour launch (programmatic dependent launch: this grid
  //    may start while it drains) before the first access to the incremented
  //    array
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (stage) gather_rows<T, LAYOUT, (RC > 0 ? RC : 1)>(sh_a, v.ind, H.staged_ids + s0, ns, v.ind_comps, v.npts, tid, nt);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if constexpr (PREFETCH_INC) gather_rows<T, LAYOUT, IC>(sh_r, v.inc, H.staged_ids + s0, ns, IC, v.npts, tid, nt);
  asm volatile("cp.async.commit_group;" ::: "memory");

  const bool active = tid < k;
  const int64_t e = (int64_t)e0 + tid;
  int ls[A];
  T d[Op::DC];
  int my_tc = -1;
  T r[A][RCN];
  if (active) {
    const SlotT* lsp = static_cast<const SlotT*>(H.local_slots) + e * A;
#pragma unroll
    for (int s = 0; s < A; ++s) ls[s] = __ldg(lsp + s);
    load_direct<Op, T>(v, e, d);
    my_tc = __ldg(H.tcol + e);
    if (RC > 0 && !stage) {  // increment-only staging: reads through the mapping (simulator.py:605-610)
#pragma unroll
      for (int s = 0; s < A; ++s) {
        const int p = map_at(v, e, s);
#pragma unroll
        for (int c = 0; c < RC; ++c) r[s][c] = __ldg(v.ind + ind_index<LAYOUT>(p, c, v.ind_comps, v.npts));
      }
    }
  }
  const int nc = __ldg(H.ncol + b);
  cp_async_wait_all();
  __syncthreads();

  // B. compute in registers
  T o[A][IC];
  if (active) {
    if (RC > 0 && stage) {
#pragma unroll
      for (int s = 0; s < A; ++s)
#pragma unroll
        for (int c = 0; c < RC; ++c) r[s][c] = sh_a[ls[s] * REG + c];
    }
    compute<Op, T>(v, r, d, o);
  }
  if (stage) __syncthreads();  // staged reads consumed: the region becomes the increment buffer

  // C. zero, then one thread colour at a time
  for (int i = tid; i < ns * REG; i += nt) sh_a[i] = T(0);
  __syncthreads();
  for (int c = 0; c < nc; ++c) {
    if (my_tc == c) {
#pragma unroll
      for (int s = 0; s < A; ++s)
#pragma unroll
        for (int cc = 0; cc < IC; ++cc) sh_a[ls[s] * REG + cc] += o[s][cc];
    }
    __syncthreads();
  }

  // D. write back
  if constexpr (DATAFLOW) {
    const int q0 = __ldg(H.pred_offsets + b), nq = __ldg(H.pred_offsets + b + 1) - q0;
    for (int i = tid; i < nq; i += nt) {
      const uint32_t* f = H.flags + __ldg(H.preds + q0 + i);
      while (ld_acquire_gpu(f) != H.epoch) __nanosleep(32);
    }
    __syncthreads();
  }
  if constexpr (WSAME) {
    if constexpr (LAYOUT == MP_AOS) {
      for (int i = tid; i < ns * IC; i += nt) {
        const int j = i / IC, c = i - j * IC;
        T* a = v.inc + (int64_t)__ldg(H.staged_ids + s0 + j) * IC + c;
        const T base = PREFETCH_INC ? sh_r[i] : ld_cg(a);
        *a = base + sh_a[j * REG + c];
      }
    } else {
      for (int i = tid; i < ns * IC; i += nt) {
        const int c = i / ns, j = i - c * ns;
        T* a = v.inc + (int64_t)c * v.npts + __ldg(H.staged_ids + s0 + j);
        const T base = PREFETCH_INC ? sh_r[j * IC + c] : ld_cg(a);
        *a = base + sh_a[j * REG + c];
      }
    }
  } else {
    const int w0 = __ldg(H.written_offsets + b), nw = __ldg(H.written_offsets + b + 1) - w0;
    for (int i = tid; i < nw * IC; i += nt) {
      int j, c;
      if (LAYOUT == MP_AOS) {
        j = i / IC;
        c = i - j * IC;
      } else {
        c = i / nw;
        j = i - c * nw;
      }
      const int p = __ldg(H.written_ids + w0 + j);
      const int sl = __ldg(H.written_slots + w0 + j);
      T* a = v.inc + ind_index<LAYOUT>(p, c, IC, v.npts);
      *a = ld_cg(a) + sh_a[sl * REG + c];
    }
  }

  if constexpr (DATAFLOW) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(H.flags + b, H.epoch);
      // the last block to finish re-arms the counters for the next launch
      if (atomicAdd(&H.tickets[1], 1u) == gridDim.x - 1) {
        H.tickets[0] = 0u;
        H.tickets[1] = 0u;
      }
    }
  }
}

template <class Op, typename T, int LAYOUT, typename SlotT, bool WSAME>
mp_status launch_sched(const LoopView<T>& v, HierView H, const mp_hier_plan& P, int32_t schedule, cudaStream_t st,
                       int threads) {
  constexpr int REG = Op::RC > Op::IC ? Op::RC : Op::IC;
  const bool df = schedule == MP_SCHED_DATAFLOW;
  const size_t smem = (size_t)P.max_staged * (REG + ((!df && WSAME) ? Op::IC : 0)) * sizeof(T);
  if (smem > 227 * 1024)
    MP_FAIL(MP_ERR_CAPACITY, "a block needs %zu shared bytes, over the 232448-byte limit", smem);
  if (df) {
    auto kern = hier_block_kernel<Op, T, LAYOUT, true, SlotT, WSAME>;
    MP_CUDA_TRY(raise_smem_limit(reinterpret_cast<const void*>(kern), smem));
    kern<<<P.num_blocks, threads, smem, st>>>(v, H);
    MP_CHECK_LAUNCH();
    return MP_OK;
  }
  auto kern = hier_block_kernel<Op, T, LAYOUT, false, SlotT, WSAME>;
  MP_CUDA_TRY(raise_smem_limit(reinterpret_cast<const void*>(kern), smem));
  static const bool no_pdl = getenv("MESHPLAN_NO_PDL") != nullptr;
  bool first = true;
  for (int c = 0; c < P.num_block_colours; ++c) {
    const int lo = P.colour_block_offsets_host[c], hi = P.colour_block_offsets_host[c + 1];
    if (hi <= lo) continue;
    H.colour_base = lo;
    // PDL only between this call's colour launches (the first one may follow
    // any other work on the stream)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(hi - lo);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (!first && !no_pdl) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, v, H));
    first = false;
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
    int threads = ((P.block_size + 31) / 32) * 32;
    if (threads < 32) threads = 32;
    if (threads > 1024) MP_FAIL(MP_ERR_CAPACITY, "block size %d exceeds the 1024-thread CTA limit", P.block_size);
    if (!P.meta) MP_FAIL(MP_ERR_KERNEL, "plan has no block descriptors");
    if (schedule == MP_SCHED_DATAFLOW && (!P.order || !P.pred_offsets || !P.flags || !P.tickets))
      MP_FAIL(MP_ERR_KERNEL, "dataflow schedule needs order/preds/flags/tickets");
    if (schedule == MP_SCHED_COLOUR && (!P.blocks_by_colour || !P.colour_block_offsets_host))
      MP_FAIL(MP_ERR_KERNEL, "colour schedule needs blocks_by_colour");
    HierView H{reinterpret_cast<const int4*>(P.meta), P.staged_ids, P.written_offsets, P.written_ids,
               P.written_slots, P.local_slots, P.thread_colours, P.colour_counts, P.blocks_by_colour,
               P.order, P.pred_offsets, P.preds, P.flags, P.tickets, 0, P.stage_reads, epoch};
    LoopView<T> v = make_view<T>(L);
    const bool u8 = P.slot_bytes == 1;
    const bool ws = P.written_is_staged != 0;
#define MP_HIER_LAYOUT(LAY)                                                                           \
  if (u8 && ws) return launch_sched<Op, T, LAY, uint8_t, true>(v, H, P, schedule, st, threads);       \
  if (u8) return launch_sched<Op, T, LAY, uint8_t, false>(v, H, P, schedule, st, threads);            \
  if (ws) return launch_sched<Op, T, LAY, uint16_t, true>(v, H, P, schedule, st, threads);            \
  return launch_sched<Op, T, LAY, uint16_t, false>(v, H, P, schedule, st, threads);
    if (L.ind_layout == MP_AOS) {
      MP_HIER_LAYOUT(MP_AOS)
    } else {
      MP_HIER_LAYOUT(MP_SOA)
    }
#undef MP_HIER_LAYOUT
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
