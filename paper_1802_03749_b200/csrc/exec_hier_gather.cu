// X2, gather form: the hierarchical executor without a thread-colour loop.
//
// Same plan and the same per-point summation order as execute_hierarchical
// (simulator.py:525-656): block colours run as one programmatic-dependent
// launch each; inside a block the staged rows are gathered into shared memory
// (cp.async ring, as in exec_hier_stream.cu), and every staged row p receives
// block_sum(p) = ((0 + x_1) + x_2) + ... over the (element, slot) refs
// writing p in thread-colour order, then res[p] = res[p] + block_sum(p) --
// the reference's zeroed shared row, per-colour np.add.at and write-back
// (simulator.py:634-643), bit for bit.
//
// What changes is who adds what.  The push form lets each element add its
// increments into shared rows one thread colour at a time (a CTA barrier and
// a shared read-modify-write per colour, conflicting quarter-warps when the
// blocks are compact 2D/3D tiles); here lanes own REFS, not elements:
//   * the plan lays each block's refs out grouped by row, in thread-colour
//     order within a row, rows never straddling a 32-lane window
//     (mp_plan_gather_refs: one 32-bit record per position: element, own row,
//     slot, position in the row's run, run end);
//   * a lane evaluates its ref's element from the staged rows (the same
//     operation on the same operands as the element's own evaluation,
//     --fmad=false) and keeps the one slot it owns;
//   * the run is summed in order with a serial shuffle chain (lane l adds its
//     x to lane l-1's partial, one step per run position), so no shared
//     increment rows, no colour barriers and no partial-warp colour passes;
//   * the lane ending a run adds the row's global value (loaded one block
//     ahead, 256-bit for 32-byte rows) and stores the row once.
// One CTA barrier per block (the stage landed); the records are loaded into
// registers one block ahead.  AoS indirect arrays, staged reads.
#include <stdlib.h>

#include <mutex>
#include <vector>

#include "mp_rows.cuh"

namespace mp {
namespace {

constexpr uint32_t GREF_INVALID = 0xFFFFFFFFu;

struct GatherView {
  const int4* __restrict__ tdesc;       // per ticket {e0, k | nc << 16, s0, ns}
  const int32_t* __restrict__ tblock;   // per ticket block id
  const int32_t* __restrict__ staged_ids;
  const unsigned char* __restrict__ emeta;  // per element: A slots (SlotT), colour, mask, pad
  const int32_t* __restrict__ roff;     // [nb+1] ref positions per block
  const uint32_t* __restrict__ refs;    // ref records
  int32_t ntickets;
  int32_t em_bytes;
  int32_t max_staged;
  int32_t max_block;
  int32_t nt;
  int32_t depth;
};

template <class Op, typename T>
struct GatherLayout {
  static constexpr int QB = RcArr<Op>::N * (int)sizeof(T);
  static constexpr int QP = Op::RC == 0 ? 0 : rows::Fmt<QB>::PITCH;
  int ids, q, dir, em, bytes;
  __host__ __device__ static int a16(int x) { return (x + 15) & ~15; }
  __host__ __device__ GatherLayout(int ms, int mb, int em_bytes) {
    ids = 16;
    q = a16(ids + ms * 4);
    dir = a16(q + (Op::RC == 0 ? 0 : ((ms + 3) & ~3) * QP));
    em = a16(dir + Op::DC * mb * (int)sizeof(T));
    bytes = a16(em + mb * em_bytes);
  }
};

template <class Op, typename T, typename SlotT, int MAXR, int RPT>
__global__ void __maxnreg__(80)
    hier_gather_kernel(LoopView<T> v, GatherView H) {
  constexpr int A = Op::ARITY, IC = Op::IC, DC = Op::DC, RCN = RcArr<Op>::N;
  using L_t = GatherLayout<Op, T>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = H.nt, D = H.depth, NS = H.depth + 1;
  const L_t L(H.max_staged, H.max_block, H.em_bytes);
  const int t = threadIdx.x;
  const int G = gridDim.x;
  const int total = H.ntickets > (int)blockIdx.x ? (H.ntickets - (int)blockIdx.x + G - 1) / G : 0;

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  auto load_desc = [&](int f) -> int4 {
    return f < total ? __ldg(H.tdesc + (int)blockIdx.x + f * G) : make_int4(0, 0, 0, 0);
  };
  auto load_block = [&](int f) -> int { return f < total ? __ldg(H.tblock + (int)blockIdx.x + f * G) : -1; };
  auto load_ids = [&](const int4& d, int (&ids)[MAXR]) {
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      ids[r] = __ldg(H.staged_ids + max(d.z + min(j, d.w - 1), 0));
    }
  };
  // the block's ref records at this thread's positions (invalid past its end)
  auto load_refs = [&](int b, uint32_t (&rec)[RPT]) {
    const int r0 = b >= 0 ? __ldg(H.roff + b) : 0, r1 = b >= 0 ? __ldg(H.roff + b + 1) : 0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int pos = r0 + t + r * NT;
      rec[r] = pos < r1 ? __ldg(H.refs + pos) : GREF_INVALID;
    }
  };
  auto issue_fill = [&](int s, const int4& d, const int (&ids)[MAXR]) {
    unsigned char* st = smem + s * L.bytes;
    const int k = d.y & 0xffff, ns = d.w;
    if (t == 0) {
      int* hdr = reinterpret_cast<int*>(st);
      hdr[0] = k;
      hdr[1] = ns;
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      if (j < ns) {
        reinterpret_cast<int*>(st + L.ids)[j] = ids[r];
        if constexpr (Op::RC > 0) rows::gather<T, RCN>(st + L.q, j, v.ind, ids[r], v.ind_comps);
      }
    }
    for (int x = t; x < k; x += NT) {
      const int64_t e = (int64_t)d.x + x;
#pragma unroll
      for (int c = 0; c < DC; ++c)
        rows::cpa<(int)sizeof(T)>(st + L.dir + (c * H.max_block + x) * (int)sizeof(T), v.dir + (int64_t)c * v.n + e);
      const unsigned char* src = H.emeta + e * H.em_bytes;
      unsigned char* dst = st + L.em + x * H.em_bytes;
      for (int o = 0; o < H.em_bytes; o += 4) rows::cpa<4>(dst + o, src + o);
    }
  };
  // global increment rows of the run-ending refs (row ids from the stage's
  // id list, stored by the fill at least one barrier ago)
  T rrow[RPT][IC];
  auto load_rows = [&](int s, const uint32_t (&rec)[RPT]) {
    const int* ids = reinterpret_cast<const int*>(smem + s * L.bytes + L.ids);
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const bool end = rec[r] != GREF_INVALID && (rec[r] >> 28 & 1u);
      const int64_t p = end ? ids[(rec[r] >> 10) & 1023u] : 0;  // unpredicated: absent rows read point 0
      rows::ldg<T, IC>(v.inc, p, rrow[r]);
    }
  };

  // prologue: fills 0 .. D-1, the first block's records and rows
  int ids_fill[MAXR];
  for (int f = 0; f < D; ++f) {
    const int4 d = load_desc(f);
    load_ids(d, ids_fill);
    issue_fill(f, d, ids_fill);
    rows::commit();
  }
  int4 d_fill = load_desc(D);
  uint32_t rec_cur[RPT], rec_next[RPT];
  load_refs(load_block(0), rec_cur);
  int b_next = load_block(1);
  __syncthreads();  // fill 0's id list (plain stores) is visible
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous colour's increments are visible
  load_rows(0, rec_cur);

  int s = 0, s_fill = D;
  for (int i = 0; i < total; ++i) {
    // a. loads for this iteration's bottom: next fill's descriptor, its ids,
    //    the next block's records
    const int4 d_next = load_desc(i + D + 1);
    load_ids(d_fill, ids_fill);
    load_refs(b_next, rec_next);
    b_next = load_block(i + 2);
    // b. block i has landed
    rows::wait_groups(D - 1);
    __syncthreads();
    const unsigned char* st = smem + s * L.bytes;
    const int* ids = reinterpret_cast<const int*>(st + L.ids);

    // c. refs: evaluate, sum each row's run in order, write the row back
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const uint32_t rec = rec_cur[r];
      const bool valid = rec != GREF_INVALID;
      const int pis = valid ? (int)(rec >> 23 & 31u) : 0;
      T x[IC];
#pragma unroll
      for (int c = 0; c < IC; ++c) x[c] = T(0);
      if (valid) {
        const int e = (int)(rec & 1023u), sq = (int)(rec >> 20 & 7u);
        const SlotT* sl = reinterpret_cast<const SlotT*>(st + L.em + e * H.em_bytes);
        T dd[DC], rr[A][RCN], o[A][IC];
#pragma unroll
        for (int c = 0; c < DC; ++c) dd[c] = reinterpret_cast<const T*>(st + L.dir)[c * H.max_block + e];
        if constexpr (Op::RC > 0) {
#pragma unroll
          for (int q = 0; q < A; ++q) rows::lds<T, RCN>(st + L.q, sl[q], rr[q]);
        }
        compute<Op, T>(v, rr, dd, o);
#pragma unroll
        for (int q = 0; q < A; ++q)
          if (q == sq) {
#pragma unroll
            for (int c = 0; c < IC; ++c) x[c] = o[q][c];
          }
      }
      T acc[IC];
#pragma unroll
      for (int c = 0; c < IC; ++c) acc[c] = pis == 0 ? x[c] + T(0) : x[c];  // a run starts from 0 + x
      const int steps = __reduce_max_sync(0xffffffffu, (unsigned)pis);
      for (int k = 1; k <= steps; ++k) {
#pragma unroll
        for (int c = 0; c < IC; ++c) {
          const T prev = __shfl_up_sync(0xffffffffu, acc[c], 1);
          if (pis == k) acc[c] = prev + x[c];
        }
      }
      if (valid && (rec >> 28 & 1u)) {
        const int64_t p = ids[(rec >> 10) & 1023u];
#pragma unroll
        for (int c = 0; c < IC; ++c) acc[c] = rrow[r][c] + acc[c];
        rows::stg<T, IC>(v.inc, p, acc);
      }
    }

    // d. refill the stage block i-1 used (every thread passed this
    //    iteration's barrier after finishing block i-1)
    issue_fill(s_fill, d_fill, ids_fill);
    rows::commit();
    // e. next block's records and increment rows (its id list was stored by
    //    its fill, issued at least one barrier ago)
    const int s_next = s + 1 == NS ? 0 : s + 1;
#pragma unroll
    for (int r = 0; r < RPT; ++r) rec_cur[r] = rec_next[r];
    if (i + 1 < total) load_rows(s_next, rec_cur);
    d_fill = d_next;
    s_fill = s;
    s = s_next;
  }
  rows::wait_groups(0);
}

template <typename K, typename... Args>
cudaError_t launch_pdl(K kern, int grid, int threads, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <class Op, typename T, typename SlotT>
mp_status launch_gather(const LoopView<T>& v, GatherView H, const mp_hier_plan& P, int32_t max_refs,
                        cudaStream_t st) {
  static const int env_depth = getenv("MESHPLAN_GATHER_DEPTH") ? atoi(getenv("MESHPLAN_GATHER_DEPTH")) : 2;
  int depth = env_depth < 2 ? 2 : (env_depth > 3 ? 3 : env_depth);
  // CTA width: enough lanes for the widest block's ref positions at RPT per
  // lane and for its staged rows at MAXR per lane
  constexpr int MAXR = 2;
  int nt = ((P.block_size + 31) / 32) * 32;
  const int nt_rows = ((P.max_staged + MAXR - 1) / MAXR + 31) / 32 * 32;
  if (nt_rows > nt) nt = nt_rows;
  int rpt = (max_refs + nt - 1) / nt;
  if (rpt > 4) {
    nt = ((max_refs + 3) / 4 + 31) / 32 * 32;
    rpt = 4;
  }
  if (nt > 512) MP_FAIL(MP_ERR_CAPACITY, "gather form: %d ref positions per block, over 4 per lane at 512 lanes", max_refs);
  if (rpt < 2) rpt = 2;
  H.nt = nt;
  H.max_block = P.block_size;
  H.max_staged = P.max_staged;
  size_t smem = 0;
  for (;; --depth) {
    const GatherLayout<Op, T> L(P.max_staged, P.block_size, P.elem_meta_bytes);
    smem = (size_t)L.bytes * (depth + 1);
    if (smem <= 227 * 1024 || depth == 2) break;
  }
  if (smem > 227 * 1024) MP_FAIL(MP_ERR_CAPACITY, "gather form needs %zu shared bytes", smem);
  H.depth = depth;
  auto kern = rpt == 2 ? hier_gather_kernel<Op, T, SlotT, MAXR, 2>
                       : (rpt == 3 ? hier_gather_kernel<Op, T, SlotT, MAXR, 3> : hier_gather_kernel<Op, T, SlotT, MAXR, 4>);
  int dev = 0, per_sm = 0, sms = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  {
    struct Entry {
      const void* k;
      size_t smem;
      int threads, dev, per_sm, sms;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    std::lock_guard<std::mutex> lock(mu);
    const void* kp = reinterpret_cast<const void*>(kern);
    bool hit = false;
    for (const auto& e : cache)
      if (e.k == kp && e.smem == smem && e.threads == nt && e.dev == dev) {
        per_sm = e.per_sm;
        sms = e.sms;
        hit = true;
      }
    if (!hit) {
      MP_CUDA_TRY(raise_smem_limit(kp, smem));
      MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
      MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      cache.push_back({kp, smem, nt, dev, per_sm, sms});
    }
  }
  if (per_sm < 1) MP_FAIL(MP_ERR_CAPACITY, "gather form does not fit on an SM (%zu shared bytes)", smem);
  const int resident = per_sm * sms;
  bool first = true;
  for (int c = 0; c < P.num_block_colours; ++c) {
    const int lo = P.colour_block_offsets_host[c], hi = P.colour_block_offsets_host[c + 1];
    if (hi <= lo) continue;
    H.tdesc = reinterpret_cast<const int4*>(P.tdesc_colour) + lo;
    H.tblock = P.tblock_colour + lo;
    H.ntickets = hi - lo;
    const int grid = (hi - lo) < resident ? (hi - lo) : resident;
    MP_CUDA_TRY(launch_pdl(kern, grid, nt, smem, st, !first, v, H));
    first = false;
  }
  return MP_OK;
}

template <class Op, typename T>
mp_status launch_gather_op(const mp_loop& Lp, const mp_hier_plan& P, const int32_t* roff, const uint32_t* refs,
                           int32_t max_refs, cudaStream_t st) {
  if constexpr (!op_supported<Op, T>() || Op::ARITY > 8) {
    MP_FAIL(MP_ERR_KERNEL, "gather form: unsupported op / element type");
  } else {
    mp_status s = check_loop_shape(Lp, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (P.num_blocks == 0) return MP_OK;
    if (Lp.ind_layout != MP_AOS) MP_FAIL(MP_ERR_KERNEL, "gather form needs AoS indirect arrays");
    if (Op::RC > 0 && !P.stage_reads) MP_FAIL(MP_ERR_KERNEL, "gather form needs staged reads");
    if (!P.written_is_staged) MP_FAIL(MP_ERR_KERNEL, "gather form needs written lists equal to staged lists");
    if (!P.tdesc_colour || !P.elem_meta || !P.tblock_colour || !roff || !refs)
      MP_FAIL(MP_ERR_KERNEL, "gather form needs ticket descriptors, element records and ref records");
    if (P.max_staged > 1024 || P.block_size > 1023)
      MP_FAIL(MP_ERR_CAPACITY, "gather form records address 1024 rows / 1023 elements per block");
    GatherView H{};
    H.staged_ids = P.staged_ids;
    H.emeta = P.elem_meta;
    H.roff = roff;
    H.refs = refs;
    H.em_bytes = P.elem_meta_bytes;
    LoopView<T> v = make_view<T>(Lp);
    if (P.slot_bytes == 1) return launch_gather<Op, T, uint8_t>(v, H, P, max_refs, st);
    return launch_gather<Op, T, uint16_t>(v, H, P, max_refs, st);
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_hier_gather(const mp_loop* loop, const mp_hier_plan* plan, const int32_t* ref_offsets,
                                         const uint32_t* refs, int32_t max_refs, void* stream) {
  mp::clear_error();
  if (!loop || !plan) MP_FAIL(MP_ERR_KERNEL, "null argument");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  const mp_hier_plan& P = *plan;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() {
      return mp::launch_gather_op<Op, scalar_t>(L, P, ref_offsets, refs, max_refs, st);
    });
  });
}
