// X2, streamed: the lean hierarchical executor (execute_hierarchical,
// simulator.py:525-656).
//
// Same block semantics as exec_hier.cu (stage -> compute -> thread-colour
// loop in shared memory -> one write-back per block; bit-identical results),
// organised for instruction efficiency.  Profiles of the warp-specialised
// executor (exec_hier_pipe.cu) showed it bound by its single producer warp
// (~750 warp instructions per block, one lane per bulk copy) and by 2-way
// shared-memory bank conflicts on 32-byte rows.  Here:
//
//   * persistent CTAs, every thread both gathers and computes: fill f of a
//     CTA takes ticket blockIdx.x + f * grid (static claims); a D-deep
//     cp.async (LDGSTS) multistage ring keeps D blocks in flight while one is
//     computed (one commit group per block, wait_group D-1, one barrier);
//   * the dependent chain ticket descriptor -> staged ids -> row gathers is
//     software-pipelined in registers one block apart, so no thread waits on
//     an index load: descriptor loads run 2 blocks ahead, id loads 1 ahead;
//   * gathers are issued by all lanes (32 rows per warp instruction), row by
//     row from the block's ascending deduplicated staged list;
//   * shared rows use an odd number of 16/8/4-byte granules as pitch
//     (32-byte rows -> 48 bytes), so consecutive slots -- the common case
//     after GPS / partition reordering -- are bank-conflict free with vector
//     accesses;
//   * per-element plan data (slots + thread colour) is one packed record
//     (plan-time), one 4-byte-granule copy per element.
//
// Schedules: MP_SCHED_COLOUR (one launch per block colour) and
// MP_SCHED_DATAFLOW (one launch; tickets in a topological order of the
// lower-colour conflict DAG).  Dataflow adds one "sync" warp per CTA that
//   - checks, in fill order and off the critical path, that every
//     lower-colour predecessor of the CTA's upcoming blocks has written back
//     (acquire loads of epoch flags) and publishes a ready count in shared
//     memory; a thread gathers a block's increment rows at fill time only if
//     the block is already ready, otherwise ("late") it reads them from L2 at
//     write-back after waiting for readiness;
//   - releases the flags of the CTA's finished blocks in batches, one gpu
//     fence per batch (never one fence per block on the compute path).
// Deadlock freedom: compute threads only wait (late write-back) for the
// readiness of the block they are writing back, whose predecessors hold
// smaller tickets; the CTA holding the smallest unfinished ticket has
// finished all its earlier ones, and sync warps keep releasing finished
// blocks while they poll, so that ticket always progresses while every CTA
// is resident (the grid is capped at the occupancy-derived resident count).
#include <stdlib.h>
#include <string.h>

#include "mp_loop.cuh"

namespace mp {
namespace {

struct StreamView {
  const int4* __restrict__ tdesc;           // per ticket {e0, k | nc << 16, s0, ns}
  const int32_t* __restrict__ tblock;       // per ticket block id (dataflow)
  const int32_t* __restrict__ staged_ids;
  const unsigned char* __restrict__ emeta;  // per element: A slots, colour byte, pad
  const int32_t* __restrict__ pred_offsets;
  const int32_t* __restrict__ preds;
  uint32_t* flags;
  uint32_t epoch;
  int32_t ntickets;
  int32_t em_bytes;
  int32_t max_staged;
  int32_t max_block;
  int32_t nt;     // compute threads (multiple of 32)
  int32_t depth;  // blocks in flight; stages = depth + 1
  int32_t stage_reads;
};

__device__ __forceinline__ unsigned saddr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <int BYTES>
__device__ __forceinline__ void cpa(void* dst, const void* src) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(dst)), "l"(src) : "memory");
  else if constexpr (BYTES == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait(int pending) {
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
  }
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(saddr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(saddr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Row format in shared memory: access granule and a pitch holding an odd
// number of granules (consecutive rows then hit disjoint banks).
template <int RB>
struct RowFmt {
  static constexpr int G = RB % 16 == 0 ? 16 : (RB % 8 == 0 ? 8 : 4);
  static constexpr int PITCH = RB == 0 ? 0 : (((RB / G) % 2 == 1) ? RB : RB + G);
};

template <int G>
struct Gran;
template <>
struct Gran<16> { using type = uint4; };
template <>
struct Gran<8> { using type = uint2; };
template <>
struct Gran<4> { using type = uint32_t; };

// shared row -> registers / registers -> shared row, granule-wide accesses
template <typename T, int N, int G>
__device__ __forceinline__ void lds_row(const unsigned char* p, T (&out)[N]) {
  using V = typename Gran<G>::type;
  constexpr int RB = N * (int)sizeof(T);
#pragma unroll
  for (int ch = 0; ch < RB / G; ++ch) {
    V x = *reinterpret_cast<const V*>(p + ch * G);
    memcpy(reinterpret_cast<unsigned char*>(out) + ch * G, &x, G);
  }
}
template <typename T, int N, int G>
__device__ __forceinline__ void sts_row(unsigned char* p, const T (&in)[N]) {
  using V = typename Gran<G>::type;
  constexpr int RB = N * (int)sizeof(T);
#pragma unroll
  for (int ch = 0; ch < RB / G; ++ch) {
    V x;
    memcpy(&x, reinterpret_cast<const unsigned char*>(in) + ch * G, G);
    *reinterpret_cast<V*>(p + ch * G) = x;
  }
}

// global row (point p) of an indirect array -> shared row (async).  AoS rows
// of `comps` components copy their first N components.
template <typename T, int N, int LAYOUT>
__device__ __forceinline__ void gather_row(unsigned char* dst, const T* g, int64_t p, int comps, int64_t npts) {
  constexpr int RB = N * (int)sizeof(T);
  constexpr int G = RowFmt<RB>::G;
  if constexpr (LAYOUT == MP_AOS) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(g + p * comps);
    if ((comps * (int)sizeof(T)) % G == 0) {
#pragma unroll
      for (int ch = 0; ch < RB / G; ++ch) cpa<G>(dst + ch * G, src + ch * G);
    } else {
#pragma unroll
      for (int c = 0; c < N; ++c) cpa<(int)sizeof(T)>(dst + c * sizeof(T), src + c * sizeof(T));
    }
  } else {
#pragma unroll
    for (int c = 0; c < N; ++c) cpa<(int)sizeof(T)>(dst + c * sizeof(T), g + (int64_t)c * npts + p);
  }
}

// Stage layout (bytes), identical on host and device.
template <class Op, typename T>
struct StreamLayout {
  static constexpr int QB = RcArr<Op>::N * (int)sizeof(T), IB = Op::IC * (int)sizeof(T);
  static constexpr int QP = RowFmt<QB>::PITCH, IP = RowFmt<IB>::PITCH;
  int ids, q, r, dir, em, bytes, inc, ctl, total;
  __host__ __device__ static int a16(int x) { return (x + 15) & ~15; }
  __host__ __device__ StreamLayout(int ms, int mb, int em_bytes, bool stage_reads, int nstage) {
    const int qrows = Op::RC == 0 ? 0 : (stage_reads ? ms : mb * Op::ARITY);
    ids = 16;
    q = a16(ids + ms * 4);
    r = a16(q + qrows * QP);
    dir = a16(r + ms * IP);
    em = a16(dir + Op::DC * mb * (int)sizeof(T));
    bytes = a16(em + mb * em_bytes);
    inc = nstage * bytes;
    ctl = a16(inc + ms * IP);
    total = ctl + 16;
  }
};

template <class Op, typename T, int LAYOUT, bool DATAFLOW, typename SlotT>
__global__ void __launch_bounds__(1024) hier_stream_kernel(LoopView<T> v, StreamView H) {
  constexpr int A = Op::ARITY, RC = Op::RC, IC = Op::IC, DC = Op::DC, RCN = RcArr<Op>::N;
  using L_t = StreamLayout<Op, T>;
  constexpr int QP = L_t::QP, IP = L_t::IP;
  constexpr int QG = RowFmt<L_t::QB>::G, IG = RowFmt<L_t::IB>::G;
  constexpr int MAXR = A;  // staged rows per thread: ns <= A * k <= A * nt
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = H.nt, D = H.depth, NS = H.depth + 1;
  const bool stage_reads = RC > 0 && H.stage_reads != 0;
  const L_t L(H.max_staged, H.max_block, H.em_bytes, stage_reads, NS);
  unsigned char* sh_inc = smem + L.inc;
  int* ctl = reinterpret_cast<int*>(smem + L.ctl);  // [0] done count, [1] ready count
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const int total = H.ntickets > (int)blockIdx.x ? (H.ntickets - (int)blockIdx.x + G - 1) / G : 0;

  for (int i = tid; i < H.max_staged * IP / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sh_inc)[i] = 0u;
  if (tid == 0) {
    ctl[0] = 0;
    ctl[1] = 0;
  }
  __syncthreads();

  if (DATAFLOW && tid >= NT) {
    // ------------------------------ sync warp ------------------------------
    const int lane = tid & 31;
    int u = 0, released = 0;
    for (;;) {
      bool progressed = false;
      const int done = ld_acquire_cta(ctl + 0);
      if (done > released) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the CTA's write-backs before the flags
        for (int f = released + lane; f < done; f += 32)
          st_relaxed_gpu(H.flags + __ldg(H.tblock + (int)blockIdx.x + f * G), H.epoch);
        released = done;
        progressed = true;
      }
      if (released >= total) break;
      if (u < total) {
        const int b = __ldg(H.tblock + (int)blockIdx.x + u * G);
        const int q0 = __ldg(H.pred_offsets + b), nq = __ldg(H.pred_offsets + b + 1) - q0;
        bool ok = true;
        for (int i = lane; i < nq; i += 32) ok &= ld_acquire_gpu(H.flags + __ldg(H.preds + q0 + i)) == H.epoch;
        if (__all_sync(0xffffffffu, ok)) {
          ++u;
          if (lane == 0) st_release_cta(ctl + 1, u);
          progressed = true;
        }
      }
      if (!progressed) __nanosleep(100);
    }
    return;
  }

  // ------------------------------ compute threads ------------------------------
  const int t = tid;
  auto ticket = [&](int f) { return (int)blockIdx.x + f * G; };
  auto load_desc = [&](int f) -> int4 {
    return f < total ? __ldg(H.tdesc + ticket(f)) : make_int4(0, 0, 0, 0);
  };
  auto load_ids = [&](const int4& d, int (&ids)[MAXR]) {
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      ids[r] = j < d.w ? __ldg(H.staged_ids + d.z + j) : 0;
    }
  };
  auto load_map = [&](const int4& d, int (&mp)[A]) {
    if (RC > 0 && !stage_reads) {
      const bool on = t < (d.y & 0xffff);
#pragma unroll
      for (int s = 0; s < A; ++s) mp[s] = on ? map_at(v, (int64_t)d.x + t, s) : 0;
    }
  };
  unsigned late_bits = 0;
  auto issue_fill = [&](int f, const int4& d, const int (&ids)[MAXR], const int (&mp)[A]) {
    const int s = f % NS;
    unsigned char* st = smem + s * L.bytes;
    const int k = d.y & 0xffff, ns = d.w;
    bool rows_ok = true;
    if constexpr (DATAFLOW) rows_ok = ld_acquire_cta(ctl + 1) > f;
    late_bits = (late_bits & ~(1u << s)) | (rows_ok ? 0u : (1u << s));
    if (t == 0) {
      int* hdr = reinterpret_cast<int*>(st);
      hdr[0] = k;
      hdr[1] = ns;
      hdr[2] = d.y >> 16;
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      if (j < ns) {
        const int p = ids[r];
        reinterpret_cast<int*>(st + L.ids)[j] = p;
        if (stage_reads) gather_row<T, RCN, LAYOUT>(st + L.q + j * QP, v.ind, p, v.ind_comps, v.npts);
        if (rows_ok) gather_row<T, IC, LAYOUT>(st + L.r + j * IP, v.inc, p, IC, v.npts);
      }
    }
    if (t < k) {
      const int64_t e = (int64_t)d.x + t;
#pragma unroll
      for (int c = 0; c < DC; ++c)
        cpa<(int)sizeof(T)>(st + L.dir + (c * H.max_block + t) * (int)sizeof(T), v.dir + (int64_t)c * v.n + e);
      const unsigned char* src = H.emeta + e * H.em_bytes;
      unsigned char* dst = st + L.em + t * H.em_bytes;
      if (H.em_bytes == 4) {
        cpa<4>(dst, src);
      } else if (H.em_bytes == 8) {
        cpa<8>(dst, src);
      } else {
        for (int o = 0; o < H.em_bytes; o += 4) cpa<4>(dst + o, src + o);
      }
      if (RC > 0 && !stage_reads) {
#pragma unroll
        for (int sl = 0; sl < A; ++sl)
          gather_row<T, RCN, LAYOUT>(st + L.q + (t * A + sl) * QP, v.ind, mp[sl], v.ind_comps, v.npts);
      }
    }
  };

  // prologue: fills 0 .. D-1, then the register pipeline for fill D, D+1
  int ids_fill[MAXR], ids_next[MAXR];
  int map_fill[A], map_next[A];
#pragma unroll
  for (int s = 0; s < A; ++s) map_fill[s] = map_next[s] = 0;
  for (int f = 0; f < D; ++f) {
    const int4 d = load_desc(f);
    load_ids(d, ids_fill);
    load_map(d, map_fill);
    issue_fill(f, d, ids_fill, map_fill);
    cp_commit();
  }
  int4 d_fill = load_desc(D);
  int4 d_next = load_desc(D + 1);
  load_ids(d_fill, ids_fill);
  load_map(d_fill, map_fill);

  auto cbar = [&]() {
    if constexpr (DATAFLOW) named_sync(1, NT);
    else __syncthreads();
  };

  for (int i = 0; i < total; ++i) {
    // a. descriptor two fills ahead, staged ids (and map rows) one fill ahead
    const int4 d_next2 = load_desc(i + D + 2);
    load_ids(d_next, ids_next);
    load_map(d_next, map_next);
    // b. block i has landed (D-1 younger groups may still be in flight)
    cp_wait(D - 1);
    cbar();
    if (DATAFLOW && t == 0) st_release_cta(ctl + 0, i);  // blocks < i are written back
    // c. refill the stage block i-1 used
    issue_fill(i + D, d_fill, ids_fill, map_fill);
    cp_commit();

    // d. compute block i
    const int s = i % NS;
    const unsigned char* st = smem + s * L.bytes;
    const int* hdr = reinterpret_cast<const int*>(st);
    const int k = hdr[0], ns = hdr[1], nc = hdr[2];
    T o[A][IC];
    int ls[A];
    int my_tc = -1;
    if (t < k) {
      const unsigned char* em = st + L.em + t * H.em_bytes;
      const SlotT* sl = reinterpret_cast<const SlotT*>(em);
#pragma unroll
      for (int q = 0; q < A; ++q) ls[q] = sl[q];
      my_tc = em[A * sizeof(SlotT)];
      T dd[DC];
#pragma unroll
      for (int c = 0; c < DC; ++c) dd[c] = reinterpret_cast<const T*>(st + L.dir)[c * H.max_block + t];
      T r[A][RCN];
      if constexpr (RC > 0) {
#pragma unroll
        for (int q = 0; q < A; ++q)
          lds_row<T, RCN, QG>(st + L.q + (stage_reads ? ls[q] : t * A + q) * QP, r[q]);
      }
      compute<Op, T>(v, r, dd, o);
    }
    // e. thread colours, one at a time
    for (int c = 0; c < nc; ++c) {
      if (my_tc == c) {
#pragma unroll
        for (int q = 0; q < A; ++q) {
          unsigned char* row = sh_inc + ls[q] * IP;
          T acc[IC];
          lds_row<T, IC, IG>(row, acc);
#pragma unroll
          for (int cc = 0; cc < IC; ++cc) acc[cc] += o[q][cc];
          sts_row<T, IC, IG>(row, acc);
        }
      }
      cbar();
    }
    // f. write back: row + increment, once per staged row; re-zero the row
    const bool late = DATAFLOW && ((late_bits >> s) & 1u);
    if (DATAFLOW && late && t < ns) {
      while (ld_acquire_cta(ctl + 1) <= i) __nanosleep(32);
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      if (j < ns) {
        const int64_t p = reinterpret_cast<const int*>(st + L.ids)[j];
        unsigned char* irow = sh_inc + j * IP;
        T acc[IC], base[IC];
        lds_row<T, IC, IG>(irow, acc);
        if (late) {
#pragma unroll
          for (int c = 0; c < IC; ++c) base[c] = ld_cg(v.inc + ind_index<LAYOUT>(p, c, IC, v.npts));
        } else {
          lds_row<T, IC, IG>(st + L.r + j * IP, base);
        }
#pragma unroll
        for (int c = 0; c < IC; ++c) acc[c] = base[c] + acc[c];
        if constexpr (LAYOUT == MP_AOS) {
          constexpr int GG = (IC * (int)sizeof(T)) % 16 == 0 ? 16 : ((IC * (int)sizeof(T)) % 8 == 0 ? 8 : 4);
          using V = typename Gran<GG>::type;
          unsigned char* dst = reinterpret_cast<unsigned char*>(v.inc + p * IC);
#pragma unroll
          for (int ch = 0; ch < IC * (int)sizeof(T) / GG; ++ch) {
            V x;
            memcpy(&x, reinterpret_cast<const unsigned char*>(acc) + ch * GG, GG);
            *reinterpret_cast<V*>(dst + ch * GG) = x;
          }
        } else {
#pragma unroll
          for (int c = 0; c < IC; ++c) v.inc[(int64_t)c * v.npts + p] = acc[c];
        }
        T z[IC];
#pragma unroll
        for (int c = 0; c < IC; ++c) z[c] = T(0);
        sts_row<T, IC, IG>(irow, z);
      }
    }
    // g. rotate the register pipeline
    d_fill = d_next;
    d_next = d_next2;
#pragma unroll
    for (int r = 0; r < MAXR; ++r) ids_fill[r] = ids_next[r];
#pragma unroll
    for (int q = 0; q < A; ++q) map_fill[q] = map_next[q];
  }
  cp_wait(0);
  if constexpr (DATAFLOW) {
    named_sync(1, NT);
    if (t == 0) st_release_cta(ctl + 0, total);
  }
}

template <class Op, typename T, int LAYOUT, typename SlotT>
mp_status launch_stream(const LoopView<T>& v, StreamView H, const mp_hier_plan& P, bool dataflow, cudaStream_t st) {
  static const int env_depth = getenv("MESHPLAN_STREAM_DEPTH") ? atoi(getenv("MESHPLAN_STREAM_DEPTH")) : 2;
  static const int env_ctas = getenv("MESHPLAN_STREAM_CTAS") ? atoi(getenv("MESHPLAN_STREAM_CTAS")) : 0;
  int depth = env_depth < 1 ? 1 : (env_depth > 4 ? 4 : env_depth);
  const int nt = ((P.block_size + 31) / 32) * 32;
  H.nt = nt;
  H.max_block = P.block_size;
  H.max_staged = P.max_staged;
  H.stage_reads = P.stage_reads;
  const bool sr = Op::RC > 0 && P.stage_reads;
  size_t smem = 0;
  for (;; --depth) {  // shrink the ring if it does not fit
    const StreamLayout<Op, T> L(P.max_staged, P.block_size, P.elem_meta_bytes, sr, depth + 1);
    smem = (size_t)L.total;
    if (smem <= 227 * 1024 || depth == 1) break;
  }
  if (smem > 227 * 1024)
    MP_FAIL(MP_ERR_CAPACITY, "streamed executor needs %zu shared bytes, over the 232448-byte limit", smem);
  H.depth = depth;
  const int threads = nt + (dataflow ? 32 : 0);
  if (threads > 1024) MP_FAIL(MP_ERR_CAPACITY, "block size %d exceeds the CTA thread limit", P.block_size);
  auto kern = dataflow ? hier_stream_kernel<Op, T, LAYOUT, true, SlotT> : hier_stream_kernel<Op, T, LAYOUT, false, SlotT>;
  MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0, dev = 0, sms = 0;
  MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  MP_CUDA_TRY(cudaGetDevice(&dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) MP_FAIL(MP_ERR_CAPACITY, "streamed executor does not fit on an SM (%zu shared bytes)", smem);
  if (env_ctas > 0 && env_ctas < per_sm) per_sm = env_ctas;
  const int resident = per_sm * sms;
  if (dataflow) {
    H.tdesc = reinterpret_cast<const int4*>(P.tdesc_order);
    H.tblock = P.order;
    H.ntickets = P.num_blocks;
    const int grid = P.num_blocks < resident ? P.num_blocks : resident;
    kern<<<grid, threads, smem, st>>>(v, H);
    MP_CHECK_LAUNCH();
    return MP_OK;
  }
  for (int c = 0; c < P.num_block_colours; ++c) {
    const int lo = P.colour_block_offsets_host[c], hi = P.colour_block_offsets_host[c + 1];
    if (hi <= lo) continue;
    H.tdesc = reinterpret_cast<const int4*>(P.tdesc_colour) + lo;
    H.tblock = P.blocks_by_colour + lo;
    H.ntickets = hi - lo;
    const int grid = (hi - lo) < resident ? (hi - lo) : resident;
    kern<<<grid, threads, smem, st>>>(v, H);
    MP_CHECK_LAUNCH();
  }
  return MP_OK;
}

template <class Op, typename T>
mp_status launch_stream_op(const mp_loop& Lp, const mp_hier_plan& P, bool dataflow, uint32_t epoch, cudaStream_t st) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(Lp, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (P.num_blocks == 0) return MP_OK;
    if (!P.written_is_staged) MP_FAIL(MP_ERR_KERNEL, "streamed executor needs written lists equal to staged lists");
    if (!P.tdesc_colour || !P.tdesc_order || !P.elem_meta)
      MP_FAIL(MP_ERR_KERNEL, "streamed executor needs the plan's ticket descriptors and element records");
    if (P.elem_meta_bytes < Op::ARITY * P.slot_bytes + 1 || P.elem_meta_bytes % 4)
      MP_FAIL(MP_ERR_KERNEL, "element records of %d bytes cannot hold %d slots and a colour", P.elem_meta_bytes,
              Op::ARITY);
    if (dataflow && (!P.order || !P.pred_offsets || !P.flags))
      MP_FAIL(MP_ERR_KERNEL, "dataflow schedule needs order/preds/flags");
    StreamView H{};
    H.staged_ids = P.staged_ids;
    H.emeta = P.elem_meta;
    H.pred_offsets = P.pred_offsets;
    H.preds = P.preds;
    H.flags = P.flags;
    H.epoch = epoch;
    H.em_bytes = P.elem_meta_bytes;
    LoopView<T> v = make_view<T>(Lp);
    const bool u8 = P.slot_bytes == 1;
    if (Lp.ind_layout == MP_AOS) {
      if (u8) return launch_stream<Op, T, MP_AOS, uint8_t>(v, H, P, dataflow, st);
      return launch_stream<Op, T, MP_AOS, uint16_t>(v, H, P, dataflow, st);
    }
    if (u8) return launch_stream<Op, T, MP_SOA, uint8_t>(v, H, P, dataflow, st);
    return launch_stream<Op, T, MP_SOA, uint16_t>(v, H, P, dataflow, st);
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_hier_stream(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule,
                                         uint32_t epoch, void* stream) {
  mp::clear_error();
  if (!loop || !plan) MP_FAIL(MP_ERR_KERNEL, "null argument");
  const bool df = (schedule & 3) == MP_SCHED_DATAFLOW;
  if (df && epoch == 0) MP_FAIL(MP_ERR_KERNEL, "dataflow epochs start at 1");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  const mp_hier_plan& P = *plan;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() { return mp::launch_stream_op<Op, scalar_t>(L, P, df, epoch, st); });
  });
}
