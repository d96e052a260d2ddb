// X2, pipelined: persistent, warp-specialised hierarchical executor.
//
// Same block semantics as exec_hier.cu (stage -> compute -> thread-colour
// loop in shared memory -> one write-back per block; bit-identical results),
// restructured the Blackwell way so that no consumer warp ever waits on HBM:
//
//   * grid = resident CTAs (persistent); each CTA = 1 producer warp + one
//     consumer thread per block element;
//   * a ring of NSTAGE shared-memory stages guarded by mbarriers
//     (full: 32 explicit + 32 cp.async.mbarrier arrivals; empty: 1 arrival);
//   * the producer warp claims the next block (colour list, or a dataflow
//     ticket), and fills a stage with cp.async (LDGSTS): the block's staged
//     ids, its staged read rows and increment rows (gathered through the
//     ascending deduplicated staged list), the element-local slot indices,
//     direct operands and thread colours -- NSTAGE blocks ahead of the
//     consumers;
//   * consumers compute from shared memory, apply increments one thread
//     colour at a time (named barrier among consumer warps only), write
//     row + increment back once, and release the stage.
//
// Dataflow schedule: one launch; CTA i takes tickets i, i+grid, i+2*grid, ...
// of a topological order of the lower-colour conflict DAG (static claims, no
// ticket atomics).  Before gathering a block's increment rows the producer
// waits (acquire) for the block's lower-colour predecessors, so the rows it
// prefetches already hold every earlier writer's contribution and consumers
// never wait.  A producer only waits on smaller tickets, and the CTA holding
// the smallest unfinished ticket has finished all its earlier ones, so that
// ticket always progresses: no deadlock while every CTA is resident (the grid
// is capped at the occupancy-derived resident count).
#include <stdlib.h>

#include <mutex>
#include <vector>

#include "mp_loop.cuh"

namespace mp {
namespace {

constexpr int MAX_STAGES = 8;  // mbarrier pairs that fit the 128-byte header
constexpr int PIPE_K = 3;  // staged-id prefetch distance (fills)

// Sanitizer controls (tools/race_control.sh; never in the shipped build):
// 1 = the producer skips its empty-barrier wait (a real write-after-read race
// on stage reuse); 2 = the producer completes its cp.async copies
// (wait_all) and arrives with a plain mbarrier.arrive instead of
// cp.async.mbarrier.arrive.noinc.
#ifndef MP_PIPE_RACE_CONTROL
#define MP_PIPE_RACE_CONTROL 0
#endif

__device__ __forceinline__ unsigned saddr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cpasync(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(
          saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int BYTES>
__device__ __forceinline__ void cpa(void* dst, const void* src) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(dst)), "l"(src) : "memory");
  else if constexpr (BYTES == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr(dst)), "l"(src) : "memory");
}

// TMA bulk copy global -> shared, completing bytes on an mbarrier transaction count
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, int bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, int bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}

constexpr int vbytes(int row_bytes) { return row_bytes % 16 == 0 ? 16 : (row_bytes % 8 == 0 ? 8 : 4); }
constexpr int align16(int x) { return (x + 15) & ~15; }

struct PipeView {
  const int4* __restrict__ meta;
  const int32_t* __restrict__ staged_ids;
  const unsigned char* __restrict__ local_slots;
  const uint8_t* __restrict__ tcol;
  const int32_t* __restrict__ ncol;
  const int32_t* __restrict__ list;  // colour: blocks of this colour; dataflow: ticket order
  int32_t list_len;
  const int32_t* __restrict__ pred_offsets;
  const int32_t* __restrict__ preds;
  uint32_t* flags;
  uint32_t* tickets;
  uint32_t epoch;
  int32_t stage_reads;
  int32_t max_staged;
  int32_t max_block;
  int32_t nstage;
  const unsigned char* __restrict__ pull_off;  // uint16 per (block, staged row) + 1
  const unsigned char* __restrict__ pull_ref;  // uint16 per (element, slot)
};

// Byte layout of one stage, computed identically on host and device.
template <class Op, typename T, typename SlotT>
struct StageLayout {
  static constexpr int A = Op::ARITY, RC = Op::RC, IC = Op::IC, DC = Op::DC;
  int hdr, ids, rows_q, rows_r, slots, dir, tc, poff, pref, bytes, dir_pitch, q_rows;
  __host__ __device__ StageLayout(int max_staged, int max_block, bool stage_reads) {
    const int qrows = RC == 0 ? 0 : (stage_reads ? max_staged : max_block * A);  // staged or per (elem, slot)
    q_rows = qrows;
    dir_pitch = ((max_block + 8) + 3) & ~3;  // + alignment slack; pitch bytes stay 16-B multiples
    hdr = 0;
    ids = 64;
    rows_q = align16(ids + max_staged * 4);
    rows_r = align16(rows_q + qrows * RC * (int)sizeof(T));
    slots = align16(rows_r + max_staged * IC * (int)sizeof(T));
    dir = align16(slots + max_block * A * (int)sizeof(SlotT) + 32);
    tc = align16(dir + DC * dir_pitch * (int)sizeof(T));
    poff = align16(tc + max_block + 32);               // pull lists (pull variant)
    pref = align16(poff + (max_staged + 1) * 2 + 32);
    bytes = align16(pref + max_block * A * 2 + 32);
  }
};

// header ints: 0 block (-1: stop), 1 e0, 2 k, 3 ns, 4 ncol, 5 slot byte delta, 6 dir elem delta, 7 tc delta

// Increment buffer: colour-loop variant [max_staged][IC] accumulators;
// pull variant [A][IC][max_block] per-(element, slot) increments.
template <class Op, typename T, bool PULL>
__host__ __device__ inline int inc_buffer_bytes(int max_staged, int max_block) {
  return align16((PULL ? max_block * Op::ARITY : max_staged) * Op::IC * (int)sizeof(T));
}

template <class Op, typename T, int LAYOUT, bool DATAFLOW, typename SlotT, bool PULL>
__global__ void __launch_bounds__(1024) hier_pipe_kernel(LoopView<T> v, PipeView H) {
  constexpr int A = Op::ARITY, RC = Op::RC, IC = Op::IC, DC = Op::DC, RCN = RcArr<Op>::N;
  extern __shared__ __align__(128) unsigned char smem[];
  const StageLayout<Op, T, SlotT> L(H.max_staged, H.max_block, H.stage_reads != 0);
  const int nthreads = blockDim.x;
  const int nc_threads = nthreads - 32;  // consumers: warps 1..
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + MAX_STAGES;
  const int NSTAGE = H.nstage;
  T* sh_inc = reinterpret_cast<T*>(smem + 128);
  unsigned char* stage0 = smem + 128 + inc_buffer_bytes<Op, T, PULL>(H.max_staged, H.max_block);
  const bool stage_reads = RC > 0 && H.stage_reads;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 64);
      mbar_init(&empty[s], 1);
    }
  }
  if (!PULL)
    for (int i = threadIdx.x; i < H.max_staged * IC; i += nthreads) sh_inc[i] = T(0);
  __syncthreads();
  // Programmatic dependent launch: the next colour's CTAs may start as this
  // grid's retire; every access to the incremented array is ordered after the
  // producer's griddepcontrol.wait, issued before its first increment-row
  // gather (consumers only write rows it has filled).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ------------------------------- producer -------------------------------
    bool pdl_waited = false;  // griddepcontrol.wait before the first increment-row gather
    // Descriptor batches + a K-deep staged-id ring keep every dependent load
    // (claim -> block id -> descriptor -> staged ids) many fills ahead of its
    // use: lane i of a batch resolves fill (base + i); the next batch is
    // issued when the current one starts; the staged ids of fill f+K are
    // cp.async'd into the ring at fill f.  Claims are taken in fill order,
    // which is the order the consumers drain the stages (dataflow proof).
    constexpr int K = PIPE_K, R = PIPE_K + 1;
    constexpr int BATCH = 32;
    const int rpitch = (H.max_staged + 11) & ~3;                      // 16-B multiple + window slack
    int* ring = reinterpret_cast<int*>(stage0 + NSTAGE * L.bytes);   // [R][rpitch] staged ids
    int* mring = ring + R * rpitch;                                  // [R][max_block*A] map rows
    const bool map_rows = RC > 0 && !H.stage_reads;
    auto load_batch = [&](int base, int& bb, int4& mdd, int& ncc) {
      // static round-robin claims (both schedules): fill f of CTA i takes list
      // entry i + f * grid -- no ticket atomics, and on the dataflow schedule
      // the claimed-but-unfinished window stays ~grid * NSTAGE tickets wide
      const int raw = blockIdx.x + (base + lane) * gridDim.x;
      bb = raw < H.list_len ? __ldg(H.list + raw) : -1;
      mdd = bb >= 0 ? __ldg(H.meta + bb) : make_int4(0, 0, 0, 0);
      ncc = bb >= 0 ? __ldg(H.ncol + bb) : 0;
    };
    int cb, cnc, xb, xnc, cbase = 0;
    int4 cmd, xmd;
    load_batch(0, cb, cmd, cnc);
    load_batch(BATCH, xb, xmd, xnc);
    auto get = [&](int f, int& bb, int4& mdd, int& ncc) {  // f in [cbase, cbase + 2*BATCH)
      const int rel = f - cbase;
      const bool cur = rel < BATCH;
      const int src = cur ? rel : rel - BATCH;
      bb = __shfl_sync(0xffffffffu, cur ? cb : xb, src);
      mdd.x = __shfl_sync(0xffffffffu, cur ? cmd.x : xmd.x, src);
      mdd.y = __shfl_sync(0xffffffffu, cur ? cmd.y : xmd.y, src);
      mdd.z = __shfl_sync(0xffffffffu, cur ? cmd.z : xmd.z, src);
      mdd.w = __shfl_sync(0xffffffffu, cur ? cmd.w : xmd.w, src);
      ncc = __shfl_sync(0xffffffffu, cur ? cnc : xnc, src);
    };
    auto prefetch_ids = [&](int f) {
      int bb, ncc;
      int4 m;
      get(f, bb, m, ncc);
      if (bb < 0) return;
      int* dst = ring + (f % R) * rpitch;  // 16-B window starting at (s0 & ~3)
      const int lo = m.z & ~3, nchunk = ((m.z & 3) + m.w + 3) >> 2;
      for (int j = lane; j < nchunk; j += 32) cpa<16>(dst + 4 * j, H.staged_ids + lo + 4 * j);
      if (map_rows) {
        int* md = mring + (f % R) * H.max_block * A;
        for (int j = lane; j < m.y * A; j += 32) cpa<4>(md + j, v.map + (int64_t)m.x * A + j);
      }
    };
    for (int j = 0; j < K; ++j) {
      prefetch_ids(j);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");  // empty "rows" group: uniform wait depth
    }
    for (int fill = 0;; ++fill) {
      const int s = fill % NSTAGE;
      unsigned char* st = stage0 + s * L.bytes;
      int* hdr = reinterpret_cast<int*>(st);
      if (fill - cbase == BATCH) {  // advance the batches; the next one lands while this one drains
        cb = xb;
        cmd = xmd;
        cnc = xnc;
        cbase += BATCH;
        load_batch(cbase + BATCH, xb, xmd, xnc);
      }
      prefetch_ids(fill + K);
      asm volatile("cp.async.commit_group;" ::: "memory");
      int b, nc0;
      int4 md;
      get(fill, b, md, nc0);
#if MP_PIPE_RACE_CONTROL != 1
      mbar_wait(&empty[s], ((fill / NSTAGE) & 1) ^ 1);
#endif
      if (b < 0) {
        if (lane == 0) hdr[0] = -1;
        mbar_arrive(&full[s]);
        mbar_arrive_cpasync(&full[s]);
        break;
      }
      const int e0 = md.x, k = md.y, ns = md.w;
      // element-local data: one TMA bulk copy per contiguous piece (16-B windows)
      int sl_delta = 0, tc_delta = 0;
      if (lane == 0) {
        const int64_t sb = (int64_t)e0 * A * (int)sizeof(SlotT), slo = sb & ~int64_t(15);
        sl_delta = (int)(sb - slo);
        const int sbytes = align16(sl_delta + k * A * (int)sizeof(SlotT));
        mbar_expect_tx(&full[s], sbytes);
        bulk_g2s(st + L.slots, H.local_slots + slo, sbytes, &full[s]);
        if constexpr (PULL) {  // pull lists instead of thread colours
          const int64_t pob = ((int64_t)md.z + b) * 2, polo = pob & ~int64_t(15);
          const int pobytes = align16((int)(pob - polo) + (ns + 1) * 2);
          const int64_t prb = (int64_t)e0 * A * 2, prlo = prb & ~int64_t(15);
          const int prbytes = align16((int)(prb - prlo) + k * A * 2);
          hdr[13] = (int)(pob - polo) / 2;
          hdr[14] = (int)(prb - prlo) / 2;
          mbar_expect_tx(&full[s], pobytes + prbytes);
          bulk_g2s(st + L.poff, H.pull_off + polo, pobytes, &full[s]);
          bulk_g2s(st + L.pref, H.pull_ref + prlo, prbytes, &full[s]);
        } else {
          const int64_t tlo = (int64_t)e0 & ~int64_t(15);
          tc_delta = (int)(e0 - tlo);
          const int tbytes = align16(tc_delta + k);
          mbar_expect_tx(&full[s], tbytes);
          bulk_g2s(st + L.tc, H.tcol + tlo, tbytes, &full[s]);
        }
        const int64_t dir_total = (int64_t)v.dir_comps * v.n * (int)sizeof(T);
        for (int c = 0; c < DC; ++c) {
          const int64_t ob = ((int64_t)c * v.n + e0) * (int)sizeof(T), olo = ob & ~int64_t(15);
          const int dbytes = align16((int)(ob - olo) + k * (int)sizeof(T));
          T* dst = reinterpret_cast<T*>(st + L.dir) + c * L.dir_pitch;
          if (olo + dbytes <= dir_total) {
            hdr[9 + c] = (int)(ob - olo) / (int)sizeof(T);
            mbar_expect_tx(&full[s], dbytes);
            bulk_g2s(dst, reinterpret_cast<const unsigned char*>(v.dir) + olo, dbytes, &full[s]);
          } else {  // tail of the array: element copies (no over-read)
            hdr[9 + c] = 0;
            for (int i = 0; i < k; ++i) cpa<(int)sizeof(T)>(dst + i, v.dir + (int64_t)c * v.n + e0 + i);
          }
        }
        hdr[0] = b;
        hdr[1] = e0;
        hdr[2] = k;
        hdr[3] = ns;
        hdr[4] = nc0;
        hdr[5] = sl_delta;
        hdr[7] = tc_delta;
      }
      // staged ids (prefetched K fills ago) -> stage; gathers of the staged rows
      asm volatile("cp.async.wait_group %0;" ::"n"(2 * PIPE_K) : "memory");  // this block's ids have landed
      __syncwarp();
      const int* rids = ring + (fill % R) * rpitch + (md.z & 3);
      const int* rmap = mring + (fill % R) * H.max_block * A;
      int* ids = reinterpret_cast<int*>(st + L.ids);
      T* rq = reinterpret_cast<T*>(st + L.rows_q);
      T* rr = reinterpret_cast<T*>(st + L.rows_r);
      // dataflow: wait (acquire) until every lower-colour predecessor has
      // written back, then gather the increment rows -- they already hold every
      // earlier writer's contribution.  A producer only waits on smaller
      // tickets; the consumers never wait, so the smallest unfinished ticket
      // always progresses (all CTAs are co-resident).
      const bool inc_rows = true;
      if (!pdl_waited) {  // descriptors, ids and map rows above are plan data
        asm volatile("griddepcontrol.wait;" ::: "memory");
        pdl_waited = true;
      }
      if constexpr (DATAFLOW) {
        const int q0 = __ldg(H.pred_offsets + b), nq = __ldg(H.pred_offsets + b + 1) - q0;
        for (int i = lane; i < nq; i += 32) {
          const uint32_t* f = H.flags + __ldg(H.preds + q0 + i);
          while (ld_acquire_gpu(f) != H.epoch) __nanosleep(64);
        }
        __syncwarp();
        asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired rows -> bulk (async-proxy) reads
      }
      constexpr bool BULK_R = LAYOUT == MP_AOS && (IC * (int)sizeof(T)) % 16 == 0;
      constexpr bool BULK_Q_T = LAYOUT == MP_AOS && RC > 0 && (RC * (int)sizeof(T)) % 16 == 0;
      const bool bulk_q = BULK_Q_T && H.stage_reads && v.ind_comps == RC;
      for (int base = 0; base < ns; base += 32) {
        const int j = base + lane;
        const bool valid = j < ns;
        const int p = valid ? rids[j] : 0;
        if (valid) ids[j] = p;
        // runs of consecutive ids -> one bulk copy per run and array
        const int prev = __shfl_up_sync(0xffffffffu, p, 1);
        const bool start = valid && (lane == 0 || p != prev + 1);
        const unsigned mask = __ballot_sync(0xffffffffu, start);
        if (start && (BULK_R || bulk_q)) {
          const unsigned above = lane == 31 ? 0u : (mask & ~((2u << lane) - 1u));
          const int lim = ns - base < 32 ? ns - base : 32;
          const int len = (above ? __ffs(above) - 1 : lim) - lane;
          if (BULK_R && inc_rows) {
            const int bytes = len * IC * (int)sizeof(T);
            mbar_expect_tx(&full[s], bytes);
            bulk_g2s(rr + j * IC, v.inc + (int64_t)p * IC, bytes, &full[s]);
          }
          if (bulk_q) {
            const int bytes = len * RC * (int)sizeof(T);
            mbar_expect_tx(&full[s], bytes);
            bulk_g2s(rq + j * RCN, v.ind + (int64_t)p * RC, bytes, &full[s]);
          }
        }
        if (!valid) continue;
        if constexpr (LAYOUT == MP_AOS) {
          if (!BULK_R && inc_rows) {
            constexpr int VR = vbytes(IC * (int)sizeof(T));
#pragma unroll
            for (int ch = 0; ch < IC * (int)sizeof(T) / VR; ++ch)
              cpa<VR>(reinterpret_cast<unsigned char*>(rr + j * IC) + ch * VR,
                      reinterpret_cast<const unsigned char*>(v.inc + (int64_t)p * IC) + ch * VR);
          }
          if (RC > 0 && H.stage_reads && !bulk_q) {
            constexpr int RCB = RC > 0 ? RC : 1;
            constexpr int VQ = vbytes(RCB * (int)sizeof(T));
            if ((v.ind_comps * (int)sizeof(T)) % VQ == 0) {
#pragma unroll
              for (int ch = 0; ch < RCB * (int)sizeof(T) / VQ; ++ch)
                cpa<VQ>(reinterpret_cast<unsigned char*>(rq + j * RCB) + ch * VQ,
                        reinterpret_cast<const unsigned char*>(v.ind + (int64_t)p * v.ind_comps) + ch * VQ);
            } else {
#pragma unroll
              for (int c = 0; c < RCB; ++c) cpa<(int)sizeof(T)>(rq + j * RCB + c, v.ind + (int64_t)p * v.ind_comps + c);
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < IC; ++c)
            if (inc_rows) cpa<(int)sizeof(T)>(rr + j * IC + c, v.inc + (int64_t)c * v.npts + p);
          if (RC > 0 && H.stage_reads) {
#pragma unroll
            for (int c = 0; c < RC; ++c) cpa<(int)sizeof(T)>(rq + j * RCN + c, v.ind + (int64_t)c * v.npts + p);
          }
        }
      }
      if (map_rows) {  // increment-only staging: read rows per (element, slot) via the mapping
        for (int i = lane; i < k * A; i += 32) {
          const int p = rmap[i];
#pragma unroll
          for (int c = 0; c < RCN; ++c) cpa<(int)sizeof(T)>(rq + i * RCN + c, v.ind + ind_index<LAYOUT>(p, c, v.ind_comps, v.npts));
        }
      }
      mbar_arrive(&full[s]);          // releases the header / ids stores
#if MP_PIPE_RACE_CONTROL == 2
      asm volatile("cp.async.wait_all;" ::: "memory");  // copies complete in this thread, then a plain arrive
      mbar_arrive(&full[s]);
#else
      mbar_arrive_cpasync(&full[s]);  // fires when this lane's copies land
#endif
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else {
    // ------------------------------- consumers ------------------------------
    const int t = threadIdx.x - 32;
    for (int use = 0;; ++use) {
      const int s = use % NSTAGE;
      unsigned char* st = stage0 + s * L.bytes;
      const int* hdr = reinterpret_cast<const int*>(st);
      mbar_wait(&full[s], (use / NSTAGE) & 1);
      const int b = hdr[0];
      if (b < 0) break;
      const int k = hdr[2], ns = hdr[3], nc = hdr[4];
      const int* ids = reinterpret_cast<const int*>(st + L.ids);
      const T* rq = reinterpret_cast<const T*>(st + L.rows_q);
      const T* rr = reinterpret_cast<const T*>(st + L.rows_r);
      T o[A][IC];
      int ls[A];
      int my_tc = -1;
      if (t < k) {
        const SlotT* sl = reinterpret_cast<const SlotT*>(st + L.slots + hdr[5]) + t * A;
#pragma unroll
        for (int q = 0; q < A; ++q) ls[q] = sl[q];
        T d[DC];
        const T* dir = reinterpret_cast<const T*>(st + L.dir) + t;
#pragma unroll
        for (int c = 0; c < DC; ++c) d[c] = dir[c * L.dir_pitch + hdr[9 + c]];
        T r[A][RCN];
        if (RC > 0) {
          if (stage_reads) {
#pragma unroll
            for (int q = 0; q < A; ++q)
#pragma unroll
              for (int c = 0; c < RC; ++c) r[q][c] = rq[ls[q] * RCN + c];
          } else {
#pragma unroll
            for (int q = 0; q < A; ++q)
#pragma unroll
              for (int c = 0; c < RC; ++c) r[q][c] = rq[(t * A + q) * RCN + c];
          }
        }
        compute<Op, T>(v, r, d, o);
        if (!PULL) my_tc = (st + L.tc)[hdr[7] + t];
      }
      if constexpr (PULL) {
        // Pull form of the colour loop: every element parks its per-slot
        // increments (conflict-free, element-fastest layout); one barrier; the
        // owner of staged row j sums the row's refs in thread-colour order
        // starting from 0 -- the same additions, in the same order, as the
        // reference's zeroed shared row + per-colour np.add.at -- and writes
        // row + sum back once.
        const int kp = H.max_block;
        if (t < k) {
#pragma unroll
          for (int q = 0; q < A; ++q)
#pragma unroll
            for (int c = 0; c < IC; ++c) sh_inc[(q * IC + c) * kp + t] = o[q][c];
        }
        named_sync(1, nc_threads);
        const uint16_t* po = reinterpret_cast<const uint16_t*>(st + L.poff) + hdr[13];
        const uint16_t* pr = reinterpret_cast<const uint16_t*>(st + L.pref) + hdr[14];
        for (int j = t; j < ns; j += nc_threads) {
          T acc[IC];
#pragma unroll
          for (int c = 0; c < IC; ++c) acc[c] = T(0);
          for (int r2 = po[j]; r2 < po[j + 1]; ++r2) {
            const int ref = pr[r2], te = ref / A, q = ref - te * A;
#pragma unroll
            for (int c = 0; c < IC; ++c) acc[c] += sh_inc[(q * IC + c) * kp + te];
          }
          const int64_t p = ids[j];
#pragma unroll
          for (int c = 0; c < IC; ++c) {
            T* a = v.inc + ind_index<LAYOUT>(p, c, IC, v.npts);
            *a = rr[j * IC + c] + acc[c];
          }
        }
        named_sync(1, nc_threads);
        if (t == 0) {
          if constexpr (DATAFLOW) {
            __threadfence();
            st_release_gpu(H.flags + b, H.epoch);
          }
          mbar_arrive(&empty[s]);
        }
        continue;
      }
      for (int c = 0; c < nc; ++c) {
        if (my_tc == c) {
#pragma unroll
          for (int q = 0; q < A; ++q)
#pragma unroll
            for (int cc = 0; cc < IC; ++cc) sh_inc[ls[q] * IC + cc] += o[q][cc];
        }
        named_sync(1, nc_threads);
      }
      if (nc == 0) named_sync(1, nc_threads);
      // write back rows + increments, re-zero the increment region
      if constexpr (LAYOUT == MP_AOS) {
        for (int i = t; i < ns * IC; i += nc_threads) {
          const int j = i / IC, c = i - j * IC;
          T* a = v.inc + (int64_t)ids[j] * IC + c;
          *a = rr[i] + sh_inc[i];
          sh_inc[i] = T(0);
        }
      } else {
        for (int i = t; i < ns * IC; i += nc_threads) {
          const int c = i / ns, j = i - c * ns;
          T* a = v.inc + (int64_t)c * v.npts + ids[j];
          *a = rr[j * IC + c] + sh_inc[j * IC + c];
        }
        named_sync(1, nc_threads);
        for (int i = t; i < ns * IC; i += nc_threads) sh_inc[i] = T(0);
      }
      named_sync(1, nc_threads);
      if (t == 0) {
        if constexpr (DATAFLOW) {
          __threadfence();
          st_release_gpu(H.flags + b, H.epoch);
        }
        mbar_arrive(&empty[s]);
      }
    }
  }
}

// resident CTAs per SM for (kernel, threads, shared bytes) on the current
// device, cached process-wide (the query costs microseconds per call); raises
// the kernel's dynamic shared-memory limit first
cudaError_t pipe_occupancy(const void* kern, int threads, size_t smem, int* occ) {
  struct Entry {
    const void* k;
    int threads, dev;
    size_t smem;
    int occ;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& c : cache)
      if (c.k == kern && c.threads == threads && c.dev == dev && c.smem == smem) {
        *occ = c.occ;
        return cudaSuccess;
      }
  }
  e = raise_smem_limit(kern, smem);
  if (e) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, threads, smem);
  if (e) return e;
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back({kern, threads, dev, smem, *occ});
  return cudaSuccess;
}

template <class Op, typename T, int LAYOUT, typename SlotT, bool PULL>
mp_status launch_pipe(const LoopView<T>& v, PipeView H, const mp_hier_plan& P, bool dataflow, cudaStream_t st) {
  const StageLayout<Op, T, SlotT> L(P.max_staged, P.block_size, P.stage_reads != 0);
  const bool map_rows = Op::RC > 0 && !P.stage_reads;
  const size_t ring = (size_t)(PIPE_K + 1) * (((P.max_staged + 11) & ~3) * 4 +
                                              (map_rows ? (size_t)P.block_size * Op::ARITY * 4 : 0));
  static const int env_stages = getenv("MESHPLAN_PIPE_STAGES") ? atoi(getenv("MESHPLAN_PIPE_STAGES")) : 0;
  static const int env_ctas = getenv("MESHPLAN_PIPE_CTAS") ? atoi(getenv("MESHPLAN_PIPE_CTAS")) : 0;
  // shared bytes per SM the resident CTAs may take: the rest stays L1 data
  // cache (on the face loop, above ~200 KB per SM every plan measured ~25 %
  // slower: C4 k-way pull 1.28 vs 1.02 ms, 4x4x8 pull 0.99 vs 0.83 ms, k-way
  // push 1.30 vs 1.03 ms, profiles/r02/pipe_stages.log, pipe_auto.log)
  static const int env_budget = getenv("MESHPLAN_PIPE_SMEM_KB") ? atoi(getenv("MESHPLAN_PIPE_SMEM_KB")) : 192;
  const int consumers = ((P.block_size + 31) / 32) * 32;
  const int threads = consumers + 32;
  auto kern = dataflow ? hier_pipe_kernel<Op, T, LAYOUT, true, SlotT, PULL>
                       : hier_pipe_kernel<Op, T, LAYOUT, false, SlotT, PULL>;
  auto smem_of = [&](int ns) {
    return 128 + inc_buffer_bytes<Op, T, PULL>(P.max_staged, P.block_size) + (size_t)ns * L.bytes + ring;
  };
  // ring depth and CTAs per SM: the most CTAs that fit the budget (and the
  // occupancy limit), then the deepest ring at that count (2..4 stages)
  int NSTAGE = 0, per_sm = 0, occ2 = 0;
  for (int ns = 2; ns <= 4; ++ns) {
    if (env_stages && ns != (env_stages < 2 ? 2 : (env_stages > MAX_STAGES ? MAX_STAGES : env_stages))) continue;
    const size_t sm = smem_of(ns);
    if (sm > 227 * 1024) break;
    int occ = 0;
    MP_CUDA_TRY(pipe_occupancy(reinterpret_cast<const void*>(kern), threads, sm, &occ));
    if (ns == 2) occ2 = occ;
    int cap = (int)(((size_t)env_budget * 1024) / (sm + 1024));
    if (env_stages || cap < 1) cap = occ;  // an explicit ring depth keeps the occupancy limit
    if (cap > occ) cap = occ;
    if (cap >= 1 && (NSTAGE == 0 || cap >= per_sm)) {
      NSTAGE = ns;
      per_sm = cap;
    }
  }
  if (!env_stages && per_sm < 2 && occ2 >= 2) {  // never one CTA per SM where two fit: two stages, two CTAs
    NSTAGE = 2;
    per_sm = 2;
  }
  if (env_stages > 4) {  // deeper rings on request
    NSTAGE = env_stages > MAX_STAGES ? MAX_STAGES : env_stages;
    MP_CUDA_TRY(pipe_occupancy(reinterpret_cast<const void*>(kern), threads, smem_of(NSTAGE), &per_sm));
  }
  if (NSTAGE == 0) MP_FAIL(MP_ERR_CAPACITY, "pipelined stages need %zu shared bytes, over the 232448-byte limit", smem_of(2));
  const size_t smem = smem_of(NSTAGE);
  H.nstage = NSTAGE;
  int dev = 0, sms = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) MP_FAIL(MP_ERR_CAPACITY, "pipelined executor does not fit on an SM (%zu shared bytes)", smem);
  if (env_ctas > 0 && env_ctas < per_sm) per_sm = env_ctas;
  if (!dataflow) {  // shared-memory carve-out for exactly the resident CTAs (the rest is L1); the
                    // static-claim dataflow grid keeps the default, which holds every CTA it counts on
    const int pct = (int)((100 * (size_t)per_sm * (smem + 1024) + 227 * 1024 - 1) / (228 * 1024));
    MP_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributePreferredSharedMemoryCarveout,
                                     pct > 100 ? 100 : pct));
  }
  if (getenv("MESHPLAN_PIPE_VERBOSE"))
    fprintf(stderr, "[pipe] pull=%d stages=%d stage_bytes=%d smem=%zu threads=%d per_sm=%d\n", (int)PULL, NSTAGE,
            (int)L.bytes, smem, threads, per_sm);
  const int resident = per_sm * sms;
  if (dataflow) {
    H.list = P.order;
    H.list_len = P.num_blocks;
    const int grid = P.num_blocks < resident ? P.num_blocks : resident;
    MP_CUDA_TRY(static_dataflow_begin(st));  // static claims: never co-resident with another such grid
    kern<<<grid, threads, smem, st>>>(v, H);
    const cudaError_t le = cudaGetLastError();
    MP_CUDA_TRY(static_dataflow_end(st));
    MP_CUDA_TRY(le);
    return MP_OK;
  }
  static const bool no_pdl = getenv("MESHPLAN_NO_PDL") != nullptr;
  bool first = true;
  for (int c = 0; c < P.num_block_colours; ++c) {
    const int lo = P.colour_block_offsets_host[c], hi = P.colour_block_offsets_host[c + 1];
    if (hi <= lo) continue;
    H.list = P.blocks_by_colour + lo;
    H.list_len = hi - lo;
    const int grid = (hi - lo) < resident ? (hi - lo) : resident;
    // PDL only between the colour launches of this call (the first one may
    // follow any other work on the stream)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
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
mp_status launch_pipe_op(const mp_loop& Lp, const mp_hier_plan& P, bool dataflow, bool pull, uint32_t epoch,
                         cudaStream_t st) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(Lp, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (P.num_blocks == 0) return MP_OK;
    if (!P.written_is_staged) MP_FAIL(MP_ERR_KERNEL, "pipelined executor needs written lists equal to staged lists");
    if (P.block_size > 992) MP_FAIL(MP_ERR_CAPACITY, "block size %d exceeds 992 (+1 producer warp)", P.block_size);
    if (pull && (!P.pull_off || !P.pull_ref)) MP_FAIL(MP_ERR_KERNEL, "pull variant needs the plan's pull lists");
    PipeView H{reinterpret_cast<const int4*>(P.meta), P.staged_ids,
               static_cast<const unsigned char*>(P.local_slots), P.thread_colours, P.colour_counts,
               nullptr, 0, P.pred_offsets, P.preds, P.flags, P.tickets, epoch, P.stage_reads, P.max_staged,
               P.block_size, 3, reinterpret_cast<const unsigned char*>(P.pull_off),
               reinterpret_cast<const unsigned char*>(P.pull_ref)};
    LoopView<T> v = make_view<T>(Lp);
    const bool u8 = P.slot_bytes == 1;
#define MP_PIPE(LAY, SL)                                                                      \
  return pull ? launch_pipe<Op, T, LAY, SL, true>(v, H, P, dataflow, st)                      \
              : launch_pipe<Op, T, LAY, SL, false>(v, H, P, dataflow, st);
    if (Lp.ind_layout == MP_AOS) {
      if (u8) { MP_PIPE(MP_AOS, uint8_t) }
      MP_PIPE(MP_AOS, uint16_t)
    }
    if (u8) { MP_PIPE(MP_SOA, uint8_t) }
    MP_PIPE(MP_SOA, uint16_t)
#undef MP_PIPE
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_hier_pipelined(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule,
                                            uint32_t epoch, void* stream) {
  mp::clear_error();
  if (!loop || !plan) MP_FAIL(MP_ERR_KERNEL, "null argument");
  const bool df = (schedule & 3) == MP_SCHED_DATAFLOW;
  const bool pull = (schedule & MP_SCHED_PULL) != 0;
  if (df && epoch == 0) MP_FAIL(MP_ERR_KERNEL, "dataflow epochs start at 1");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  const mp_hier_plan& P = *plan;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() { return mp::launch_pipe_op<Op, scalar_t>(L, P, df, pull, epoch, st); });
  });
}
