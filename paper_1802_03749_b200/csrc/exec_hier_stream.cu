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
//     software-pipelined in registers: an iteration's top loads the next
//     fill's descriptor and this fill's ids, its bottom issues the gathers,
//     so no thread waits on an index load;
//   * gathers are issued by all lanes (32 rows per warp instruction), row by
//     row from the block's ascending deduplicated staged list;
//   * shared rows hold an odd number of 16/8/4-byte granules, or are
//     XOR-swizzled when the granule count is a power of two (32-byte rows),
//     so consecutive slots -- the common case after GPS / partition
//     reordering -- are bank-conflict free with vector accesses;
//   * increment rows are loaded into registers one block ahead (not staged);
//     the first writer of each staged row stores 0 + x (plan-time mask), so
//     the shared increment rows are never re-zeroed;
//   * per-element plan data (slots, thread colour, first-writer mask) is one
//     packed record (plan-time), one 4-byte-granule copy per element;
//   * increment-only staging reads the element's rows straight into
//     registers through its mapping row (issued before the stage wait);
//   * CTAs are widened when the widest staged list needs more than 2 (4 for
//     arity 8) rows per thread; 72-register cap -> 7 CTAs of 128 per SM.
//
// Schedules: MP_SCHED_COLOUR (one programmatic-dependent launch per block
// colour: a colour's prologue overlaps the previous colour's tail), its pull
// form (| MP_SCHED_PULL: elements park their per-slot increments, one
// barrier, the owner of each staged row sums its refs in thread-colour order
// from the plan pull lists), and MP_SCHED_DATAFLOW (one launch; tickets in a
// topological order of the lower-colour conflict DAG).  Dataflow adds one
// "sync" warp per CTA that
//   - checks, in fill order and off the critical path, that every
//     lower-colour predecessor of the CTA's upcoming blocks has written back
//     (relaxed polls of epoch flags from ticket-ordered padded lists, one gpu
//     fence per productive pass) and publishes a ready count in shared
//     memory; a block's increment rows are trusted only if the block was
//     ready when they were loaded, otherwise ("late") they are re-read from
//     L2 at write-back after waiting for readiness;
//   - releases the flags of the CTA's finished blocks (per-warp write-back
//     counters) in batches, one gpu fence per batch.
// Deadlock freedom: compute threads only wait (late write-back) for the
// readiness of the block they are writing back, whose predecessors hold
// smaller tickets; the CTA holding the smallest unfinished ticket has
// finished all its earlier ones, and sync warps keep releasing finished
// blocks while they poll, so that ticket always progresses while every CTA
// is resident (the grid is capped at the occupancy-derived resident count,
// and static-claim dataflow grids on a device are chained one after another,
// mp_common.cuh static_dataflow_begin).
// An opt-in variant (MESHPLAN_STREAM_TMA=1) gathers read rows with TMA
// tile::gather4 into per-stage mbarriers (measured slower).
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "mp_loop.cuh"

#ifndef MP_ROW256
#define MP_ROW256 1  // 256-bit global accesses for 32-byte increment rows
#endif
#ifndef MP_STREAM_MAXREG
#define MP_STREAM_MAXREG 72  // 7 CTAs of 128 threads per SM
#endif
#ifndef MP_STREAM_MAXREG_EXPORT
#define MP_STREAM_MAXREG_EXPORT 72  // fused halo export: 7 CTAs/SM (24 bytes of spill; C5 at world size 1: 1.296 vs 1.295 ms without the export)
#endif
#ifndef MP_STREAM_MAXREG_DF
#define MP_STREAM_MAXREG_DF 72  // dataflow: 128 + 32 threads, 5 CTAs/SM (64 spills on the critical path)
#endif

namespace mp {
namespace {

// staged entry -> (owner peer << 24 | row of the owner's mailbox slot), -1 =
// none; per peer the owner's export slot for this rank (parity 0) and the
// bytes between its two parity slots; the device step epoch
struct ExportDesc {
  const int32_t* dest;
  unsigned long long base[8];
  long long stride[8];
  const uint32_t* epoch;
};

struct StreamView {
  const int4* __restrict__ tdesc;           // per ticket {e0, k | nc << 16, s0, ns}
  const int32_t* __restrict__ tblock;       // per ticket block id (dataflow)
  const int32_t* __restrict__ staged_ids;
  const unsigned char* __restrict__ emeta;  // per element: A slots, colour byte, pad
  const int32_t* __restrict__ pred_offsets;
  const int32_t* __restrict__ preds;
  union {                                   // (one kernel parameter slot: the struct's size is tuned)
    const int32_t* __restrict__ pred_pad;   // [ntickets][8] (dataflow schedules)
    const struct ExportDesc* xdesc;         // fused halo export (EXPORT, colour schedules): the block that
  };                                        // writes a halo row last stores it into the owner's mailbox
  uint32_t* flags;
  uint32_t epoch;
  const uint16_t* __restrict__ pull_off;  // pull variant: plan pull lists
  const uint16_t* __restrict__ pull_ref;
  int32_t ntickets;
  int32_t em_bytes;
  int32_t max_staged;
  int32_t max_block;
  int32_t nt;     // compute threads (multiple of 32)
  int32_t depth;  // blocks in flight; stages = depth + 1
  int32_t stage_reads;
  int32_t bulk_rows;  // TMA path: per-lane 1D bulk copies of 32-byte rows instead of tensor gather4
  uint32_t* stats;  // optional (MESHPLAN_STREAM_STATS): [0] late blocks
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
__device__ __forceinline__ void red_release_cta_add(int* p, int v) {
  asm volatile("red.release.cta.shared::cta.add.s32 [%0], %1;" ::"r"(saddr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- mbarrier / TMA gather4 (staged read rows through the tensor engine) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(
          saddr(bar)),
      "r"(parity)
      : "memory");
}
// four rows (r0..r3) of a 2D tensor map, {comps x 1} box each, into 4
// consecutive shared rows (the map's swizzle applies), completing on `bar`
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(saddr(bar))
      : "memory");
}

// one contiguous global -> shared copy through the TMA unit, completing on `bar`
__device__ __forceinline__ void tma_bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}

// Row format in shared memory.  A row of RB bytes is accessed in granules of
// G = 16/8/4 bytes (the widest dividing RB); N = RB/G granules.  Rows are
// packed at pitch RB when N is odd (consecutive rows then start in distinct
// bank groups); when N is a power of two >= 2 (16-byte granules: 32-, 64-,
// 128-byte rows) granule c of row r is stored at slot c ^ ((r / (8/N)) % N),
// an XOR swizzle that keeps any 8 consecutive rows' granules in distinct
// 16-byte bank groups without padding; other even N are padded by one granule.
template <int RB>
struct RowFmt {
  static constexpr int G = RB % 16 == 0 ? 16 : (RB % 8 == 0 ? 8 : 4);
  static constexpr int N = RB / G;
  static constexpr bool SWZ = G == 16 && N >= 2 && N <= 8 && (N & (N - 1)) == 0;
  static constexpr int PITCH = RB == 0 ? 0 : ((N % 2 == 1 || SWZ) ? RB : RB + G);
  __device__ __forceinline__ static int slot(int r, int c) {
    constexpr int SHIFT = N == 2 ? 2 : (N == 4 ? 1 : 0);
    if constexpr (SWZ) return r * PITCH + ((c ^ ((r >> SHIFT) & (N - 1))) * G);
    else return r * PITCH + c * G;
  }
};

template <int G>
struct Gran;
template <>
struct Gran<16> { using type = uint4; };
template <>
struct Gran<8> { using type = uint2; };
template <>
struct Gran<4> { using type = uint32_t; };

// shared row r -> registers / registers -> shared row r (granule accesses)
template <typename T, int NC>
__device__ __forceinline__ void lds_row(const unsigned char* base, int r, T (&out)[NC]) {
  using F = RowFmt<NC * (int)sizeof(T)>;
  using V = typename Gran<F::G>::type;
#pragma unroll
  for (int c = 0; c < F::N; ++c) {
    V x = *reinterpret_cast<const V*>(base + F::slot(r, c));
    memcpy(reinterpret_cast<unsigned char*>(out) + c * F::G, &x, F::G);
  }
}
template <typename T, int NC>
__device__ __forceinline__ void sts_row(unsigned char* base, int r, const T (&in)[NC]) {
  using F = RowFmt<NC * (int)sizeof(T)>;
  using V = typename Gran<F::G>::type;
#pragma unroll
  for (int c = 0; c < F::N; ++c) {
    V x;
    memcpy(&x, reinterpret_cast<const unsigned char*>(in) + c * F::G, F::G);
    *reinterpret_cast<V*>(base + F::slot(r, c)) = x;
  }
}

// global row (point p) of an indirect array -> shared row r (async).  AoS rows
// of `comps` components copy their first NC components.
template <typename T, int NC, int LAYOUT>
__device__ __forceinline__ void gather_row(unsigned char* base, int r, const T* g, int64_t p, int comps,
                                           int64_t npts) {
  using F = RowFmt<NC * (int)sizeof(T)>;
  if constexpr (LAYOUT == MP_AOS) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(g + p * comps);
    if ((comps * (int)sizeof(T)) % F::G == 0) {
#pragma unroll
      for (int c = 0; c < F::N; ++c) cpa<F::G>(base + F::slot(r, c), src + c * F::G);
      return;
    }
  }
  // element-wise (SoA planes, or AoS rows whose stride breaks the granule)
  constexpr int PER = F::G / (int)sizeof(T);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const T* s = LAYOUT == MP_AOS ? g + p * comps + c : g + (int64_t)c * npts + p;
    cpa<(int)sizeof(T)>(base + F::slot(r, c / PER) + (c % PER) * (int)sizeof(T), s);
  }
}

// global row of an incremented array -> registers (L2 path when `cg`)
template <typename T, int NC, int LAYOUT>
__device__ __forceinline__ void ldg_row(const T* g, int64_t p, int64_t npts, bool cg, T (&out)[NC]) {
  constexpr int RB = NC * (int)sizeof(T);
  if constexpr (LAYOUT == MP_AOS && RB == 32 && MP_ROW256) {
    // one 256-bit access per 32-byte row (LDG.E.ENL2.256): one LSU request
    // per lane instead of two 16-byte ones
    const T* src = g + p * NC;
    unsigned long long a, b, c, d;
    if (cg)
      asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(src));
    else
      asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(src));
    const unsigned long long w[4] = {a, b, c, d};
    memcpy(out, w, 32);
  } else if constexpr (LAYOUT == MP_AOS) {
    constexpr int G = RB % 16 == 0 ? 16 : (RB % 8 == 0 ? 8 : 4);
    using V = typename Gran<G>::type;
    const V* src = reinterpret_cast<const V*>(g + p * NC);
#pragma unroll
    for (int c = 0; c < RB / G; ++c) {
      V x = cg ? __ldcg(src + c) : *(src + c);
      memcpy(reinterpret_cast<unsigned char*>(out) + c * G, &x, G);
    }
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = cg ? __ldcg(g + (int64_t)c * npts + p) : g[(int64_t)c * npts + p];
  }
}

// Control block: int counters [0] done fills, [1] ready fills (dataflow),
// then one "rows landed" mbarrier per stage (TMA path).
constexpr int CTL_RING = 8;
constexpr int MAX_NS = 6;
constexpr int CTL_BYTES = CTL_RING * 4 + MAX_NS * 8;

// registers -> global row (point p) of the incremented array
template <typename T, int NC, int LAYOUT>
__device__ __forceinline__ void stg_row(T* g, int64_t p, int64_t npts, const T (&in)[NC]) {
  if constexpr (LAYOUT == MP_AOS && NC * (int)sizeof(T) == 32 && MP_ROW256) {
    unsigned long long w[4];
    memcpy(w, in, 32);
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(g + p * NC), "l"(w[0]), "l"(w[1]), "l"(w[2]),
                 "l"(w[3])
                 : "memory");
  } else if constexpr (LAYOUT == MP_AOS) {
    constexpr int RB = NC * (int)sizeof(T);
    constexpr int GG = RB % 16 == 0 ? 16 : (RB % 8 == 0 ? 8 : 4);
    using V = typename Gran<GG>::type;
    unsigned char* dst = reinterpret_cast<unsigned char*>(g + p * NC);
#pragma unroll
    for (int ch = 0; ch < RB / GG; ++ch) {
      V x;
      memcpy(&x, reinterpret_cast<const unsigned char*>(in) + ch * GG, GG);
      *reinterpret_cast<V*>(dst + ch * GG) = x;
    }
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) g[(int64_t)c * npts + p] = in[c];
  }
}

// Stage layout (bytes), identical on host and device.
template <class Op, typename T>
struct StreamLayout {
  static constexpr int QB = RcArr<Op>::N * (int)sizeof(T), IB = Op::IC * (int)sizeof(T);
  static constexpr int QP = RowFmt<QB>::PITCH, IP = RowFmt<IB>::PITCH;
  int ids, q, dir, em, poff, pref, bytes, inc, ctl, total;
  __host__ __device__ static int a16(int x) { return (x + 15) & ~15; }
  // stage_reads: staged read rows [ms (+3)][QP]; increment-only staging: the
  // block's mapping rows [mb][ARITY] int32 (reads go straight to registers).
  // tma: 1024-byte aligned read rows (TMA swizzle atoms).  pull: the block's
  // pull lists (u16 offsets per staged row, u16 refs per (element, slot),
  // 4-byte windows) and a parking buffer [mb*ARITY][IP] instead of the
  // shared increment rows [ms][IP].
  __host__ __device__ StreamLayout(int ms, int mb, int em_bytes, bool stage_reads, int nstage, bool tma = false,
                                   bool pull = false) {
    const int qbytes = Op::RC == 0 ? 0 : (stage_reads ? ((ms + 3) & ~3) * QP : mb * Op::ARITY * 4);
    const int al = tma ? 1023 : 15;
    ids = 16;
    q = (ids + ms * 4 + al) & ~al;
    dir = a16(q + qbytes);
    em = a16(dir + Op::DC * mb * (int)sizeof(T));
    poff = a16(em + mb * em_bytes);
    pref = a16(poff + (pull ? (ms + 1) * 2 + 8 : 0));
    bytes = (pref + (pull ? mb * Op::ARITY * 2 + 8 : 0) + al) & ~al;
    inc = nstage * bytes;
    ctl = a16(inc + (pull ? mb * Op::ARITY : ms) * IP);
    total = ctl + CTL_BYTES;
  }
};

template <class Op, typename T, int LAYOUT, bool DATAFLOW, typename SlotT, int MAXR, bool TMAQ, bool SR, bool PULL,
          bool EXPORT = false>
__global__ void __maxnreg__(DATAFLOW ? MP_STREAM_MAXREG_DF : (EXPORT ? MP_STREAM_MAXREG_EXPORT : MP_STREAM_MAXREG))
    hier_stream_kernel(LoopView<T> v, StreamView H, const __grid_constant__ CUtensorMap qmap) {
  constexpr int A = Op::ARITY, RC = Op::RC, IC = Op::IC, DC = Op::DC, RCN = RcArr<Op>::N;
  using L_t = StreamLayout<Op, T>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int NT = H.nt, D = H.depth, NS = H.depth + 1;
  constexpr bool stage_reads = RC > 0 && SR;  // staged read rows (else reads via the mapping)
  const L_t L(H.max_staged, H.max_block, H.em_bytes, stage_reads, NS, TMAQ, PULL);
  unsigned char* sh_inc = smem + L.inc;
  int* ctl = reinterpret_cast<int*>(smem + L.ctl);  // [0] done count, [1] ready count
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  // static claims: fill f of CTA c takes ticket c + f * grid
  const int total = H.ntickets > (int)blockIdx.x ? (H.ntickets - (int)blockIdx.x + G - 1) / G : 0;

  for (int i = tid; i < (PULL ? 0 : H.max_staged * L_t::IP / 4); i += blockDim.x) reinterpret_cast<uint32_t*>(sh_inc)[i] = 0u;
  if (tid < CTL_RING) ctl[tid] = 0;
  uint64_t* qbar = reinterpret_cast<uint64_t*>(ctl + CTL_RING);  // [NS] staged read rows landed
  if (TMAQ && tid == 0) {
    for (int b = 0; b < NS; ++b) mbar_init(qbar + b, NT >> 5);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Programmatic dependent launch: let the next launch on the stream start
  // its CTAs (prologue gathers of read-only data) as this grid's CTAs retire;
  // griddepcontrol.wait below guards every access to the incremented array.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (DATAFLOW && tid >= NT) {
    // ------------------------------ sync warp ------------------------------
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // Readiness: lanes = 4 fills x 8 predecessor slots; the predecessor ids of
    // the window [u, u+4) come from the ticket-ordered padded lists (-1 = none,
    // -2 in slot 7 = more in the CSR) and stay in registers while the window
    // waits, so a pass costs one round trip of relaxed flag loads.  One gpu
    // fence per productive pass turns the observed flags into acquires (before
    // the ready count is published) and the CTA's finished write-backs
    // (counted per warp in shared memory) into releases (before their flags).
    const int lane = tid & 31, fo = lane >> 3, slot = lane & 7;
    int u = 0, released = 0, win = -1;
    int pid = -1;
    for (;;) {
      if (win != u) {  // (re)load the window's predecessor ids
        const int f = u + fo;
        pid = f < total ? __ldg(H.pred_pad + (int64_t)((int)blockIdx.x + f * G) * 8 + slot) : -1;
        win = u;
      }
      bool ok = pid < 0 || ld_relaxed_gpu(H.flags + pid) == H.epoch;
      if (pid == -2) {  // overflow: the block's 8th and later predecessors from the CSR
        const int tk = (int)blockIdx.x + (u + fo) * G;
        const int q1 = __ldg(H.pred_offsets + tk + 1);
        for (int q = __ldg(H.pred_offsets + tk) + 7; q < q1; ++q)
          ok &= ld_relaxed_gpu(H.flags + __ldg(H.preds + q)) == H.epoch;
      }
      const int done = ld_acquire_cta(ctl + 0);
      const unsigned bad = __ballot_sync(0xffffffffu, !ok);
      int nu = u + (bad ? (__ffs(bad) - 1) / 8 : 4);
      nu = nu < total ? nu : total;
      if (done > released || nu > u) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int g = released + lane; g < done; g += 32)
          st_relaxed_gpu(H.flags + __ldg(H.tblock + (int)blockIdx.x + g * G), H.epoch);
        released = done;
        if (nu > u && lane == 0) st_release_cta(ctl + 1, nu);
        u = nu;
      } else {
        __nanosleep(32);
      }
      if (released >= total) break;
    }
    return;
  }

  // ------------------------------ compute threads ------------------------------
  const int t = tid;
  auto load_desc = [&](int f) -> int4 {
    return f < total ? __ldg(H.tdesc + (int)blockIdx.x + f * G) : make_int4(0, 0, 0, 0);
  };
  auto load_block = [&](int f) -> int { return (PULL && f < total) ? __ldg(H.tblock + (int)blockIdx.x + f * G) : 0; };
  auto load_ids = [&](const int4& d, int (&ids)[MAXR]) {
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {  // unpredicated (clamped) loads: no merge copies
      const int j = t + r * NT;
      ids[r] = __ldg(H.staged_ids + max(d.z + min(j, d.w - 1), 0));
    }
  };
  auto load_map = [&](const int4& d, int (&mp)[A]) {
    if (RC > 0 && !stage_reads) {
      const bool on = t < (d.y & 0xffff);
#pragma unroll
      for (int s = 0; s < A; ++s) mp[s] = on ? map_at(v, (int64_t)d.x + t, s) : 0;
    }
  };
  uint64_t row_bits = 0;  // bit s*MAXR + r: this thread's row r of the block in stage s exists
  auto issue_fill = [&](int s, const int4& d, int blk, const int (&ids)[MAXR], const int (&mp)[A]) {
    unsigned char* st = smem + s * L.bytes;
    const int k = d.y & 0xffff, ns = d.w;
    if constexpr (PULL) {  // 4-byte windows over the u16 lists; the u16 deltas go to the header
      const int64_t ob = ((int64_t)d.z + blk) * 2, olo = ob & ~int64_t(3);
      const int ow = ns > 0 ? (int)((ob - olo) + (ns + 1) * 2 + 3) / 4 : 0;
      const int64_t rb = (int64_t)d.x * A * 2, rlo = rb & ~int64_t(3);
      const int rw = k > 0 ? (int)((rb - rlo) + k * A * 2 + 3) / 4 : 0;
      for (int w = t; w < ow + rw; w += NT) {
        if (w < ow)
          cpa<4>(st + L.poff + 4 * w, reinterpret_cast<const unsigned char*>(H.pull_off) + olo + 4 * w);
        else
          cpa<4>(st + L.pref + 4 * (w - ow), reinterpret_cast<const unsigned char*>(H.pull_ref) + rlo + 4 * (w - ow));
      }
      if (t == 0) {
        reinterpret_cast<int*>(st)[3] = (int)(ob - olo) / 2 | ((int)(rb - rlo) / 2) << 16;
      }
    }
    uint64_t bits = 0;
#pragma unroll
    for (int r = 0; r < MAXR; ++r) bits |= (uint64_t)(t + r * NT < ns) << r;
    row_bits = (row_bits & ~(((uint64_t(1) << MAXR) - 1) << (s * MAXR))) | (bits << (s * MAXR));
    if (t == 0) {
      int* hdr = reinterpret_cast<int*>(st);
      hdr[0] = k;
      hdr[1] = ns;
      hdr[2] = d.y >> 16;
      if constexpr (EXPORT) ctl[2 + s] = d.z;  // staged offset of the stage's block (fused export)
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      if (j < ns) {
        const int p = ids[r];
        reinterpret_cast<int*>(st + L.ids)[j] = p;
        if (!TMAQ && stage_reads) gather_row<T, RCN, LAYOUT>(st + L.q, j, v.ind, p, v.ind_comps, v.npts);
      }
    }
    if constexpr (TMAQ) if (H.bulk_rows) {
      // every lane copies its own 32-byte rows with 1D bulk copies through the
      // TMA unit (no LSU instructions): one copy per row, or its two 16-byte
      // granules swapped where the row format's XOR swizzle exchanges them
      const int lane = t & 31;
      unsigned nrow = 0;
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        const int left = ns - ((t & ~31) + r * NT);
        nrow += left <= 0 ? 0u : (unsigned)(left > 32 ? 32 : left);
      }
      if (lane == 0) mbar_arrive_expect(qbar + s, nrow * (unsigned)L_t::QB);
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        const int j = t + r * NT;
        if (j < ns) {
          const unsigned char* src = reinterpret_cast<const unsigned char*>(v.ind + (int64_t)ids[r] * v.ind_comps);
          unsigned char* row = st + L.q;
          using F = RowFmt<L_t::QB>;
          if (F::slot(j, 0) == j * F::PITCH) {
            tma_bulk(row + F::slot(j, 0), src, (unsigned)L_t::QB, qbar + s);
          } else {
#pragma unroll
            for (int c = 0; c < F::N; ++c) tma_bulk(row + F::slot(j, c), src + c * F::G, (unsigned)F::G, qbar + s);
          }
        }
      }
    } else {
      // each warp gathers its own rows, four per lane-quad leader; rows past
      // ns repeat the warp's last valid id (the q area holds ns rounded up to
      // 4 rows).  The transaction bytes are announced before any copy issues.
      const int lane = t & 31;
      unsigned groups = 0;
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        const int nrow = ns - ((t & ~31) + r * NT);
        groups += nrow <= 0 ? 0u : (unsigned)((nrow > 32 ? 32 : nrow) + 3) / 4;
      }
      if (lane == 0) mbar_arrive_expect(qbar + s, groups * 4u * (unsigned)L_t::QB);
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the stage before async writes
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        const int base = (t & ~31) + r * NT;
        const int last = ns - 1 - base;  // lane holding the block's last id, if in this warp
        const int pl = __shfl_sync(0xffffffffu, ids[r], last < 0 ? 0 : (last > 31 ? 31 : last));
        const int pp = (base + lane) < ns ? ids[r] : pl;
        const int p1 = __shfl_down_sync(0xffffffffu, pp, 1), p2 = __shfl_down_sync(0xffffffffu, pp, 2),
                  p3 = __shfl_down_sync(0xffffffffu, pp, 3);
        if ((lane & 3) == 0 && base + lane < ns)
          tma_gather4(st + L.q + (base + lane) * L_t::QP, &qmap, pp, p1, p2, p3, qbar + s);
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
    }
    if (RC > 0 && !stage_reads && t < H.max_block) {  // this thread's own mapping row (-1: no element)
#pragma unroll
      for (int sl = 0; sl < A; ++sl) reinterpret_cast<int*>(st + L.q)[t * A + sl] = t < k ? mp[sl] : -1;
    }
  };
  // increment rows of block f (staged ids of stage s) -> registers; on the
  // dataflow schedule only once the block's predecessors are known done
  // fused halo export (EXPORT instantiations only): the block that writes a
  // halo row last stores the row's final value into the owner's mailbox slot
  // instead of the local row (which is re-zeroed after the step and never
  // read again): one 256-bit P2P store in place of the local one
  auto write_row = [&](int s_, int j, int64_t p, const T (&val)[IC]) {
    if constexpr (EXPORT) {
      const ExportDesc* X = H.xdesc;
      const int dst = __ldg(X->dest + ctl[2 + s_] + j);
      T* base = v.inc;
      int64_t row = p;
      if (dst >= 0) {
        const int peer = dst >> 24;
        base = reinterpret_cast<T*>(__ldg(&X->base[peer]) +
                                    (unsigned long long)(__ldg(X->epoch) & 1u) * (unsigned long long)__ldg(&X->stride[peer]));
        row = dst & 0xFFFFFF;
      }
      stg_row<T, IC, MP_AOS>(base, row, 0, val);
    } else {
      stg_row<T, IC, LAYOUT>(v.inc, p, v.npts, val);
    }
  };
  T rrow[MAXR][IC];
  bool rows_late = false;
  auto load_rows = [&](int f, int s) {
    const unsigned char* st = smem + s * L.bytes;
    rows_late = false;
    if constexpr (DATAFLOW) rows_late = ld_acquire_cta(ctl + 1) <= f;
    // unpredicated loads (absent rows read point 0; a late block's rows are
    // re-read after its wait), so the values land straight in rrow
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      const int p = ((row_bits >> (s * MAXR + r)) & 1u) ? reinterpret_cast<const int*>(st + L.ids)[j] : 0;
      ldg_row<T, IC, LAYOUT>(v.inc, p, v.npts, DATAFLOW, rrow[r]);
    }
  };

  // Prologue: fills 0 .. D-1 and block 0's increment rows.  Steady state,
  // iteration i: the top loads the descriptor of fill i+D+1 and the staged
  // ids (map rows) of fill i+D (descriptor loaded one iteration earlier); the
  // bottom issues fill i+D and loads block i+1's increment rows.  Every
  // register load has a whole iteration to land before its first use.
  int ids_fill[MAXR];
  int map_fill[A];
#pragma unroll
  for (int s = 0; s < A; ++s) map_fill[s] = 0;
  for (int f = 0; f < D; ++f) {
    const int4 d = load_desc(f);
    load_ids(d, ids_fill);
    load_map(d, map_fill);
    issue_fill(f, d, load_block(f), ids_fill, map_fill);
    cp_commit();
  }
  int4 d_fill = load_desc(D);
  int b_fill = load_block(D);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous launch's increments are visible
  load_rows(0, 0);  // the ids are this thread's own shared stores: no wait

  auto cbar = [&]() {
    if constexpr (DATAFLOW) named_sync(1, NT);
    else __syncthreads();
  };

  int s = 0;       // stage of block i
  int s_fill = D;  // stage of fill i+D (= stage of block i-1)
  unsigned qphase = 0;  // TMA path: expected parity of each stage's mbarrier
  for (int i = 0; i < total; ++i) {
    // a. loads for the bottom of this iteration and the next one
    const int4 d_next = load_desc(i + D + 1);
    const int b_next = load_block(i + D + 1);
    load_ids(d_fill, ids_fill);
    load_map(d_fill, map_fill);
    // increment-only staging: this thread's element reads through its own
    // mapping row (stored by this thread at fill time), issued before the wait
    T r[A][RCN];
    if constexpr (RC > 0 && !stage_reads) if (t < H.max_block) {
      const int* mrow = reinterpret_cast<const int*>(smem + s * L.bytes + L.q) + t * A;
#pragma unroll
      for (int q = 0; q < A; ++q) {
        const int p = max(mrow[q], 0);
#pragma unroll
        for (int c = 0; c < RCN; ++c) r[q][c] = __ldg(v.ind + ind_index<LAYOUT>(p, c, v.ind_comps, v.npts));
      }
    }
    // b. block i has landed (D-1 younger groups may still be in flight)
    cp_wait(D - 1);
    if constexpr (TMAQ) {
      mbar_wait(qbar + s, (qphase >> s) & 1u);
      qphase ^= 1u << s;
    }
    cbar();
    if (DATAFLOW && t == 0) st_release_cta(ctl + 0, i);  // blocks < i are written back (this barrier)
    const unsigned char* st = smem + s * L.bytes;
    const int* hdr = reinterpret_cast<const int*>(st);

    // c. compute block i
    const int k = hdr[0], ns = hdr[1], nc = hdr[2];
    T o[A][IC];
    int ls[A];
    int my_tc = -1;
    unsigned fmask = 0;  // slots whose row this element writes first (store, no load)
    if (t < k) {
      const unsigned char* em = st + L.em + t * H.em_bytes;
      const SlotT* sl = reinterpret_cast<const SlotT*>(em);
#pragma unroll
      for (int q = 0; q < A; ++q) ls[q] = sl[q];
      my_tc = em[A * sizeof(SlotT)];
      fmask = em[A * sizeof(SlotT) + 1];
      T dd[DC];
#pragma unroll
      for (int c = 0; c < DC; ++c) dd[c] = reinterpret_cast<const T*>(st + L.dir)[c * H.max_block + t];
      if (RC > 0 && stage_reads) {
#pragma unroll
        for (int q = 0; q < A; ++q) lds_row<T, RCN>(st + L.q, ls[q], r[q]);
      }
      compute<Op, T>(v, r, dd, o);
    }
    if constexpr (PULL) {
      // d'. pull form of the colour loop: park every element's increments
      //     (one barrier), then the owner of staged row j sums the row's refs
      //     in thread-colour order starting from 0 -- the reference's zeroed
      //     shared row + per-colour np.add.at (simulator.py:634-643), bit for
      //     bit -- and writes row + sum back once.
      if (t < k) {
#pragma unroll
        for (int q = 0; q < A; ++q) sts_row<T, IC>(sh_inc, t * A + q, o[q]);
      }
      cbar();
      const int dl = hdr[3];
      const uint16_t* po = reinterpret_cast<const uint16_t*>(st + L.poff) + (dl & 0xffff);
      const uint16_t* pr = reinterpret_cast<const uint16_t*>(st + L.pref) + (dl >> 16);
      if (DATAFLOW && rows_late && t < ns) {
        while (ld_acquire_cta(ctl + 1) <= i) __nanosleep(32);
      }
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        const int j = t + r * NT;
        if (j < ns) {
          const int64_t p = reinterpret_cast<const int*>(st + L.ids)[j];
          const int lo = po[j], hi = po[j + 1];
          T acc[IC], x[IC];
          lds_row<T, IC>(sh_inc, pr[lo], x);
#pragma unroll
          for (int c = 0; c < IC; ++c) acc[c] = x[c] + T(0);  // 0 + x
          for (int rr = lo + 1; rr < hi; ++rr) {
            lds_row<T, IC>(sh_inc, pr[rr], x);
#pragma unroll
            for (int c = 0; c < IC; ++c) acc[c] += x[c];
          }
          if (DATAFLOW && rows_late) ldg_row<T, IC, LAYOUT>(v.inc, p, v.npts, true, rrow[r]);
#pragma unroll
          for (int c = 0; c < IC; ++c) acc[c] = rrow[r][c] + acc[c];
          write_row(s, j, p, acc);
        }
      }
    } else {
    // d. thread colours, one at a time
    for (int c = 0; c < nc; ++c) {
      if (my_tc == c) {
#pragma unroll
        for (int q = 0; q < A; ++q) {
          T acc[IC];
          if ((fmask >> q) & 1u) {  // 0 + x, the reference's zeroed shared row (simulator.py:634-643)
#pragma unroll
            for (int cc = 0; cc < IC; ++cc) acc[cc] = o[q][cc] + T(0);
          } else {
            lds_row<T, IC>(sh_inc, ls[q], acc);
#pragma unroll
            for (int cc = 0; cc < IC; ++cc) acc[cc] += o[q][cc];
          }
          sts_row<T, IC>(sh_inc, ls[q], acc);
        }
      }
      cbar();
    }
    // e. write back: row + increment, once per staged row (every staged row has
    //    a first writer, so the shared rows need no re-zeroing)
    if (DATAFLOW && rows_late && t < ns) {
      if (H.stats && t == 0) atomicAdd(H.stats, 1u);
      while (ld_acquire_cta(ctl + 1) <= i) __nanosleep(32);
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int j = t + r * NT;
      if (j < ns) {
        const int64_t p = reinterpret_cast<const int*>(st + L.ids)[j];
        T acc[IC];
        lds_row<T, IC>(sh_inc, j, acc);
        if (DATAFLOW && rows_late) ldg_row<T, IC, LAYOUT>(v.inc, p, v.npts, true, rrow[r]);
#pragma unroll
        for (int c = 0; c < IC; ++c) acc[c] = rrow[r][c] + acc[c];
        write_row(s, j, p, acc);
      }
    }
    }  // push form
    // f. issue fill i+D into the stage block i-1 used (every thread passed
    //    this iteration's barrier after finishing block i-1); load block
    //    i+1's increment rows (its ids were stored by this thread)
    issue_fill(s_fill, d_fill, b_fill, ids_fill, map_fill);
    cp_commit();
    const int s_next = s + 1 == NS ? 0 : s + 1;
    load_rows(i + 1, s_next);
    d_fill = d_next;
    b_fill = b_next;
    s_fill = s;
    s = s_next;
  }
  cp_wait(0);
  if constexpr (DATAFLOW) {
    named_sync(1, NT);
    if (t == 0) st_release_cta(ctl + 0, total);
  }
}

// ---- host: 2D row tensor maps for TMA gather4 ----
template <typename T> constexpr int dtype_code() {
  return std::is_same<T, double>::value ? (int)CU_TENSOR_MAP_DATA_TYPE_FLOAT64
       : std::is_same<T, float>::value  ? (int)CU_TENSOR_MAP_DATA_TYPE_FLOAT32
       : sizeof(T) == 8                 ? (int)CU_TENSOR_MAP_DATA_TYPE_INT64
                                        : (int)CU_TENSOR_MAP_DATA_TYPE_INT32;
}
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
#define MP_CUDA_TRY_DRV(expr)                                              \
  do {                                                                     \
    int _r = (expr);                                                       \
    if (_r != 0) MP_FAIL(MP_ERR_CUDA, "tensor map encode failed (%d)", _r); \
  } while (0)
// rows of `comps` elements (stride comps*esize bytes), boxes of `used`
// elements x 1 row, swizzle matching RowFmt (32/64/128-byte rows)
inline int encode_row_map(CUtensorMap* map, const void* base, int esize, int dtype, int comps, int64_t rows,
                          int used) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) return -1;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  const int rb = used * esize;
  const CUtensorMapSwizzle sw = rb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                               : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                               : rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE;
  cuuint64_t dims[2] = {(cuuint64_t)comps, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)comps * esize};
  cuuint32_t box[2] = {(cuuint32_t)used, 1};
  cuuint32_t estr[2] = {1, 1};
  return (int)fn(map, (CUtensorMapDataType)dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// Launch with programmatic stream serialization (PDL): consecutive colour
// launches of one loop execution overlap one grid's tail with the next grid's
// prologue, which gathers the loop's read-only data (read rows, direct
// operands, plan records) before griddepcontrol.wait.  Only colour launches
// after the first of a call use it: the first launch of a call may follow
// any other work on the stream (e.g. a loop that writes this loop's read
// array), so it is fully serialised.
template <typename K, typename... Args>
cudaError_t launch_pdl(K kern, int grid, int threads, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  static const bool off = getenv("MESHPLAN_NO_PDL") != nullptr;
  pdl = pdl && !off;
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

template <class Op, typename T, int LAYOUT, typename SlotT>
mp_status launch_stream(const LoopView<T>& v, StreamView H, const mp_hier_plan& P, bool dataflow, bool pull,
                        cudaStream_t st, bool exporting_req = false) {
  static const int env_depth = getenv("MESHPLAN_STREAM_DEPTH") ? atoi(getenv("MESHPLAN_STREAM_DEPTH")) : 2;
  static const int env_ctas = getenv("MESHPLAN_STREAM_CTAS") ? atoi(getenv("MESHPLAN_STREAM_CTAS")) : 0;
  int depth = env_depth < 2 ? 2 : (env_depth > 4 ? 4 : env_depth);
  // CTA width: one thread per block element, widened (idle in the element
  // phases) when the widest staged list would need more than R_LO rows per
  // thread -- arity-8 loops stage ~4 rows per element
  constexpr int R_LO0 = Op::ARITY <= 2 ? 2 : 4;
  int nt = ((P.block_size + 31) / 32) * 32;
  const int nt_rows = ((P.max_staged + R_LO0 - 1) / R_LO0 + 31) / 32 * 32;
  if (nt_rows > nt) nt = nt_rows < 480 ? nt_rows : 480;
  H.nt = nt;
  H.max_block = P.block_size;
  H.max_staged = P.max_staged;
  H.stage_reads = P.stage_reads;
  static uint32_t* stats = nullptr;
  if (getenv("MESHPLAN_STREAM_STATS") && !stats) {
    MP_CUDA_TRY(cudaMallocManaged(&stats, 64));
    memset(stats, 0, 64);
  }
  if (stats && dataflow) {
    MP_CUDA_TRY(cudaStreamSynchronize(st));
    if (stats[1]++ > 0) fprintf(stderr, "[stream stats] late blocks last run: %u\n", stats[0]);
    stats[0] = 0;
  }
  H.stats = stats;
  const bool sr = Op::RC > 0 && P.stage_reads;
  // staged read rows through TMA gather4 when the rows are 32/64/128-byte
  // AoS rows with a 16-byte-multiple stride (else LDGSTS gathers)
  constexpr int QB = Op::RC * (int)sizeof(T);
  // opt-in (MESHPLAN_STREAM_TMA=1): measured slower than the LDGSTS gathers on
  // B200 (C5 1.55 vs 1.39 ms; per-lane coordinates serialise through uniform
  // registers, one gather4 per 4 rows), kept as the TMA-gather variant
  static const bool env_tma = getenv("MESHPLAN_STREAM_TMA") && atoi(getenv("MESHPLAN_STREAM_TMA")) != 0;
  // per-lane 1D bulk copies of the read rows through the TMA unit (takes the
  // q gathers off the LSU pipe)
  static const bool env_bulk = getenv("MESHPLAN_STREAM_BULK") && atoi(getenv("MESHPLAN_STREAM_BULK")) != 0;
  CUtensorMap qmap;
  memset(&qmap, 0, sizeof(qmap));
  bool tma = false;
  H.bulk_rows = 0;
  if constexpr (LAYOUT == MP_AOS && (QB == 32 || QB == 64 || QB == 128)) {  // 4-row groups stay 128-B aligned
    const bool rows_ok = sr && v.n > 0 && (v.ind_comps * (int)sizeof(T)) % 16 == 0 &&
                         (reinterpret_cast<uintptr_t>(v.ind) & 15) == 0;
    if (rows_ok && env_bulk) {
      tma = true;
      H.bulk_rows = 1;
    } else {
      tma = env_tma && rows_ok;
      if (tma)
        MP_CUDA_TRY_DRV(encode_row_map(&qmap, v.ind, (int)sizeof(T), dtype_code<T>(), v.ind_comps, v.npts, Op::RC));
    }
  }
  if (exporting_req) {  // the fused export lives in the LDGSTS instantiations
    tma = false;
    H.bulk_rows = 0;
  }
  size_t smem = 0;
  for (;; --depth) {  // shrink the ring if it does not fit
    const StreamLayout<Op, T> L(P.max_staged, P.block_size, P.elem_meta_bytes, sr, depth + 1, tma, pull);
    smem = (size_t)L.total;
    if (smem <= 227 * 1024 || depth == 2) break;
  }
  if (smem > 227 * 1024)
    MP_FAIL(MP_ERR_CAPACITY, "streamed executor needs %zu shared bytes, over the 232448-byte limit", smem);
  H.depth = depth;
  const int threads = nt + (dataflow ? 32 : 0);
  if (threads > 512) MP_FAIL(MP_ERR_CAPACITY, "block size %d exceeds the streamed executor limit of 480", P.block_size);
  // staged rows per thread (ns <= ARITY * k): 2 for pair loops, 4 or 8 otherwise
  constexpr int R_LO = Op::ARITY <= 2 ? 2 : 4, R_HI = Op::ARITY <= 2 ? 2 : 8;
  const bool hi = P.max_staged > R_LO * nt;
  if (P.max_staged > R_HI * nt) MP_FAIL(MP_ERR_CAPACITY, "block stages %d rows, over %d per CTA", P.max_staged, R_HI * nt);
  using TT = std::true_type;
  using FF = std::false_type;
  constexpr bool TMA_OK = LAYOUT == MP_AOS && (QB == 32 || QB == 64 || QB == 128);
  const bool exporting = exporting_req;
  auto pick_r = [&](auto dflow, auto tmaq, auto sread, auto pl) {
    constexpr bool DF = decltype(dflow)::value, TQ = decltype(tmaq)::value, S = decltype(sread)::value,
                   PU = decltype(pl)::value;
    if constexpr (!DF && !TQ && LAYOUT == MP_AOS) {
      if (exporting)
        return hi ? hier_stream_kernel<Op, T, LAYOUT, DF, SlotT, R_HI, TQ, S, PU, true>
                  : hier_stream_kernel<Op, T, LAYOUT, DF, SlotT, R_LO, TQ, S, PU, true>;
    }
    return hi ? hier_stream_kernel<Op, T, LAYOUT, DF, SlotT, R_HI, TQ, S, PU>
              : hier_stream_kernel<Op, T, LAYOUT, DF, SlotT, R_LO, TQ, S, PU>;
  };
  auto pick_s = [&](auto dflow, auto pl) {  // staging-mode / TMA variants
    if constexpr (Op::RC == 0) return pick_r(dflow, FF{}, FF{}, pl);
    else if constexpr (TMA_OK && !decltype(pl)::value)
      return tma ? pick_r(dflow, TT{}, TT{}, pl) : (sr ? pick_r(dflow, FF{}, TT{}, pl) : pick_r(dflow, FF{}, FF{}, pl));
    else return sr ? pick_r(dflow, FF{}, TT{}, pl) : pick_r(dflow, FF{}, FF{}, pl);
  };
  // pull form: colour schedule only
  auto kern = dataflow ? pick_s(TT{}, FF{}) : (pull ? pick_s(FF{}, TT{}) : pick_s(FF{}, FF{}));
  // attribute + occupancy queries cost microseconds of host time per call:
  // cache them per (kernel, shared bytes, threads, device), process-wide
  int per_sm = 0, dev = 0, sms = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  {
    struct Entry {
      const void* k;
      size_t smem;
      int threads, dev, per_sm, sms;
    };
    struct Limit {
      const void* k;
      int dev;
      size_t smem;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    static std::vector<Limit> limits;  // per (kernel, device): largest dynamic smem limit set
    std::lock_guard<std::mutex> lock(mu);
    const void* kp = reinterpret_cast<const void*>(kern);
    Limit* lim = nullptr;
    for (auto& e : limits)
      if (e.k == kp && e.dev == dev) lim = &e;
    if (!lim) {
      limits.push_back({kp, dev, 0});
      lim = &limits.back();
    }
    if (lim->smem < smem) {  // a larger limit stays valid for smaller launches
      MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      lim->smem = smem;
    }
    bool hit = false;
    for (const auto& e : cache)
      if (e.k == kp && e.smem == smem && e.threads == threads && e.dev == dev) {
        per_sm = e.per_sm;
        sms = e.sms;
        hit = true;
        break;
      }
    if (!hit) {
      MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
      MP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      cache.push_back({kp, smem, threads, dev, per_sm, sms});
    }
  }
  if (per_sm < 1) MP_FAIL(MP_ERR_CAPACITY, "streamed executor does not fit on an SM (%zu shared bytes)", smem);
  if (env_ctas > 0 && env_ctas < per_sm) per_sm = env_ctas;
  const int resident = per_sm * sms;
  if (dataflow) {
    H.tdesc = reinterpret_cast<const int4*>(P.tdesc_order);
    H.tblock = P.order;
    H.pred_offsets = P.tpred_offsets;  // ticket-ordered predecessor CSR
    H.preds = P.tpreds;
    H.pred_pad = P.tpred_pad;
    H.ntickets = P.num_blocks;
    const int grid = P.num_blocks < resident ? P.num_blocks : resident;
    MP_CUDA_TRY(static_dataflow_begin(st));
    const cudaError_t le = launch_pdl(kern, grid, threads, smem, st, false, v, H, qmap);
    MP_CUDA_TRY(static_dataflow_end(st));
    MP_CUDA_TRY(le);
    return MP_OK;
  }
  bool first = true;
  for (int c = 0; c < P.num_block_colours; ++c) {
    const int lo = P.colour_block_offsets_host[c], hi = P.colour_block_offsets_host[c + 1];
    if (hi <= lo) continue;
    H.tdesc = reinterpret_cast<const int4*>(P.tdesc_colour) + lo;
    H.tblock = P.tblock_colour + lo;
    H.ntickets = hi - lo;
    const int grid = (hi - lo) < resident ? (hi - lo) : resident;
    MP_CUDA_TRY(launch_pdl(kern, grid, threads, smem, st, !first, v, H, qmap));
    first = false;
  }
  return MP_OK;
}

struct ExportArgs {
  const void* desc;  // device ExportDesc
};

template <class Op, typename T>
mp_status launch_stream_op(const mp_loop& Lp, const mp_hier_plan& P, bool dataflow, bool pull, uint32_t epoch,
                           cudaStream_t st, const ExportArgs* ex = nullptr) {
  if constexpr (!op_supported<Op, T>()) {
    MP_FAIL(MP_ERR_KERNEL, "heavy face flux needs float data");
  } else {
    mp_status s = check_loop_shape(Lp, Op::ARITY, Op::RC, Op::DC, Op::IC);
    if (s) return s;
    if (P.num_blocks == 0) return MP_OK;
    if (!P.written_is_staged) MP_FAIL(MP_ERR_KERNEL, "streamed executor needs written lists equal to staged lists");
    if (!P.tdesc_colour || !P.tdesc_order || !P.elem_meta || !P.tblock_colour)
      MP_FAIL(MP_ERR_KERNEL, "streamed executor needs the plan's ticket descriptors and element records");
    if (Op::ARITY > 8 || P.elem_meta_bytes < Op::ARITY * P.slot_bytes + 2 || P.elem_meta_bytes % 4)
      MP_FAIL(MP_ERR_KERNEL, "element records of %d bytes cannot hold %d slots, a colour and a first-writer mask", P.elem_meta_bytes,
              Op::ARITY);
    if (dataflow && (!P.order || !P.tpred_offsets || !P.tpreds || !P.tpred_pad || !P.flags))
      MP_FAIL(MP_ERR_KERNEL, "dataflow schedule needs order/preds/flags");
    StreamView H{};
    H.staged_ids = P.staged_ids;
    H.pull_off = P.pull_off;
    H.pull_ref = P.pull_ref;
    H.emeta = P.elem_meta;
    H.pred_offsets = P.pred_offsets;
    H.preds = P.preds;
    H.flags = P.flags;
    H.epoch = epoch;
    H.em_bytes = P.elem_meta_bytes;
    const bool xp = ex && ex->desc;
    if (xp) {
      if (dataflow) MP_FAIL(MP_ERR_KERNEL, "fused halo export runs under the colour schedules");
      if (Lp.ind_layout != MP_AOS) MP_FAIL(MP_ERR_KERNEL, "fused halo export needs AoS increment rows");
      H.xdesc = static_cast<const ExportDesc*>(ex->desc);
    }
    LoopView<T> v = make_view<T>(Lp);
    const bool u8 = P.slot_bytes == 1;
    if (Lp.ind_layout == MP_AOS) {
      if (u8) return launch_stream<Op, T, MP_AOS, uint8_t>(v, H, P, dataflow, pull, st, xp);
      return launch_stream<Op, T, MP_AOS, uint16_t>(v, H, P, dataflow, pull, st, xp);
    }
    if (u8) return launch_stream<Op, T, MP_SOA, uint8_t>(v, H, P, dataflow, pull, st);
    return launch_stream<Op, T, MP_SOA, uint16_t>(v, H, P, dataflow, pull, st);
  }
}

}  // namespace
}  // namespace mp

extern "C" mp_status mp_exec_hier_stream(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule,
                                         uint32_t epoch, void* stream) {
  mp::clear_error();
  if (!loop || !plan) MP_FAIL(MP_ERR_KERNEL, "null argument");
  const bool df = (schedule & 3) == MP_SCHED_DATAFLOW;
  const bool pull = !df && (schedule & MP_SCHED_PULL) != 0;
  if (pull && plan->num_blocks > 0 && (!plan->pull_off || !plan->pull_ref))
    MP_FAIL(MP_ERR_KERNEL, "pull form needs the plan's pull lists");
  if (df && epoch == 0) MP_FAIL(MP_ERR_KERNEL, "dataflow epochs start at 1");
  cudaStream_t st = mp::as_stream(stream);
  const mp_loop& L = *loop;
  const mp_hier_plan& P = *plan;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() { return mp::launch_stream_op<Op, scalar_t>(L, P, df, pull, epoch, st); });
  });
}

extern "C" mp_status mp_export_desc_bytes(void) { return (mp_status)sizeof(mp::ExportDesc); }

extern "C" mp_status mp_exec_hier_stream_export(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule,
                                                const void* export_desc, void* stream) {
  mp::clear_error();
  if (!loop || !plan || !export_desc) MP_FAIL(MP_ERR_KERNEL, "null argument");
  if ((schedule & 3) == MP_SCHED_DATAFLOW) MP_FAIL(MP_ERR_KERNEL, "fused halo export runs under the colour schedules");
  const bool pull = (schedule & MP_SCHED_PULL) != 0;
  if (pull && plan->num_blocks > 0 && (!plan->pull_off || !plan->pull_ref))
    MP_FAIL(MP_ERR_KERNEL, "pull form needs the plan's pull lists");
  cudaStream_t st = mp::as_stream(stream);
  const mp::ExportArgs ex{export_desc};
  const mp_loop& L = *loop;
  const mp_hier_plan& P = *plan;
  return MP_DISPATCH_OP(L.op, [&]() {
    return MP_DISPATCH_DTYPE(L.dtype, [&]() { return mp::launch_stream_op<Op, scalar_t>(L, P, false, pull, 0, st, &ex); });
  });
}
