// Block-local planner kernels (one CTA per plan block):
//   * staged / written point lists  (plan.py:582-603)
//   * shared-slot tables            (plan.py:168-182, materialised)
//   * thread colouring + colour sort (plan.py:260-284, 508-517)
// Blocks are independent, so these are embarrassingly parallel and
// bit-exact with the reference's per-block Python loops.
#include <limits.h>

#include "mp_block_sort.cuh"

namespace mp {
namespace {

__device__ __forceinline__ int32_t map_entry(const int32_t* map, int64_t n, int arity, int layout, int64_t e, int s) {
  return __ldg(layout == MP_AOS ? map + e * arity + s : map + (int64_t)s * n + e);
}

__device__ __forceinline__ int nth_slot(uint32_t mask, int i) {
  // index of the i-th set bit of mask
  for (int s = 0; s < 32; ++s)
    if (mask >> s & 1u) {
      if (i == 0) return s;
      --i;
    }
  return -1;
}

// ---- per-block ascending unique point lists ---------------------------------
__global__ void block_points_kernel(int32_t nb, const int32_t* __restrict__ block_offsets,
                                    const int32_t* __restrict__ map, int64_t n, int arity, int layout,
                                    uint32_t mask, int32_t* counts, const int32_t* __restrict__ offsets,
                                    int32_t* ids) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int warp_tmp[32];
  const int b = blockIdx.x;
  const int e0 = block_offsets[b], k = block_offsets[b + 1] - e0;
  const int nsl = __popc(mask);
  const int cnt = k * nsl, m = next_pow2(cnt > 0 ? cnt : 1);
  int32_t* keys = reinterpret_cast<int32_t*>(smem);
  int* flag = reinterpret_cast<int*>(keys + m);
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    if (i < cnt) {
      int j = i / nsl, s = nth_slot(mask, i - j * nsl);
      keys[i] = map_entry(map, n, arity, layout, (int64_t)e0 + j, s);
    } else {
      keys[i] = INT_MAX;
    }
  }
  bitonic_sort_shared(keys, m);
  for (int i = threadIdx.x; i < m; i += blockDim.x) flag[i] = (i < cnt) && (i == 0 || keys[i] != keys[i - 1]);
  __syncthreads();
  int total = block_exclusive_scan(flag, flag, m, warp_tmp);
  if (ids == nullptr) {
    if (threadIdx.x == 0) counts[b] = total;
    return;
  }
  const int base = offsets[b];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x)
    if (i == 0 || keys[i] != keys[i - 1]) ids[base + flag[i]] = keys[i];
}

// ---- shared-slot tables -------------------------------------------------------
__device__ __forceinline__ int find_sorted(const int32_t* a, int len, int32_t x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return (lo < len && a[lo] == x) ? lo : -1;
}

__global__ void local_slots_kernel(int32_t nb, const int32_t* __restrict__ block_offsets,
                                   const int32_t* __restrict__ map, int64_t n, int arity, int layout, uint32_t mask,
                                   const int32_t* __restrict__ st_off, const int32_t* __restrict__ st_ids,
                                   uint16_t* local_slots, const int32_t* __restrict__ wr_off,
                                   const int32_t* __restrict__ wr_ids, uint16_t* written_slots, int* miss_block) {
  extern __shared__ __align__(16) unsigned char smem[];
  int32_t* lst = reinterpret_cast<int32_t*>(smem);
  const int b = blockIdx.x;
  const int e0 = block_offsets[b], k = block_offsets[b + 1] - e0;
  const int s0 = st_off[b], ns = st_off[b + 1] - s0;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) lst[i] = st_ids[s0 + i];
  __syncthreads();
  for (int i = threadIdx.x; i < k * arity; i += blockDim.x) {
    int j = i / arity, s = i - j * arity;
    int64_t e = (int64_t)e0 + j;
    uint16_t out = 0xFFFFu;
    if (mask >> s & 1u) {
      int pos = find_sorted(lst, ns, map_entry(map, n, arity, layout, e, s));
      if (pos < 0) atomicMin(miss_block, b); else out = (uint16_t)pos;
    }
    local_slots[e * arity + s] = out;
  }
  if (written_slots != nullptr) {
    const int w0 = wr_off[b], nw = wr_off[b + 1] - w0;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
      int pos = find_sorted(lst, ns, wr_ids[w0 + i]);
      if (pos < 0) atomicMin(miss_block, b);
      written_slots[w0 + i] = pos < 0 ? 0xFFFFu : (uint16_t)pos;
    }
  }
}

// ---- thread colouring: one warp per block ----------------------------------
// Conflict graph (elements sharing a written point) as a bit matrix,
// smallest-last elimination order (numpy_impl.py:95-111), first-fit greedy in
// that order (numpy_impl.py:62-92, plan.py:284 passes least_loaded=False),
// then a stable counting sort by colour (plan.py:514).
constexpr int kMaxThreadColours = 256;

__global__ void __launch_bounds__(32) thread_colour_kernel(int32_t nb, const int32_t* __restrict__ block_offsets,
                                                           const int32_t* __restrict__ map, int64_t n, int arity,
                                                           int layout, uint32_t mask, int32_t max_block,
                                                           int32_t* colours, int32_t* counts, int32_t* sorted_order,
                                                           int* overflow_block) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.x, lane = threadIdx.x;
  const int e0 = block_offsets[b], k = block_offsets[b + 1] - e0;
  const int nsl = __popc(mask);
  const int mmax = next_pow2(max_block * nsl > 0 ? max_block * nsl : 1);
  const int W = (max_block + 31) / 32;  // row words (sized for the widest block)
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint32_t* adj = reinterpret_cast<uint32_t*>(keys + mmax);  // [max_block][W]
  int32_t* deg = reinterpret_cast<int32_t*>(adj + (size_t)max_block * W);
  int32_t* col = deg + max_block;
  int32_t* order = col + max_block;
  uint32_t* removed = reinterpret_cast<uint32_t*>(order + max_block);  // [W]

  const int cnt = k * nsl, m = next_pow2(cnt > 0 ? cnt : 1);
  for (int i = lane; i < m; i += 32) {
    if (i < cnt) {
      int j = i / nsl, s = nth_slot(mask, i - j * nsl);
      uint32_t p = (uint32_t)map_entry(map, n, arity, layout, (int64_t)e0 + j, s);
      keys[i] = ((uint64_t)p << 32) | (uint32_t)j;
    } else {
      keys[i] = ~0ull;
    }
  }
  for (int i = lane; i < k * W; i += 32) adj[i] = 0u;
  for (int i = lane; i < W; i += 32) removed[i] = 0u;
  bitonic_sort_shared(keys, m);
  for (int i = lane; i < cnt; i += 32) {
    uint32_t p = (uint32_t)(keys[i] >> 32), u = (uint32_t)keys[i];
    for (int j = i + 1; j < cnt && (uint32_t)(keys[j] >> 32) == p; ++j) {
      uint32_t v = (uint32_t)keys[j];
      if (v == u) continue;
      atomicOr(&adj[u * W + (v >> 5)], 1u << (v & 31));
      atomicOr(&adj[v * W + (u >> 5)], 1u << (u & 31));
    }
  }
  __syncwarp();
  for (int u = lane; u < k; u += 32) {
    int d = 0;
    for (int w = 0; w < W; ++w) d += __popc(adj[u * W + w]);
    deg[u] = d;
    col[u] = -1;
  }
  __syncwarp();
  // smallest-last: remove min (remaining degree, index), place last
  for (int pos = k - 1; pos >= 0; --pos) {
    uint64_t best = ~0ull;
    for (int u = lane; u < k; u += 32)
      if (!(removed[u >> 5] >> (u & 31) & 1u)) {
        uint64_t key = ((uint64_t)(uint32_t)deg[u] << 32) | (uint32_t)u;
        best = key < best ? key : best;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    const int u = (int)(uint32_t)best;
    if (lane == 0) {
      order[pos] = u;
      removed[u >> 5] |= 1u << (u & 31);
    }
    __syncwarp();
    for (int w = lane; w < W; w += 32) {
      uint32_t bits = adj[u * W + w] & ~removed[w];
      while (bits) {
        int t = __ffs(bits) - 1;
        bits &= bits - 1;
        deg[w * 32 + t] -= 1;
      }
    }
    __syncwarp();
  }
  // first-fit greedy in elimination order
  int ncol = 0;
  for (int step = 0; step < k; ++step) {
    const int u = order[step];
    uint64_t forb[kMaxThreadColours / 64] = {0, 0, 0, 0};
    for (int w = lane; w < W; w += 32) {
      uint32_t bits = adj[u * W + w];
      while (bits) {
        int t = __ffs(bits) - 1;
        bits &= bits - 1;
        int c = col[w * 32 + t];
        if (c >= 0 && c < kMaxThreadColours) forb[c >> 6] |= 1ull << (c & 63);
      }
    }
    int chosen = -1;
#pragma unroll
    for (int q = 0; q < kMaxThreadColours / 64; ++q) {
      uint64_t f = forb[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) f |= __shfl_xor_sync(0xffffffffu, f, o);
      if (chosen < 0 && ~f != 0ull) chosen = q * 64 + (__ffsll((long long)~f) - 1);
    }
    if (chosen < 0 || chosen >= kMaxThreadColours) {
      if (lane == 0) atomicMin(overflow_block, b);
      chosen = kMaxThreadColours - 1;
    }
    if (lane == 0) col[u] = chosen;
    ncol = chosen + 1 > ncol ? chosen + 1 : ncol;
    __syncwarp();
  }
  // stable counting sort by colour (lane 0; k <= 1024)
  if (lane == 0) {
    int* start = deg;  // reuse: deg no longer needed, ncol <= k
    for (int c = 0; c < ncol; ++c) start[c] = 0;
    for (int i = 0; i < k; ++i) start[col[i]]++;
    int acc = 0;
    for (int c = 0; c < ncol; ++c) {
      int t = start[c];
      start[c] = acc;
      acc += t;
    }
    for (int i = 0; i < k; ++i) sorted_order[e0 + start[col[i]]++] = e0 + i;
    counts[b] = ncol;
  }
  for (int i = lane; i < k; i += 32) colours[e0 + i] = col[i];
}

size_t thread_colour_smem(int max_block, int nsl) {
  int mmax = next_pow2(max_block * nsl > 0 ? max_block * nsl : 1);
  int W = (max_block + 31) / 32;
  return (size_t)mmax * 8 + (size_t)max_block * W * 4 + (size_t)max_block * 12 + (size_t)W * 4 + 16;
}


// ---- shared-memory row placement (executor layout; the plan is unchanged) -----------
// The executors keep staged row j of a block at shared row j, 32-byte rows
// swizzled so that any 8 rows with distinct j mod 8 fall in 8 distinct 16-byte
// bank groups (exec_hier_stream.cu RowFmt).  A quarter-warp (8 lanes) access
// of 16-byte granules is conflict-free exactly when its rows are distinct mod
// 8.  Blocks whose elements touch staged rows in strided patterns (compact
// tiles: an edge colour class visits every other cell) conflict 2-4 ways.
// This pass renumbers each block's staged rows so that the rows of each
// quarter-warp access group land in distinct classes mod 8: groups are the
// colour-loop read-modify-writes (lanes t..t+7 of one thread colour, one
// slot) and then the element reads (lanes t..t+7, one slot); a greedy
// assigns each unplaced row the class with the most room not yet used in its
// group.  Class c holds positions c, c+8, ... (ns/8 rounded per class), so the
// renumbering is a permutation of 0..ns-1; perm[s0 + position] = old row.
constexpr int RP_MAXS = 4096;

__global__ void row_placement_kernel(int32_t nb, const int32_t* __restrict__ bo, const int32_t* __restrict__ st_off,
                                     const uint16_t* __restrict__ ls, int arity, const uint8_t* __restrict__ tcol,
                                     int32_t* perm) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int e0 = bo[b], k = bo[b + 1] - e0, s0 = st_off[b], ns = st_off[b + 1] - s0;
  if (ns > RP_MAXS) {  // identity (the host checks the maximum first)
    for (int r = 0; r < ns; ++r) perm[s0 + r] = r;
    return;
  }
  int8_t cls[RP_MAXS];
  for (int r = 0; r < ns; ++r) cls[r] = -1;
  int cap[8];
  for (int c = 0; c < 8; ++c) cap[c] = ns / 8 + (c < ns % 8 ? 1 : 0);
  auto place = [&](const int* rows, int n) {
    unsigned used = 0;
    for (int i = 0; i < n; ++i)
      if (cls[rows[i]] >= 0) used |= 1u << cls[rows[i]];
    for (int i = 0; i < n; ++i) {
      const int r = rows[i];
      if (cls[r] >= 0) continue;
      int best = -1;
      for (int pass = 0; pass < 2 && best < 0; ++pass)
        for (int c = 0; c < 8; ++c)
          if (cap[c] > 0 && (pass == 1 || !(used >> c & 1u)) && (best < 0 || cap[c] > cap[best])) best = c;
      cls[r] = (int8_t)best;
      --cap[best];
      used |= 1u << best;
    }
  };
  int rows[8];
  for (int pass = 0; pass < 2; ++pass)  // 0: colour-loop groups, 1: element reads
    for (int q = 0; q < arity; ++q)
      for (int t0 = 0; t0 < k; t0 += 8) {
        const int t1 = t0 + 8 < k ? t0 + 8 : k;
        int t = t0;
        while (t < t1) {  // runs of one thread colour (colour-sorted elements)
          const int c = tcol[e0 + t];
          int n = 0;
          for (; t < t1 && (pass == 1 || tcol[e0 + t] == c); ++t) {
            const int r = ls[(int64_t)(e0 + t) * arity + q];
            if (r == 0xFFFF || r >= ns) continue;
            bool dup = false;
            for (int i = 0; i < n; ++i) dup |= rows[i] == r;
            if (!dup) rows[n++] = r;
          }
          place(rows, n);
        }
      }
  int idx[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = 0; r < ns; ++r) {
    int c = cls[r];
    if (c < 0) {  // a staged row no element touches through a staged slot
      c = 0;
      for (int d = 1; d < 8; ++d)
        if (cap[d] > cap[c]) c = d;
      --cap[c];
    }
    perm[s0 + c + 8 * idx[c]++] = r;
  }
}

// ---- gather-form ref records (exec_hier_gather.cu) ----------------------------
// Per block, the pull lists' (element, slot) refs of each staged row (thread-
// colour order) laid out row after row, a row never straddling a 32-lane
// window (padding positions stay 0xFFFFFFFF).  Record: element (10 bits), own
// row (10), slot (3), position in the row's run (5), run end (1).  Pass 1
// (rec == NULL) counts positions per block (rounded up to 4).
__global__ void gather_refs_kernel(int32_t nb, const int32_t* __restrict__ bo, const int32_t* __restrict__ st_off,
                                   const uint16_t* __restrict__ poff, const uint16_t* __restrict__ pref, int arity,
                                   const int32_t* __restrict__ roff, int32_t* counts, uint32_t* rec, int* bad) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int e0 = bo[b], s0 = st_off[b], ns = st_off[b + 1] - s0;
  const uint16_t* po = poff + s0 + b;
  const uint16_t* pr = pref + (int64_t)e0 * arity;
  int pos = 0;
  for (int j = 0; j < ns; ++j) {
    const int lo = po[j], len = (int)po[j + 1] - lo;
    if (len <= 0) continue;
    if (len > 32 || j > 1023) {
      atomicMin(bad, b);
      return;
    }
    if ((pos & 31) + len > 32) pos = (pos + 31) & ~31;
    if (rec) {
      for (int q = 0; q < len; ++q) {
        const int ref = pr[lo + q], e = ref / arity, sl = ref - e * arity;
        if (e > 1022) {
          atomicMin(bad, b);
          return;
        }
        rec[roff[b] + pos + q] = (uint32_t)e | (uint32_t)j << 10 | (uint32_t)sl << 20 | (uint32_t)q << 23 |
                                 (uint32_t)(q == len - 1) << 28;
      }
    }
    pos += len;
  }
  if (!rec) counts[b] = (pos + 3) & ~3;
}
}  // namespace
}  // namespace mp

using namespace mp;

extern "C" mp_status mp_plan_block_points(int32_t nb, const int32_t* block_offsets, const int32_t* map, int64_t n,
                                          int32_t arity, int32_t layout, uint32_t mask, int32_t max_block,
                                          int32_t* counts, const int32_t* offsets, int32_t* ids, void* stream) {
  clear_error();
  if (nb == 0) return MP_OK;
  int m = next_pow2(max_block * __builtin_popcount(mask) > 0 ? max_block * __builtin_popcount(mask) : 1);
  size_t smem = (size_t)m * 8;
  if (smem > 227 * 1024) MP_FAIL(MP_ERR_CAPACITY, "block of %d elements x %d slots too large to plan", max_block, arity);
  MP_CUDA_TRY(raise_smem_limit(reinterpret_cast<const void*>(block_points_kernel), smem));
  block_points_kernel<<<nb, 256, smem, as_stream(stream)>>>(nb, block_offsets, map, n, arity, layout, mask, counts,
                                                            offsets, ids);
  MP_CHECK_LAUNCH();
  return MP_OK;
}

extern "C" mp_status mp_plan_local_slots(int32_t nb, const int32_t* block_offsets, const int32_t* map, int64_t n,
                                         int32_t arity, int32_t layout, uint32_t mask, const int32_t* st_off,
                                         const int32_t* st_ids, uint16_t* local_slots, const int32_t* wr_off,
                                         const int32_t* wr_ids, uint16_t* written_slots, void* stream) {
  clear_error();
  if (nb == 0) return MP_OK;
  cudaStream_t st = as_stream(stream);
  if (arity > 32) MP_FAIL(MP_ERR_CAPACITY, "arity %d exceeds 32", arity);
  int32_t* d_miss = nullptr;
  MP_CUDA_TRY(cudaMallocAsync(&d_miss, sizeof(int32_t), st));
  int32_t big = INT_MAX;
  MP_CUDA_TRY(cudaMemcpyAsync(d_miss, &big, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  // a staged list holds at most block_size x arity <= 8192 points
  const size_t smem = 8192 * sizeof(int32_t);
  MP_CUDA_TRY(raise_smem_limit(reinterpret_cast<const void*>(local_slots_kernel), smem));
  local_slots_kernel<<<nb, 256, smem, st>>>(nb, block_offsets, map, n, arity, layout, mask, st_off, st_ids,
                                            local_slots, wr_off, wr_ids, written_slots, d_miss);
  MP_CHECK_LAUNCH();
  int32_t miss = INT_MAX;
  MP_CUDA_TRY(cudaMemcpyAsync(&miss, d_miss, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaFreeAsync(d_miss, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  if (miss != INT_MAX) MP_FAIL(MP_ERR_CAPACITY, "block %d: access to a point missing from its staging list", miss);
  return MP_OK;
}

extern "C" mp_status mp_plan_thread_colours(int32_t nb, const int32_t* block_offsets, const int32_t* map, int64_t n,
                                            int32_t arity, int32_t layout, uint32_t mask, int32_t max_block,
                                            int32_t* colours, int32_t* counts, int32_t* sorted_order, void* stream) {
  clear_error();
  if (nb == 0) return MP_OK;
  if (max_block > 1024) MP_FAIL(MP_ERR_CAPACITY, "block of %d elements exceeds 1024", max_block);
  cudaStream_t st = as_stream(stream);
  size_t smem = thread_colour_smem(max_block, __builtin_popcount(mask));
  if (smem > 227 * 1024) MP_FAIL(MP_ERR_CAPACITY, "thread colouring of %d-element blocks needs %zu shared bytes", max_block, smem);
  int32_t* d_over = nullptr;
  MP_CUDA_TRY(cudaMallocAsync(&d_over, sizeof(int32_t), st));
  int32_t big = INT_MAX;
  MP_CUDA_TRY(cudaMemcpyAsync(d_over, &big, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  MP_CUDA_TRY(raise_smem_limit(reinterpret_cast<const void*>(thread_colour_kernel), smem));
  thread_colour_kernel<<<nb, 32, smem, st>>>(nb, block_offsets, map, n, arity, layout, mask, max_block, colours, counts,
                                             sorted_order, d_over);
  MP_CHECK_LAUNCH();
  int32_t over = INT_MAX;
  MP_CUDA_TRY(cudaMemcpyAsync(&over, d_over, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaFreeAsync(d_over, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  if (over != INT_MAX) MP_FAIL(MP_ERR_CAPACITY, "block %d needs more than 256 thread colours", over);
  return MP_OK;
}

extern "C" mp_status mp_plan_row_placement(int32_t nb, const int32_t* block_offsets, const int32_t* staged_offsets,
                                          const uint16_t* local_slots, int32_t arity, const uint8_t* thread_colours,
                                          int32_t* perm, void* stream) {
  clear_error();
  if (nb == 0) return MP_OK;
  mp::row_placement_kernel<<<(nb + 127) / 128, 128, 0, as_stream(stream)>>>(nb, block_offsets, staged_offsets,
                                                                            local_slots, arity, thread_colours, perm);
  MP_CHECK_LAUNCH();
  return MP_OK;
}

extern "C" mp_status mp_plan_gather_refs(int32_t nb, const int32_t* block_offsets, const int32_t* staged_offsets,
                                        const uint16_t* pull_off, const uint16_t* pull_ref, int32_t arity,
                                        const int32_t* ref_offsets, int32_t* counts, uint32_t* refs, void* stream) {
  clear_error();
  if (nb == 0) return MP_OK;
  cudaStream_t st = as_stream(stream);
  int* d_bad = nullptr;
  MP_CUDA_TRY(cudaMallocAsync(&d_bad, sizeof(int), st));
  int big = INT_MAX;
  MP_CUDA_TRY(cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  mp::gather_refs_kernel<<<(nb + 127) / 128, 128, 0, st>>>(nb, block_offsets, staged_offsets, pull_off, pull_ref,
                                                            arity, ref_offsets, counts, refs, d_bad);
  MP_CHECK_LAUNCH();
  int bad = INT_MAX;
  MP_CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaFreeAsync(d_bad, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  if (bad != INT_MAX)
    MP_FAIL(MP_ERR_CAPACITY, "block %d: gather records need <= 32 refs per row, <= 1024 rows, <= 1023 elements", bad);
  return MP_OK;
}
