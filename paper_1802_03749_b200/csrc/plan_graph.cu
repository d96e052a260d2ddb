// Graph-wide planner and checker kernels (CUB radix sorts + custom passes):
//   * race check            (simulator.py:245-261, 446-469)
//   * block conflict DAG + topological schedule for the dataflow executor
//   * level-synchronous BFS (numpy_impl.py:114-131; levels are visit-order
//     independent, so GPS levels equal the reference's)
//   * heavy-edge matching (numpy_impl.py:134-157) in dependency rounds, equal
//     to the reference's sequential visit-order greedy
#include <cub/cub.cuh>
#include <limits.h>
#include <stdlib.h>

#include <vector>

#include "mp_common.cuh"

namespace mp {
namespace {

// RAII scratch on the stream-ordered allocator
struct Scratch {
  void* p = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes > 0 ? bytes : 1, st); }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
  template <typename T> T* as() { return static_cast<T*>(p); }
};

template <typename K>
cudaError_t sort_keys(K* keys, K* tmp_keys, int64_t n, cudaStream_t st, int end_bit = sizeof(K) * 8) {
  cub::DoubleBuffer<K> db(keys, tmp_keys);
  size_t bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, n, 0, end_bit, st);
  if (e) return e;
  Scratch tmp(st);
  if ((e = tmp.alloc(bytes))) return e;
  if ((e = cub::DeviceRadixSort::SortKeys(tmp.p, bytes, db, n, 0, end_bit, st))) return e;
  if (db.Current() != keys) e = cudaMemcpyAsync(keys, db.Current(), n * sizeof(K), cudaMemcpyDeviceToDevice, st);
  return e;
}

int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b)) ++b;
  return b;
}

// ---- race check ----------------------------------------------------------------
__global__ void race_keys_kernel(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ refs,
                                 const int64_t* __restrict__ groups, int64_t span, uint64_t* keys, int32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = groups[i];
    for (int64_t j = off[i]; j < off[i + 1]; ++j) {
      keys[j] = (uint64_t)(g * span + refs[j]);
      vals[j] = (int32_t)i;
    }
  }
}

__global__ void first_dup_kernel(int64_t m, const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals,
                                 unsigned long long* first) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j + 1 < m; j += (int64_t)gridDim.x * blockDim.x)
    if (keys[j] == keys[j + 1] && vals[j] != vals[j + 1]) atomicMin(first, (unsigned long long)j);
}

// ---- block DAG ------------------------------------------------------------------
__global__ void point_block_keys(int32_t nb, const int32_t* __restrict__ off, const int32_t* __restrict__ ids,
                                 uint64_t* keys) {
  for (int b = blockIdx.x; b < nb; b += gridDim.x)
    for (int j = off[b] + threadIdx.x; j < off[b + 1]; j += blockDim.x)
      keys[j] = ((uint64_t)(uint32_t)ids[j] << 32) | (uint32_t)b;
}

// For each segment start (new point) count the block pairs of the segment.
__global__ void seg_pair_count(int64_t m, const uint64_t* __restrict__ keys, int64_t* cnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    if (j == 0 || (keys[j] >> 32) != (keys[j - 1] >> 32)) {
      int64_t e = j + 1;
      while (e < m && (keys[e] >> 32) == (keys[j] >> 32)) ++e;
      int64_t L = e - j;
      c = L * (L - 1) / 2;
    }
    cnt[j] = c;
  }
}

__global__ void seg_pair_emit(int64_t m, const uint64_t* __restrict__ keys, const int64_t* __restrict__ pos,
                              const int32_t* __restrict__ colour, uint64_t* edges) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    if (!(j == 0 || (keys[j] >> 32) != (keys[j - 1] >> 32))) continue;
    int64_t e = j + 1;
    while (e < m && (keys[e] >> 32) == (keys[j] >> 32)) ++e;
    int64_t w = pos[j];
    for (int64_t a = j; a < e; ++a)
      for (int64_t c = a + 1; c < e; ++c) {
        uint32_t x = (uint32_t)keys[a], y = (uint32_t)keys[c];  // x < y (sorted by block)
        // edge from the lower (colour, id) block to the higher one (by id alone
        // when no colours are given)
        bool x_first = colour == nullptr || colour[x] < colour[y] || (colour[x] == colour[y] && x < y);
        uint32_t src = x_first ? x : y, dst = x_first ? y : x;
        edges[w++] = ((uint64_t)dst << 32) | src;
      }
  }
}

__global__ void pred_offsets_kernel(int32_t nb, int64_t E, const uint64_t* __restrict__ edges, int32_t* off,
                                    int32_t* preds) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nb; i += (int64_t)gridDim.x * blockDim.x) {
    // first edge with dst >= i
    int64_t lo = 0, hi = E;
    const uint64_t key = (uint64_t)i << 32;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (edges[mid] < key) lo = mid + 1; else hi = mid;
    }
    off[i] = (int32_t)lo;
  }
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < E; j += (int64_t)gridDim.x * blockDim.x)
    preds[j] = (int32_t)(uint32_t)edges[j];
}

__global__ void colour_keys_kernel(int32_t nb, const int32_t* __restrict__ colour, uint64_t* keys) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    keys[b] = ((uint64_t)(uint32_t)colour[b] << 32) | (uint32_t)b;
}

// key(b) = max(b, max over preds key(p) + 1) for the blocks of one colour
__global__ void dag_key_kernel(int32_t lo, int32_t hi, const uint64_t* __restrict__ by_colour,
                               const int32_t* __restrict__ off, const int32_t* __restrict__ preds, uint32_t* key,
                               uint32_t lag) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)by_colour[i];
    uint32_t k = b;
    for (int j = off[b]; j < off[b + 1]; ++j) {
      uint32_t q = key[preds[j]] + lag;
      k = q > k ? q : k;
    }
    key[b] = k;
  }
}

__global__ void order_keys_kernel(int32_t nb, const uint32_t* __restrict__ key, uint64_t* keys) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    keys[b] = ((uint64_t)key[b] << 32) | (uint32_t)b;
}

__global__ void low_words_kernel(int64_t n, const uint64_t* __restrict__ keys, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)(uint32_t)keys[i];
}

// ---- BFS --------------------------------------------------------------------------
__global__ void bfs_init(int32_t n, int32_t* levels, int32_t start, int32_t* frontier) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    levels[i] = (i == start) ? 0 : -1;
  if (blockIdx.x == 0 && threadIdx.x == 0) frontier[0] = start;
}

__global__ void bfs_expand(int32_t fsize, const int32_t* __restrict__ frontier, const int64_t* __restrict__ indptr,
                           const int32_t* __restrict__ indices, int32_t* levels, int32_t next_level, int32_t* next,
                           int32_t* next_size) {
  // one warp per frontier node, lanes over its neighbours
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < fsize;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t u = frontier[w];
    for (int64_t j = indptr[u] + lane; j < indptr[u + 1]; j += 32) {
      const int32_t v = indices[j];
      if (levels[v] < 0 && atomicCAS(&levels[v], -1, next_level) == -1) next[atomicAdd(next_size, 1)] = v;
    }
  }
}

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}


// ---- heavy-edge matching ------------------------------------------------------------
// The reference visits nodes in a random order; an unmatched node takes its
// heaviest available neighbour (ties: lowest id).  Node u's turn reads only
// the matched state of its neighbours, which the earlier turns of nodes within
// two hops decide.  So u can act as soon as every earlier-ranked node within
// two hops of it has been matched: all such "ready" nodes act together on the
// previous round's state (two ready nodes are more than two hops apart, so
// they never pick the same partner or each other), and the result is the
// sequential one.  The earliest unmatched node is always ready.
__global__ void hem_rank_kernel(int32_t n, const int64_t* __restrict__ visit, int32_t* rank, int32_t* work,
                                int64_t* match) {
  for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    rank[visit[s]] = s;
    work[s] = s;
    match[s] = -1;
  }
}

__global__ void hem_round_kernel(int32_t m, const int32_t* __restrict__ work, const int64_t* __restrict__ indptr,
                                 const int64_t* __restrict__ indices, const int64_t* __restrict__ weights,
                                 const int64_t* __restrict__ node_w, const int32_t* __restrict__ rank,
                                 int64_t max_cluster, const int64_t* __restrict__ match, int64_t* __restrict__ dec) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int64_t u = work[i];
    if (match[u] >= 0) {  // taken as a partner last round
      dec[i] = -3;
      continue;
    }
    const int32_t r = rank[u];
    const int64_t a = indptr[u], z = indptr[u + 1];
    bool ready = true;
    for (int64_t j = a; j < z && ready; ++j) {
      const int64_t v = indices[j];
      if (v == u || match[v] >= 0) continue;  // a matched neighbour stays unavailable
      if (rank[v] < r) {
        ready = false;
        break;
      }
      for (int64_t k = indptr[v]; k < indptr[v + 1]; ++k) {
        const int64_t x = indices[k];
        if (x != u && rank[x] < r && match[x] < 0) {
          ready = false;
          break;
        }
      }
    }
    if (!ready) {
      dec[i] = -2;
      continue;
    }
    int64_t best = u, best_w = -1;
    for (int64_t j = a; j < z; ++j) {
      const int64_t v = indices[j];
      if (match[v] >= 0 || v == u) continue;
      if (node_w[u] + node_w[v] > max_cluster) continue;
      const int64_t w = weights[j];
      if (w > best_w || (w == best_w && v < best)) {
        best = v;
        best_w = w;
      }
    }
    dec[i] = best;
  }
}

__global__ void hem_apply_kernel(int32_t m, const int32_t* __restrict__ work, const int64_t* __restrict__ dec,
                                 int64_t* match, int32_t* next, int32_t* count) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int64_t u = work[i], d = dec[i];
    if (d >= 0) {
      match[u] = d;
      if (d != u) match[d] = u;
    } else if (d == -2) {
      next[atomicAdd(count, 1)] = (int32_t)u;
    }
  }
}


// ---- sequential greedy block colouring (numpy_impl.py:12-60 over blocks) -------------
// The least-loaded choice of block i depends on the colour counts after blocks
// 0..i-1, so the pass is sequential by definition.  Its per-block work is
// short once the conflict structure is known: the colours forbidden to block i
// are exactly those of its lower-id conflict neighbours (blocks < i writing a
// common point), a CSR built in parallel by sorts beforehand.  One warp then
// walks the blocks in id order: lanes fetch neighbour colours (recent ones
// from a shared-memory ring, older ones from L2), OR them into per-lane bit
// words (lane l owns colours l, l+32, ...), and two warp min-reductions pick
// the admissible colour with the fewest blocks (ties: lowest id) -- the
// reference's choice.  The other warps stage the next chunk of the CSR into
// shared memory meanwhile (double buffer, one CTA barrier per chunk).
constexpr int GC_THREADS = 128;
constexpr int GC_CH = 2048;     // blocks per chunk (at most)
constexpr int GC_PCAP = 12288;  // neighbour entries per chunk buffer
constexpr int GC_RING = 16384;  // colours of the most recent blocks
constexpr size_t GC_SMEM = (2 * (GC_CH + 1) + 2 * GC_PCAP) * 4 + GC_RING * 2;

__device__ __forceinline__ int32_t gc_chunk_end(int32_t nb, const int32_t* __restrict__ off, int32_t lo) {
  // largest hi <= lo + GC_CH with off[hi] - off[lo] <= GC_PCAP, at least lo + 1
  int32_t hi = lo + GC_CH < nb ? lo + GC_CH : nb;
  const int32_t base = off[lo];
  if (off[hi] - base <= GC_PCAP) return hi;
  int32_t a = lo + 1, b = hi;  // off[a]-base may exceed the cap: a one-block chunk reads global
  while (a < b) {
    int32_t mid = (a + b + 1) >> 1;
    if (off[mid] - base <= GC_PCAP) a = mid; else b = mid - 1;
  }
  return a;
}

template <int K>
__global__ void __launch_bounds__(GC_THREADS, 1)
    greedy_blocks_kernel(int32_t nb, const int32_t* __restrict__ off, const int32_t* __restrict__ preds,
                         int32_t least_loaded, int32_t* colours, int32_t* result /* [0] colours, [1] overflow */) {
  extern __shared__ __align__(16) int32_t gsm[];
  int32_t* soff = gsm;                                             // 2 x (GC_CH + 1)
  int32_t* spred = soff + 2 * (GC_CH + 1);                         // 2 x GC_PCAP
  uint16_t* ring = reinterpret_cast<uint16_t*>(spred + 2 * GC_PCAP);  // GC_RING
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  auto stage = [&](int buf, int32_t lo, int32_t hi, int t0, int nt) {
    const int32_t base = off[lo];
    for (int32_t i = t0; i <= hi - lo; i += nt) soff[buf * (GC_CH + 1) + i] = off[lo + i];
    const int32_t np = off[hi] - base;
    if (np <= GC_PCAP)
      for (int32_t j = t0; j < np; j += nt) spred[buf * GC_PCAP + j] = preds[base + j];
  };

  int32_t lo = 0, hi = gc_chunk_end(nb, off, 0);
  stage(0, lo, hi, tid, GC_THREADS);
  __syncthreads();
  uint32_t cnt[K];
#pragma unroll
  for (int k = 0; k < K; ++k) cnt[k] = 0;
  uint32_t ncol = 0;
  int buf = 0;
  while (lo < nb) {
    const int32_t nlo = hi, nhi = nlo < nb ? gc_chunk_end(nb, off, nlo) : nlo;
    if (warp == 0) {
      const int32_t* so = soff + buf * (GC_CH + 1);
      const int32_t base = so[0];
      const bool glob = so[hi - lo] - base > GC_PCAP;
      const int32_t* sp = spred + buf * GC_PCAP;
      for (int32_t i = lo; i < hi; ++i) {
        const int32_t s = so[i - lo], e = so[i - lo + 1];
        uint32_t bits[K];
#pragma unroll
        for (int k = 0; k < K; ++k) bits[k] = 0;
        for (int32_t t = s + lane; t < e; t += 32) {
          const int32_t j = glob ? __ldg(preds + t) : sp[t - base];
          const uint32_t c = j > i - GC_RING ? ring[j % GC_RING] : (uint32_t)__ldcg(colours + j);
#pragma unroll
          for (int k = 0; k < K; ++k) bits[k] |= (c >> 5) == (uint32_t)k ? 1u << (c & 31) : 0u;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) bits[k] = __reduce_or_sync(0xffffffffu, bits[k]);
        uint32_t cand = 0xffffffffu;
        if (least_loaded) {
          uint32_t mc = 0xffffffffu;
#pragma unroll
          for (int k = 0; k < K; ++k)
            if ((uint32_t)(lane + 32 * k) < ncol && !(bits[k] >> lane & 1u) && cnt[k] < mc) mc = cnt[k];
          mc = __reduce_min_sync(0xffffffffu, mc);
#pragma unroll
          for (int k = K - 1; k >= 0; --k)
            if ((uint32_t)(lane + 32 * k) < ncol && !(bits[k] >> lane & 1u) && cnt[k] == mc) cand = lane + 32 * k;
        } else {
#pragma unroll
          for (int k = K - 1; k >= 0; --k)
            if ((uint32_t)(lane + 32 * k) < ncol && !(bits[k] >> lane & 1u)) cand = lane + 32 * k;
        }
        uint32_t best = __reduce_min_sync(0xffffffffu, cand);
        if (best == 0xffffffffu) {
          best = ncol++;
          if (ncol > 32u * K) {  // every lane sees it: leave together
            if (lane == 0) result[1] = 1;
            break;
          }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) cnt[k] += (best == (uint32_t)(lane + 32 * k)) ? 1u : 0u;
        if (lane == 0) {
          ring[i % GC_RING] = (uint16_t)best;
          colours[i] = (int32_t)best;
        }
        __syncwarp();
      }
    } else if (nlo < nb) {
      stage(buf ^ 1, nlo, nhi, tid - 32, GC_THREADS - 32);
    }
    __syncthreads();
    if (*(volatile int32_t*)&result[1]) return;
    lo = nlo;
    hi = nhi;
    buf ^= 1;
  }
  if (tid == 0) result[0] = (int32_t)ncol;
}
}  // namespace
}  // namespace mp

using namespace mp;

extern "C" mp_status mp_race_check(int64_t n, const int64_t* ref_offsets, const int32_t* refs, const int64_t* groups,
                                   int64_t key_span, int64_t* first_pair, void* stream) {
  clear_error();
  first_pair[0] = first_pair[1] = -1;
  if (n == 0) return MP_OK;
  cudaStream_t st = as_stream(stream);
  int64_t m = 0;
  MP_CUDA_TRY(cudaMemcpyAsync(&m, ref_offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  if (m < 2) return MP_OK;
  Scratch keys(st), keys2(st), vals(st), vals2(st), tmp(st), first(st);
  MP_CUDA_TRY(keys.alloc(m * 8));
  MP_CUDA_TRY(keys2.alloc(m * 8));
  MP_CUDA_TRY(vals.alloc(m * 4));
  MP_CUDA_TRY(vals2.alloc(m * 4));
  MP_CUDA_TRY(first.alloc(8));
  race_keys_kernel<<<grid_for(n), 256, 0, st>>>(n, ref_offsets, refs, groups, key_span, keys.as<uint64_t>(),
                                                 vals.as<int32_t>());
  MP_CHECK_LAUNCH();
  cub::DoubleBuffer<uint64_t> dk(keys.as<uint64_t>(), keys2.as<uint64_t>());
  cub::DoubleBuffer<int32_t> dv(vals.as<int32_t>(), vals2.as<int32_t>());
  size_t bytes = 0;
  MP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, m, 0, 64, st));
  MP_CUDA_TRY(tmp.alloc(bytes));
  MP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, m, 0, 64, st));
  unsigned long long none = ~0ull;
  MP_CUDA_TRY(cudaMemcpyAsync(first.p, &none, 8, cudaMemcpyHostToDevice, st));
  first_dup_kernel<<<grid_for(m), 256, 0, st>>>(m, dk.Current(), dv.Current(), first.as<unsigned long long>());
  MP_CHECK_LAUNCH();
  unsigned long long j = none;
  MP_CUDA_TRY(cudaMemcpyAsync(&j, first.p, 8, cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  if (j != none) {
    int32_t pair[2];
    MP_CUDA_TRY(cudaMemcpyAsync(pair, dv.Current() + j, 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaStreamSynchronize(st));
    first_pair[0] = pair[0];
    first_pair[1] = pair[1];
  }
  return MP_OK;
}

// Unique conflict edges (dst << 32 | src) between blocks writing a common point,
// sorted: src is the lower (colour, id) block, or the lower id when colour is
// null.  `uniq` receives U edges.
static mp_status block_conflict_edges(int32_t nb, const int32_t* written_offsets, const int32_t* written_ids,
                                      const int32_t* block_colours, cudaStream_t st, Scratch& uniq, int64_t* num) {
  *num = 0;
  int32_t m32 = 0;
  MP_CUDA_TRY(cudaMemcpyAsync(&m32, written_offsets + nb, 4, cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t m = m32;
  Scratch keys(st), keys2(st), cnt(st), pos(st), tmp(st);
  MP_CUDA_TRY(keys.alloc(m * 8));
  MP_CUDA_TRY(keys2.alloc(m * 8));
  point_block_keys<<<grid_for(nb, 1), 128, 0, st>>>(nb, written_offsets, written_ids, keys.as<uint64_t>());
  MP_CHECK_LAUNCH();
  MP_CUDA_TRY(sort_keys(keys.as<uint64_t>(), keys2.as<uint64_t>(), m, st));
  MP_CUDA_TRY(cnt.alloc((m + 1) * 8));
  MP_CUDA_TRY(pos.alloc((m + 1) * 8));
  seg_pair_count<<<grid_for(m), 256, 0, st>>>(m, keys.as<uint64_t>(), cnt.as<int64_t>());
  MP_CHECK_LAUNCH();
  MP_CUDA_TRY(cudaMemsetAsync(cnt.as<int64_t>() + m, 0, 8, st));
  size_t bytes = 0;
  MP_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.as<int64_t>(), pos.as<int64_t>(), m + 1, st));
  MP_CUDA_TRY(tmp.alloc(bytes));
  MP_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.as<int64_t>(), pos.as<int64_t>(), m + 1, st));
  int64_t E = 0;
  MP_CUDA_TRY(cudaMemcpyAsync(&E, pos.as<int64_t>() + m, 8, cudaMemcpyDeviceToHost, st));
  MP_CUDA_TRY(cudaStreamSynchronize(st));

  Scratch edges(st), edges2(st), nuniq(st), tmp2(st);
  MP_CUDA_TRY(edges.alloc(E * 8));
  MP_CUDA_TRY(edges2.alloc(E * 8));
  if (E > 0) {
    seg_pair_emit<<<grid_for(m), 256, 0, st>>>(m, keys.as<uint64_t>(), pos.as<int64_t>(), block_colours,
                                                edges.as<uint64_t>());
    MP_CHECK_LAUNCH();
    MP_CUDA_TRY(sort_keys(edges.as<uint64_t>(), edges2.as<uint64_t>(), E, st));
  }
  MP_CUDA_TRY(uniq.alloc(E * 8));
  MP_CUDA_TRY(nuniq.alloc(8));
  int64_t U = 0;
  if (E > 0) {
    bytes = 0;
    MP_CUDA_TRY(cub::DeviceSelect::Unique(nullptr, bytes, edges.as<uint64_t>(), uniq.as<uint64_t>(),
                                          nuniq.as<int64_t>(), E, st));
    MP_CUDA_TRY(tmp2.alloc(bytes));
    MP_CUDA_TRY(cub::DeviceSelect::Unique(tmp2.p, bytes, edges.as<uint64_t>(), uniq.as<uint64_t>(),
                                          nuniq.as<int64_t>(), E, st));
    MP_CUDA_TRY(cudaMemcpyAsync(&U, nuniq.p, 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaStreamSynchronize(st));
  }
  *num = U;
  return MP_OK;
}

extern "C" mp_status mp_plan_block_dag(int32_t nb, const int32_t* written_offsets, const int32_t* written_ids,
                                       int64_t n_points, const int32_t* block_colours, int32_t num_colours, int32_t lag,
                                       int32_t* pred_offsets, int32_t* preds, int64_t preds_capacity,
                                       int64_t* num_preds, int32_t* order, void* stream) {
  clear_error();
  *num_preds = 0;
  if (nb == 0) return MP_OK;
  cudaStream_t st = as_stream(stream);
  Scratch uniq(st);
  int64_t U = 0;
  {
    mp_status rc = block_conflict_edges(nb, written_offsets, written_ids, block_colours, st, uniq, &U);
    if (rc != MP_OK) return rc;
  }
  *num_preds = U;
  if (U > preds_capacity) return MP_OK;  // caller grows the buffer and calls again
  pred_offsets_kernel<<<grid_for(nb + 1 > U ? nb + 1 : U), 256, 0, st>>>(nb, U, uniq.as<uint64_t>(), pred_offsets,
                                                                          preds);
  MP_CHECK_LAUNCH();

  // blocks grouped by colour, then keys colour by colour
  Scratch ck(st), ck2(st), key(st);
  MP_CUDA_TRY(ck.alloc(nb * 8));
  MP_CUDA_TRY(ck2.alloc(nb * 8));
  MP_CUDA_TRY(key.alloc(nb * 4));
  colour_keys_kernel<<<grid_for(nb), 256, 0, st>>>(nb, block_colours, ck.as<uint64_t>());
  MP_CHECK_LAUNCH();
  MP_CUDA_TRY(sort_keys(ck.as<uint64_t>(), ck2.as<uint64_t>(), nb, st));
  // host copy of colour boundaries
  uint64_t* hk = (uint64_t*)malloc(nb * 8);
  if (!hk) MP_FAIL(MP_ERR_CUDA, "host allocation failed");
  cudaError_t ce = cudaMemcpyAsync(hk, ck.p, nb * 8, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) {
    free(hk);
    MP_CUDA_TRY(ce);
  }
  int32_t lo = 0;
  while (lo < nb) {
    uint32_t c = (uint32_t)(hk[lo] >> 32);
    int32_t hi = lo;
    while (hi < nb && (uint32_t)(hk[hi] >> 32) == c) ++hi;
    dag_key_kernel<<<grid_for(hi - lo), 256, 0, st>>>(lo, hi, ck.as<uint64_t>(), pred_offsets, preds,
                                                     key.as<uint32_t>(), (uint32_t)(lag > 0 ? lag : 1));
    ce = cudaGetLastError();
    if (ce != cudaSuccess) break;
    lo = hi;
  }
  free(hk);
  MP_CUDA_TRY(ce);
  order_keys_kernel<<<grid_for(nb), 256, 0, st>>>(nb, key.as<uint32_t>(), ck.as<uint64_t>());
  MP_CHECK_LAUNCH();
  MP_CUDA_TRY(sort_keys(ck.as<uint64_t>(), ck2.as<uint64_t>(), nb, st));
  low_words_kernel<<<grid_for(nb), 256, 0, st>>>(nb, ck.as<uint64_t>(), order);
  MP_CHECK_LAUNCH();
  MP_CUDA_TRY(cudaStreamSynchronize(st));
  (void)n_points;
  (void)num_colours;
  return MP_OK;
}

extern "C" mp_status mp_plan_block_colours(int32_t nb, const int32_t* written_offsets, const int32_t* written_ids,
                                           int32_t least_loaded, int32_t* colours, int32_t* num_colours,
                                           void* stream) {
  clear_error();
  *num_colours = 0;
  if (nb <= 0) return MP_OK;
  cudaStream_t st = as_stream(stream);
  Scratch uniq(st), poff(st), preds(st), res(st);
  int64_t U = 0;
  {
    mp_status rc = block_conflict_edges(nb, written_offsets, written_ids, nullptr, st, uniq, &U);
    if (rc != MP_OK) return rc;
  }
  if (U > INT32_MAX) MP_FAIL(MP_ERR_CAPACITY, "%lld block conflicts exceed the int32 CSR", (long long)U);
  MP_CUDA_TRY(poff.alloc((size_t)(nb + 1) * 4));
  MP_CUDA_TRY(preds.alloc((size_t)U * 4));
  pred_offsets_kernel<<<grid_for(nb + 1 > U ? nb + 1 : U), 256, 0, st>>>(nb, U, uniq.as<uint64_t>(),
                                                                          poff.as<int32_t>(), preds.as<int32_t>());
  MP_CHECK_LAUNCH();
  MP_CUDA_TRY(res.alloc(8));
  int32_t h[2] = {0, 0};
  for (int pass = 0; pass < 2; ++pass) {
    MP_CUDA_TRY(cudaMemsetAsync(res.p, 0, 8, st));
    if (pass == 0) {  // up to 64 colours
      MP_CUDA_TRY(raise_smem_limit((const void*)greedy_blocks_kernel<2>, GC_SMEM));
      greedy_blocks_kernel<2><<<1, GC_THREADS, GC_SMEM, st>>>(nb, poff.as<int32_t>(), preds.as<int32_t>(),
                                                              least_loaded, colours, res.as<int32_t>());
    } else {  // up to 1024
      MP_CUDA_TRY(raise_smem_limit((const void*)greedy_blocks_kernel<32>, GC_SMEM));
      greedy_blocks_kernel<32><<<1, GC_THREADS, GC_SMEM, st>>>(nb, poff.as<int32_t>(), preds.as<int32_t>(),
                                                               least_loaded, colours, res.as<int32_t>());
    }
    MP_CHECK_LAUNCH();
    MP_CUDA_TRY(cudaMemcpyAsync(h, res.p, 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaStreamSynchronize(st));
    if (!h[1]) break;
  }
  if (h[1]) MP_FAIL(MP_ERR_CAPACITY, "block colouring needs more than 1024 colours");
  *num_colours = h[0];
  return MP_OK;
}

extern "C" mp_status mp_bfs_levels(int32_t n, const int64_t* indptr, const int32_t* indices, int32_t start,
                                   int32_t* levels, int32_t* ecc, int32_t* visited, void* stream) {
  clear_error();
  *ecc = 0;
  *visited = 0;
  if (n == 0) return MP_OK;
  if (start < 0 || start >= n) MP_FAIL(MP_ERR_VALIDATION, "bfs start %d out of range", start);
  cudaStream_t st = as_stream(stream);
  Scratch fa(st), fb(st), cnt(st);
  MP_CUDA_TRY(fa.alloc((size_t)n * 4));
  MP_CUDA_TRY(fb.alloc((size_t)n * 4));
  MP_CUDA_TRY(cnt.alloc(4));
  int32_t* pinned = nullptr;
  MP_CUDA_TRY(cudaMallocHost(&pinned, 4));
  bfs_init<<<grid_for(n), 256, 0, st>>>(n, levels, start, fa.as<int32_t>());
  cudaError_t ce = cudaGetLastError();
  int32_t fsize = 1, total = 1, level = 0;
  int32_t *cur = fa.as<int32_t>(), *nxt = fb.as<int32_t>();
  while (ce == cudaSuccess && fsize > 0) {
    ce = cudaMemsetAsync(cnt.p, 0, 4, st);
    if (ce) break;
    int64_t threads = (int64_t)fsize * 32;
    int grid = (int)((threads + 255) / 256 < 148 * 16 ? (threads + 255) / 256 : 148 * 16);
    bfs_expand<<<grid, 256, 0, st>>>(fsize, cur, indptr, indices, levels, level + 1, nxt, cnt.as<int32_t>());
    if ((ce = cudaGetLastError())) break;
    if ((ce = cudaMemcpyAsync(pinned, cnt.p, 4, cudaMemcpyDeviceToHost, st))) break;
    if ((ce = cudaStreamSynchronize(st))) break;
    fsize = *pinned;
    if (fsize > 0) {
      ++level;
      total += fsize;
      int32_t* t = cur;
      cur = nxt;
      nxt = t;
    }
  }
  cudaFreeHost(pinned);
  MP_CUDA_TRY(ce);
  *ecc = level;
  *visited = total;
  return MP_OK;
}

static int32_t hem_round_cap() {
  const char* e = getenv("MESHPLAN_MATCH_ROUNDS");  // test hook: force the host finish
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : 4096;
}

extern "C" mp_status mp_heavy_edge_matching_device(int32_t n, const int64_t* indptr, const int64_t* indices,
                                                   const int64_t* weights, const int64_t* node_w,
                                                   const int64_t* visit, int64_t max_cluster, int64_t* match,
                                                   int32_t* rounds, void* stream) {
  clear_error();
  *rounds = 0;
  if (n < 0) MP_FAIL(MP_ERR_VALIDATION, "negative node count");
  if (n == 0) return MP_OK;
  cudaStream_t st = as_stream(stream);
  Scratch rk(st), wa(st), wb(st), dec(st), cnt(st);
  MP_CUDA_TRY(rk.alloc((size_t)n * 4));
  MP_CUDA_TRY(wa.alloc((size_t)n * 4));
  MP_CUDA_TRY(wb.alloc((size_t)n * 4));
  MP_CUDA_TRY(dec.alloc((size_t)n * 8));
  MP_CUDA_TRY(cnt.alloc(4));
  int32_t* pinned = nullptr;
  MP_CUDA_TRY(cudaMallocHost(&pinned, 4));
  hem_rank_kernel<<<grid_for(n), 256, 0, st>>>(n, visit, rk.as<int32_t>(), wa.as<int32_t>(), match);
  cudaError_t ce = cudaGetLastError();
  int32_t m = n, r = 0;
  int32_t *cur = wa.as<int32_t>(), *nxt = wb.as<int32_t>();
  const int32_t cap = hem_round_cap();
  while (ce == cudaSuccess && m > 0 && r < cap) {
    if ((ce = cudaMemsetAsync(cnt.p, 0, 4, st))) break;
    hem_round_kernel<<<grid_for(m), 256, 0, st>>>(m, cur, indptr, indices, weights, node_w, rk.as<int32_t>(),
                                                  max_cluster, match, dec.as<int64_t>());
    hem_apply_kernel<<<grid_for(m), 256, 0, st>>>(m, cur, dec.as<int64_t>(), match, nxt, cnt.as<int32_t>());
    if ((ce = cudaGetLastError())) break;
    if ((ce = cudaMemcpyAsync(pinned, cnt.p, 4, cudaMemcpyDeviceToHost, st))) break;
    if ((ce = cudaStreamSynchronize(st))) break;
    m = *pinned;
    ++r;
    std::swap(cur, nxt);
  }
  cudaFreeHost(pinned);
  MP_CUDA_TRY(ce);
  *rounds = r;
  if (m > 0) {
    // A dependency chain longer than the round cap (adversarial visit orders;
    // random ones need O(log n) rounds): finish sequentially on the host.  The
    // decided nodes are the sequential outcomes and no decided node lies within
    // two hops of an undecided one with a lower rank, so the remaining turns in
    // visit order see exactly the sequential state.
    std::vector<int64_t> ip(n + 1), w_match(n), vis(n), nw(n);
    MP_CUDA_TRY(cudaMemcpyAsync(ip.data(), indptr, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaMemcpyAsync(w_match.data(), match, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaMemcpyAsync(vis.data(), visit, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaMemcpyAsync(nw.data(), node_w, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    MP_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<int64_t> ix(ip[n]), ew(ip[n]);
    MP_CUDA_TRY(cudaMemcpy(ix.data(), indices, ip[n] * 8, cudaMemcpyDeviceToHost));
    MP_CUDA_TRY(cudaMemcpy(ew.data(), weights, ip[n] * 8, cudaMemcpyDeviceToHost));
    for (int32_t step = 0; step < n; ++step) {
      const int64_t u = vis[step];
      if (w_match[u] >= 0) continue;
      int64_t best = u, best_w = -1;
      for (int64_t j = ip[u]; j < ip[u + 1]; ++j) {
        const int64_t v = ix[j];
        if (w_match[v] >= 0 || v == u) continue;
        if (nw[u] + nw[v] > max_cluster) continue;
        if (ew[j] > best_w || (ew[j] == best_w && v < best)) {
          best = v;
          best_w = ew[j];
        }
      }
      w_match[u] = best;
      if (best != u) w_match[best] = u;
    }
    MP_CUDA_TRY(cudaMemcpyAsync(match, w_match.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
    MP_CUDA_TRY(cudaStreamSynchronize(st));
    *rounds = -r;  // negative: finished on the host after r rounds
  }
  return MP_OK;
}
