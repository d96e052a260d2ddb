// Sequential planner kernels that the reference defines by a strictly
// sequential greedy order, in native host C++.
//
// These are the Seam A (_accel) functions whose result depends on the
// global processing order (least-loaded colour choice over all earlier
// items, smallest-last argmin chains, in-place refinement sweeps).  They are
// restated loop for loop from the reference semantics
// (pkg/src/meshplan/_accel/numpy_impl.py) and are bit-identical to it; the
// parallel-friendly planner steps run on the GPU (plan_*.cu).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <set>
#include <thread>
#include <utility>
#include <vector>
#include <cstdint>
#include <climits>

#include "../../include/meshplan_b200.h"

namespace mp {
void set_error(const char* fmt, ...);
void clear_error();
}  // namespace mp

// numpy_impl.py:12-60 -- items in index order, per-point colour lists,
// least-loaded (strict <, lowest colour on ties) or first-fit choice.
extern "C" mp_status mp_greedy_colour_csr(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t n_points,
                                          int32_t least_loaded, int64_t* colours) {
  mp::clear_error();
  if (n < 0 || n_points < 0) {
    mp::set_error("negative size");
    return MP_ERR_VALIDATION;
  }
  if (n == 0) return MP_OK;
  const int64_t nref = indptr[n];
  // per-point slots for the colours of its writers, filled in item order
  std::vector<int64_t> start(n_points + 1, 0);
  for (int64_t j = 0; j < nref; ++j) {
    int64_t p = indices[j];
    if (p < 0 || p >= n_points) {
      mp::set_error("point %lld out of range 0..%lld", (long long)p, (long long)n_points - 1);
      return MP_ERR_VALIDATION;
    }
    start[p + 1]++;
  }
  for (int64_t p = 0; p < n_points; ++p) start[p + 1] += start[p];
  std::vector<int32_t> fill(n_points, 0);
  std::vector<int32_t> pcol(nref > 0 ? nref : 1);
  std::vector<int64_t> stamp;  // stamp[c] == i  <=> colour c forbidden for item i
  std::vector<int64_t> count;
  int64_t ncol = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = indptr[i], z = indptr[i + 1];
    for (int64_t j = a; j < z; ++j) {
      const int64_t p = indices[j];
      const int32_t* lst = pcol.data() + start[p];
      for (int32_t t = 0; t < fill[p]; ++t) stamp[lst[t]] = i;
    }
    int64_t best = -1;
    if (least_loaded) {
      int64_t best_count = std::numeric_limits<int64_t>::max();
      for (int64_t c = 0; c < ncol; ++c)
        if (stamp[c] != i && count[c] < best_count) {
          best = c;
          best_count = count[c];
        }
    } else {
      for (int64_t c = 0; c < ncol; ++c)
        if (stamp[c] != i) {
          best = c;
          break;
        }
    }
    if (best < 0) {
      best = ncol++;
      stamp.push_back(-1);
      count.push_back(0);
    }
    colours[i] = best;
    count[best]++;
    for (int64_t j = a; j < z; ++j) {
      const int64_t p = indices[j];
      pcol[start[p] + fill[p]] = (int32_t)best;
      fill[p]++;
    }
  }
  return MP_OK;
}

// numpy_impl.py:62-92 -- greedy over an adjacency CSR in a given order.
extern "C" mp_status mp_greedy_colour_adj(int64_t n, const int64_t* indptr, const int64_t* indices,
                                          const int64_t* order, int32_t least_loaded, int64_t* colours) {
  mp::clear_error();
  for (int64_t u = 0; u < n; ++u) colours[u] = -1;
  std::vector<int64_t> stamp, count;
  int64_t ncol = 0;
  for (int64_t step = 0; step < n; ++step) {
    const int64_t u = order[step];
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t c = colours[indices[j]];
      if (c >= 0) stamp[c] = u;
    }
    int64_t best = -1;
    if (least_loaded) {
      int64_t best_count = std::numeric_limits<int64_t>::max();
      for (int64_t c = 0; c < ncol; ++c)
        if (stamp[c] != u && count[c] < best_count) {
          best = c;
          best_count = count[c];
        }
    } else {
      for (int64_t c = 0; c < ncol; ++c)
        if (stamp[c] != u) {
          best = c;
          break;
        }
    }
    if (best < 0) {
      best = ncol++;
      stamp.push_back(-1);
      count.push_back(0);
    }
    colours[u] = best;
    count[best]++;
  }
  return MP_OK;
}

// numpy_impl.py:95-111 -- repeatedly remove the minimum (remaining degree,
// index) node and place it last.  An ordered set gives the same argmin as
// the reference's key = deg*(n+1)+u scan.
extern "C" mp_status mp_smallest_last_order(int64_t n, const int64_t* indptr, const int64_t* indices,
                                            int64_t* order) {
  mp::clear_error();
  std::vector<int64_t> deg(n);
  std::vector<char> removed(n, 0);
  std::set<std::pair<int64_t, int64_t>> live;
  for (int64_t u = 0; u < n; ++u) {
    deg[u] = indptr[u + 1] - indptr[u];
    live.insert({deg[u], u});
  }
  for (int64_t pos = n - 1; pos >= 0; --pos) {
    auto it = live.begin();
    const int64_t u = it->second;
    live.erase(it);
    removed[u] = 1;
    order[pos] = u;
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t v = indices[j];
      if (removed[v]) continue;
      live.erase({deg[v], v});
      deg[v]--;
      live.insert({deg[v], v});
    }
  }
  return MP_OK;
}

// ---- multilevel k-way partitioner pieces (partition.py:173-350) -------------------------

// numpy_impl.py:134-157 -- greedy heavy-edge matching in a given visit order.
extern "C" mp_status mp_heavy_edge_matching(int64_t n, const int64_t* indptr, const int64_t* indices,
                                            const int64_t* weights, const int64_t* node_w, const int64_t* visit,
                                            int64_t max_cluster, int64_t* match) {
  mp::clear_error();
  for (int64_t u = 0; u < n; ++u) match[u] = -1;
  for (int64_t step = 0; step < n; ++step) {
    const int64_t u = visit[step];
    if (match[u] >= 0) continue;
    int64_t best = u, best_w = -1;
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t v = indices[j];
      if (match[v] >= 0 || v == u) continue;
      if (node_w[u] + node_w[v] > max_cluster) continue;
      const int64_t w = weights[j];
      if (w > best_w || (w == best_w && v < best)) {
        best = v;
        best_w = w;
      }
    }
    match[u] = best;
    if (best != u) match[best] = u;
  }
  return MP_OK;
}

// numpy_impl.py:197-206
extern "C" mp_status mp_cut_weight(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                                   const int64_t* assignment, int32_t use_w, int64_t* cut) {
  mp::clear_error();
  int64_t c = 0;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t v = indices[j];
      if (u < v && assignment[u] != assignment[v]) c += use_w ? weights[j] : 1;
    }
  *cut = c;
  return MP_OK;
}

// numpy_impl.py:160-194 -- one in-place boundary refinement sweep.
extern "C" mp_status mp_refine_boundary_pass(int64_t n, const int64_t* indptr, const int64_t* indices,
                                             const int64_t* weights, int64_t* assignment, int64_t* block_w,
                                             int64_t num_blocks, const int64_t* node_w, int64_t cap, int32_t use_w,
                                             int64_t* moves_out) {
  mp::clear_error();
  std::vector<int64_t> conn(num_blocks, 0), touched(num_blocks);
  int64_t moves = 0;
  for (int64_t u = 0; u < n; ++u) {
    const int64_t own = assignment[u];
    int64_t nt = 0;
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t b = assignment[indices[j]];
      if (conn[b] == 0) touched[nt++] = b;
      conn[b] += use_w ? weights[j] : 1;
    }
    int64_t best = own, best_gain = 0;
    for (int64_t k = 0; k < nt; ++k) {
      const int64_t b = touched[k];
      if (b == own) continue;
      const int64_t gain = conn[b] - conn[own];
      if (gain > best_gain || (gain == best_gain && best != own && b < best)) {
        if (block_w[b] + node_w[u] <= cap && block_w[own] - node_w[u] > 0) {
          best = b;
          best_gain = gain;
        }
      }
    }
    if (best != own) {
      assignment[u] = best;
      block_w[own] -= node_w[u];
      block_w[best] += node_w[u];
      ++moves;
    }
    for (int64_t k = 0; k < nt; ++k) conn[touched[k]] = 0;
  }
  *moves_out = moves;
  return MP_OK;
}

// partition.py:326-337 -- up to `max_passes` boundary sweeps (stopping after a
// sweep with no move), the same decisions as repeated mp_refine_boundary_pass
// calls but with every sweep after the first visiting only the nodes whose
// decision can differ.  A node can move only if some neighbouring block beats
// its own block's connectivity (a positive-gain candidate); whether it has one
// depends only on its neighbours' blocks.  So a node that last saw no such
// candidate keeps that outcome until a neighbour moves, and a node that had
// one but was blocked by the weight cap is re-checked every sweep.  Visited in
// ascending order (the reference's order) with the flags maintained as moves
// happen: a move flags the mover and all its neighbours for the next sweep,
// and its later-ordered neighbours for the current one.  For large graphs the
// first sweep's flags come from a multi-threaded scan of the starting state.
extern "C" mp_status mp_refine_boundary(int64_t n, const int64_t* indptr, const int64_t* indices,
                                        const int64_t* weights, int64_t* assignment, int64_t* block_w,
                                        int64_t num_blocks, const int64_t* node_w, int64_t cap, int32_t use_w,
                                        int32_t max_passes, int64_t* moves_out) {
  mp::clear_error();
  const int64_t nbk = num_blocks > 0 ? num_blocks : 1, nwords = (n + 63) / 64;
  std::vector<int64_t> conn(nbk, 0), touched(nbk);
  // flag bitsets: a sweep clears the bits it visits, so both are all-zero
  // again when it ends and need no O(n) reset
  std::vector<uint64_t> cur(nwords, ~0ull), nxt(nwords, 0);
  if (n % 64) cur[nwords - 1] = (1ull << (n % 64)) - 1;
  // Positive-gain test for the first sweep's flags (multi-threaded, each
  // thread owning whole words of the bitset).
  auto positive_at = [&](int64_t u, int64_t* c, int64_t* tch) {
    const int64_t own = assignment[u];
    int64_t nt = 0;
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t b = assignment[indices[j]];
      if (c[b] == 0) tch[nt++] = b;
      c[b] += use_w ? weights[j] : 1;
    }
    bool positive = false;
    for (int64_t k = 0; k < nt; ++k) positive |= tch[k] != own && c[tch[k]] > c[own];
    for (int64_t k = 0; k < nt; ++k) c[tch[k]] = 0;
    return positive;
  };
  if (n >= (1 << 16) && max_passes > 0) {
    const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t)
      pool.emplace_back([&, t]() {
        std::vector<int64_t> c(nbk, 0), tch(nbk);
        for (int64_t wi = nwords * t / nth; wi < nwords * (t + 1) / nth; ++wi) {
          uint64_t bits = 0;
          for (int64_t u = wi * 64; u < std::min(n, wi * 64 + 64); ++u)
            if (positive_at(u, c.data(), tch.data())) bits |= 1ull << (u - wi * 64);
          cur[wi] = bits;
        }
      });
    for (auto& th : pool) th.join();
  }
  int64_t total = 0;
  for (int pass = 0; pass < max_passes; ++pass) {
    int64_t moves = 0;
    for (int64_t wi = 0; wi < nwords; ++wi) {
      while (uint64_t bits = cur[wi]) {  // re-read: a move may flag later nodes of this word
        cur[wi] = bits & (bits - 1);
        const int64_t u = wi * 64 + __builtin_ctzll(bits);
        const int64_t own = assignment[u];
        int64_t nt = 0;
        for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
          const int64_t b = assignment[indices[j]];
          if (conn[b] == 0) touched[nt++] = b;
          conn[b] += use_w ? weights[j] : 1;
        }
        int64_t best = own, best_gain = 0;
        bool positive = false;
        for (int64_t k = 0; k < nt; ++k) {
          const int64_t b = touched[k];
          if (b == own) continue;
          const int64_t gain = conn[b] - conn[own];
          positive |= gain > 0;
          if (gain > best_gain || (gain == best_gain && best != own && b < best)) {
            if (block_w[b] + node_w[u] <= cap && block_w[own] - node_w[u] > 0) {
              best = b;
              best_gain = gain;
            }
          }
        }
        for (int64_t k = 0; k < nt; ++k) conn[touched[k]] = 0;
        if (best != own) {
          assignment[u] = best;
          block_w[own] -= node_w[u];
          block_w[best] += node_w[u];
          ++moves;
          nxt[u >> 6] |= 1ull << (u & 63);
          for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
            const int64_t v = indices[j];
            nxt[v >> 6] |= 1ull << (v & 63);
            if (v > u) cur[v >> 6] |= 1ull << (v & 63);
          }
        } else if (positive) {
          nxt[u >> 6] |= 1ull << (u & 63);
        }
      }
    }
    total += moves;
    cur.swap(nxt);
    if (moves == 0) break;
  }
  *moves_out = total;
  return MP_OK;
}

// partition.py:255-285 -- push members out of over-cap blocks (best effort).
//
// Same decisions as the reference, in O(n + moves * (degree + log nb)):
// * blocks never become over-cap (a destination must have room), so the
//   over-cap set only shrinks and its lowest id never decreases, and an
//   over-cap block never gains members: its member list is the initial one
//   (ascending, like np.flatnonzero) minus the nodes already moved out;
// * a candidate's connectivity is 0 unless it is a neighbouring block, so the
//   reference's lexsort((id, -conn)) picks the best-connected neighbouring
//   block with room (ties: lowest id) or, when none has room, the lowest-id
//   block with room -- found with a min segment tree over block weights.
extern "C" mp_status mp_rebalance(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                                  int64_t* assignment, int64_t* block_w, int64_t num_blocks, const int64_t* node_w,
                                  int64_t cap, int32_t use_w) {
  mp::clear_error();
  if (num_blocks <= 0) return MP_OK;
  // members per block (counting sort: ascending node ids)
  std::vector<int64_t> moff(num_blocks + 1, 0), mem(n);
  for (int64_t u = 0; u < n; ++u) ++moff[assignment[u] + 1];
  for (int64_t k = 0; k < num_blocks; ++k) moff[k + 1] += moff[k];
  {
    std::vector<int64_t> pos(moff.begin(), moff.end() - 1);
    for (int64_t u = 0; u < n; ++u) mem[pos[assignment[u]]++] = u;
  }
  // min segment tree over block weights
  int64_t size = 1;
  while (size < num_blocks) size <<= 1;
  const int64_t INF = INT64_MAX;
  std::vector<int64_t> tree(2 * size, INF);
  for (int64_t k = 0; k < num_blocks; ++k) tree[size + k] = block_w[k];
  for (int64_t i = size - 1; i >= 1; --i) tree[i] = std::min(tree[2 * i], tree[2 * i + 1]);
  auto update = [&](int64_t k) {
    int64_t i = size + k;
    tree[i] = block_w[k];
    for (i >>= 1; i >= 1; i >>= 1) tree[i] = std::min(tree[2 * i], tree[2 * i + 1]);
  };
  auto first_at_most = [&](int64_t limit) -> int64_t {  // lowest k with block_w[k] <= limit
    if (tree[1] > limit) return -1;
    int64_t i = 1;
    while (i < size) i = tree[2 * i] <= limit ? 2 * i : 2 * i + 1;
    return i - size < num_blocks ? i - size : -1;
  };
  std::vector<int64_t> conn(num_blocks, 0), touched;
  int64_t guard = 0, scan = 0;
  while (true) {
    while (scan < num_blocks && block_w[scan] <= cap) ++scan;
    if (scan >= num_blocks || guard > n * 4) break;
    ++guard;
    const int64_t b = scan;
    bool moved = false;
    for (int64_t m = moff[b]; m < moff[b + 1]; ++m) {
      const int64_t u = mem[m];
      if (assignment[u] != b) continue;  // moved out in an earlier pass over b
      if (block_w[b] <= cap) break;
      touched.clear();
      for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
        const int64_t c = assignment[indices[j]];
        if (conn[c] == 0) touched.push_back(c);
        conn[c] += use_w ? weights[j] : 1;
      }
      int64_t best = -1;
      for (int64_t c : touched) {
        if (c == b || block_w[c] + node_w[u] > cap) continue;
        if (best < 0 || conn[c] > conn[best] || (conn[c] == conn[best] && c < best)) best = c;
      }
      for (int64_t c : touched) conn[c] = 0;
      if (best < 0) best = first_at_most(cap - node_w[u]);  // lightest-id block with room (b is over cap)
      if (best < 0) continue;
      assignment[u] = best;
      block_w[b] -= node_w[u];
      block_w[best] += node_w[u];
      update(b);
      update(best);
      moved = true;
    }
    if (!moved) break;
  }
  return MP_OK;
}

namespace {
// partition.py:198-236 -- region-growing bisection of `subset` (ascending).
void grow_bisection(const int64_t* indptr, const int64_t* indices, const int64_t* node_w,
                    const std::vector<int64_t>& subset, int64_t k1, int64_t k2, int64_t cap, std::vector<char>& in_sub,
                    std::vector<char>& taken, std::vector<int64_t>& left, std::vector<int64_t>& right) {
  int64_t total = 0;
  for (int64_t u : subset) total += node_w[u];
  const int64_t lower = std::max<int64_t>(0, total - k2 * cap);
  const int64_t upper = std::min<int64_t>(k1 * cap, total);
  // Python: int(round(total * k1 / (k1 + k2))) -- true division, round half to even
  const double q = (double)(total * k1) / (double)(k1 + k2);
  int64_t target = (int64_t)std::nearbyint(q);
  target = std::min(std::max(target, lower), upper);
  for (int64_t u : subset) in_sub[u] = 1;
  std::vector<int64_t> queue;
  queue.reserve(subset.size());
  left.clear();
  int64_t w = 0;
  size_t seed_pos = 0, head = 0;
  while (w < target) {
    if (head >= queue.size()) {
      while (seed_pos < subset.size() && taken[subset[seed_pos]]) ++seed_pos;
      if (seed_pos >= subset.size()) break;
      queue.push_back(subset[seed_pos]);
      taken[subset[seed_pos]] = 1;
    }
    const int64_t u = queue[head++];
    if (w + node_w[u] > upper) continue;
    left.push_back(u);
    w += node_w[u];
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t v = indices[j];
      if (in_sub[v] && !taken[v]) {
        taken[v] = 1;
        queue.push_back(v);
      }
    }
  }
  std::sort(left.begin(), left.end());
  // right = subset minus left, subset order
  right.clear();
  std::vector<int64_t>::const_iterator it = left.begin();
  for (int64_t u : subset) {
    while (it != left.end() && *it < u) ++it;
    if (it != left.end() && *it == u) continue;
    right.push_back(u);
  }
  for (int64_t u : subset) {
    in_sub[u] = 0;
    taken[u] = 0;
  }
  for (int64_t u : queue) taken[u] = 0;
}
}  // namespace

// partition.py:239-252 -- recursive bisection seeding of num_blocks blocks.
extern "C" mp_status mp_initial_partition(int64_t n, const int64_t* indptr, const int64_t* indices,
                                          const int64_t* node_w, int64_t num_blocks, int64_t cap,
                                          int64_t* assignment) {
  mp::clear_error();
  for (int64_t u = 0; u < n; ++u) assignment[u] = -1;
  std::vector<char> in_sub(n, 0), taken(n, 0);
  struct Job {
    std::vector<int64_t> subset;
    int64_t first, k;
  };
  std::vector<Job> stack;
  Job root;
  root.subset.resize(n);
  for (int64_t u = 0; u < n; ++u) root.subset[u] = u;
  root.first = 0;
  root.k = num_blocks;
  stack.push_back(std::move(root));
  std::vector<int64_t> left, right;
  while (!stack.empty()) {
    Job job = std::move(stack.back());
    stack.pop_back();
    if (job.k == 1 || job.subset.empty()) {
      for (int64_t u : job.subset) assignment[u] = job.first;
      continue;
    }
    const int64_t k1 = (job.k + 1) / 2;
    grow_bisection(indptr, indices, node_w, job.subset, k1, job.k - k1, cap, in_sub, taken, left, right);
    Job a, b;
    a.subset = left;
    a.first = job.first;
    a.k = k1;
    b.subset = right;
    b.first = job.first + k1;
    b.k = job.k - k1;
    stack.push_back(std::move(b));
    stack.push_back(std::move(a));
  }
  return MP_OK;
}

// numpy_impl.py:114-131 -- FIFO breadth-first search from `start`: levels
// (-1 unreached), the visit queue (first *tail entries valid) and its tail.
// The queue order follows the adjacency order, as the reference's does.
extern "C" mp_status mp_bfs_levels_host(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t start,
                                        int64_t* levels, int64_t* queue, int64_t* tail) {
  mp::clear_error();
  if (n <= 0 || start < 0 || start >= n) {
    mp::set_error("start node %lld out of range 0..%lld", (long long)start, (long long)n - 1);
    return MP_ERR_VALIDATION;
  }
  for (int64_t v = 0; v < n; ++v) levels[v] = -1;
  levels[start] = 0;
  queue[0] = start;
  int64_t head = 0, t = 1;
  while (head < t) {
    const int64_t u = queue[head++];
    for (int64_t j = indptr[u]; j < indptr[u + 1]; ++j) {
      const int64_t v = indices[j];
      if (levels[v] < 0) {
        levels[v] = levels[u] + 1;
        queue[t++] = v;
      }
    }
  }
  *tail = t;
  return MP_OK;
}

// numpy_impl.py:231-259 -- every unordered pair inside each segment
// seg_values[seg_indptr[s] .. seg_indptr[s+1]), as (min, max).  The reference
// leaves the pair order unspecified; here segments come in order and, within
// one, pairs in (i, j) position order.  With us == NULL only *num_pairs is
// written (size query); otherwise us / vs must hold *num_pairs entries.
extern "C" mp_status mp_pairs_from_segments(int64_t num_segments, const int64_t* seg_indptr, const int64_t* seg_values,
                                            int64_t* us, int64_t* vs, int64_t* num_pairs) {
  mp::clear_error();
  if (num_segments < 0) {
    mp::set_error("negative segment count");
    return MP_ERR_VALIDATION;
  }
  int64_t total = 0;
  for (int64_t s = 0; s < num_segments; ++s) {
    const int64_t k = seg_indptr[s + 1] - seg_indptr[s];
    if (k < 0) {
      mp::set_error("segment %lld has negative length", (long long)s);
      return MP_ERR_VALIDATION;
    }
    total += k * (k - 1) / 2;
  }
  if (!us) {
    *num_pairs = total;
    return MP_OK;
  }
  if (*num_pairs < total) {
    mp::set_error("pair buffers hold %lld entries, %lld needed", (long long)*num_pairs, (long long)total);
    return MP_ERR_VALIDATION;
  }
  int64_t o = 0;
  for (int64_t s = 0; s < num_segments; ++s) {
    const int64_t a = seg_indptr[s], z = seg_indptr[s + 1];
    for (int64_t i = a; i < z; ++i)
      for (int64_t j = i + 1; j < z; ++j) {
        const int64_t x = seg_values[i], y = seg_values[j];
        us[o] = x < y ? x : y;
        vs[o] = x < y ? y : x;
        ++o;
      }
  }
  *num_pairs = total;
  return MP_OK;
}
