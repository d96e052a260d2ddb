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
#include <limits>
#include <set>
#include <utility>
#include <vector>

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
