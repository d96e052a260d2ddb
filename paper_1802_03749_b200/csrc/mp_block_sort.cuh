// Small CTA-local helpers for the planner: in-shared-memory bitonic sort
// and exclusive scan.  Sizes are bounded by one block (<= 1024 elements x
// arity 8), so an O(m log^2 m) network is cheap and deterministic.
#pragma once

#include "mp_common.cuh"

namespace mp {

__host__ __device__ inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Sorts keys[0..m) ascending; m must be a power of two (pad with max).
template <typename K>
__device__ void bitonic_sort_shared(K* keys, int m) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = tid; i < (m >> 1); i += nt) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        K a = keys[lo], b = keys[hi];
        if ((a > b) == up) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

// Block-wide exclusive scan of flags[0..m) into out[0..m); returns total.
// `tmp` holds one int per warp.
__device__ inline int block_exclusive_scan(const int* in, int* out, int m, int* tmp) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = (nt + 31) >> 5;
  __shared__ int s_carry;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < m; base += nt) {
    int i = base + tid;
    int x = i < m ? in[i] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? tmp[lane] : 0;
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < nw) tmp[lane] = wi - w;  // exclusive warp offsets
    }
    __syncthreads();
    int carry = s_carry;
    if (i < m) out[i] = carry + tmp[warp] + incl - x;
    __syncthreads();
    if (tid == nt - 1) s_carry = carry + tmp[warp] + incl;
    __syncthreads();
  }
  return s_carry;
}

}  // namespace mp
