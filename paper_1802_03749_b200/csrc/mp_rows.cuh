// Shared-memory row staging helpers (cp.async gathers, swizzled row format,
// 256-bit global row accesses), used by the gather-form executor.
#pragma once

#include <string.h>

#include "mp_loop.cuh"

namespace mp {
namespace rows {

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
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_groups(int pending) {
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

// A row of RB bytes in granules of G = 16/8/4 bytes; N = RB/G.  Odd N: rows
// packed at pitch RB; power-of-two N (16-byte granules): granule c of row r at
// c ^ ((r / (8/N)) % N), so any 8 consecutive rows fill 8 distinct 16-byte
// bank groups; other even N padded by one granule.
template <int RB>
struct Fmt {
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
template <int G> struct Gran;
template <> struct Gran<16> { using type = uint4; };
template <> struct Gran<8> { using type = uint2; };
template <> struct Gran<4> { using type = uint32_t; };

template <typename T, int NC>
__device__ __forceinline__ void lds(const unsigned char* base, int r, T (&out)[NC]) {
  using F = Fmt<NC * (int)sizeof(T)>;
  using V = typename Gran<F::G>::type;
#pragma unroll
  for (int c = 0; c < F::N; ++c) {
    V x = *reinterpret_cast<const V*>(base + F::slot(r, c));
    memcpy(reinterpret_cast<unsigned char*>(out) + c * F::G, &x, F::G);
  }
}

// global AoS row p (first NC of `comps` components) -> shared row r, async
template <typename T, int NC>
__device__ __forceinline__ void gather(unsigned char* base, int r, const T* g, int64_t p, int comps) {
  using F = Fmt<NC * (int)sizeof(T)>;
  const unsigned char* src = reinterpret_cast<const unsigned char*>(g + p * comps);
  if ((comps * (int)sizeof(T)) % F::G == 0) {
#pragma unroll
    for (int c = 0; c < F::N; ++c) cpa<F::G>(base + F::slot(r, c), src + c * F::G);
  } else {
    constexpr int PER = F::G / (int)sizeof(T);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      cpa<(int)sizeof(T)>(base + F::slot(r, c / PER) + (c % PER) * (int)sizeof(T), g + p * comps + c);
  }
}

// global AoS row p of NC components <-> registers; 32-byte rows as one
// 256-bit access (LDG/STG.E.ENL2.256)
template <typename T, int NC>
__device__ __forceinline__ void ldg(const T* g, int64_t p, T (&out)[NC]) {
  constexpr int RB = NC * (int)sizeof(T);
  if constexpr (RB == 32) {
    unsigned long long a, b, c, d;
    asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(g + p * NC));
    const unsigned long long w[4] = {a, b, c, d};
    memcpy(out, w, 32);
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = g[p * NC + c];
  }
}
template <typename T, int NC>
__device__ __forceinline__ void stg(T* g, int64_t p, const T (&in)[NC]) {
  constexpr int RB = NC * (int)sizeof(T);
  if constexpr (RB == 32) {
    unsigned long long w[4];
    memcpy(w, in, 32);
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(g + p * NC), "l"(w[0]), "l"(w[1]), "l"(w[2]),
                 "l"(w[3])
                 : "memory");
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) g[p * NC + c] = in[c];
  }
}

}  // namespace rows
}  // namespace mp
