// Element functors of the five registered loops.
//
// Each functor states its shape (arity, indirect-read components it
// consumes, direct components it consumes, increment components) and maps
// one element's inputs to its per-slot increments.  Operation order is the
// numpy expression order of the reference kernels
// (pkg/src/meshplan/bench_kernels.py:170-181, 196-201, 226-238) and the
// library is compiled with --fmad=false, so element results are bit-equal
// to the reference in every dtype; only the accumulation order of a plan
// can differ, and the executors reproduce the reference's.
#pragma once

#include "mp_common.cuh"

namespace mp {

template <typename T> __device__ __forceinline__ T one() { return T(1); }

template <typename T> __device__ __forceinline__ T sqrt_rn(T x);
template <> __device__ __forceinline__ double sqrt_rn<double>(double x) { return __dsqrt_rn(x); }
template <> __device__ __forceinline__ float sqrt_rn<float>(float x) { return __fsqrt_rn(x); }
template <typename T> __device__ __forceinline__ T div_rn(T a, T b);
template <> __device__ __forceinline__ double div_rn<double>(double a, double b) { return __ddiv_rn(a, b); }
template <> __device__ __forceinline__ float div_rn<float>(float a, float b) { return __fdiv_rn(a, b); }
template <typename T> __device__ __forceinline__ T abs_(T x) { return x < T(0) ? -x : x; }
template <> __device__ __forceinline__ double abs_<double>(double x) { return fabs(x); }
template <> __device__ __forceinline__ float abs_<float>(float x) { return fabsf(x); }

// left = (q1 - q0) * w0 ; right = -left
struct OpFlux {
  static constexpr int ARITY = 2, RC = 4, DC = 1, IC = 4;
  template <typename T>
  __device__ __forceinline__ static void apply(const T (&r)[ARITY][RC], const T (&d)[DC], T (&o)[ARITY][IC]) {
#pragma unroll
    for (int c = 0; c < IC; ++c) {
      T l = (r[1][c] - r[0][c]) * d[0];
      o[0][c] = l;
      o[1][c] = -l;
    }
  }
};

// no indirect read: left = w0 (x4), right = w1 (x4)
struct OpFluxNoRead {
  static constexpr int ARITY = 2, RC = 0, DC = 2, IC = 4;
  template <typename T>
  __device__ __forceinline__ static void apply(const T (&)[ARITY][1], const T (&d)[DC], T (&o)[ARITY][IC]) {
#pragma unroll
    for (int c = 0; c < IC; ++c) {
      o[0][c] = d[0];
      o[1][c] = d[1];
    }
  }
};

// v = [s0+s1, s1*s2, s3-s0] to all eight corners
struct OpScatter8 {
  static constexpr int ARITY = 8, RC = 0, DC = 4, IC = 3;
  template <typename T>
  __device__ __forceinline__ static void apply(const T (&)[ARITY][1], const T (&d)[DC], T (&o)[ARITY][IC]) {
    T v0 = d[0] + d[1], v1 = d[1] * d[2], v2 = d[3] - d[0];
#pragma unroll
    for (int s = 0; s < ARITY; ++s) {
      o[s][0] = v0;
      o[s][1] = v1;
      o[s][2] = v2;
    }
  }
};

// phi = (sr[:5] - sl[:5]) * fw0 ; +phi / -phi
struct OpFaceFlux {
  static constexpr int ARITY = 2, RC = 5, DC = 1, IC = 5;
  template <typename T>
  __device__ __forceinline__ static void apply(const T (&r)[ARITY][RC], const T (&d)[DC], T (&o)[ARITY][IC]) {
#pragma unroll
    for (int c = 0; c < IC; ++c) {
      T phi = (r[1][c] - r[0][c]) * d[0];
      o[0][c] = phi;
      o[1][c] = -phi;
    }
  }
};

// heavy: phi = phi * (sqrt(|sl5|+1) + sqrt(|sr6|+2)) / sqrt(fw1*fw1 + 1)
struct OpFaceFluxHeavy {
  static constexpr int ARITY = 2, RC = 7, DC = 2, IC = 5;
  template <typename T>
  __device__ __forceinline__ static void apply(const T (&r)[ARITY][RC], const T (&d)[DC], T (&o)[ARITY][IC]) {
    T scale = sqrt_rn<T>(abs_<T>(r[0][5]) + T(1)) + sqrt_rn<T>(abs_<T>(r[1][6]) + T(2));
    T den = sqrt_rn<T>(d[1] * d[1] + T(1));
#pragma unroll
    for (int c = 0; c < IC; ++c) {
      T phi = (r[1][c] - r[0][c]) * d[0];
      phi = div_rn<T>(phi * scale, den);
      o[0][c] = phi;
      o[1][c] = -phi;
    }
  }
};

template <class Op> struct RcArr { static constexpr int N = Op::RC > 0 ? Op::RC : 1; };

// Address of (point, component) in an indirect array of `comps` components.
template <int LAYOUT>
__device__ __forceinline__ int64_t ind_index(int64_t p, int c, int comps, int64_t npts) {
  return LAYOUT == MP_AOS ? p * comps + c : (int64_t)c * npts + p;
}

}  // namespace mp

// op dispatch: binds `Op` and calls the body
#define MP_DISPATCH_OP(op, ...)                                              \
  [&]() -> mp_status {                                                       \
    switch (op) {                                                            \
      case MP_OP_FLUX: { using Op = ::mp::OpFlux; return __VA_ARGS__(); }    \
      case MP_OP_FLUX_NOREAD: { using Op = ::mp::OpFluxNoRead; return __VA_ARGS__(); } \
      case MP_OP_SCATTER8: { using Op = ::mp::OpScatter8; return __VA_ARGS__(); }      \
      case MP_OP_FACE_FLUX: { using Op = ::mp::OpFaceFlux; return __VA_ARGS__(); }     \
      case MP_OP_FACE_FLUX_HEAVY: { using Op = ::mp::OpFaceFluxHeavy; return __VA_ARGS__(); } \
      default: MP_FAIL(MP_ERR_KERNEL, "no device functor for op %d", (int)(op));     \
    }                                                                        \
  }()
