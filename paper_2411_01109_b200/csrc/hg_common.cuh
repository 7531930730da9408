// Shared helpers for the halfgnn sm_100a kernels: error plumbing, workspace
// carving, and the two precision modes (binary16 / binary32) behind one set of
// templates.  Rounding-sensitive arithmetic always goes through explicit
// round-to-nearest intrinsics so that FMA contraction can never change a
// reference-order result.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "halfgnn.h"

namespace hg {

// Rows per packed work unit (hg_schedule_build pack_rows upper bound; the
// SpMM team keeps one end offset per packed row in its lanes' registers).
constexpr int kPackRows = 16;

void set_error(const char* fmt, ...);

#define HG_REQUIRE(cond, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      ::hg::set_error(__VA_ARGS__);    \
      return HG_EINVAL;                \
    }                                  \
  } while (0)

#define HG_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t hg_e_ = (call);                                                        \
    if (hg_e_ != cudaSuccess) {                                                        \
      ::hg::set_error("CUDA error '%s' at %s:%d", cudaGetErrorString(hg_e_), __FILE__, \
                      __LINE__);                                                       \
      return HG_ECUDA;                                                                 \
    }                                                                                  \
  } while (0)

#define HG_LAUNCHED() HG_CUDA(cudaGetLastError())

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// Bump allocator over a caller-supplied workspace.  In "sizing" mode (base ==
// nullptr) it only accumulates the bytes needed.
struct Carver {
  char* base;
  size_t cap;
  size_t used = 0;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    size_t off = align_up(used);
    used = off + align_up(count * sizeof(T));
    return base ? reinterpret_cast<T*>(base + off) : nullptr;
  }
  bool fits() const { return used <= cap; }
};

inline int grid_for(int64_t work_items, int per_block, int64_t cap = (1LL << 31) - 1) {
  int64_t g = (work_items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------- numerics
// Num<T>: scalar ops with exactly one round-to-nearest-even per call.

template <typename T>
struct Num;

template <>
struct Num<__half> {
  using T2 = __half2;
  static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
  static __device__ __forceinline__ double to_d(__half v) { return (double)__half2float(v); }
  static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ __half from_d(double v) { return __double2half(v); }
  static __device__ __forceinline__ __half add(__half a, __half b) { return __hadd_rn(a, b); }
  static __device__ __forceinline__ __half sub(__half a, __half b) { return __hsub_rn(a, b); }
  static __device__ __forceinline__ __half mul(__half a, __half b) { return __hmul_rn(a, b); }
  static __device__ __forceinline__ __half zero() { return __ushort_as_half(0); }
  static __device__ __forceinline__ bool gt0(__half a) { return __hgt(a, zero()); }
  // pairs (two adjacent feature columns)
  static __device__ __forceinline__ __half2 fma2(__half2 a, __half2 b, __half2 c) {
    return __hfma2(a, b, c);
  }
  static __device__ __forceinline__ __half2 add2(__half2 a, __half2 b) { return __hadd2_rn(a, b); }
  static __device__ __forceinline__ __half2 mul2(__half2 a, __half2 b) { return __hmul2_rn(a, b); }
  static __device__ __forceinline__ __half2 bcast(__half a) { return __half2half2(a); }
  static __device__ __forceinline__ __half2 pack2(__half a, __half b) { return __halves2half2(a, b); }
  static __device__ __forceinline__ __half2 zero2() { return __halves2half2(zero(), zero()); }
  static __device__ __forceinline__ __half lo(__half2 v) { return __low2half(v); }
  static __device__ __forceinline__ __half hi(__half2 v) { return __high2half(v); }
};

template <>
struct Num<float> {
  using T2 = float2;
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ double to_d(float v) { return (double)v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
  static __device__ __forceinline__ float from_d(double v) { return __double2float_rn(v); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float zero() { return 0.0f; }
  static __device__ __forceinline__ bool gt0(float a) { return a > 0.0f; }
  static __device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    return make_float2(__fmaf_rn(a.x, b.x, c.x), __fmaf_rn(a.y, b.y, c.y));
  }
  static __device__ __forceinline__ float2 add2(float2 a, float2 b) {
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
  }
  static __device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
  }
  static __device__ __forceinline__ float2 bcast(float a) { return make_float2(a, a); }
  static __device__ __forceinline__ float2 pack2(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ float2 zero2() { return make_float2(0.0f, 0.0f); }
  static __device__ __forceinline__ float lo(float2 v) { return v.x; }
  static __device__ __forceinline__ float hi(float2 v) { return v.y; }
};

// 2^x for x <= 0 as one MUFU.EX2 (flush-to-zero).  Equal to exp2f for every
// x >= -126; below, both are < 2^-126 and every use (alpha = 2^(l - m) / s with
// s >= 1, rounded to binary16) rounds them to zero alike.
__device__ __forceinline__ float ex2_neg(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Largest r with offsets[r] <= e (offsets non-decreasing, n+1 entries, e < offsets[n]).
__device__ __forceinline__ int64_t row_of_edge(const int64_t* __restrict__ offsets, int64_t n,
                                               int64_t e) {
  int64_t lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(offsets + mid) <= e) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace hg
