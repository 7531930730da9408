// fp32-guarded GAT attention for numerics="fast" (the row-owned B200 path; the
// bit-exact reference chain stays in sddmm_softmax.cu):
//
//  * k_gat_fwd_*   alpha[e, h] = rnd(softmax_r(leaky(s_l[r, h] + s_r[c, h])))
//                  -- attention_scores + leaky_relu + edge_softmax
//                  (models.py:188-200, 317-326, 382-401) in one pass: fp32
//                  logits (never rounded) kept in the log2 domain (leaky
//                  commutes with the positive log2(e) scale), fp32 online
//                  max / sum with exp2 (MUFU.EX2), one rounding of alpha.  No E x H logits array is written.
//  * k_gat_bwd_*   de'[e, h] = rnd(alpha (dalpha - sum_r alpha dalpha) *
//                  leaky'(e)) and ds_l[r, h] = rnd(sum_r de') -- edge_softmax
//                  backward (403-410), leaky backward and the row-sum half of
//                  attention_scores backward (329-333) in one pass.
//  * k_gat_sums_*  out[r, h] = rnd(sum_e v[idx(e), h]) with idx = perm (CSC
//                  gather: the column-sum half of attention_scores backward,
//                  335-337) or identity.
//
// Rows are split by length: <= short_max edges -> one thread per (row, head);
// medium rows (listed) -> one warp per row, lanes over (edge, head); rows
// longer than long_min (listed) -> one 256-thread CTA per row.  All sums are
// fp32 in a fixed order per launch configuration: deterministic.
#include "hg_common.cuh"

namespace hg {

__device__ __forceinline__ float leaky_f(float v, float slope) { return v > 0.0f ? v : v * slope; }

constexpr float kLog2e = 1.4426950408889634f;

// merge two online-softmax states (m, s), s = sum exp(v - m)
__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  if (mm == -INFINITY) return;
  s = (m == -INFINITY ? 0.0f : s * exp2f(m - mm)) + (m2 == -INFINITY ? 0.0f : s2 * exp2f(m2 - mm));
  m = mm;
}

// combine (m, s) over lanes with the same lane % H
template <int H>
__device__ __forceinline__ void ms_warp(float& m, float& s) {
#pragma unroll
  for (int o = 16; o >= H; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    ms_merge(m, s, m2, s2);
  }
}

template <int H>
__device__ __forceinline__ float sum_warp(float v) {
#pragma unroll
  for (int o = 16; o >= H; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// All edge loops below visit edges e = first, first + step, ... in groups of
// U (independent column-id loads, then independent gathers: the dependent
// cols -> s_r chain is the latency that bounds these kernels).
constexpr int U = 4;

// online (max, sum) over the logits of the edges this thread visits
template <typename T, int H>
__device__ __forceinline__ void fwd_pass1(const int32_t* __restrict__ cols, const T* __restrict__ sr,
                                          int64_t first, int64_t end, int64_t step, int h,
                                          float a, float slope, float& m, float& s) {
  for (int64_t e0 = first; e0 < end; e0 += step * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = e0 + u * step < end ? __ldg(cols + e0 + u * step) : -1;
    float v[U];
    float mu = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = c[u] >= 0 ? leaky_f(fmaf(Num<T>::to_f(sr[(size_t)(unsigned)c[u] * H + h]), kLog2e, a), slope)
                       : -INFINITY;
      mu = fmaxf(mu, v[u]);
    }
    if (mu > m) {
      s = m == -INFINITY ? 0.0f : s * exp2f(m - mu);
      m = mu;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) s += exp2f(v[u] - m);
  }
}

template <typename T, int H>
__device__ __forceinline__ void fwd_pass2(const int32_t* __restrict__ cols, const T* __restrict__ sr,
                                          int64_t first, int64_t end, int64_t step, int h,
                                          float a, float slope, float m, float inv,
                                          T* __restrict__ alpha, int ald) {
  for (int64_t e0 = first; e0 < end; e0 += step * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = e0 + u * step < end ? __ldg(cols + e0 + u * step) : -1;
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = c[u] >= 0 ? leaky_f(fmaf(Num<T>::to_f(sr[(size_t)(unsigned)c[u] * H + h]), kLog2e, a), slope)
                       : 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) alpha[(e0 + u * step) * ald + h] = Num<T>::from_f(ex2_neg(v[u] - m) * inv);
  }
}

// D = sum alpha * dalpha over the visited edges
template <typename T, int H>
__device__ __forceinline__ float bwd_pass1(const T* __restrict__ alpha, const T* __restrict__ dalpha,
                                           int64_t first, int64_t end, int64_t step, int h, int ald) {
  float d = 0.0f;
  for (int64_t e0 = first; e0 < end; e0 += step * U) {
    float x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * step;
      x[u] = e < end ? Num<T>::to_f(alpha[e * ald + h]) : 0.0f;
      y[u] = e < end ? Num<T>::to_f(dalpha[e * H + h]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) d = fmaf(x[u], y[u], d);
  }
  return d;
}

// de = alpha (dalpha - D) leaky'(l); returns the thread's sum of de
template <typename T, int H>
__device__ __forceinline__ float bwd_pass2(const int32_t* __restrict__ cols, const T* __restrict__ sr,
                                           const T* __restrict__ alpha, const T* __restrict__ dalpha,
                                           int64_t first, int64_t end, int64_t step, int h, float a,
                                           float slope, float d, T* __restrict__ de, int ald) {
  float acc = 0.0f;
  for (int64_t e0 = first; e0 < end; e0 += step * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = e0 + u * step < end ? __ldg(cols + e0 + u * step) : -1;
    float sv[U], x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * step;
      sv[u] = c[u] >= 0 ? Num<T>::to_f(sr[(size_t)(unsigned)c[u] * H + h]) : 0.0f;
      x[u] = c[u] >= 0 ? Num<T>::to_f(alpha[e * ald + h]) : 0.0f;
      y[u] = c[u] >= 0 ? Num<T>::to_f(dalpha[e * H + h]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c[u] >= 0) {
        float g = x[u] * (y[u] - d);
        g = a + sv[u] > 0.0f ? g : g * slope;
        de[(e0 + u * step) * ald + h] = Num<T>::from_f(g);
        acc += g;
      }
    }
  }
  return acc;
}

template <typename T, int H>
__device__ __forceinline__ float sums_pass(const T* __restrict__ v, const int32_t* __restrict__ perm,
                                           int64_t first, int64_t end, int64_t step, int h) {
  float acc = 0.0f;
  for (int64_t e0 = first; e0 < end; e0 += step * U) {
    int64_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * step;
      idx[u] = e < end ? (perm ? (int64_t)__ldg(perm + e) : e) : -1;
    }
    float x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = idx[u] >= 0 ? Num<T>::to_f(v[idx[u] * H + h]) : 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) acc += x[u];
  }
  return acc;
}

// ---------------------------------------------------------------- forward

template <typename T, int H>
__device__ __forceinline__ void
d_gat_fwd_thread(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
                 int64_t n_rows, const T* __restrict__ sl, const T* __restrict__ sr, float slope,
                 T* __restrict__ alpha, int short_max, int ald, float2* __restrict__ stats) {
  const int64_t t = blk * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_rows * H) return;
  const int64_t r = t / H;
  const int h = (int)(t - r * H);
  const int64_t beg = offsets[r], end = offsets[r + 1];
  if (end == beg || end - beg > short_max) return;
  const float a = Num<T>::to_f(sl[t]) * kLog2e;  // log2 domain
  if (end - beg <= U) {
    // one chunk (most rows of a power-law graph): the logits and their
    // exponentials stay in registers between the two passes -- the same
    // operations in the same order as fwd_pass1 + fwd_pass2, so bitwise equal
    int c[U];
    float v[U], p[U];
    float mu = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = beg + u < end ? __ldg(cols + beg + u) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = c[u] >= 0 ? leaky_f(fmaf(Num<T>::to_f(sr[(size_t)(unsigned)c[u] * H + h]), kLog2e, a), slope)
                       : -INFINITY;
      mu = fmaxf(mu, v[u]);
    }
    float s1 = 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      p[u] = c[u] >= 0 ? ex2_neg(v[u] - mu) : 0.0f;
      if (c[u] >= 0) s1 += p[u];
    }
    const float inv = 1.0f / s1;
    if (stats) {  // hg_gat_attention_stats: alpha = rnd(exp2(l - m) * inv) later, in hg_gat_aggregate
      stats[t] = make_float2(mu, inv);
      return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) alpha[(beg + u) * ald + h] = Num<T>::from_f(p[u] * inv);
    return;
  }
  float m = -INFINITY, s = 0.0f;
  fwd_pass1<T, H>(cols, sr, beg, end, 1, h, a, slope, m, s);
  if (stats) {
    stats[t] = make_float2(m, 1.0f / s);
    return;
  }
  fwd_pass2<T, H>(cols, sr, beg, end, 1, h, a, slope, m, 1.0f / s, alpha, ald);
}

template <typename T, int H>
__device__ __forceinline__ void
d_gat_fwd_warp(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
               const int32_t* __restrict__ rows, int64_t n_list, const T* __restrict__ sl,
               const T* __restrict__ sr, float slope, T* __restrict__ alpha, int ald,
               float2* __restrict__ stats) {
  constexpr int EPB = 32 / H;
  const int lane = threadIdx.x & 31, j = lane / H, h = lane % H;
  const int64_t nwarps = (int64_t)nblk * (blockDim.x >> 5);
  for (int64_t w = blk * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_list;
       w += nwarps) {
    const int64_t r = rows[w];
    const int64_t beg = offsets[r], end = offsets[r + 1];
    const float a = Num<T>::to_f(sl[r * H + h]) * kLog2e;
    float m = -INFINITY, s = 0.0f;
    fwd_pass1<T, H>(cols, sr, beg + j, end, EPB, h, a, slope, m, s);
    ms_warp<H>(m, s);
    if (stats) {
      if (j == 0) stats[r * H + h] = make_float2(m, 1.0f / s);
      continue;
    }
    fwd_pass2<T, H>(cols, sr, beg + j, end, EPB, h, a, slope, m, 1.0f / s, alpha, ald);
  }
}

template <typename T, int H>
__device__ __forceinline__ void
d_gat_fwd_cta(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
              const int32_t* __restrict__ rows, const T* __restrict__ sl,
              const T* __restrict__ sr, float slope, T* __restrict__ alpha, int ald,
              float2* __restrict__ stats) {
  constexpr int EPB = 256 / H;
  __shared__ float sm[8][H], ss[8][H];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, j = tid / H, h = tid % H;
  const int64_t r = rows[blk];
  const int64_t beg = offsets[r], end = offsets[r + 1];
  const float a = Num<T>::to_f(sl[r * H + h]) * kLog2e;
  float m = -INFINITY, s = 0.0f;
  fwd_pass1<T, H>(cols, sr, beg + j, end, EPB, h, a, slope, m, s);
  ms_warp<H>(m, s);
  if (lane < H) { sm[warp][lane] = m; ss[warp][lane] = s; }
  __syncthreads();
  float mt = sm[0][h], st = ss[0][h];
#pragma unroll
  for (int k = 1; k < 8; ++k) ms_merge(mt, st, sm[k][h], ss[k][h]);
  if (stats) {
    if (j == 0) stats[r * H + h] = make_float2(mt, 1.0f / st);
    return;
  }
  fwd_pass2<T, H>(cols, sr, beg + j, end, EPB, h, a, slope, mt, 1.0f / st, alpha, ald);
}

// --------------------------------------------------------------- backward

template <typename T, int H>
__device__ __forceinline__ void
d_gat_bwd_thread(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
                 int64_t n_rows, const T* __restrict__ sl, const T* __restrict__ sr, float slope,
                 const T* __restrict__ alpha, const T* __restrict__ dalpha, T* __restrict__ de,
                 T* __restrict__ dsl, int short_max, int ald) {
  const int64_t t = blk * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_rows * H) return;
  const int64_t r = t / H;
  const int h = (int)(t - r * H);
  const int64_t beg = offsets[r], end = offsets[r + 1];
  if (end - beg > short_max) return;
  const float a = Num<T>::to_f(sl[t]);
  if (end - beg <= U) {
    // one chunk: alpha / dalpha / s_r read once (bwd_pass1 + bwd_pass2 in the
    // same order, bitwise equal)
    int c[U];
    float sv[U], x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = beg + u < end ? __ldg(cols + beg + u) : -1;
    float d = 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = beg + u;
      x[u] = c[u] >= 0 ? Num<T>::to_f(alpha[e * ald + h]) : 0.0f;
      y[u] = c[u] >= 0 ? Num<T>::to_f(dalpha[e * H + h]) : 0.0f;
      sv[u] = c[u] >= 0 ? Num<T>::to_f(sr[(size_t)(unsigned)c[u] * H + h]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) d = fmaf(x[u], y[u], d);
    float acc = 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c[u] >= 0) {
        float g = x[u] * (y[u] - d);
        g = a + sv[u] > 0.0f ? g : g * slope;
        de[(beg + u) * ald + h] = Num<T>::from_f(g);
        acc += g;
      }
    }
    dsl[t] = Num<T>::from_f(acc);
    return;
  }
  const float d = bwd_pass1<T, H>(alpha, dalpha, beg, end, 1, h, ald);
  dsl[t] = Num<T>::from_f(bwd_pass2<T, H>(cols, sr, alpha, dalpha, beg, end, 1, h, a, slope, d, de, ald));
}

template <typename T, int H>
__device__ __forceinline__ void
d_gat_bwd_warp(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
               const int32_t* __restrict__ rows, int64_t n_list, const T* __restrict__ sl,
               const T* __restrict__ sr, float slope, const T* __restrict__ alpha,
               const T* __restrict__ dalpha, T* __restrict__ de, T* __restrict__ dsl, int ald) {
  constexpr int EPB = 32 / H;
  const int lane = threadIdx.x & 31, j = lane / H, h = lane % H;
  const int64_t nwarps = (int64_t)nblk * (blockDim.x >> 5);
  for (int64_t w = blk * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_list;
       w += nwarps) {
    const int64_t r = rows[w];
    const int64_t beg = offsets[r], end = offsets[r + 1];
    const float d = sum_warp<H>(bwd_pass1<T, H>(alpha, dalpha, beg + j, end, EPB, h, ald));
    const float a = Num<T>::to_f(sl[r * H + h]);
    const float acc = sum_warp<H>(
        bwd_pass2<T, H>(cols, sr, alpha, dalpha, beg + j, end, EPB, h, a, slope, d, de, ald));
    if (lane < H) dsl[r * H + lane] = Num<T>::from_f(acc);
  }
}

template <int H>
__device__ __forceinline__ float block_sum_h(float v, float (*red)[H]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, h = tid % H;
  v = sum_warp<H>(v);
  if (lane < H) red[warp][lane] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) t += red[k][h];
  __syncthreads();
  return t;
}

template <typename T, int H>
__device__ __forceinline__ void
d_gat_bwd_cta(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
              const int32_t* __restrict__ rows, const T* __restrict__ sl,
              const T* __restrict__ sr, float slope, const T* __restrict__ alpha,
              const T* __restrict__ dalpha, T* __restrict__ de, T* __restrict__ dsl, int ald) {
  constexpr int EPB = 256 / H;
  __shared__ float red[8][H];
  const int tid = threadIdx.x, j = tid / H, h = tid % H;
  const int64_t r = rows[blk];
  const int64_t beg = offsets[r], end = offsets[r + 1];
  const float d = block_sum_h<H>(bwd_pass1<T, H>(alpha, dalpha, beg + j, end, EPB, h, ald), red);
  const float a = Num<T>::to_f(sl[r * H + h]);
  const float acc = block_sum_h<H>(
      bwd_pass2<T, H>(cols, sr, alpha, dalpha, beg + j, end, EPB, h, a, slope, d, de, ald), red);
  if (tid < H) dsl[r * H + tid] = Num<T>::from_f(acc);
}

// ------------------------------------------------------------- edge sums

template <typename T, int H>
__device__ __forceinline__ void
d_gat_sums_thread(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ v,
                  const int32_t* __restrict__ perm, T* __restrict__ out, int short_max) {
  const int64_t t = blk * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_rows * H) return;
  const int64_t r = t / H;
  const int h = (int)(t - r * H);
  const int64_t beg = offsets[r], end = offsets[r + 1];
  if (end - beg > short_max) return;
  out[t] = Num<T>::from_f(sums_pass<T, H>(v, perm, beg, end, 1, h));
}

template <typename T, int H>
__device__ __forceinline__ void
d_gat_sums_warp(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ rows,
                int64_t n_list, const T* __restrict__ v, const int32_t* __restrict__ perm,
                T* __restrict__ out) {
  constexpr int EPB = 32 / H;
  const int lane = threadIdx.x & 31, j = lane / H, h = lane % H;
  const int64_t nwarps = (int64_t)nblk * (blockDim.x >> 5);
  for (int64_t w = blk * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_list;
       w += nwarps) {
    const int64_t r = rows[w];
    const int64_t beg = offsets[r], end = offsets[r + 1];
    const float acc = sum_warp<H>(sums_pass<T, H>(v, perm, beg + j, end, EPB, h));
    if (lane < H) out[r * H + lane] = Num<T>::from_f(acc);
  }
}

template <typename T, int H>
__device__ __forceinline__ void
d_gat_sums_cta(int64_t blk, int64_t nblk, const int64_t* __restrict__ offsets, const int32_t* __restrict__ rows,
               const T* __restrict__ v, const int32_t* __restrict__ perm, T* __restrict__ out) {
  constexpr int EPB = 256 / H;
  __shared__ float red[8][H];
  const int tid = threadIdx.x, j = tid / H, h = tid % H;
  const int64_t r = rows[blk];
  const int64_t beg = offsets[r], end = offsets[r + 1];
  const float acc = block_sum_h<H>(sums_pass<T, H>(v, perm, beg + j, end, EPB, h), red);
  if (tid < H) out[r * H + tid] = Num<T>::from_f(acc);
}


// One launch per operation: blocks [0, n_long) take the long rows (one CTA each,
// dispatched first so the hub rows start early and overlap everything else),
// the next b_med blocks the medium rows (warp per row), the rest one thread per
// (row, head) for the short rows.
template <typename T, int H>
__global__ void __launch_bounds__(256)
k_gat_fwd_all(const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
              int64_t n_rows, const int32_t* __restrict__ medium, int64_t n_medium,
              const int32_t* __restrict__ longr, int64_t n_long, int64_t b_med,
              const T* __restrict__ sl, const T* __restrict__ sr, float slope,
              T* __restrict__ alpha, int short_max, int ald, float2* __restrict__ stats) {
  int64_t b = blockIdx.x;
  if (b < n_long)
    return d_gat_fwd_cta<T, H>(b, n_long, offsets, cols, longr, sl, sr, slope, alpha, ald, stats);
  b -= n_long;
  if (b < b_med)
    return d_gat_fwd_warp<T, H>(b, b_med, offsets, cols, medium, n_medium, sl, sr, slope, alpha,
                                ald, stats);
  b -= b_med;
  d_gat_fwd_thread<T, H>(b, 0, offsets, cols, n_rows, sl, sr, slope, alpha, short_max, ald, stats);
}

template <typename T, int H>
__global__ void __launch_bounds__(256, 5)
k_gat_bwd_all(const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
              int64_t n_rows, const int32_t* __restrict__ medium, int64_t n_medium,
              const int32_t* __restrict__ longr, int64_t n_long, int64_t b_med,
              const T* __restrict__ sl, const T* __restrict__ sr, float slope,
              const T* __restrict__ alpha, const T* __restrict__ dalpha, T* __restrict__ de,
              T* __restrict__ dsl, int short_max, int ald) {
  int64_t b = blockIdx.x;
  if (b < n_long)
    return d_gat_bwd_cta<T, H>(b, n_long, offsets, cols, longr, sl, sr, slope, alpha, dalpha, de,
                               dsl, ald);
  b -= n_long;
  if (b < b_med)
    return d_gat_bwd_warp<T, H>(b, b_med, offsets, cols, medium, n_medium, sl, sr, slope, alpha,
                                dalpha, de, dsl, ald);
  b -= b_med;
  d_gat_bwd_thread<T, H>(b, 0, offsets, cols, n_rows, sl, sr, slope, alpha, dalpha, de, dsl,
                         short_max, ald);
}

template <typename T, int H>
__global__ void __launch_bounds__(256)
k_gat_sums_all(const int64_t* __restrict__ offsets, int64_t n_rows,
               const int32_t* __restrict__ medium, int64_t n_medium,
               const int32_t* __restrict__ longr, int64_t n_long, int64_t b_med,
               const T* __restrict__ v, const int32_t* __restrict__ perm, T* __restrict__ out,
               int short_max) {
  int64_t b = blockIdx.x;
  if (b < n_long) return d_gat_sums_cta<T, H>(b, n_long, offsets, longr, v, perm, out);
  b -= n_long;
  if (b < b_med) return d_gat_sums_warp<T, H>(b, b_med, offsets, medium, n_medium, v, perm, out);
  b -= b_med;
  d_gat_sums_thread<T, H>(b, 0, offsets, n_rows, v, perm, out, short_max);
}

// -------------------------------------------------------------- head mean

// out[n, f] = rnd(sum_h y[n, h, f] / H): the H fp16 values sum exactly in fp64
// (models.py mean of concatenated heads; _HeadMeanFn).  Backward:
// g_in[n, h, f] = rnd(g[n, f] / H).
template <typename T>
__global__ void k_head_mean(const T* __restrict__ y, int64_t n, int heads, int f,
                            T* __restrict__ out) {
  const int64_t total = n * (int64_t)f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / f;
    const int c = (int)(i - r * f);
    double s = 0.0;
    for (int h = 0; h < heads; ++h) s += Num<T>::to_d(y[(r * heads + h) * f + c]);
    out[i] = Num<T>::from_d(s / heads);
  }
}

template <typename T>
__global__ void k_head_mean_bwd(const T* __restrict__ g, int64_t n, int heads, int f,
                                T* __restrict__ gin) {
  const int64_t total = n * (int64_t)f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / f;
    const int c = (int)(i - r * f);
    const T v = Num<T>::from_d(Num<T>::to_d(g[i]) / heads);
    for (int h = 0; h < heads; ++h) gin[(r * heads + h) * f + c] = v;
  }
}

// 8-column vector versions (binary16, f % 8 == 0, 16-byte aligned).
__global__ void k_head_mean_v8(const __half* __restrict__ y, int64_t n, int heads, int f,
                               __half* __restrict__ out) {
  const int C = f / 8;
  const int64_t total = n * (int64_t)C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = (int)(i - r * C);
    double s[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = 0.0;
    // up to 8 heads loaded before any add (the head loop was one dependent
    // load per step); sums in head order as before
    for (int h0 = 0; h0 < heads; h0 += 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (h0 + u < heads) v[u] = *reinterpret_cast<const uint4*>(y + (r * heads + h0 + u) * f + c * 8);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (h0 + u >= heads) break;
        const __half* e = reinterpret_cast<const __half*>(&v[u]);
#pragma unroll
        for (int k = 0; k < 8; ++k) s[k] += (double)__half2float(e[k]);
      }
    }
    __align__(16) __half o[8];
    // power-of-two head counts: the quotient is an exact scaling
    const bool p2 = (heads & (heads - 1)) == 0;
    const double inv = 1.0 / heads;
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = __double2half(p2 ? s[k] * inv : s[k] / heads);
    *reinterpret_cast<uint4*>(out + r * f + c * 8) = *reinterpret_cast<const uint4*>(o);
  }
}

__global__ void k_head_mean_bwd_v8(const __half* __restrict__ g, int64_t n, int heads, int f,
                                   __half* __restrict__ gin) {
  const int C = f / 8;
  const int64_t total = n * (int64_t)C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = (int)(i - r * C);
    const uint4 v = *reinterpret_cast<const uint4*>(g + r * f + c * 8);
    const __half* e = reinterpret_cast<const __half*>(&v);
    __align__(16) __half o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = __double2half((double)__half2float(e[k]) / heads);
    for (int h = 0; h < heads; ++h)
      *reinterpret_cast<uint4*>(gin + (r * heads + h) * f + c * 8) = *reinterpret_cast<const uint4*>(o);
  }
}

struct GatRows {
  const int64_t* offsets;
  const int32_t* cols;
  int64_t n_rows;
  const int32_t* medium;
  int64_t n_medium;
  const int32_t* longr;
  int64_t n_long;
  int short_max;
  cudaStream_t st;
  int ald;  // row stride (elements) of alpha and d_e: H, or 2H for interleaved rows
};

static inline int64_t med_blocks(const GatRows& g) {
  return g.n_medium ? grid_for(g.n_medium, 8, 148 * 32) : 0;
}

static inline unsigned all_blocks(const GatRows& g, int H) {
  return (unsigned)(g.n_long + med_blocks(g) + grid_for(g.n_rows * H, 256));
}

template <typename T, int H>
static void gat_fwd(const GatRows& g, const void* sl, const void* sr, float slope, void* alpha,
                    float2* stats) {
  k_gat_fwd_all<T, H><<<all_blocks(g, H), 256, 0, g.st>>>(
      g.offsets, g.cols, g.n_rows, g.medium, g.n_medium, g.longr, g.n_long, med_blocks(g),
      (const T*)sl, (const T*)sr, slope, (T*)alpha, g.short_max, g.ald, stats);
}

template <typename T, int H>
static void gat_bwd(const GatRows& g, const void* sl, const void* sr, float slope,
                    const void* alpha, const void* dalpha, void* de, void* dsl) {
  k_gat_bwd_all<T, H><<<all_blocks(g, H), 256, 0, g.st>>>(
      g.offsets, g.cols, g.n_rows, g.medium, g.n_medium, g.longr, g.n_long, med_blocks(g),
      (const T*)sl, (const T*)sr, slope, (const T*)alpha, (const T*)dalpha, (T*)de, (T*)dsl,
      g.short_max, g.ald);
}

template <typename T, int H>
static void gat_sums(const GatRows& g, const void* v, const int32_t* perm, void* out) {
  k_gat_sums_all<T, H><<<all_blocks(g, H), 256, 0, g.st>>>(
      g.offsets, g.n_rows, g.medium, g.n_medium, g.longr, g.n_long, med_blocks(g),
      (const T*)v, perm, (T*)out, g.short_max);
}

#define HG_GAT_HEADS(FN, T, ...)                  \
  switch (heads) {                                \
    case 1: FN<T, 1>(__VA_ARGS__); break;         \
    case 2: FN<T, 2>(__VA_ARGS__); break;         \
    case 4: FN<T, 4>(__VA_ARGS__); break;         \
    case 8: FN<T, 8>(__VA_ARGS__); break;         \
    default: FN<T, 16>(__VA_ARGS__); break;       \
  }

}  // namespace hg

using namespace hg;

static int gat_rows_check(int heads, int dtype, int64_t n_medium, const int32_t* medium,
                          int64_t n_long, const int32_t* longr, int short_max) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1 && heads <= 16 && (heads & (heads - 1)) == 0,
             "heads must be a power of two <= 16, got %d", heads);
  HG_REQUIRE((n_medium == 0 || medium) && (n_long == 0 || longr),
             "row classes listed without index arrays");
  HG_REQUIRE(short_max >= 0, "short_max must be >= 0");
  return HG_OK;
}

extern "C" int hg_gat_attention_fwd(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                                    const void* s_l, const void* s_r, int32_t heads, float slope,
                                    void* alpha, int64_t alpha_ld, const int32_t* medium_rows,
                                    int64_t n_medium, const int32_t* long_rows, int64_t n_long,
                                    int32_t short_max, int dtype, void* stream) {
  int rc = gat_rows_check(heads, dtype, n_medium, medium_rows, n_long, long_rows, short_max);
  if (rc) return rc;
  HG_REQUIRE(alpha_ld == 0 || (alpha_ld >= heads && alpha_ld <= INT32_MAX), "bad alpha row stride");
  if (n_rows == 0) return HG_OK;
  GatRows g{offsets, cols, n_rows, medium_rows, n_medium, long_rows, n_long, short_max,
            as_stream(stream), (int)(alpha_ld ? alpha_ld : heads)};
  if (dtype == HG_F16) { HG_GAT_HEADS(gat_fwd, __half, g, s_l, s_r, slope, alpha, nullptr) }
  else { HG_GAT_HEADS(gat_fwd, float, g, s_l, s_r, slope, alpha, nullptr) }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_gat_attention_stats(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                                      const void* s_l, const void* s_r, int32_t heads, float slope,
                                      float* stats, const int32_t* medium_rows, int64_t n_medium,
                                      const int32_t* long_rows, int64_t n_long, int32_t short_max,
                                      int dtype, void* stream) {
  int rc = gat_rows_check(heads, dtype, n_medium, medium_rows, n_long, long_rows, short_max);
  if (rc) return rc;
  if (n_rows == 0) return HG_OK;
  HG_REQUIRE(stats && (reinterpret_cast<uintptr_t>(stats) & 7) == 0, "hg_gat_attention_stats: stats must be 8-byte aligned");
  GatRows g{offsets, cols, n_rows, medium_rows, n_medium, long_rows, n_long, short_max,
            as_stream(stream), heads};
  float2* st = reinterpret_cast<float2*>(stats);
  if (dtype == HG_F16) { HG_GAT_HEADS(gat_fwd, __half, g, s_l, s_r, slope, nullptr, st) }
  else { HG_GAT_HEADS(gat_fwd, float, g, s_l, s_r, slope, nullptr, st) }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_gat_attention_bwd(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                                    const void* s_l, const void* s_r, int32_t heads, float slope,
                                    const void* alpha, const void* dalpha, void* de, int64_t ae_ld,
                                    void* ds_l, const int32_t* medium_rows, int64_t n_medium,
                                    const int32_t* long_rows, int64_t n_long, int32_t short_max,
                                    int dtype, void* stream) {
  int rc = gat_rows_check(heads, dtype, n_medium, medium_rows, n_long, long_rows, short_max);
  if (rc) return rc;
  HG_REQUIRE(ae_ld == 0 || (ae_ld >= heads && ae_ld <= INT32_MAX), "bad alpha / d_e row stride");
  if (n_rows == 0) return HG_OK;
  GatRows g{offsets, cols, n_rows, medium_rows, n_medium, long_rows, n_long, short_max,
            as_stream(stream), (int)(ae_ld ? ae_ld : heads)};
  if (dtype == HG_F16) { HG_GAT_HEADS(gat_bwd, __half, g, s_l, s_r, slope, alpha, dalpha, de, ds_l) }
  else { HG_GAT_HEADS(gat_bwd, float, g, s_l, s_r, slope, alpha, dalpha, de, ds_l) }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_edge_sums_fast(const int64_t* offsets, int64_t n_rows, const void* vals,
                                 const int32_t* perm, int32_t heads, void* out,
                                 const int32_t* medium_rows, int64_t n_medium,
                                 const int32_t* long_rows, int64_t n_long, int32_t short_max,
                                 int dtype, void* stream) {
  int rc = gat_rows_check(heads, dtype, n_medium, medium_rows, n_long, long_rows, short_max);
  if (rc) return rc;
  if (n_rows == 0) return HG_OK;
  GatRows g{offsets, nullptr, n_rows, medium_rows, n_medium, long_rows, n_long, short_max,
            as_stream(stream), heads};
  if (dtype == HG_F16) { HG_GAT_HEADS(gat_sums, __half, g, vals, perm, out) }
  else { HG_GAT_HEADS(gat_sums, float, g, vals, perm, out) }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_head_mean(const void* y, int64_t n, int32_t heads, int32_t f, void* out,
                            int dtype, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1 && f >= 1, "hg_head_mean: bad shape");
  if (n == 0) return HG_OK;
  const int g = grid_for(n * f, 256, 148 * 16);
  const bool v8 = dtype == HG_F16 && f % 8 == 0 &&
                  ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (v8)
    k_head_mean_v8<<<grid_for(n * (f / 8), 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        (const __half*)y, n, heads, f, (__half*)out);
  else if (dtype == HG_F16)
    k_head_mean<__half><<<g, 256, 0, as_stream(stream)>>>((const __half*)y, n, heads, f, (__half*)out);
  else
    k_head_mean<float><<<g, 256, 0, as_stream(stream)>>>((const float*)y, n, heads, f, (float*)out);
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_head_mean_bwd(const void* g, int64_t n, int32_t heads, int32_t f, void* gin,
                                int dtype, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1 && f >= 1, "hg_head_mean_bwd: bad shape");
  if (n == 0) return HG_OK;
  const int gr = grid_for(n * f, 256, 148 * 16);
  const bool v8 = dtype == HG_F16 && f % 8 == 0 &&
                  ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(gin)) & 15) == 0;
  if (v8)
    k_head_mean_bwd_v8<<<grid_for(n * (f / 8), 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        (const __half*)g, n, heads, f, (__half*)gin);
  else if (dtype == HG_F16)
    k_head_mean_bwd<__half><<<gr, 256, 0, as_stream(stream)>>>((const __half*)g, n, heads, f, (__half*)gin);
  else
    k_head_mean_bwd<float><<<gr, 256, 0, as_stream(stream)>>>((const float*)g, n, heads, f, (float*)gin);
  HG_LAUNCHED();
  return HG_OK;
}
