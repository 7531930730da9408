// Row/column helpers around the dense per-layer GEMM (the GCN layer's
// epilogue side), memory-bound, 16-byte vectors:
//
//  * k_bias_scale  out = rnd(rnd(x + b[col]) * s[row])  -- models.add_bias
//                  (models.py:161-166) fused with the SpMM's left-norm input
//                  scaling X' = rnd(X * in_scale) (kernels.py:358-361).  Both
//                  roundings are the hardware's correctly rounded HADD / HMUL,
//                  i.e. the reference's fp64-then-round for two fp16 operands.
//  * k_col_sums    out[f] = rnd(sum_r x[r, f]) with fp32 accumulation
//                  (add_bias backward, models.py:168-170: fp32 sum over axis 0,
//                  one rounding); deterministic two-pass reduction.
#include "hg_common.cuh"

namespace hg {

template <typename T, int V>
struct Vec;
template <> struct Vec<__half, 8> { using raw = uint4; };
template <> struct Vec<__half, 1> { using raw = __half; };
template <> struct Vec<float, 4> { using raw = float4; };
template <> struct Vec<float, 1> { using raw = float; };

// One thread per V-element chunk of a row.
template <typename T, int V>
__global__ void __launch_bounds__(256)
k_bias_scale(const T* __restrict__ x, const T* __restrict__ b, const T* __restrict__ s,
             int64_t rows, int F, T* __restrict__ out) {
  using Raw = typename Vec<T, V>::raw;
  const int C = F / V;
  const int64_t total = rows * (int64_t)C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = (int)(i - r * C);
    Raw xv = reinterpret_cast<const Raw*>(x)[i];
    T* xe = reinterpret_cast<T*>(&xv);
    if (b != nullptr) {
      const Raw bv = reinterpret_cast<const Raw*>(b)[c];
      const T* be = reinterpret_cast<const T*>(&bv);
#pragma unroll
      for (int k = 0; k < V; ++k) xe[k] = Num<T>::add(xe[k], be[k]);
    }
    if (s != nullptr) {
      const T sv = s[r];
#pragma unroll
      for (int k = 0; k < V; ++k) xe[k] = Num<T>::mul(xe[k], sv);
    }
    reinterpret_cast<Raw*>(out)[i] = xv;
  }
}

template <typename T>
static void launch_bias_scale(const void* x, const void* b, const void* s, int64_t rows, int F,
                              void* out, cudaStream_t st) {
  constexpr int VB = 16 / sizeof(T);
  const bool vec = F % VB == 0 &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) |
                     reinterpret_cast<uintptr_t>(b)) % 16 == 0);
  if (vec) {
    const int g = grid_for(rows * (F / VB), 256, 148 * 16);
    k_bias_scale<T, VB><<<g, 256, 0, st>>>((const T*)x, (const T*)b, (const T*)s, rows, F, (T*)out);
  } else {
    const int g = grid_for(rows * F, 256, 148 * 16);
    k_bias_scale<T, 1><<<g, 256, 0, st>>>((const T*)x, (const T*)b, (const T*)s, rows, F, (T*)out);
  }
}

// Pass 1: block k sums rows [k*rpb, (k+1)*rpb); thread t owns column chunk
// t % C of row lane t / C (C = F / V chunks, RL = 256 / C lanes); lanes are
// folded in a fixed order through shared memory -> part[k, F] (fp32).
constexpr int kColBlocks = 148 * 4;

template <typename T, int V>
__global__ void __launch_bounds__(256)
k_col_sums_part(const T* __restrict__ x, int64_t rows, int F, int64_t rpb,
                float* __restrict__ part) {
  using Raw = typename Vec<T, V>::raw;
  extern __shared__ float sh[];  // [RL][F]
  const int C = F / V;
  const int RL = C <= 256 ? 256 / C : 1;
  const int t = threadIdx.x;
  const int64_t r0 = blockIdx.x * rpb;
  const int64_t r1 = r0 + rpb < rows ? r0 + rpb : rows;
  for (int cb = 0; cb < C; cb += 256) {  // column sweep when C > 256
    const int c = cb + (C <= 256 ? t % C : t);
    const int rl = C <= 256 ? t / C : 0;
    const bool active = rl < RL && c < C;
    float acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.0f;
    if (active) {
      for (int64_t r = r0 + rl; r < r1; r += RL) {
        const Raw v = reinterpret_cast<const Raw*>(x + r * F)[c];
        const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __fadd_rn(acc[k], Num<T>::to_f(e[k]));
      }
#pragma unroll
      for (int k = 0; k < V; ++k) sh[rl * F + c * V + k] = acc[k];
    }
    __syncthreads();
    const int width = C <= 256 ? F : (C - cb < 256 ? C - cb : 256) * V;
    for (int f = t; f < width; f += blockDim.x) {
      const int col = (C <= 256 ? 0 : cb * V) + f;
      float s = 0.0f;
      for (int l = 0; l < RL; ++l) s = __fadd_rn(s, sh[l * F + col]);
      part[(int64_t)blockIdx.x * F + col] = s;
    }
    __syncthreads();
  }
}

// Pass 2: warp per column; lane l folds partials l, l+32, ... in order, then
// a fixed xor-shuffle tree: out[f] = rnd(sum_k part[k, f]), deterministic.
template <typename T>
__global__ void k_col_sums_final(const float* __restrict__ part, int nb, int F,
                                 T* __restrict__ out) {
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (f >= F) return;
  float s = 0.0f;
  for (int k = lane; k < nb; k += 32) s = __fadd_rn(s, part[(int64_t)k * F + f]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) out[f] = Num<T>::from_f(s);
}

template <typename T>
static int launch_col_sums(const void* x, int64_t rows, int F, void* out, float* part,
                           cudaStream_t st) {
  constexpr int VB = 16 / sizeof(T);
  const bool vec = F % VB == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
  int64_t nb = rows < kColBlocks ? (rows > 0 ? rows : 1) : kColBlocks;
  const int64_t rpb = (rows + nb - 1) / nb;
  nb = rows > 0 ? (rows + rpb - 1) / rpb : 1;
  const int V = vec ? VB : 1;
  const int C = F / V;
  const int RL = C <= 256 ? 256 / C : 1;
  const size_t smem = (size_t)RL * F * sizeof(float);
  HG_REQUIRE(smem <= 227 * 1024, "hg_col_sums: F=%d too wide", F);
  if (vec) {
    if (smem > 48 * 1024)
      HG_CUDA(cudaFuncSetAttribute(k_col_sums_part<T, VB>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_col_sums_part<T, VB><<<(unsigned)nb, 256, smem, st>>>((const T*)x, rows, F, rpb, part);
  } else {
    if (smem > 48 * 1024)
      HG_CUDA(cudaFuncSetAttribute(k_col_sums_part<T, 1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_col_sums_part<T, 1><<<(unsigned)nb, 256, smem, st>>>((const T*)x, rows, F, rpb, part);
  }
  HG_LAUNCHED();
  k_col_sums_final<T><<<(F + 7) / 8, 256, 0, st>>>(part, (int)nb, F, (T*)out);
  HG_LAUNCHED();
  return HG_OK;
}

// GIN combine (models.py:220-240): out = rnd(rnd(x * ope) + rnd(a * lam)), the
// products formed in fp64 (lam is a Python float; x * ope of two fp16 values is
// exact in fp32 already).  Backward: gx = rnd(g * ope), ga = rnd(g * lam) and
// the (1 + eps) gradient rnd(sum x * g) with an fp64 sum (per-block partials,
// fixed-order final fold: deterministic).
template <typename T, int V>
__global__ void __launch_bounds__(256)
k_scale_combine(const T* __restrict__ x, const T* __restrict__ a, const T* __restrict__ ope,
                double lam, int64_t count, T* __restrict__ out) {
  using Raw = typename Vec<T, V>::raw;
  const double o = Num<T>::to_d(*ope);
  const int64_t nv = count / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    Raw xv = reinterpret_cast<const Raw*>(x)[i];
    const Raw av = reinterpret_cast<const Raw*>(a)[i];
    T* xe = reinterpret_cast<T*>(&xv);
    const T* ae = reinterpret_cast<const T*>(&av);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const T u = Num<T>::from_d(Num<T>::to_d(xe[k]) * o);
      const T v = Num<T>::from_d(Num<T>::to_d(ae[k]) * lam);
      xe[k] = Num<T>::add(u, v);
    }
    reinterpret_cast<Raw*>(out)[i] = xv;
  }
}

constexpr int kCombBlocks = 148 * 8;

template <typename T, int V>
__global__ void __launch_bounds__(256)
k_scale_combine_bwd(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ ope,
                    double lam, int64_t count, T* __restrict__ gx, T* __restrict__ ga,
                    double* __restrict__ part) {
  using Raw = typename Vec<T, V>::raw;
  __shared__ double red[8];
  const double o = Num<T>::to_d(*ope);
  const int64_t nv = count / V;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Raw gv = reinterpret_cast<const Raw*>(g)[i];
    const T* ge = reinterpret_cast<const T*>(&gv);
    if (part) {
      const Raw xv = reinterpret_cast<const Raw*>(x)[i];
      const T* xe = reinterpret_cast<const T*>(&xv);
#pragma unroll
      for (int k = 0; k < V; ++k) acc = fma(Num<T>::to_d(xe[k]), Num<T>::to_d(ge[k]), acc);
    }
    if (gx) {
      Raw r;
      T* re = reinterpret_cast<T*>(&r);
#pragma unroll
      for (int k = 0; k < V; ++k) re[k] = Num<T>::from_d(Num<T>::to_d(ge[k]) * o);
      reinterpret_cast<Raw*>(gx)[i] = r;
    }
    if (ga) {
      Raw r;
      T* re = reinterpret_cast<T*>(&r);
#pragma unroll
      for (int k = 0; k < V; ++k) re[k] = Num<T>::from_d(Num<T>::to_d(ge[k]) * lam);
      reinterpret_cast<Raw*>(ga)[i] = r;
    }
  }
  if (!part) return;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

template <typename T>
__global__ void k_scale_combine_fold(const double* __restrict__ part, int nb, T* __restrict__ gope) {
  __shared__ double red[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) t += part[i];
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) u += red[w];
    *gope = Num<T>::from_d(u);
  }
}

}  // namespace hg

using namespace hg;

extern "C" int hg_scale_combine(const void* x, const void* a, const void* one_plus_eps,
                                double lam, int64_t count, void* out, int dtype, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(count >= 0 && one_plus_eps, "hg_scale_combine: bad arguments");
  if (count == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = count % 8 == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(a) |
                                       reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (dtype == HG_F16) {
    if (vec) k_scale_combine<__half, 8><<<grid_for(count / 8, 256, 148 * 16), 256, 0, st>>>(
        (const __half*)x, (const __half*)a, (const __half*)one_plus_eps, lam, count, (__half*)out);
    else k_scale_combine<__half, 1><<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(
        (const __half*)x, (const __half*)a, (const __half*)one_plus_eps, lam, count, (__half*)out);
  } else {
    if (vec) k_scale_combine<float, 4><<<grid_for(count / 4, 256, 148 * 16), 256, 0, st>>>(
        (const float*)x, (const float*)a, (const float*)one_plus_eps, lam, count, (float*)out);
    else k_scale_combine<float, 1><<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(
        (const float*)x, (const float*)a, (const float*)one_plus_eps, lam, count, (float*)out);
  }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_scale_combine_bwd_workspace(size_t* bytes) {
  HG_REQUIRE(bytes, "hg_scale_combine_bwd_workspace: bad arguments");
  *bytes = (size_t)kCombBlocks * sizeof(double);
  return HG_OK;
}

extern "C" int hg_scale_combine_bwd(const void* x, const void* g, const void* one_plus_eps,
                                    double lam, int64_t count, void* gx, void* ga, void* gope,
                                    int dtype, void* ws, size_t ws_bytes, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(count >= 0 && one_plus_eps, "hg_scale_combine_bwd: bad arguments");
  if (count == 0) {
    if (gope) HG_CUDA(cudaMemsetAsync(gope, 0, dtype == HG_F16 ? 2 : 4, as_stream(stream)));
    return HG_OK;
  }
  HG_REQUIRE(g, "hg_scale_combine_bwd: null gradient");
  HG_REQUIRE(!gope || (x && ws && ws_bytes >= (size_t)kCombBlocks * sizeof(double)),
             "hg_scale_combine_bwd: the (1+eps) gradient needs x and a workspace");
  cudaStream_t st = as_stream(stream);
  double* part = gope ? (double*)ws : nullptr;
  const int64_t V = dtype == HG_F16 ? 8 : 4;
  const bool vec = count % V == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) |
                                       reinterpret_cast<uintptr_t>(gx) | reinterpret_cast<uintptr_t>(ga)) & 15) == 0;
  const int nb = grid_for(vec ? count / V : count, 256, kCombBlocks);
  if (dtype == HG_F16) {
    if (vec) k_scale_combine_bwd<__half, 8><<<nb, 256, 0, st>>>(
        (const __half*)x, (const __half*)g, (const __half*)one_plus_eps, lam, count, (__half*)gx,
        (__half*)ga, part);
    else k_scale_combine_bwd<__half, 1><<<nb, 256, 0, st>>>(
        (const __half*)x, (const __half*)g, (const __half*)one_plus_eps, lam, count, (__half*)gx,
        (__half*)ga, part);
  } else {
    if (vec) k_scale_combine_bwd<float, 4><<<nb, 256, 0, st>>>(
        (const float*)x, (const float*)g, (const float*)one_plus_eps, lam, count, (float*)gx,
        (float*)ga, part);
    else k_scale_combine_bwd<float, 1><<<nb, 256, 0, st>>>(
        (const float*)x, (const float*)g, (const float*)one_plus_eps, lam, count, (float*)gx,
        (float*)ga, part);
  }
  HG_LAUNCHED();
  if (gope) {
    if (dtype == HG_F16) k_scale_combine_fold<__half><<<1, 1024, 0, st>>>(part, nb, (__half*)gope);
    else k_scale_combine_fold<float><<<1, 1024, 0, st>>>(part, nb, (float*)gope);
    HG_LAUNCHED();
  }
  return HG_OK;
}

namespace hg {
// relu backward (models.py:176-185) from the ReLU's output: g where y > 0, else 0.
template <typename T, int V>
__global__ void k_relu_grad(const T* __restrict__ y, const T* __restrict__ g, int64_t count,
                            T* __restrict__ out) {
  using Raw = typename Vec<T, V>::raw;
  const int64_t nv = count / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Raw yv = reinterpret_cast<const Raw*>(y)[i];
    Raw gv = reinterpret_cast<const Raw*>(g)[i];
    const T* ye = reinterpret_cast<const T*>(&yv);
    T* ge = reinterpret_cast<T*>(&gv);
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (!Num<T>::gt0(ye[k])) ge[k] = Num<T>::zero();
    reinterpret_cast<Raw*>(out)[i] = gv;
  }
}
}  // namespace hg

extern "C" int hg_relu_grad(const void* y, const void* g, int64_t count, void* out, int dtype,
                            void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  if (count == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t V = dtype == HG_F16 ? 8 : 4;
  const bool vec = count % V == 0 && ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(g) |
                                       reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (dtype == HG_F16) {
    if (vec) k_relu_grad<__half, 8><<<grid_for(count / 8, 256, 148 * 16), 256, 0, st>>>(
        (const __half*)y, (const __half*)g, count, (__half*)out);
    else k_relu_grad<__half, 1><<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(
        (const __half*)y, (const __half*)g, count, (__half*)out);
  } else {
    if (vec) k_relu_grad<float, 4><<<grid_for(count / 4, 256, 148 * 16), 256, 0, st>>>(
        (const float*)y, (const float*)g, count, (float*)out);
    else k_relu_grad<float, 1><<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(
        (const float*)y, (const float*)g, count, (float*)out);
  }
  HG_LAUNCHED();
  return HG_OK;
}

namespace hg {
// dst[i, :] = src[idx[i], :] in words W (wpr words per row).  Each thread keeps
// 8 independent gathers in flight (the idx -> src chain is latency-bound).
template <typename W>
__global__ void __launch_bounds__(256)
k_gather_rows_bytes(const W* __restrict__ src, const int32_t* __restrict__ idx, int64_t rows,
                    int wpr, W* __restrict__ dst) {
  constexpr int U = 8;
  const int64_t total = rows * (int64_t)wpr;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U; base < total;
       base += (int64_t)gridDim.x * blockDim.x * U) {
    int64_t pos[U];
    W v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x + threadIdx.x;
      pos[u] = -1;
      if (i < total) {
        const int64_t r = i / wpr;
        pos[u] = (int64_t)__ldg(idx + r) * wpr + (i - r * wpr);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pos[u] >= 0) v[u] = __ldg(src + pos[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x + threadIdx.x;
      if (i < total) dst[i] = v[u];
    }
  }
}
}  // namespace hg

extern "C" int hg_gather_rows(const void* src, const int32_t* idx, int64_t rows,
                              int32_t row_bytes, void* dst, void* stream) {
  HG_REQUIRE(rows >= 0 && row_bytes > 0 && row_bytes % 2 == 0, "hg_gather_rows: bad shape");
  if (rows == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const bool a8 = row_bytes % 8 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7) == 0;
  const bool a4 = row_bytes % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3) == 0;
  if (a8) {
    const int wpr = row_bytes / 8;
    k_gather_rows_bytes<uint2><<<grid_for(rows * wpr, 256 * 8, 148 * 16), 256, 0, st>>>(
        (const uint2*)src, idx, rows, wpr, (uint2*)dst);
  } else if (a4) {
    const int wpr = row_bytes / 4;
    k_gather_rows_bytes<uint32_t><<<grid_for(rows * wpr, 256 * 8, 148 * 16), 256, 0, st>>>(
        (const uint32_t*)src, idx, rows, wpr, (uint32_t*)dst);
  } else {
    const int wpr = row_bytes / 2;
    k_gather_rows_bytes<uint16_t><<<grid_for(rows * wpr, 256 * 8, 148 * 16), 256, 0, st>>>(
        (const uint16_t*)src, idx, rows, wpr, (uint16_t*)dst);
  }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_bias_scale_rows(const void* x, const void* bias, const void* row_scale,
                                  int64_t rows, int32_t F, void* out, int dtype, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(rows >= 0 && F > 0, "hg_bias_scale_rows: bad shape");
  if (rows == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == HG_F16) launch_bias_scale<__half>(x, bias, row_scale, rows, F, out, st);
  else launch_bias_scale<float>(x, bias, row_scale, rows, F, out, st);
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_col_sums_workspace(int64_t rows, int32_t F, size_t* bytes) {
  HG_REQUIRE(bytes && rows >= 0 && F > 0, "hg_col_sums_workspace: bad arguments");
  *bytes = (size_t)kColBlocks * F * sizeof(float);
  return HG_OK;
}

extern "C" int hg_col_sums(const void* x, int64_t rows, int32_t F, void* out, int dtype, void* ws,
                           size_t ws_bytes, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(rows >= 0 && F > 0, "hg_col_sums: bad shape");
  HG_REQUIRE(ws && ws_bytes >= (size_t)kColBlocks * F * sizeof(float),
             "hg_col_sums: workspace too small");
  cudaStream_t st = as_stream(stream);
  if (rows == 0) {
    HG_CUDA(cudaMemsetAsync(out, 0, (size_t)F * (dtype == HG_F16 ? 2 : 4), st));
    return HG_OK;
  }
  return dtype == HG_F16 ? launch_col_sums<__half>(x, rows, F, out, (float*)ws, st)
                         : launch_col_sums<float>(x, rows, F, out, (float*)ws, st);
}
