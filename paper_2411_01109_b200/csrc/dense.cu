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

}  // namespace hg

using namespace hg;

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
