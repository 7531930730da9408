// Experiment (not product code): random-row gather throughput with 16-byte vs
// 32-byte (LDG.256) lane loads, same access pattern as hg_gather_probe.
#include <cstdint>
#include <cuda_runtime.h>

struct V8 { uint32_t a[8]; };

template <int MODE>
__device__ __forceinline__ V8 ld256(const void* p) {
  V8 v;
  if constexpr (MODE == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]),
                   "=r"(v.a[5]), "=r"(v.a[6]), "=r"(v.a[7])
                 : "l"(p));
    return v;
  }
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]),
                 "=r"(v.a[5]), "=r"(v.a[6]), "=r"(v.a[7])
               : "l"(p));
  return v;
}

template <int TEAM, int BYTES, int MODE = 0>
__global__ void __launch_bounds__(256) k_probe(const int* __restrict__ cols, int64_t E,
                                               const char* __restrict__ x, int64_t ld,
                                               unsigned* out) {
  constexpr int RPL = 32 / TEAM;
  const int lane = threadIdx.x & 31, sub = lane % TEAM, slot = lane / TEAM;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned acc = 0;
  for (int64_t base = warp * 32; base < E; base += nw * 32) {
    const int c = base + lane < E ? __ldg(cols + base + lane) : -1;
    if constexpr (BYTES == 32) {
      V8 v[TEAM];
#pragma unroll
      for (int k = 0; k < TEAM; ++k) {
        const int r = __shfl_sync(0xffffffffu, c, k * RPL + slot);
        if (r >= 0) v[k] = ld256<MODE>(x + (int64_t)r * ld + sub * 32);
        else for (int i = 0; i < 8; ++i) v[k].a[i] = 0;
      }
#pragma unroll
      for (int k = 0; k < TEAM; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc ^= v[k].a[i];
    } else {
      int4 v[TEAM];
#pragma unroll
      for (int k = 0; k < TEAM; ++k) {
        const int r = __shfl_sync(0xffffffffu, c, k * RPL + slot);
        v[k] = r >= 0 ? __ldg(reinterpret_cast<const int4*>(x + (int64_t)r * ld + sub * 16))
                      : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < TEAM; ++k) acc ^= (unsigned)(v[k].x ^ v[k].y ^ v[k].z ^ v[k].w);
    }
  }
  for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc == 0x9e3779b9u) atomicXor(out, acc);
}

extern "C" int probe(const int* cols, int64_t E, const void* x, int64_t ld, int row_bytes,
                     int lane_bytes, unsigned* out, int blocks, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const char* xb = (const char*)x;
  if (lane_bytes == 33) {
    switch (row_bytes / 32) {
      case 2: k_probe<2, 32, 1><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      case 4: k_probe<4, 32, 1><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      case 8: k_probe<8, 32, 1><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      default: return 1;
    }
  } else if (lane_bytes == 32) {
    switch (row_bytes / 32) {
      case 2: k_probe<2, 32><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      case 4: k_probe<4, 32><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      case 8: k_probe<8, 32><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      default: return 1;
    }
  } else {
    switch (row_bytes / 16) {
      case 4: k_probe<4, 16><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      case 8: k_probe<8, 16><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      case 16: k_probe<16, 16><<<blocks, 256, 0, st>>>(cols, E, xb, ld, out); break;
      default: return 1;
    }
  }
  return (int)cudaGetLastError();
}
