// Experiment (not product code): random-row gather throughput through the
// TMA engine instead of the LSU.  Same access pattern as hg_gather_probe (the
// C3 column stream, rows of X), three front ends:
//   mode 0: LDG.256 team loads (the product probe's scheme, for reference)
//   mode 1: tile::gather4 TMA (cp.async.bulk.tensor.2d ... gather4): one
//           instruction fetches 4 rows into shared memory
//   mode 2: cp.async.bulk (non-tensor) per row
// Each warp pipelines its own ring of NST stages of 128 rows (lane j fetches
// rows 4j..4j+3), waits on the stage's mbarrier and XORs the rows out of
// shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                        int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2),
      "r"(r3)
      : "memory");
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int NST>
__global__ void __launch_bounds__(128) k_tma_gather(const int* __restrict__ cols, int64_t E,
                                                    const __grid_constant__ CUtensorMap map,
                                                    const char* __restrict__ x, int64_t ld,
                                                    int row_bytes, int mode,
                                                    unsigned* out) {
  extern __shared__ __align__(128) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int stage_bytes = 128 * row_bytes;
  char* ring = smem + 1024 + (size_t)warp * NST * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * NST;
  if (lane == 0)
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t tw = (int64_t)gridDim.x * nwarps;
  const int64_t nb = (E + 127) / 128;  // batches of 128 edges
  unsigned acc = 0;
  uint32_t phase[NST];
  for (int s = 0; s < NST; ++s) phase[s] = 0;
  auto issue = [&](int64_t b, int s) {
    const int64_t e0 = b * 128 + lane * 4;
    int r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = e0 + q < E ? __ldg(cols + e0 + q) : 0;
    if (lane == 0) mbar_expect_tx(&bars[s], (uint32_t)stage_bytes);
    __syncwarp();
    char* dst = ring + (size_t)s * stage_bytes + (size_t)lane * 4 * row_bytes;
    if (mode == 1) {
      gather4(dst, &map, &bars[s], 0, r[0], r[1], r[2], r[3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        bulk_row(dst + q * row_bytes, x + (int64_t)r[q] * ld, (uint32_t)row_bytes, &bars[s]);
    }
  };
  int64_t b = gw;
  // prologue
  for (int s = 0; s < NST; ++s)
    if (b + (int64_t)s * tw < nb) issue(b + (int64_t)s * tw, s);
  int s = 0;
  for (; b < nb; b += tw) {
    mbar_wait(&bars[s], phase[s]);
    phase[s] ^= 1;
    const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * stage_bytes);
    const int words = stage_bytes / 16;
    for (int i = lane; i < words; i += 32) {
      uint4 v = st[i];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncwarp();
    const int64_t nxt = b + (int64_t)NST * tw;
    if (nxt < nb) issue(nxt, s);
    s = s + 1 == NST ? 0 : s + 1;
  }
  for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc == 0x9e3779b9u) atomicXor(out, acc);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int tma_probe(const int* cols, int64_t E, const void* x, int64_t rows,
                         int64_t ld_bytes, int row_bytes, int mode, int ctas_per_sm, int nst,
                         unsigned* out, void* stream) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess)
      return -1;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)(row_bytes / 2), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)(row_bytes / 2), 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(x), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 1000 + (int)r;
  const int warps = 4;
  size_t smem = 1024 + (size_t)warps * nst * 128 * row_bytes;
  cudaStream_t st = (cudaStream_t)stream;
  int grid = 148 * ctas_per_sm;
  cudaError_t e;
#define L(N)                                                                                  \
  e = cudaFuncSetAttribute(k_tma_gather<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           (int)smem);                                                        \
  if (e != cudaSuccess) return 2000 + (int)e;                                                 \
  k_tma_gather<N><<<grid, warps * 32, smem, st>>>(cols, E, map, (const char*)x, ld_bytes,      \
                                                   row_bytes, mode, out);
  if (nst == 2) { L(2) } else if (nst == 3) { L(3) } else { L(4) }
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 3000 + (int)e;
}
