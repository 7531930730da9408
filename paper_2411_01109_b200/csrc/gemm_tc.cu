// Dense per-layer feature GEMM on the 5th-generation tensor cores with the GCN
// epilogue fused in:
//
//   out[m, n] = rnd(rnd(rnd(sum_k A[m, k] Bt[n, k]) + bias[n]) * row_scale[m])
//
// i.e. models.matmul (fp32 accumulation, one rounding, models.py:141-158) ->
// add_bias (161-166) -> the aggregation's left-norm input scaling
// (kernels.py:358-361), each rounding exactly where the reference rounds.
//
// Persistent, one CTA (320 threads) per SM over 128-row tiles:
//   warp 0 / lane 0   TMA producer: 64-wide K slabs of A (128 x 64) and Bt
//                     (N x 64) into a 3-8 deep shared-memory ring
//                     (cp.async.bulk.tensor, SWIZZLE_128B, OOB -> zeros),
//                     running ahead across tile boundaries;
//   warp 1 / lane 0   MMA issuer: 4 x tcgen05.mma.cta_group::1.kind::f16
//                     (M=128, N, K=16) per slab into one of two fp32 TMEM
//                     accumulators; tcgen05.commit frees the slab / hands the
//                     accumulator to the epilogue;
//   warps 2-9         epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes
//                     32(w%4)..+31 = rows; the two warps of a quarter split
//                     the 16-column chunks), fp16x2 rounding, bias, row scale,
//                     staged in shared memory, coalesced 16-byte stores; it
//                     overlaps the next tile's MMAs.
// Fed by TMA and drained from TMEM, the kernel is bound by reading A once
// (HBM), which is what the GCN layer-1 GEMM (233K x 608 x 64) costs.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "hg_common.cuh"

namespace hg {

constexpr int kTcBM = 128;  // rows per tile (UMMA M)
constexpr int kTcBK = 64;   // fp16 K elements per slab = one 128-byte swizzle row

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
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand in a 128-byte-swizzled tile: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_kmajor_desc(const void* tile) {
  const uint64_t addr = smem_u32(tile);
  uint64_t d = (addr >> 4) & 0x3FFFull;  // start address
  d |= 1ull << 16;                       // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;      // stride byte offset: 8 rows x 128 B
  d |= 1ull << 46;                       // descriptor version (sm_100)
  d |= 2ull << 61;                       // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_f16_f32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ void epi_bar_n(int threads) {  // named barrier over the epilogue warps
  asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
}

// packed fp32 FMA (FFMA2): d = a * b + c on both lanes, each lane one IEEE fma
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long x, y, z, d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(z) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}

// smem ring depth for a given N (the ring plus the output staging tile fit ~200 KB)
template <int N, bool RESB>
struct TcCfg {
  static constexpr uint32_t kABytes = kTcBM * kTcBK * 2;
  static constexpr uint32_t kBBytes = N * kTcBK * 2;
  // RESB: all of Bt (<= kMaxResKb slabs) stays resident in shared memory for
  // the CTA's lifetime; the ring then streams A only
  static constexpr int kMaxResKb = RESB ? (int)((32u * 1024u) / kBBytes) : 0;
  static constexpr uint32_t kRes = (uint32_t)kMaxResKb * kBBytes;
  static constexpr uint32_t kSlot = kABytes + (RESB ? 0 : kBBytes);  // ring bytes per stage
  // N % 64 == 0: two 128-byte-swizzled staging tiles written back by TMA
  // stores (double-buffered); otherwise one padded tile + coalesced stores
  static constexpr bool kTmaStore = N % 64 == 0;
  static constexpr uint32_t kPitch = N * 2 + 16;  // padded staging row pitch (bytes)
  static constexpr uint32_t kBufs = (kTmaStore && N <= 128) ? 2 : 1;
  // (a width n_out < N, i.e. N padded up from 8 mod 16, takes the padded tile)
  static constexpr uint32_t kStageT = kTmaStore ? kBufs * kTcBM * N * 2 : 0;
  static constexpr uint32_t kStage = kStageT > kTcBM * kPitch ? kStageT : kTcBM * kPitch;
  static constexpr int kStages0 = (int)((200u * 1024u - kStage - kRes) / kSlot);
  static constexpr int kStages = kStages0 > 8 ? 8 : kStages0;
  static constexpr uint32_t kCols = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 2 * N <= 256 ? 256 : 512;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kSlot + kRes + kStage +
                                  (2 * kStages + 5) * 8 + 16 + N * 2 + N * 8;
};

// Epilogue: kEpiWarps warps, two per TMEM lane quarter (warp w reads lanes
// 32 (w % 4) ..); the pair splits the tile's 16-column chunks between them.
constexpr int kEpiWarps = 8;
constexpr int kTcThreads = 64 + 32 * kEpiWarps;

// Persistent: one CTA per SM loops over 128-row tiles.  Warp 0 = TMA producer
// (runs ahead across tile boundaries through the ring), warp 1 = MMA issuer,
// warps 2-5 = epilogue.  Two TMEM accumulators: the epilogue of tile i
// overlaps the MMAs of tile i+1.  The epilogue stages the fp16 tile in shared
// memory and writes it back with coalesced 16-byte stores.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

template <int N, bool RESB>
__global__ void __launch_bounds__(kTcThreads, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
          const __grid_constant__ CUtensorMap map_o, int64_t m, int num_kb, const __half* __restrict__ bias,
          const __half* __restrict__ row_scale, __half* __restrict__ out, int64_t ldo, int relu,
          int n_out, const __half* __restrict__ dot_a, const __half* __restrict__ dot_b,
          int dot_heads, int dot_fh, __half* __restrict__ dot_out_a, __half* __restrict__ dot_out_b,
          const __half* __restrict__ mask, int64_t ldm) {
  using C = TcCfg<N, RESB>;
  constexpr int S = C::kStages;
  constexpr int kEpiThreads = 32 * kEpiWarps;
  // instruction descriptor: f16 x f16 -> f32, both K-major, M = 128, N
  constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcBM >> 4) << 24);

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-aligned, offset from smem_raw so the compiler keeps the shared state
  // space (LDS / STS, not generic LD / ST)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sa = base;                          // [S][128 x 128 B]
  unsigned char* sb = base + S * C::kABytes;         // ring: [S][N x 128 B]; RESB: [kb][N x 128 B]
  unsigned char* stage = sb + (RESB ? C::kRes : S * C::kBBytes);  // output staging
  // head vectors for the epilogue's dots: [N / 2] column pairs as fp32
  // (a_l[2p], a_l[2p + 1], a_r[2p], a_r[2p + 1])
  float4* svec = reinterpret_cast<float4*>(stage + C::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + C::kStage + N * 8);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;                       // [2]
  uint64_t* tempty = tfull + 2;                      // [2]
  uint64_t* bfull = tempty + 2;                      // resident B landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  __half* sbias = reinterpret_cast<__half*>(tmem_slot + 4);  // [N], zero past n_out

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = (m + kTcBM - 1) / kTcBM;
  // TMA-store epilogue only when every one of the N columns is stored
  const bool tstore = C::kTmaStore && n_out == N;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiThreads);
    }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  for (int j = threadIdx.x; j < N; j += blockDim.x)
    sbias[j] = (bias && j < n_out) ? bias[j] : __ushort_as_half(0);
  if (dot_out_a) {  // head vectors by column pair, fp32, for the epilogue's dots
    for (int p = threadIdx.x; p < N / 2; p += blockDim.x)
      svec[p] = make_float4(__half2float(dot_a[2 * p]), __half2float(dot_a[2 * p + 1]),
                            __half2float(dot_b[2 * p]), __half2float(dot_b[2 * p + 1]));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      if (RESB) {
        mbar_expect_tx(bfull, (uint32_t)num_kb * C::kBBytes);
        for (int kb = 0; kb < num_kb; ++kb)
          tma_load_2d(sb + kb * C::kBBytes, &map_b, bfull, kb * kTcBK, 0);
      }
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          mbar_expect_tx(&full[s], RESB ? C::kABytes : C::kABytes + C::kBBytes);
          tma_load_2d(sa + s * C::kABytes, &map_a, &full[s], kb * kTcBK, (int)(tile * kTcBM));
          if (!RESB) tma_load_2d(sb + s * C::kBBytes, &map_b, &full[s], kb * kTcBK, 0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      if (RESB) mbar_wait(bfull, 0);
      uint32_t it = 0, tc = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
        const uint32_t a = tc & 1;
        mbar_wait(&tempty[a], ((tc >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + a * N;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = sw128_kmajor_desc(sa + s * C::kABytes);
          const uint64_t db = sw128_kmajor_desc(sb + (RESB ? kb : s) * C::kBBytes);
#pragma unroll
          for (int k = 0; k < kTcBK / 16; ++k)  // 16 fp16 = 32 B steps inside the swizzle row
            umma_f16_f32(acc, da + 2 * k, db + 2 * k, kIdesc, (kb | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[a]);
      }
    }
    __syncwarp();
  } else {  // epilogue warps 2..: TMEM lane quarter = warp % 4, chunk parity = pair member
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;  // 0 / 1: 16-column chunks of this parity
    const int r = q * 32 + lane;       // tile row = TMEM lane
    const int et = threadIdx.x - 64;   // 0 .. kEpiThreads - 1
    const __half2 z2 = __half2half2(__ushort_as_half(0));
    const __half2* bias2 = reinterpret_cast<const __half2*>(sbias);
    constexpr int kChunks = N / 16;
    constexpr int kPer = (kChunks + 1) / 2;  // chunks per warp half (the last may be absent)
    // this warp half's 16-column chunks, in column order: whole groups of G
    // chunks alternate between the halves -- G = 1 (chunk parity) normally, a
    // head's width with the head dots so each thread owns whole heads
    const int G = dot_out_a ? dot_fh >> 4 : 1;
    int mych[kPer], myhd[kPer];
    unsigned last = 0;  // bit k: chunk k completes its head (for this thread)
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      mych[k] = (2 * (k / G) + half) * G + k % G;
      myhd[k] = 2 * (k / G) + half;
      if (k % G == G - 1 || k == kPer - 1) last |= 1u << k;
    }
    // ReLU backward folded in (mask != NULL): out = mask > 0 ? out : +0, the
    // mask chunks of this thread's columns loaded one tile ahead into registers
    // (issued when a tile's chunks are done; a second register set loaded a
    // whole tile period ahead and moved over measured slower: 2.86 vs 2.09 ms)
    uint4 ym[kPer][2];
#define HG_LOAD_MASK(dst, t)                                                                  \
  do {                                                                                        \
    const int64_t mr_ = (t) * kTcBM + r;                                                      \
    _Pragma("unroll") for (int k = 0; k < kPer; ++k) {                                        \
      const bool ok_ = (t) < num_tiles && mr_ < m && (kChunks % 2 == 0 || mych[k] < kChunks); \
      _Pragma("unroll") for (int hh = 0; hh < 2; ++hh) dst[k][hh] =                           \
          ok_ ? __ldg(reinterpret_cast<const uint4*>(mask + mr_ * ldm + mych[k] * 16 + hh * 8))  \
              : make_uint4(0, 0, 0, 0);                                                       \
    }                                                                                         \
  } while (0)
    if (mask) HG_LOAD_MASK(ym, (int64_t)blockIdx.x);
    uint32_t tc = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
      const uint32_t a = tc & 1;
      const int64_t m0 = tile * kTcBM;
      const int64_t row = m0 + r;
      const bool live = row < m;
      mbar_wait(&tfull[a], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      unsigned char* sbuf = stage + (tstore ? (tc % C::kBufs) * (kTcBM * N * 2) : 0);
      if (tstore) {
        // the TMA store issued from this buffer kBufs tiles ago has read it
        if (et == 0) {
          if constexpr (C::kBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        epi_bar_n(kEpiThreads);
      }
      unsigned char* srow = sbuf + r * (tstore ? 128 : C::kPitch);
      // head dots (GAT s_l / s_r): this thread owns whole heads and meets their
      // chunks in column order -- one running register pair (even / odd column
      // lanes) per head, rounded and stored when the head is complete
      float2 run_l = make_float2(0.0f, 0.0f), run_r = run_l;
      // TMEM loads two chunks per wait
#pragma unroll
      for (int k0 = 0; k0 < kPer; k0 += 2) {
        if constexpr (kChunks % 2 == 1) {  // warp-uniform: half 1 has one chunk fewer
          if (mych[k0] >= kChunks) break;
        }
        uint32_t vv[2][16];
        const bool two = k0 + 1 < kPer && (kChunks % 2 == 0 || mych[k0 + 1] < kChunks);
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + a * N + mych[k0] * 16, vv[0]);
        if (two) tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + a * N + mych[k0 + 1] * 16, vv[1]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int c0 = mych[k0 + u] * 16;
          __align__(16) __half2 h[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            h[j] = __floats2half2_rn(__uint_as_float(vv[u][2 * j]), __uint_as_float(vv[u][2 * j + 1]));
          if (bias) {
#pragma unroll
            for (int j = 0; j < 8; ++j) h[j] = __hadd2_rn(h[j], bias2[c0 / 2 + j]);
          }
          if (row_scale) {
            // loaded here, not at the tile start: a load there waited on the
            // previous tile's in-flight mask prefetch (register reuse)
            const __half2 sv2 = __half2half2(live ? __ldg(row_scale + row) : __float2half_rn(1.0f));
#pragma unroll
            for (int j = 0; j < 8; ++j) h[j] = __hmul2_rn(h[j], sv2);  // (loaded per chunk: L1)
          }
          if (dot_out_a) {  // z . a over this chunk's 16 columns (exact products, fp32 sum)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v = svec[c0 / 2 + j];
              const float2 zf = __half22float2(h[j]);
              run_l = ffma2(zf, make_float2(v.x, v.y), run_l);
              run_r = ffma2(zf, make_float2(v.z, v.w), run_r);
            }
            if ((last >> (k0 + u)) & 1) {  // head complete: one rounding, then restart
              if (live) {
                const int hd = myhd[k0 + u];
                dot_out_a[row * dot_heads + hd] = __float2half_rn(run_l.x + run_l.y);
                dot_out_b[row * dot_heads + hd] = __float2half_rn(run_r.x + run_r.y);
              }
              run_l = run_r = make_float2(0.0f, 0.0f);
            }
          }
          if (mask) {  // relu backward: y > 0 ? g : +0 (NaN y -> 0), y = this chunk's mask
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4 yq = ym[k0 + u][j >> 2];  // (no address taken: stays in registers)
              const uint32_t yw = (j & 3) == 0 ? yq.x : (j & 3) == 1 ? yq.y : (j & 3) == 2 ? yq.z : yq.w;
              const unsigned mk = __hgt2_mask(*reinterpret_cast<const __half2*>(&yw), z2);
              h[j] = __halves2half2(__ushort_as_half((unsigned short)(__half_as_ushort(__low2half(h[j])) & mk)),
                                    __ushort_as_half((unsigned short)(__half_as_ushort(__high2half(h[j])) & (mk >> 16))));
            }
          }
          if (relu) {  // models.relu: x > 0 ? x : +0 (NaN -> 0)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const unsigned mk = __hgt2_mask(h[j], z2);
              h[j] = __halves2half2(__ushort_as_half((unsigned short)(__half_as_ushort(__low2half(h[j])) & mk)),
                                    __ushort_as_half((unsigned short)(__half_as_ushort(__high2half(h[j])) & (mk >> 16))));
            }
          }
          if (tstore) {
            // 64-column boxes of 128 rows x 128 B, 16-byte chunk c of row r at c ^ (r & 7)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int c = c0 / 8 + hh;
              unsigned char* dst = sbuf + (c / 8) * (kTcBM * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
              *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&h[4 * hh]);
            }
          } else {
            reinterpret_cast<uint4*>(srow + c0 * 2)[0] = *reinterpret_cast<const uint4*>(&h[0]);
            reinterpret_cast<uint4*>(srow + c0 * 2)[1] = *reinterpret_cast<const uint4*>(&h[4]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[a]);  // accumulator drained: the MMA warp may reuse it
      if (mask) HG_LOAD_MASK(ym, tile + gridDim.x);  // in flight over the store and the next MMA
      if (tstore) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> TMA
        epi_bar_n(kEpiThreads);
        if (et == 0) {
#pragma unroll
          for (int bx = 0; bx < N / 64; ++bx)
            tma_store_2d(&map_o, sbuf + bx * (kTcBM * 128), bx * 64, (int)m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else {
        epi_bar_n(kEpiThreads);
        // coalesced write-back of the live rows: 16-byte chunks, row-major
        const int rows = (int)((m - m0) < kTcBM ? (m - m0) : kTcBM);
        const int CPR = n_out / 8;  // n_out <= N: columns past n_out are padding
        for (int ch = et; ch < rows * CPR; ch += kEpiThreads) {
          const int rr = ch / CPR, c8 = ch - rr * CPR;
          *reinterpret_cast<uint4*>(out + (m0 + rr) * ldo + c8 * 8) =
              *reinterpret_cast<const uint4*>(sbuf + rr * C::kPitch + c8 * 16);
        }
        epi_bar_n(kEpiThreads);
      }
    }
    if (tstore && et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kCols));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;  // process-wide driver entry point cache
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D fp16 tensor [rows, cols] with row pitch ld (elements), box {64 cols, box_rows}.
static int g_tma_err = 0;
static bool make_map_box(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                         uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) {
    g_tma_err = -1;
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  g_tma_err = (int)r;
  return r == CUDA_SUCCESS;
}

static bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                     uint32_t box_rows) {
  return make_map_box(map, ptr, rows, cols, ld, (uint32_t)kTcBK, box_rows);
}

struct Dots {  // epilogue extras: GAT head dots (NULL out_a: off), ReLU-backward mask (NULL: off)
  const void* a;
  const void* b;
  int heads, fh;
  void* out_a;
  void* out_b;
  const void* mask;
  int64_t ldm;
};

template <int N, bool RESB>
static int launch_gemm_tc_v(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                            int64_t m, int num_kb, const void* bias, const void* row_scale,
                            void* out, int64_t ldo, int relu, int n_out, const Dots& dt,
                            cudaStream_t st) {
  constexpr size_t smem = TcCfg<N, RESB>::kSmem;
  static_assert(smem <= 227 * 1024, "gemm_tc shared memory budget");
  static_assert(TcCfg<N, RESB>::kStages >= 2, "gemm_tc ring too shallow");
  HG_CUDA(cudaFuncSetAttribute(k_gemm_tc<N, RESB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tiles = (m + kTcBM - 1) / kTcBM;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  k_gemm_tc<N, RESB><<<grid, kTcThreads, smem, st>>>(
      ma, mb, mo, m, num_kb, (const __half*)bias, (const __half*)row_scale, (__half*)out, ldo, relu,
      n_out, (const __half*)dt.a, (const __half*)dt.b, dt.heads, dt.fh, (__half*)dt.out_a,
      (__half*)dt.out_b, (const __half*)dt.mask, dt.ldm);
  HG_LAUNCHED();
  return HG_OK;
}

template <int N>
static int launch_gemm_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                          int64_t m, int64_t k, const void* bias, const void* row_scale, void* out,
                          int64_t ldo, int relu, int n_out, const Dots& dt, cudaStream_t st) {
  const int num_kb = (int)((k + kTcBK - 1) / kTcBK);
  if (num_kb <= TcCfg<N, true>::kMaxResKb)
    return launch_gemm_tc_v<N, true>(ma, mb, mo, m, num_kb, bias, row_scale, out, ldo, relu,
                                     n_out, dt, st);
  return launch_gemm_tc_v<N, false>(ma, mb, mo, m, num_kb, bias, row_scale, out, ldo, relu,
                                    n_out, dt, st);
}


// ---------------------------------------------------------------------------
// Weight gradient of the per-layer GEMM (matmul's backward, models.py:151-155):
//
//   out[m, n] = rnd(sum_k A[k, m] B[k, n])        A = x [K, M], B = g [K, N]
//
// The contraction runs over the vertices (K = 233K .. 16.7M rows) while the
// output is tiny (M, N <= a few hundred), so the kernel splits K across the
// SMs: CTA (group, split) streams its slab range of A and B once through a
// TMA ring and keeps one fp32 TMEM accumulator per 128-row tile of M (up to
// 512 TMEM columns), then writes its fp32 partial tile; hg_wgrad_reduce sums
// the partials in split order (deterministic) and rounds once.  The bias
// gradient (add_bias backward, models.py:168-170: column sums of g) rides
// along as one more accumulator fed by a constant all-ones A tile, so g is
// read once for both.  Both operands
// are row-major in HBM, i.e. MN-major for the MMA: 64-element-wide x 32-row
// TMA boxes with 128-byte swizzle are exactly the canonical MN-major SW128
// atoms (8 K-rows of 128 B, 1024 B apart; the next 64 MN elements one box on).
// Bound by reading A and B once from HBM.
// K rows per slab: 32, 64 or 128 (the deepest that leaves >= 3 ring stages);
// one TMA box = 64 (MN) x bk (K) fp16 = 128 * bk bytes
constexpr uint32_t kWgOnes = 4096;                // all-ones A tile: 2 x 16 K-rows x 128 B
constexpr int kWgMaxMT = 8;                       // 128-row M tiles per CTA

// MN-major, 128-byte-swizzled operand: LBO = next 64-element MN block,
// SBO = next 8-row K group.
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(const void* tile, uint32_t lbo) {
  const uint64_t addr = smem_u32(tile);
  uint64_t d = (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

template <int NB>
__global__ void __launch_bounds__(192, 1)
k_gemm_wgrad(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
             int64_t m, int n, int mt_total, int mt_group, int64_t slabs, int64_t slabs_per_split,
             int splits, int stages, int bk, int a_boxes, uint32_t tmem_cols, int with_bias,
             float* __restrict__ part) {
  constexpr int UN = 64 * NB;  // UMMA N
  // f16 x f16 -> f32, A and B MN-major, M = 128, N = UN
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(UN >> 3) << 17) |
                              ((uint32_t)(kTcBM >> 4) << 24);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-aligned, offset from smem_raw so the compiler keeps the shared state
  // space (LDS / STS, not generic LD / ST)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int group = blockIdx.x / splits, split = blockIdx.x - group * splits;
  const int t0 = group * mt_group;
  const int mt = min(mt_group, mt_total - t0);
  const uint32_t box = 128u * (uint32_t)bk;
  // a stage: a_boxes A half-tiles (64 M columns each; halves wholly past M are
  // neither loaded nor stored: their MMA rows only feed output rows >= M,
  // which are dropped) then NB boxes of B
  const uint32_t stage_bytes = (uint32_t)(a_boxes + NB) * box;
  unsigned char* ones = base + (size_t)stages * stage_bytes;  // kWgOnes bytes of 1.0
  uint64_t* full = reinterpret_cast<uint64_t*>(ones + kWgOnes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  // slabs split, split + splits, ...: the CTAs sweep A and B together, front
  // to back (one moving window of DRAM pages instead of a stream per CTA)
  const int64_t nkb = split < slabs ? (slabs - split + splits - 1) / splits : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the bias accumulator: rows of the all-ones tile times B = column sums of B
  const bool bias_acc = with_bias && group == 0;
  if (bias_acc) {
    for (int i = threadIdx.x; i < (int)(kWgOnes / 16); i += blockDim.x)
      reinterpret_cast<uint4*>(ones)[i] = make_uint4(0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u);
  }
  const int64_t lh = (m - (int64_t)t0 * kTcBM + 63) / 64;
  const int live_halves = lh < 2 * mt ? (int)lh : 2 * mt;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // ones tile -> tensor core

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: per slab, the live A half-tiles and NB boxes of B
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < nkb; ++it) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], (uint32_t)(live_halves + NB) * box);
        unsigned char* st = base + (size_t)s * stage_bytes;
        const int krow = (int)((split + it * splits) * bk);
        for (int hb = 0; hb < live_halves; ++hb)
          tma_load_2d(st + hb * box, &map_a, &full[s], t0 * kTcBM + 64 * hb, krow);
        for (int b = 0; b < NB; ++b)
          tma_load_2d(st + (a_boxes + b) * box, &map_b, &full[s], 64 * b, krow);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < nkb; ++it) {
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        unsigned char* st = base + (size_t)s * stage_bytes;
        unsigned char* sbt = st + a_boxes * box;
        for (int k = 0; k < bk / 16; ++k) {  // 16 K rows = 2 swizzle atoms = 2048 B
          const uint64_t db = sw128_mnmajor_desc(sbt + k * 2048, box);
          const uint32_t accum = (it | k) != 0;
          for (int t = 0; t < mt; ++t)
            umma_f16_f32(tmem + (uint32_t)(t * UN), sw128_mnmajor_desc(st + 2 * t * box + k * 2048, box),
                         db, kIdesc, accum);
          if (bias_acc)
            umma_f16_f32(tmem + (uint32_t)(mt * UN), sw128_mnmajor_desc(ones, 2048), db, kIdesc, accum);
        }
        umma_commit(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
      umma_commit(tfull);
    }
    __syncwarp();
  } else {  // epilogue warps 2..5: TMEM lane quarter q = rows 32q..32q+31 of each tile
    const int q = warp & 3;
    if (nkb > 0) {
      mbar_wait(tfull, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // tile mt (bias_acc only): any one TMEM lane holds the column sums; lane 0 -> row m
    const int tiles = mt + (bias_acc && q == 0 ? 1 : 0);
    for (int t = 0; t < tiles; ++t) {
      const bool brow = t == mt;
      const int64_t row = brow ? (lane == 0 ? m : m + 1) : (int64_t)(t0 + t) * kTcBM + q * 32 + lane;
      float* dst = part + ((int64_t)split * (m + 1) + row) * n;
#pragma unroll 1
      for (int cb = 0; cb < UN; cb += 32) {
        uint32_t v[32];
        if (nkb > 0) {
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + t * UN + cb, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + t * UN + cb + 16,
                    *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0u;
        }
        if (row < m || (brow && lane == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (cb + j < n)  // n is a multiple of 8 (and so of 4)
              *reinterpret_cast<float4*>(dst + cb + j) =
                  make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                              __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// out[m, n] = rnd(sum_s part[s, m, n]) in a fixed order; with accumulate,
// out = rnd(out + that) (autograd's in-place gradient accumulation).
// Partials are [splits][m + 1][n]; row m holds the bias column sums (written
// to bias_out when it is non-null).  Block = 32 float4 columns x kRedY split
// lanes: lane y folds splits y, y + kRedY, ... in order, then the kRedY
// partial sums are added in y order through shared memory (deterministic).
constexpr int kRedY = 16;
__global__ void __launch_bounds__(32 * kRedY)
k_wgrad_reduce(const float* __restrict__ part, int splits, int64_t m, int n,
               __half* __restrict__ out, int64_t ldo, __half* __restrict__ bias_out,
               int accumulate) {
  __shared__ float4 sh[kRedY][32];
  const int64_t n4 = n / 4;
  const int64_t total = (m + (bias_out ? 1 : 0)) * n4;
  const int64_t i = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int y = threadIdx.y;
  const int64_t r = i / n4, c = (i - r * n4) * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < total) {
    for (int s = y; s < splits; s += kRedY) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(part + ((int64_t)s * (m + 1) + r) * n + c));
      acc.x = __fadd_rn(acc.x, v.x);
      acc.y = __fadd_rn(acc.y, v.y);
      acc.z = __fadd_rn(acc.z, v.z);
      acc.w = __fadd_rn(acc.w, v.w);
    }
  }
  sh[y][threadIdx.x] = acc;
  __syncthreads();
  if (y != 0 || i >= total) return;
#pragma unroll
  for (int k = 1; k < kRedY; ++k) {
    const float4 v = sh[k][threadIdx.x];
    acc.x = __fadd_rn(acc.x, v.x);
    acc.y = __fadd_rn(acc.y, v.y);
    acc.z = __fadd_rn(acc.z, v.z);
    acc.w = __fadd_rn(acc.w, v.w);
  }
  __half h[4] = {__float2half_rn(acc.x), __float2half_rn(acc.y), __float2half_rn(acc.z),
                 __float2half_rn(acc.w)};
  __half* o = r < m ? out + r * ldo + c : bias_out + c;
  if (accumulate) {
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __hadd_rn(o[j], h[j]);
  }
  *reinterpret_cast<uint2*>(o) = *reinterpret_cast<const uint2*>(h);
}

static int launch_wgrad_reduce(const float* part, int splits, int64_t m, int n, void* out,
                               int64_t ldo, void* bias_out, int accumulate, cudaStream_t st) {
  const int64_t total = (m + (bias_out ? 1 : 0)) * (n / 4);
  k_wgrad_reduce<<<(unsigned)((total + 31) / 32), dim3(32, kRedY), 0, st>>>(
      part, splits, m, n, (__half*)out, ldo, (__half*)bias_out, accumulate);
  HG_LAUNCHED();
  return HG_OK;
}

struct WgradPlan {
  int nb, mt_total, mt_group, groups, splits, stages, bk, a_boxes;
  int64_t slabs, sps;
  uint32_t tmem_cols;
  size_t smem, part_bytes;
};

static WgradPlan wgrad_plan(int64_t k, int64_t m, int n, int sms) {
  WgradPlan p{};

  p.nb = (n + 63) / 64;
  p.mt_total = (int)((m + kTcBM - 1) / kTcBM);
  // TMEM: one 64*nb-column accumulator per tile, plus the bias accumulator
  const int mt_cap = std::min(kWgMaxMT, 512 / (64 * p.nb) - 1);
  p.groups = (p.mt_total + mt_cap - 1) / mt_cap;
  if (const char* e = getenv("HG_WG_GROUPS"))  // measurement knob (A/B runs only)
    p.groups = std::max(p.groups, std::min(p.mt_total, atoi(e)));
  p.mt_group = (p.mt_total + p.groups - 1) / p.groups;
  const uint32_t cols = (uint32_t)((p.mt_group + 1) * 64 * p.nb);
  p.tmem_cols = 32;
  while (p.tmem_cols < cols) p.tmem_cols <<= 1;
  p.a_boxes = (int)std::min<int64_t>(2 * p.mt_group, (m + 63) / 64);
  // narrow operands (<= 3 boxes per slab): two CTAs per SM -- one CTA's ring
  // streams ~25 GB/s whatever its depth (C4 GIN dW: 171 -> 132 us); wide ones
  // need the whole shared memory for depth.  HG_WG_CTAS overrides (A/B runs).
  int cps = p.a_boxes + p.nb <= 3 ? 2 : 1;
  if (const char* e = getenv("HG_WG_CTAS")) cps = std::max(1, atoi(e));
  const uint32_t budget = (200u * 1024u) / (uint32_t)cps;
  // deepest slab that keeps >= 3 stages in ~200 KB of shared memory
  p.bk = 32;
  for (int cand : {128, 64})
    if ((uint32_t)(p.a_boxes + p.nb) * 128u * cand * 3 <= budget) { p.bk = cand; break; }
  // measurement knobs (A/B runs only): HG_WG_BK = slab rows, HG_WG_STAGES = ring depth
  if (const char* e = getenv("HG_WG_BK")) p.bk = atoi(e);
  p.slabs = (k + p.bk - 1) / p.bk;
  // >= 512 rows per split keeps the partials small next to A
  const int64_t min_slabs = 512 / p.bk;
  int64_t want = std::max<int64_t>(1, std::min<int64_t>(cps * sms / p.groups, (p.slabs + min_slabs - 1) / min_slabs));
  p.sps = (p.slabs + want - 1) / want;
  p.splits = (int)((p.slabs + p.sps - 1) / p.sps);
  if (p.splits < 1) p.splits = 1;
  const uint32_t stage = (uint32_t)(p.a_boxes + p.nb) * 128u * (uint32_t)p.bk;
  p.stages = (int)std::min<uint32_t>(16, budget / stage);
  if (const char* e = getenv("HG_WG_STAGES")) p.stages = std::min(p.stages, atoi(e));
  p.smem = 1024 + (size_t)p.stages * stage + kWgOnes + (2 * p.stages + 1) * 8 + 16;
  p.part_bytes = align_up((size_t)p.splits * (size_t)(m + 1) * (size_t)n * sizeof(float));
  return p;
}

static int device_sms() {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int NB>
static int launch_wgrad(const CUtensorMap& ma, const CUtensorMap& mb, const WgradPlan& p, int64_t m,
                        int n, int with_bias, float* part, cudaStream_t st) {
  HG_CUDA(cudaFuncSetAttribute(k_gemm_wgrad<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)p.smem));
  k_gemm_wgrad<NB><<<p.groups * p.splits, 192, p.smem, st>>>(
      ma, mb, m, n, p.mt_total, p.mt_group, p.slabs, p.sps, p.splits, p.stages, p.bk, p.a_boxes, p.tmem_cols,
      with_bias, part);
  HG_LAUNCHED();
  return HG_OK;
}

}  // namespace hg

using namespace hg;

static int gemm_tc_impl(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt,
                        int32_t n, int64_t ldb, const void* bias, const void* row_scale,
                        int32_t relu, void* out, int64_t ldo, void* stream, const Dots& dots);

extern "C" int hg_gemm_tc(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt,
                          int32_t n, int64_t ldb, const void* bias, const void* row_scale,
                          int32_t relu, void* out, int64_t ldo, void* stream) {
  return gemm_tc_impl(a, m, k, lda, bt, n, ldb, bias, row_scale, relu, out, ldo, stream, Dots{});
}

extern "C" int hg_gemm_tc_dots(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt,
                               int32_t n, int64_t ldb, void* out, int64_t ldo, const void* dot_a,
                               const void* dot_b, int32_t heads, void* dot_out_a, void* dot_out_b,
                               void* stream) {
  HG_REQUIRE(heads >= 1 && heads <= 8 && n % heads == 0 && (n / heads) % 16 == 0,
             "hg_gemm_tc_dots: heads=%d must split N=%d into multiples of 16 (<= 8 heads)", heads, n);
  // each epilogue thread owns whole heads: an even head count, or 16-wide heads
  HG_REQUIRE(heads % 2 == 0 || n / heads == 16,
             "hg_gemm_tc_dots: %d heads of width %d: odd head counts need 16-wide heads", heads,
             n / heads);
  HG_REQUIRE(dot_a && dot_b && dot_out_a && dot_out_b &&
                 ((reinterpret_cast<uintptr_t>(dot_a) | reinterpret_cast<uintptr_t>(dot_b)) & 3) == 0,
             "hg_gemm_tc_dots: null or misaligned head vectors / outputs");
  return gemm_tc_impl(a, m, k, lda, bt, n, ldb, nullptr, nullptr, 0, out, ldo, stream,
                      Dots{dot_a, dot_b, heads, n / heads, dot_out_a, dot_out_b, nullptr, 0});
}

extern "C" int hg_gemm_tc_masked(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt,
                                 int32_t n, int64_t ldb, void* out, int64_t ldo, const void* mask,
                                 int64_t ldm, void* stream) {
  HG_REQUIRE(mask && ldm >= n && ldm % 8 == 0 && (reinterpret_cast<uintptr_t>(mask) & 15) == 0 &&
                 n % 16 == 0,
             "hg_gemm_tc_masked: the mask must be [m, n] binary16, 16-byte aligned rows, n %% 16 == 0");
  return gemm_tc_impl(a, m, k, lda, bt, n, ldb, nullptr, nullptr, 0, out, ldo, stream,
                      Dots{nullptr, nullptr, 1, 16, nullptr, nullptr, mask, ldm});
}

static int gemm_tc_impl(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt,
                        int32_t n, int64_t ldb, const void* bias, const void* row_scale,
                        int32_t relu, void* out, int64_t ldo, void* stream, const Dots& dots) {
  HG_REQUIRE(m >= 0 && k > 0, "hg_gemm_tc: bad arguments");
  if (m == 0) return HG_OK;
  HG_REQUIRE(a && bt && out, "hg_gemm_tc: null operand");
  HG_REQUIRE(n >= 8 && n <= 256 && n % 8 == 0, "hg_gemm_tc: N=%d must be a multiple of 8 in [8, 256]", n);
  // UMMA N is a multiple of 16: a width of 8 (mod 16) runs as the next
  // multiple, its extra Bt rows zero-filled by TMA and its columns not stored
  const int n16 = (n + 15) / 16 * 16;
  HG_REQUIRE(lda >= k && ldb >= k && ldo >= n && lda % 8 == 0 && ldb % 8 == 0 && ldo % 8 == 0,
             "hg_gemm_tc: row pitches must cover K / N and be multiples of 8 elements");
  HG_REQUIRE(((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(bt) |
               reinterpret_cast<uintptr_t>(out)) & 15) == 0,
             "hg_gemm_tc: operands must be 16-byte aligned");
  if (m == 0) return HG_OK;
  // the tensor-map encoder is a driver call: bind the runtime's primary context
  // to this thread first (autograd runs backward on its own worker threads)
  int dev = 0;
  HG_CUDA(cudaGetDevice(&dev));
  HG_CUDA(cudaSetDevice(dev));
  CUtensorMap ma, mb;
  HG_REQUIRE(make_map(&ma, a, m, k, lda, kTcBM),
             "hg_gemm_tc: cuTensorMapEncodeTiled(A [%lld x %lld], pitch %lld, ptr %p) failed: %d",
             (long long)m, (long long)k, (long long)lda, a, g_tma_err);
  HG_REQUIRE(make_map(&mb, bt, n, k, ldb, (uint32_t)n16),
             "hg_gemm_tc: cuTensorMapEncodeTiled(Bt [%d x %lld], pitch %lld, ptr %p) failed: %d",
             n, (long long)k, (long long)ldb, bt, g_tma_err);
  CUtensorMap mo = ma;  // TMA-store epilogue (N % 64 == 0): 64-column boxes of the output
  if (n % 64 == 0)
    HG_REQUIRE(make_map(&mo, out, m, n, ldo, kTcBM),
               "hg_gemm_tc: cuTensorMapEncodeTiled(out [%lld x %d], pitch %lld) failed: %d",
               (long long)m, n, (long long)ldo, g_tma_err);
  cudaStream_t st = as_stream(stream);
  switch (n16) {
#define HG_TC(NN) case NN: return launch_gemm_tc<NN>(ma, mb, mo, m, k, bias, row_scale, out, ldo, relu, n, dots, st);
    HG_TC(16) HG_TC(32) HG_TC(48) HG_TC(64) HG_TC(80) HG_TC(96) HG_TC(112) HG_TC(128)
    HG_TC(144) HG_TC(160) HG_TC(176) HG_TC(192) HG_TC(208) HG_TC(224) HG_TC(240) HG_TC(256)
#undef HG_TC
    default: break;
  }
  HG_REQUIRE(false, "hg_gemm_tc: unsupported N=%d", n);
}

extern "C" int hg_gemm_wgrad_workspace(int64_t k, int64_t m, int32_t n, size_t* bytes) {
  HG_REQUIRE(bytes && k >= 0 && m >= 0 && n >= 8 && n <= 256 && n % 8 == 0,
             "hg_gemm_wgrad_workspace: bad arguments (N=%d must be a multiple of 8 in [8, 256])", n);
  *bytes = (k == 0 || m == 0) ? 0 : wgrad_plan(k, m, n, device_sms()).part_bytes;
  return HG_OK;
}

extern "C" int hg_gemm_wgrad(const void* a, int64_t k, int64_t m, int64_t lda, const void* b,
                             int32_t n, int64_t ldb, void* out, int64_t ldo, void* bias_out,
                             int32_t accumulate, void* ws, size_t ws_bytes, void* stream) {
  HG_REQUIRE(k >= 0 && m >= 0, "hg_gemm_wgrad: bad arguments");
  HG_REQUIRE(n >= 8 && n <= 256 && n % 8 == 0, "hg_gemm_wgrad: N=%d must be a multiple of 8 in [8, 256]", n);
  if (m == 0) return HG_OK;
  HG_REQUIRE(out, "hg_gemm_wgrad: null output");
  HG_REQUIRE(m % 8 == 0 && lda >= m && ldb >= n && ldo >= n && lda % 8 == 0 && ldb % 8 == 0 && ldo % 4 == 0,
             "hg_gemm_wgrad: M must be a multiple of 8 and pitches cover M / N (multiples of 8)");
  cudaStream_t st = as_stream(stream);
  if (k == 0) {  // empty sum: zeros (or out unchanged when accumulating)
    return launch_wgrad_reduce(nullptr, 0, m, n, out, ldo, bias_out, accumulate, st);
  }
  HG_REQUIRE(a && b, "hg_gemm_wgrad: null operand");
  HG_REQUIRE(((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0 &&
                 ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(bias_out)) & 7) == 0,
             "hg_gemm_wgrad: operands must be 16-byte aligned, out 8-byte aligned");
  const WgradPlan p = wgrad_plan(k, m, n, device_sms());
  HG_REQUIRE(ws && ws_bytes >= p.part_bytes, "hg_gemm_wgrad: workspace too small (%zu < %zu)",
             ws_bytes, p.part_bytes);
  int dev = 0;
  HG_CUDA(cudaGetDevice(&dev));
  HG_CUDA(cudaSetDevice(dev));
  CUtensorMap ma, mb;
  // A = x [k rows, m cols]: boxes of 64 columns x 32 rows; B = g [k, n] likewise
  HG_REQUIRE(make_map_box(&ma, a, k, m, lda, 64, (uint32_t)p.bk),
             "hg_gemm_wgrad: cuTensorMapEncodeTiled(A [%lld x %lld]) failed: %d", (long long)k,
             (long long)m, g_tma_err);
  HG_REQUIRE(make_map_box(&mb, b, k, n, ldb, 64, (uint32_t)p.bk),
             "hg_gemm_wgrad: cuTensorMapEncodeTiled(B [%lld x %d]) failed: %d", (long long)k, n,
             g_tma_err);
  float* part = static_cast<float*>(ws);
  int rc = HG_OK;
  switch (p.nb) {
    case 1: rc = launch_wgrad<1>(ma, mb, p, m, n, bias_out != nullptr, part, st); break;
    case 2: rc = launch_wgrad<2>(ma, mb, p, m, n, bias_out != nullptr, part, st); break;
    case 3: rc = launch_wgrad<3>(ma, mb, p, m, n, bias_out != nullptr, part, st); break;
    default: rc = launch_wgrad<4>(ma, mb, p, m, n, bias_out != nullptr, part, st); break;
  }
  if (rc != HG_OK) return rc;
  return launch_wgrad_reduce(part, p.splits, m, n, out, ldo, bias_out, accumulate, st);
}
