// SDDMM, GAT attention scores and edge softmax (forward/backward) for sm_100a.
// All of these reproduce the reference's rounding sequence bit for bit:
//   sddmm           kernels.py:407-455 (products rounded, pair sums, adjacent-pair tree)
//   attention       models.py:317-326 + leaky_relu 188-200
//   edge softmax    models.py:382-412 (row max, rnd(exp), tree sum, rnd(ex/den))
// The adjacent-pair tree with pass-through of a lone right-most element is the
// implicit binary tree over power-of-two aligned index ranges; warps evaluate it
// with predicated shuffle-down levels and combine 32-element block roots with a
// binary-counter stack, so any row length reproduces the same tree.
#include <cstdlib>

#include "hg_common.cuh"

namespace hg {

template <int BYTES> struct RawV;
struct alignas(32) SdU32x8 { uint32_t a[8]; };
template <> struct RawV<32> { using type = SdU32x8; };
template <> struct RawV<16> { using type = uint4; };

// Read-only gather of one lane chunk (32 bytes: one LDG.256).
template <typename R>
__device__ __forceinline__ R ldg_chunk(const R* p) {
  if constexpr (sizeof(R) == 32) {
    R v;
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]), "=r"(v.a[5]),
          "=r"(v.a[6]), "=r"(v.a[7])
        : "l"(p));
    return v;
  } else {
    return __ldg(p);
  }
}
template <> struct RawV<4> { using type = uint32_t; };
template <> struct RawV<8> { using type = uint2; };

// ------------------------------------------------------------------- SDDMM

// Tree value of one V-element chunk: per-pair sums v_i = rnd(rnd(x0*y0) + rnd(x1*y1)),
// then the adjacent-pair tree over the V/2 sums (a power of two: all present).
template <typename T, int V>
__device__ __forceinline__ T chunk_dot(const typename RawV<V * sizeof(T)>::type& xr,
                                       const typename RawV<V * sizeof(T)>::type& yr) {
  using N = Num<T>;
  const T* xa = reinterpret_cast<const T*>(&xr);
  const T* ya = reinterpret_cast<const T*>(&yr);
  T v[V / 2];
#pragma unroll
  for (int i = 0; i < V / 2; ++i)
    v[i] = N::add(N::mul(xa[2 * i], ya[2 * i]), N::mul(xa[2 * i + 1], ya[2 * i + 1]));
#pragma unroll
  for (int s = 1; s < V / 2; s <<= 1)
#pragma unroll
    for (int i = 0; i + s < V / 2; i += 2 * s) v[i] = N::add(v[i], v[i + s]);
  return v[0];
}

template <typename T>
__device__ __forceinline__ T shfl_down_t(unsigned mask, T v, int s, int width) {
  if constexpr (sizeof(T) == 2) {
    unsigned short b = __half_as_ushort(v);
    return __ushort_as_half((unsigned short)__shfl_down_sync(mask, (unsigned)b, s, width));
  } else {
    return __shfl_down_sync(mask, v, s, width);
  }
}

// Team of TEAM lanes per unit (row slice); lane owns chunks c = tl + k*TEAM of V
// elements; lph = chunks per head (fh / V).  Requires lph % 32 == 0 or 32 % lph == 0
// when NCH > 1.
template <typename T, int V, int TEAM, int NCH>
__global__ void __launch_bounds__(256)
k_sddmm(const int4* __restrict__ units, int64_t num_units, const int32_t* __restrict__ cols,
        const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ out, int F, int heads) {
  using N = Num<T>;
  using Raw = typename RawV<V * sizeof(T)>::type;
  constexpr int EB = NCH >= 2 ? 4 : 8;
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TEAM - 1);
  const unsigned tmask =
      TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << (lane & ~(TEAM - 1)));
  const int64_t team = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
  if (team >= num_units) return;
  const int4 un = units[team];
  const int row = un.x, beg = un.y, end = un.z;
  const int fh = F / heads, lph = fh / V, nvec = F / V;

  Raw xr[NCH];
  bool cval[NCH];
  int q[NCH], hd[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int c = tl + k * TEAM;
    cval[k] = c < nvec;
    hd[k] = c / lph;
    q[k] = c - hd[k] * lph;
    if (cval[k]) xr[k] = *reinterpret_cast<const Raw*>(x + (int64_t)row * F + c * V);
  }
  // column ids of the next batch are fetched while the current batch computes
  int cj[EB];
#pragma unroll
  for (int j = 0; j < EB; ++j) cj[j] = beg + j < end ? __ldg(cols + beg + j) : 0;
  for (int base = beg; base < end; base += EB) {
    int nj[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      const int e = base + EB + j;
      nj[j] = e < end ? __ldg(cols + e) : 0;
    }
    Raw yr[EB][NCH];
#pragma unroll
    for (int j = 0; j < EB; ++j) {
#pragma unroll
      for (int k = 0; k < NCH; ++k)
        if (base + j < end && cval[k])
          yr[j][k] = __ldg(reinterpret_cast<const Raw*>(y + (int64_t)cj[j] * F + (tl + k * TEAM) * V));
    }
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      const int64_t e = base + j;
      if (e >= end) break;  // uniform across the team
      T part[NCH];
#pragma unroll
      for (int k = 0; k < NCH; ++k) part[k] = cval[k] ? chunk_dot<T, V>(xr[k], yr[j][k]) : N::zero();
      // shuffle levels inside each k-slice (q and q+s share the slice)
#pragma unroll
      for (int s = 1; s < TEAM; s <<= 1) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const T o = shfl_down_t(tmask, part[k], s, TEAM);
          if ((q[k] & (2 * s - 1)) == 0 && q[k] + s < lph && (tl + s) < TEAM) part[k] = N::add(part[k], o);
        }
      }
      // levels across k-slices (heads wider than one slice: lph multiple of TEAM)
      if (NCH > 1 && lph > TEAM) {
        const int spr = lph / TEAM;  // slices per head
#pragma unroll
        for (int s = 1; s < NCH; s <<= 1)
#pragma unroll
          for (int k = 0; k + s < NCH; k += 2 * s)
            if ((k % spr) % (2 * s) == 0 && (k % spr) + s < spr) part[k] = N::add(part[k], part[k + s]);
      }
#pragma unroll
      for (int k = 0; k < NCH; ++k)
        if (cval[k] && q[k] == 0) out[e * heads + hd[k]] = part[k];
    }
#pragma unroll
    for (int j = 0; j < EB; ++j) cj[j] = nj[j];
  }
}

// fp32-guarded SDDMM (numerics="fast"): out[e, h] = rnd(sum_f x[r, hf] y[c, hf])
// with exact f16 products accumulated in fp32 (fma.rn.f32.f16), one rounding.
// Team of TEAM = F/V lanes per unit, G = fh/V lanes per head (power of two,
// G <= TEAM).  The EB per-edge partial dots of a batch are reduced across the
// G lanes of a head with a reduce-scatter butterfly: each level halves the
// values a lane carries, so EB edges cost ~EB + log2(G) shuffles instead of
// EB * log2(G).
template <typename T, int V>
__device__ __forceinline__ float chunk_dot_f32(const typename RawV<V * sizeof(T)>::type& xr,
                                               const typename RawV<V * sizeof(T)>::type& yr) {
  float acc = 0.0f;
  if constexpr (sizeof(T) == 2) {
    const unsigned short* xa = reinterpret_cast<const unsigned short*>(&xr);
    const unsigned short* ya = reinterpret_cast<const unsigned short*>(&yr);
#pragma unroll
    for (int i = 0; i < V; ++i)
      asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(xa[i]), "h"(ya[i]));
  } else {
    const float* xa = reinterpret_cast<const float*>(&xr);
    const float* ya = reinterpret_cast<const float*>(&yr);
#pragma unroll
    for (int i = 0; i < V; ++i) acc = fmaf(xa[i], ya[i], acc);
  }
  return acc;
}

template <typename T, int V, int TEAM, int G>
#ifndef HG_SDDMM_OCC
#define HG_SDDMM_OCC 3   // resident 256-thread blocks per SM (A/B builds)
#endif
__global__ void __launch_bounds__(256, HG_SDDMM_OCC)
k_sddmm_fast(const int4* __restrict__ units, int64_t num_units, const int32_t* __restrict__ cols,
             const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ out, int F,
             int heads) {
  using Raw = typename RawV<V * sizeof(T)>::type;
  constexpr int EB = V * sizeof(T) == 32 ? 4 : 8;
  constexpr int LV = (G < EB ? G : EB);  // butterfly levels that halve the batch: log2(LV)
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TEAM - 1);
  const unsigned tmask =
      TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << (lane & ~(TEAM - 1)));
  const int nvec = F / V;
  const bool cval = tl < nvec;
  const int hd = tl / G, gp = tl & (G - 1);  // head, position inside the head's lane group
  // Persistent teams walk the unit list with stride nteams; the next unit's
  // descriptor is fetched before the current one is processed.
  const int64_t nteams = ((int64_t)gridDim.x * blockDim.x) / TEAM;
  int64_t team = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
  if (team >= num_units) return;
  int4 un = units[team];
  for (;;) {
  const int64_t nxt_team = team + nteams;
  const int4 nxt = nxt_team < num_units ? units[nxt_team] : make_int4(0, 0, 0, 0);
  const int row = un.x, beg = un.y, end = un.z;
  Raw xr;
  if (cval) xr = *reinterpret_cast<const Raw*>(x + (int64_t)row * F + tl * V);
  // column ids spread over the team: lane tl holds edges base + tl + q*TEAM
  constexpr int IDS = (EB + TEAM - 1) / TEAM;
  const int tb = lane & ~(TEAM - 1);
  int cq[IDS];
#pragma unroll
  for (int q = 0; q < IDS; ++q) {
    const int j = tl + q * TEAM;
    cq[q] = (j < EB && beg + j < end) ? __ldcs(cols + beg + j) : 0;
  }
  for (int base = beg; base < end; base += EB) {
    int nq[IDS];
#pragma unroll
    for (int q = 0; q < IDS; ++q) {
      const int j = tl + q * TEAM;
      nq[q] = (j < EB && base + EB + j < end) ? __ldcs(cols + base + EB + j) : 0;
    }
    Raw yr[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      const int c = __shfl_sync(tmask, cq[j / TEAM], tb + j % TEAM);
      if (base + j < end && cval) yr[j] = ldg_chunk(reinterpret_cast<const Raw*>(y + (int64_t)c * F + tl * V));
    }
    float v[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) v[j] = (base + j < end && cval) ? chunk_dot_f32<T, V>(xr, yr[j]) : 0.0f;
    // reduce-scatter over the G lanes of each head (xor partners stay in the group)
    int eoff = 0;
#pragma unroll
    for (int s = G / 2, cnt = EB; s >= 1 && cnt > 1; s >>= 1, cnt >>= 1) {
      const bool up = (gp & s) != 0;
#pragma unroll
      for (int i = 0; i < cnt / 2; ++i) {
        const float send = up ? v[i] : v[i + cnt / 2];
        const float keep = up ? v[i + cnt / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(tmask, send, s);
      }
      if (up) eoff += cnt / 2;
    }
    // heads wider than the batch: finish with plain xor sums (G > EB)
#pragma unroll
    for (int s = G / (2 * LV) > 0 ? (G / LV) / 2 : 0; s >= 1; s >>= 1)
      v[0] += __shfl_xor_sync(tmask, v[0], s);
    constexpr int KEEP = EB / LV;  // values per lane after the butterfly
    const bool writer = G <= EB || (gp & (G / LV - 1)) == 0;
    if (cval && writer) {
#pragma unroll
      for (int i = 0; i < KEEP; ++i) {
        const int e = base + eoff + i;
        if (e < end) out[(int64_t)e * heads + hd] = Num<T>::from_f(v[i]);
      }
    }
#pragma unroll
    for (int q = 0; q < IDS; ++q) cq[q] = nq[q];
  }
  if (nxt_team >= num_units) break;
  team = nxt_team;
  un = nxt;
  }
}

// Packs (hg_schedule_build): an aligned block of short rows walked as one edge
// stream in 4-edge batches, each edge's X row picked by its row id (reused
// from the previous edge of the batch when the row repeats).  Per-edge
// arithmetic and the butterfly grouping are k_sddmm_fast's: bitwise equal.
template <typename T, int V, int TEAM, int G>
__global__ void __launch_bounds__(256, V * sizeof(T) == 32 ? 2 : 4)
k_sddmm_packed(const int4* __restrict__ packs, int64_t num_packs, const int32_t* __restrict__ rowid,
               const int32_t* __restrict__ cols, const T* __restrict__ x,
               const T* __restrict__ y, T* __restrict__ out, int F, int heads) {
  using Raw = typename RawV<V * sizeof(T)>::type;
  constexpr int EB = 4;
  constexpr int LV = (G < EB ? G : EB);
  constexpr int IDS = (EB + TEAM - 1) / TEAM;
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TEAM - 1);
  const int tb = lane & ~(TEAM - 1);
  const unsigned tmask = TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << tb);
  const int nvec = F / V;
  const bool cval = tl < nvec;
  const int hd = tl / G, gp = tl & (G - 1);
  const int64_t team = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
  if (team >= num_packs) return;
  const int4 pk = packs[team];
  const int beg = pk.y, end = pk.z;
  int cq[IDS], rq[IDS];
#pragma unroll
  for (int q = 0; q < IDS; ++q) {
    const int j = tl + q * TEAM;
    const bool in = j < EB && beg + j < end;
    cq[q] = in ? __ldcs(cols + beg + j) : 0;
    rq[q] = in ? __ldcs(rowid + beg + j) : -1;
  }
  for (int base = beg; base < end; base += EB) {
    int nc[IDS], nr[IDS];
#pragma unroll
    for (int q = 0; q < IDS; ++q) {
      const int j = tl + q * TEAM;
      const bool in = j < EB && base + EB + j < end;
      nc[q] = in ? __ldcs(cols + base + EB + j) : 0;
      nr[q] = in ? __ldcs(rowid + base + EB + j) : -1;
    }
    Raw xr[EB], yr[EB];
    int rj[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      const int c = __shfl_sync(tmask, cq[j / TEAM], tb + j % TEAM);
      rj[j] = __shfl_sync(tmask, rq[j / TEAM], tb + j % TEAM);
      if (rj[j] >= 0 && cval) {
        yr[j] = ldg_chunk(reinterpret_cast<const Raw*>(y + (int64_t)c * F + tl * V));
        if (j == 0 || rj[j] != rj[j - 1])
          xr[j] = ldg_chunk(reinterpret_cast<const Raw*>(x + (int64_t)rj[j] * F + tl * V));
      }
    }
#pragma unroll
    for (int j = 1; j < EB; ++j)
      if (rj[j] == rj[j - 1]) xr[j] = xr[j - 1];
    float v[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) v[j] = (rj[j] >= 0 && cval) ? chunk_dot_f32<T, V>(xr[j], yr[j]) : 0.0f;
    int eoff = 0;
#pragma unroll
    for (int s = G / 2, cnt = EB; s >= 1 && cnt > 1; s >>= 1, cnt >>= 1) {
      const bool up = (gp & s) != 0;
#pragma unroll
      for (int i = 0; i < cnt / 2; ++i) {
        const float send = up ? v[i] : v[i + cnt / 2];
        const float keep = up ? v[i + cnt / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(tmask, send, s);
      }
      if (up) eoff += cnt / 2;
    }
#pragma unroll
    for (int s = G / (2 * LV) > 0 ? (G / LV) / 2 : 0; s >= 1; s >>= 1)
      v[0] += __shfl_xor_sync(tmask, v[0], s);
    constexpr int KEEP = EB / LV;
    const bool writer = G <= EB || (gp & (G / LV - 1)) == 0;
    if (cval && writer) {
#pragma unroll
      for (int i = 0; i < KEEP; ++i) {
        const int e = base + eoff + i;
        if (e < end) out[(int64_t)e * heads + hd] = Num<T>::from_f(v[i]);
      }
    }
#pragma unroll
    for (int q = 0; q < IDS; ++q) { cq[q] = nc[q]; rq[q] = nr[q]; }
  }
}

}  // namespace hg

using namespace hg;

struct SdPacks {
  const int4* packs;
  int64_t np;
  const int32_t* rowid;
};

template <typename T, int V, int TEAM, int G>
static int launch_sddmm_fast(const int4* units, int64_t nu, const SdPacks& pk, const int32_t* cols,
                             const void* x, const void* y, void* out, int F, int heads,
                             cudaStream_t st) {
  constexpr int tpb = 256 / TEAM;
  if (pk.np > 0) {
    k_sddmm_packed<T, V, TEAM, G><<<(unsigned)((pk.np + tpb - 1) / tpb), 256, 0, st>>>(
        pk.packs, pk.np, pk.rowid, cols, (const T*)x, (const T*)y, (T*)out, F, heads);
    HG_LAUNCHED();
  }
  if (nu == 0) return HG_OK;
  int sms = 148, dev = 0, occ = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sddmm_fast<T, V, TEAM, G>, 256, 0);
  const int64_t need = (nu + tpb - 1) / tpb;
  const int64_t cap = (int64_t)sms * (occ > 0 ? occ : 4);
  k_sddmm_fast<T, V, TEAM, G><<<(unsigned)(need < cap ? need : cap), 256, 0, st>>>(
      units, nu, cols, (const T*)x, (const T*)y, (T*)out, F, heads);
  HG_LAUNCHED();
  return HG_OK;
}

template <typename T, int V, int TEAM>
static int dispatch_sddmm_fast_g(const int4* units, int64_t nu, const SdPacks& pk,
                                 const int32_t* cols, const void* x, const void* y, void* out,
                                 int F, int heads, int g, cudaStream_t st) {
  switch (g) {
    case 1: return launch_sddmm_fast<T, V, TEAM, 1>(units, nu, pk, cols, x, y, out, F, heads, st);
    case 2: if constexpr (TEAM >= 2) return launch_sddmm_fast<T, V, TEAM, 2>(units, nu, pk, cols, x, y, out, F, heads, st); break;
    case 4: if constexpr (TEAM >= 4) return launch_sddmm_fast<T, V, TEAM, 4>(units, nu, pk, cols, x, y, out, F, heads, st); break;
    case 8: if constexpr (TEAM >= 8) return launch_sddmm_fast<T, V, TEAM, 8>(units, nu, pk, cols, x, y, out, F, heads, st); break;
    case 16: if constexpr (TEAM >= 16) return launch_sddmm_fast<T, V, TEAM, 16>(units, nu, pk, cols, x, y, out, F, heads, st); break;
    case 32: if constexpr (TEAM >= 32) return launch_sddmm_fast<T, V, TEAM, 32>(units, nu, pk, cols, x, y, out, F, heads, st); break;
    default: break;
  }
  HG_REQUIRE(false, "hg_sddmm_fast: head group %d unsupported", g);
}

// Returns -1 when the layout is not covered (caller falls back to the exact kernel).
template <typename T, int V>
static int dispatch_sddmm_fast(const int4* units, int64_t nu, const SdPacks& pk,
                               const int32_t* cols, const void* x, const void* y, void* out,
                               int F, int heads, cudaStream_t st) {
  const int nvec = F / V, g = F / heads / V;
  if (nvec > 32 || g < 1 || (g & (g - 1)) != 0 || nvec % g != 0) return -1;
  const int team = nvec <= 1 ? 1 : nvec <= 2 ? 2 : nvec <= 4 ? 4 : nvec <= 8 ? 8 : nvec <= 16 ? 16 : 32;
  switch (team) {
    case 1: return dispatch_sddmm_fast_g<T, V, 1>(units, nu, pk, cols, x, y, out, F, heads, g, st);
    case 2: return dispatch_sddmm_fast_g<T, V, 2>(units, nu, pk, cols, x, y, out, F, heads, g, st);
    case 4: return dispatch_sddmm_fast_g<T, V, 4>(units, nu, pk, cols, x, y, out, F, heads, g, st);
    case 8: return dispatch_sddmm_fast_g<T, V, 8>(units, nu, pk, cols, x, y, out, F, heads, g, st);
    case 16: return dispatch_sddmm_fast_g<T, V, 16>(units, nu, pk, cols, x, y, out, F, heads, g, st);
    default: return dispatch_sddmm_fast_g<T, V, 32>(units, nu, pk, cols, x, y, out, F, heads, g, st);
  }
}

template <typename T, int V, int TEAM, int NCH>
static int launch_sddmm(const int4* units, int64_t nu, const int32_t* cols, const void* x,
                        const void* y, void* out, int F, int heads, cudaStream_t st) {
  constexpr int tpb = 256 / TEAM;
  if (nu == 0) return HG_OK;
  k_sddmm<T, V, TEAM, NCH><<<(unsigned)((nu + tpb - 1) / tpb), 256, 0, st>>>(
      units, nu, cols, (const T*)x, (const T*)y, (T*)out, F, heads);
  HG_LAUNCHED();
  return HG_OK;
}

template <typename T, int V>
static int dispatch_sddmm(const int4* units, int64_t nu, const int32_t* cols, const void* x,
                          const void* y, void* out, int F, int heads, cudaStream_t st) {
  const int nvec = F / V, lph = F / heads / V;
#define HG_SD(TM, NC) return launch_sddmm<T, V, TM, NC>(units, nu, cols, x, y, out, F, heads, st)
  if (nvec <= 1) HG_SD(1, 1);
  if (nvec <= 2) HG_SD(2, 1);
  if (nvec <= 4) HG_SD(4, 1);
  if (nvec <= 8) HG_SD(8, 1);
  if (nvec <= 16) HG_SD(16, 1);
  if (nvec <= 32) HG_SD(32, 1);
  HG_REQUIRE(lph % 32 == 0 || 32 % lph == 0,
             "hg_sddmm: head width %d does not tile 32-lane slices", F / heads);
  HG_REQUIRE(nvec % 32 == 0, "hg_sddmm: feature length %d unsupported", F);
  if (nvec <= 64) HG_SD(32, 2);
  if (nvec <= 128) HG_SD(32, 4);
  if (nvec <= 256) HG_SD(32, 8);
#undef HG_SD
  HG_REQUIRE(false, "hg_sddmm: feature length %d too large", F);
}

// 32-byte lanes for binary16 rows of 64..512 elements with 16-element heads
// (A/B switch for measurement: HG_SPMM_LANE32=0, as for hg_spmm).
static bool sd_lane32() {
  static const bool on = [] {
    const char* e = getenv("HG_SPMM_LANE32");
    return !(e && e[0] == '0');
  }();
  return on;
}

extern "C" int hg_sddmm_fast(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                             int64_t num_edges, const int32_t* units, int64_t num_units,
                             const int32_t* packs, int64_t num_packs, const int32_t* pack_rowid,
                             const void* x, const void* y, void* out, int32_t F, int32_t heads,
                             int dtype, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(F > 0 && F % 2 == 0, "feature length %d must be even and positive", F);
  HG_REQUIRE(heads >= 1 && F % heads == 0 && (F / heads) % 2 == 0,
             "feature length %d does not split into %d even heads", F, heads);
  cudaStream_t st = as_stream(stream);
  const int fh = F / heads;
  const int4* u = reinterpret_cast<const int4*>(units);
  const bool aligned = reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0;
  SdPacks pk{reinterpret_cast<const int4*>(packs), packs && num_edges > 0 ? num_packs : 0,
             pack_rowid};
  HG_REQUIRE(pk.np == 0 || pack_rowid, "hg_sddmm_fast: packs need pack_rowid");
  int rc = -1;
  const bool aligned32 = reinterpret_cast<uintptr_t>(x) % 32 == 0 && reinterpret_cast<uintptr_t>(y) % 32 == 0;
  if (dtype == HG_F16 && aligned32 && fh % 16 == 0 && F >= 64 && F <= 512 && sd_lane32())
    rc = dispatch_sddmm_fast<__half, 16>(u, num_units, pk, cols, x, y, out, F, heads, st);
  else if (dtype == HG_F16 && aligned && fh % 8 == 0)
    rc = dispatch_sddmm_fast<__half, 8>(u, num_units, pk, cols, x, y, out, F, heads, st);
  else if (dtype == HG_F16)
    rc = dispatch_sddmm_fast<__half, 2>(u, num_units, pk, cols, x, y, out, F, heads, st);
  else if (aligned && fh % 4 == 0)
    rc = dispatch_sddmm_fast<float, 4>(u, num_units, pk, cols, x, y, out, F, heads, st);
  else
    rc = dispatch_sddmm_fast<float, 2>(u, num_units, pk, cols, x, y, out, F, heads, st);
  if (rc >= 0) return rc;
  HG_REQUIRE(pk.np == 0, "hg_sddmm_fast: layout F=%d heads=%d is outside the butterfly kernel; "
             "build the schedule without packs", F, heads);
  // layouts outside the butterfly kernel (F/V > 32, non-power-of-two heads):
  // the exact kernel (its result is within the fast tolerance by definition)
  return hg_sddmm(offsets, cols, n_rows, num_edges, units, num_units, x, y, out, F, heads,
                  dtype, stream);
}

extern "C" int hg_sddmm(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                        int64_t num_edges, const int32_t* units, int64_t num_units,
                        const void* x, const void* y, void* out, int32_t F, int32_t heads,
                        int dtype, void* stream) {
  (void)offsets; (void)n_rows; (void)num_edges;
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(F > 0 && F % 2 == 0, "feature length %d must be even and positive", F);
  HG_REQUIRE(heads >= 1 && F % heads == 0 && (F / heads) % 2 == 0,
             "feature length %d does not split into %d even heads", F, heads);
  cudaStream_t st = as_stream(stream);
  const int fh = F / heads;
  const int4* u = reinterpret_cast<const int4*>(units);
  const bool aligned = reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0;
  if (dtype == HG_F16) {
    if (aligned && fh % 8 == 0) return dispatch_sddmm<__half, 8>(u, num_units, cols, x, y, out, F, heads, st);
    return dispatch_sddmm<__half, 2>(u, num_units, cols, x, y, out, F, heads, st);
  }
  if (aligned && fh % 4 == 0) return dispatch_sddmm<float, 4>(u, num_units, cols, x, y, out, F, heads, st);
  return dispatch_sddmm<float, 2>(u, num_units, cols, x, y, out, F, heads, st);
}

// --------------------------------------------------------- attention scores

namespace hg {

// Edge-parallel: 256 consecutive edges per block, rows located by a block-local
// binary search between the block's first and last rows.
template <typename T>
__global__ void k_attn_scores(const int64_t* __restrict__ offsets, const int32_t* __restrict__ cols,
                              int64_t n_rows, int64_t num_edges, const T* __restrict__ sl,
                              const T* __restrict__ sr, int heads, double slope,
                              T* __restrict__ out) {
  using N = Num<T>;
  __shared__ int64_t rng[2];
  const int64_t e0 = (int64_t)blockIdx.x * blockDim.x;
  if (e0 >= num_edges) return;
  const int64_t elast = e0 + blockDim.x - 1 < num_edges ? e0 + blockDim.x - 1 : num_edges - 1;
  if (threadIdx.x == 0) rng[0] = row_of_edge(offsets, n_rows, e0);
  if (threadIdx.x == 1 || blockDim.x == 1) rng[1] = row_of_edge(offsets, n_rows, elast);
  __syncthreads();
  const int64_t e = e0 + threadIdx.x;
  if (e >= num_edges) return;
  int64_t lo = rng[0], hi = rng[1] + 1;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (offsets[mid] <= e) lo = mid; else hi = mid;
  }
  const int64_t r = lo, c = cols[e];
  for (int h = 0; h < heads; ++h) {
    const T s = N::add(sl[r * heads + h], sr[c * heads + h]);
    out[e * heads + h] = N::gt0(s) ? s : N::from_d(N::to_d(s) * slope);
  }
}

// ------------------------------------------------------------ edge softmax

// rnd(exp(x)) for binary16 x: table of all 65536 inputs, generated at build
// time from numpy's float64 exp (exact by construction); binary32 uses fp64 exp.
__device__ const unsigned short kExp16[65536] = {
#include "hg_exp16.inc"
};

template <typename T>
__device__ __forceinline__ T exp_rnd(T x) {
  if constexpr (sizeof(T) == 2) return __ushort_as_half(__ldg(&kExp16[__half_as_ushort(x)]));
  else return Num<T>::from_d(exp(Num<T>::to_d(x)));
}

// rnd(a / b): for binary16 an fp32 IEEE quotient rounded once more is the
// correctly rounded half quotient (24 >= 2*11 + 2); binary32 divides in fp64.
template <typename T>
__device__ __forceinline__ T div_rnd(T a, T b) {
  if constexpr (sizeof(T) == 2) return __float2half_rn(__fdiv_rn(__half2float(a), __half2float(b)));
  else return Num<T>::from_d(Num<T>::to_d(a) / Num<T>::to_d(b));
}

// Adjacent-pair tree over a row's values, evaluated 32 at a time.
template <typename T>
struct RowTree {
  T stk[40];
  int64_t blocks = 0;
  // v: lane's element of the block starting at `base`; valid iff base + lane < len.
  __device__ __forceinline__ void push(T v, int64_t base, int64_t len, int lane) {
    using N = Num<T>;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const T o = shfl_down_t(0xffffffffu, v, s, 32);
      if ((lane & (2 * s - 1)) == 0 && base + lane + s < len) v = N::add(v, o);
    }
    T cur = shfl_t(v);
    int64_t t = blocks;
    int lvl = 0;
    while (t & 1) {
      cur = N::add(stk[lvl], cur);
      t >>= 1;
      ++lvl;
    }
    stk[lvl] = cur;
    ++blocks;
  }
  // Push the root of the next aligned block (computed elsewhere).
  __device__ __forceinline__ void push_root(T cur) {
    using N = Num<T>;
    int64_t t = blocks;
    int lvl = 0;
    while (t & 1) {
      cur = N::add(stk[lvl], cur);
      t >>= 1;
      ++lvl;
    }
    stk[lvl] = cur;
    ++blocks;
  }
  __device__ __forceinline__ T root() const {
    using N = Num<T>;
    T acc = N::zero();
    bool have = false;
    for (int lvl = 0; (blocks >> lvl) != 0; ++lvl) {
      if ((blocks >> lvl) & 1) {
        acc = have ? N::add(stk[lvl], acc) : stk[lvl];
        have = true;
      }
    }
    return acc;
  }
  static __device__ __forceinline__ T shfl_t(T v) {
    if constexpr (sizeof(T) == 2)
      return __ushort_as_half((unsigned short)__shfl_sync(0xffffffffu, (unsigned)__half_as_ushort(v), 0));
    else
      return __shfl_sync(0xffffffffu, v, 0);
  }
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, s));
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_softmax_fwd(const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ e,
              T* __restrict__ alpha, int heads, int64_t long_thresh) {
  using N = Num<T>;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], len = offsets[r + 1] - beg;
    if (len == 0 || len > long_thresh) continue;
    for (int h = 0; h < heads; ++h) {
      float m = -INFINITY;
      bool nan = false;
      for (int64_t i = lane; i < len; i += 32) {
        const float v = N::to_f(e[(beg + i) * heads + h]);
        nan |= v != v;
        m = fmaxf(m, v);
      }
      m = warp_max(m);
      nan = __any_sync(0xffffffffu, nan);
      const T mt = nan ? N::from_f(NAN) : N::from_f(m);  // np.maximum propagates NaN
      RowTree<T> tree;
      for (int64_t b = 0; b < len; b += 32) {
        const int64_t i = b + lane;
        T ex = N::zero();
        if (i < len) {
          const T s = N::sub(e[(beg + i) * heads + h], mt);
          ex = exp_rnd<T>(s);
          alpha[(beg + i) * heads + h] = ex;
        }
        tree.push(ex, b, len, lane);
      }
      const T den = tree.root();
      for (int64_t i = lane; i < len; i += 32) {
        const int64_t k = (beg + i) * heads + h;
        alpha[k] = div_rnd<T>(alpha[k], den);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_softmax_bwd(const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ alpha,
              const T* __restrict__ g, T* __restrict__ de, int heads, int64_t long_thresh) {
  using N = Num<T>;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], len = offsets[r + 1] - beg;
    if (len == 0 || len > long_thresh) continue;
    for (int h = 0; h < heads; ++h) {
      RowTree<T> tree;
      for (int64_t b = 0; b < len; b += 32) {
        const int64_t i = b + lane;
        T p = N::zero();
        if (i < len) {
          const int64_t k = (beg + i) * heads + h;
          p = N::mul(alpha[k], g[k]);
        }
        tree.push(p, b, len, lane);
      }
      const T s = tree.root();
      for (int64_t i = lane; i < len; i += 32) {
        const int64_t k = (beg + i) * heads + h;
        de[k] = N::mul(alpha[k], N::sub(g[k], s));
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_edge_rowsum(const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ v,
              const int32_t* __restrict__ perm, int heads, T* __restrict__ out,
              int64_t long_thresh) {
  using N = Num<T>;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], end = offsets[r + 1];
    if (end - beg > long_thresh) continue;
    for (int h = 0; h < heads; ++h) {
      float s = 0.0f;
      for (int64_t i = beg + lane; i < end; i += 32) {
        const int64_t idx = perm ? (int64_t)perm[i] : i;
        s += N::to_f(v[idx * heads + h]);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) out[r * heads + h] = N::from_f(s);
    }
  }
}

// ------------------------------------ short rows, all heads per warp pass
// Lane l works on edge (l / H) of the current 32/H-edge block and head l % H
// (edge-major [E, H] storage: a warp reads 64 contiguous bytes).  Per-head
// trees combine lanes at stride H; block roots are pushed on a per-lane
// binary-counter stack (replicated across the lanes of a head).

template <typename T, int H>
struct HeadTree {
  T stk[40];
  int64_t blocks = 0;
  static constexpr int EPB = 32 / H;  // edges per block
  // v: this lane's element (edge base + lane/H, head lane%H); returns nothing,
  // pushes the block root for this lane's head.
  __device__ __forceinline__ void push(T v, int64_t base, int64_t len, int lane) {
    using N = Num<T>;
    const int j = lane / H;
#pragma unroll
    for (int s = 1; s < EPB; s <<= 1) {
      const T o = shfl_down_t(0xffffffffu, v, s * H, 32);
      if ((j & (2 * s - 1)) == 0 && base + j + s < len) v = N::add(v, o);
    }
    T cur;
    if constexpr (sizeof(T) == 2)
      cur = __ushort_as_half((unsigned short)__shfl_sync(0xffffffffu, (unsigned)__half_as_ushort(v), lane % H));
    else
      cur = __shfl_sync(0xffffffffu, v, lane % H);
    int64_t t = blocks;
    int lvl = 0;
    while (t & 1) {
      cur = N::add(stk[lvl], cur);
      t >>= 1;
      ++lvl;
    }
    stk[lvl] = cur;
    ++blocks;
  }
  __device__ __forceinline__ T root() const {
    using N = Num<T>;
    T acc = N::zero();
    bool have = false;
    for (int lvl = 0; (blocks >> lvl) != 0; ++lvl) {
      if ((blocks >> lvl) & 1) {
        acc = have ? N::add(stk[lvl], acc) : stk[lvl];
        have = true;
      }
    }
    return acc;
  }
};

template <int H>
__device__ __forceinline__ float head_max(float v) {
#pragma unroll
  for (int s = 16; s >= H; s >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, s));
  return v;
}

template <typename T, int H>
__global__ void __launch_bounds__(256)
k_softmax_fwd_h(const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ e,
                T* __restrict__ alpha, int64_t long_thresh) {
  using N = Num<T>;
  constexpr int EPB = 32 / H;
  const int lane = threadIdx.x & 31;
  const int j = lane / H;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], len = offsets[r + 1] - beg;
    if (len == 0 || len > long_thresh) continue;
    const T* er = e + beg * H;
    T* ar = alpha + beg * H;
    float m = -INFINITY;
    bool nan = false;
    for (int64_t i = lane; i < len * H; i += 32) {
      const float v = N::to_f(er[i]);
      nan |= v != v;
      m = fmaxf(m, v);
    }
    m = head_max<H>(m);
    nan = head_max<H>(nan ? 1.0f : 0.0f) > 0.0f;
    const T mt = nan ? N::from_f(NAN) : N::from_f(m);
    HeadTree<T, H> tree;
    for (int64_t b = 0; b < len; b += EPB) {
      const int64_t i = b + j;
      T ex = N::zero();
      if (i < len) {
        ex = exp_rnd<T>(N::sub(er[i * H + lane % H], mt));
        ar[i * H + lane % H] = ex;
      }
      tree.push(ex, b, len, lane);
    }
    const T den = tree.root();
    for (int64_t i = lane; i < len * H; i += 32) ar[i] = div_rnd<T>(ar[i], den);
  }
}

template <typename T, int H>
__global__ void __launch_bounds__(256)
k_softmax_bwd_h(const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ alpha,
                const T* __restrict__ g, T* __restrict__ de, int64_t long_thresh) {
  using N = Num<T>;
  constexpr int EPB = 32 / H;
  const int lane = threadIdx.x & 31;
  const int j = lane / H;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], len = offsets[r + 1] - beg;
    if (len == 0 || len > long_thresh) continue;
    const T* a = alpha + beg * H;
    const T* gr = g + beg * H;
    HeadTree<T, H> tree;
    for (int64_t b = 0; b < len; b += EPB) {
      const int64_t i = b + j;
      T p = N::zero();
      if (i < len) p = N::mul(a[i * H + lane % H], gr[i * H + lane % H]);
      tree.push(p, b, len, lane);
    }
    const T sv = tree.root();  // this lane's head
    // lanes of a head hold its root; element k = (edge, head) reads head k % H,
    // which for the strided loop below is again lane % H (32 % H == 0)
    for (int64_t k = lane; k < len * H; k += 32) de[beg * H + k] = N::mul(a[k], N::sub(gr[k], sv));
  }
}

template <typename T, int H>
__global__ void __launch_bounds__(256)
k_edge_rowsum_h(const int64_t* __restrict__ offsets, int64_t n_rows, const T* __restrict__ v,
                const int32_t* __restrict__ perm, T* __restrict__ out, int64_t long_thresh) {
  const int lane = threadIdx.x & 31;
  constexpr int EPB = 32 / H;
  const int j = lane / H, h = lane % H;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], end = offsets[r + 1];
    if (end - beg > long_thresh) continue;
    float s = 0.0f;
    for (int64_t i = beg + j; i < end; i += EPB) {
      const int64_t idx = perm ? (int64_t)perm[i] : i;
      s += Num<T>::to_f(v[idx * H + h]);
    }
#pragma unroll
    for (int o = 16; o >= H; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane < H) out[r * H + lane] = Num<T>::from_f(s);
  }
}

// ------------------------------------------------ long rows: one CTA per row
// 1024 threads cover a 1024-element superblock per step: each warp reduces its
// aligned 32-element block (predicated shuffles), warp 0 reduces the 32 block
// roots the same way, and thread 0 pushes the superblock root onto the
// binary-counter stack -- the same implicit aligned tree as the warp path.

template <typename T>
__device__ __forceinline__ T superblock_root(T v, int64_t sb, int64_t len, T* roots) {
  using N = Num<T>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = sb + (int64_t)warp * 32;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const T o = shfl_down_t(0xffffffffu, v, s, 32);
    if ((lane & (2 * s - 1)) == 0 && base + lane + s < len) v = N::add(v, o);
  }
  if (lane == 0) roots[warp] = v;
  __syncthreads();
  T r = N::zero();
  if (warp == 0) {
    r = roots[lane];
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const T o = shfl_down_t(0xffffffffu, r, s, 32);
      if ((lane & (2 * s - 1)) == 0 && sb + 32 * (int64_t)(lane + s) < len) r = N::add(r, o);
    }
  }
  __syncthreads();
  return r;  // valid in thread 0
}

__device__ __forceinline__ float block_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = warp_max(red[lane]);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const float r = red[0];
  __syncthreads();
  return r;
}

template <typename T>
__global__ void __launch_bounds__(1024)
k_softmax_fwd_long(const int64_t* __restrict__ offsets, const int32_t* __restrict__ rows,
                   const T* __restrict__ e, T* __restrict__ alpha, int heads) {
  using N = Num<T>;
  __shared__ T roots[32];
  __shared__ float red[32];
  __shared__ T den_s;
  const int64_t r = rows[blockIdx.x];
  const int64_t beg = offsets[r], len = offsets[r + 1] - beg;
  for (int h = 0; h < heads; ++h) {
    float m = -INFINITY, nanf_ = 0.0f;
    for (int64_t i = threadIdx.x; i < len; i += 1024) {
      const float v = N::to_f(e[(beg + i) * heads + h]);
      if (v != v) nanf_ = 1.0f;
      m = fmaxf(m, v);
    }
    m = block_max(m, red);
    const bool nan = block_max(nanf_, red) > 0.0f;
    const T mt = nan ? N::from_f(NAN) : N::from_f(m);
    RowTree<T> tree;
    for (int64_t sb = 0; sb < len; sb += 1024) {
      const int64_t i = sb + threadIdx.x;
      T ex = N::zero();
      if (i < len) {
        const T sv = N::sub(e[(beg + i) * heads + h], mt);
        ex = exp_rnd<T>(sv);
        alpha[(beg + i) * heads + h] = ex;
      }
      const T rt = superblock_root(ex, sb, len, roots);
      if (threadIdx.x == 0) tree.push_root(rt);
    }
    if (threadIdx.x == 0) den_s = tree.root();
    __syncthreads();
    const T den = den_s;
    for (int64_t i = threadIdx.x; i < len; i += 1024) {
      const int64_t k = (beg + i) * heads + h;
      alpha[k] = div_rnd<T>(alpha[k], den);
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(1024)
k_softmax_bwd_long(const int64_t* __restrict__ offsets, const int32_t* __restrict__ rows,
                   const T* __restrict__ alpha, const T* __restrict__ g, T* __restrict__ de,
                   int heads) {
  using N = Num<T>;
  __shared__ T roots[32];
  __shared__ T s_s;
  const int64_t r = rows[blockIdx.x];
  const int64_t beg = offsets[r], len = offsets[r + 1] - beg;
  for (int h = 0; h < heads; ++h) {
    RowTree<T> tree;
    for (int64_t sb = 0; sb < len; sb += 1024) {
      const int64_t i = sb + threadIdx.x;
      T p = N::zero();
      if (i < len) {
        const int64_t k = (beg + i) * heads + h;
        p = N::mul(alpha[k], g[k]);
      }
      const T rt = superblock_root(p, sb, len, roots);
      if (threadIdx.x == 0) tree.push_root(rt);
    }
    if (threadIdx.x == 0) s_s = tree.root();
    __syncthreads();
    const T sv = s_s;
    for (int64_t i = threadIdx.x; i < len; i += 1024) {
      const int64_t k = (beg + i) * heads + h;
      de[k] = N::mul(alpha[k], N::sub(g[k], sv));
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(1024)
k_edge_rowsum_long(const int64_t* __restrict__ offsets, const int32_t* __restrict__ rows,
                   const T* __restrict__ v, const int32_t* __restrict__ perm, int heads,
                   T* __restrict__ out) {
  __shared__ float red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = rows[blockIdx.x];
  const int64_t beg = offsets[r], end = offsets[r + 1];
  for (int h = 0; h < heads; ++h) {
    float s = 0.0f;
    for (int64_t i = beg + threadIdx.x; i < end; i += 1024) {
      const int64_t idx = perm ? (int64_t)perm[i] : i;
      s += Num<T>::to_f(v[idx * heads + h]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (warp == 0) {
      s = red[lane];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) out[r * heads + h] = Num<T>::from_f(s);
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void k_scale_f64(const T* __restrict__ x, double s, T* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = Num<T>::from_d(Num<T>::to_d(x[i]) * s);
}

}  // namespace hg

extern "C" int hg_attn_scores(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                              int64_t num_edges, const void* s_l, const void* s_r,
                              int32_t heads, double slope, void* out, int dtype, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1, "heads must be positive");
  if (num_edges == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const unsigned g = (unsigned)((num_edges + 255) / 256);
  if (dtype == HG_F16)
    k_attn_scores<__half><<<g, 256, 0, st>>>(offsets, cols, n_rows, num_edges, (const __half*)s_l,
                                             (const __half*)s_r, heads, slope, (__half*)out);
  else
    k_attn_scores<float><<<g, 256, 0, st>>>(offsets, cols, n_rows, num_edges, (const float*)s_l,
                                            (const float*)s_r, heads, slope, (float*)out);
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_edge_softmax_fwd(const int64_t* offsets, int64_t n_rows, int64_t num_edges,
                                   const void* e, void* alpha, int32_t heads,
                                   const int32_t* long_rows, int64_t n_long, int64_t long_thresh,
                                   int dtype, void* stream) {
  (void)num_edges;
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1, "heads must be positive");
  HG_REQUIRE(n_long == 0 || long_rows, "long rows listed without an index array");
  if (n_rows == 0) return HG_OK;
  if (n_long == 0) long_thresh = INT64_MAX;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(n_rows, 8, 148 * 64);
  const bool pow2 = heads <= 16 && (heads & (heads - 1)) == 0;
#define HG_SMF(TT)                                                                          \
  switch (heads) {                                                                          \
    case 1: k_softmax_fwd_h<TT, 1><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)e, (TT*)alpha, long_thresh); break; \
    case 2: k_softmax_fwd_h<TT, 2><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)e, (TT*)alpha, long_thresh); break; \
    case 4: k_softmax_fwd_h<TT, 4><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)e, (TT*)alpha, long_thresh); break; \
    case 8: k_softmax_fwd_h<TT, 8><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)e, (TT*)alpha, long_thresh); break; \
    default: k_softmax_fwd_h<TT, 16><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)e, (TT*)alpha, long_thresh); \
  }
  if (dtype == HG_F16 && pow2) {
    HG_SMF(__half)
    if (n_long)
      k_softmax_fwd_long<__half><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const __half*)e, (__half*)alpha, heads);
  } else if (dtype == HG_F32 && pow2) {
    HG_SMF(float)
    if (n_long)
      k_softmax_fwd_long<float><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const float*)e, (float*)alpha, heads);
  } else if (dtype == HG_F16) {
    k_softmax_fwd<__half><<<g, 256, 0, st>>>(offsets, n_rows, (const __half*)e, (__half*)alpha,
                                             heads, long_thresh);
    if (n_long)
      k_softmax_fwd_long<__half><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const __half*)e, (__half*)alpha, heads);
  } else {
    k_softmax_fwd<float><<<g, 256, 0, st>>>(offsets, n_rows, (const float*)e, (float*)alpha,
                                            heads, long_thresh);
    if (n_long)
      k_softmax_fwd_long<float><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const float*)e, (float*)alpha, heads);
  }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_edge_softmax_bwd(const int64_t* offsets, int64_t n_rows, int64_t num_edges,
                                   const void* alpha, const void* grad, void* de, int32_t heads,
                                   const int32_t* long_rows, int64_t n_long, int64_t long_thresh,
                                   int dtype, void* stream) {
  (void)num_edges;
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1, "heads must be positive");
  HG_REQUIRE(n_long == 0 || long_rows, "long rows listed without an index array");
  if (n_rows == 0) return HG_OK;
  if (n_long == 0) long_thresh = INT64_MAX;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(n_rows, 8, 148 * 64);
  const bool pow2 = heads <= 16 && (heads & (heads - 1)) == 0;
#define HG_SMB(TT)                                                                          \
  switch (heads) {                                                                          \
    case 1: k_softmax_bwd_h<TT, 1><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)alpha, (const TT*)grad, (TT*)de, long_thresh); break; \
    case 2: k_softmax_bwd_h<TT, 2><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)alpha, (const TT*)grad, (TT*)de, long_thresh); break; \
    case 4: k_softmax_bwd_h<TT, 4><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)alpha, (const TT*)grad, (TT*)de, long_thresh); break; \
    case 8: k_softmax_bwd_h<TT, 8><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)alpha, (const TT*)grad, (TT*)de, long_thresh); break; \
    default: k_softmax_bwd_h<TT, 16><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)alpha, (const TT*)grad, (TT*)de, long_thresh); \
  }
  if (dtype == HG_F16 && pow2) {
    HG_SMB(__half)
    if (n_long)
      k_softmax_bwd_long<__half><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const __half*)alpha, (const __half*)grad, (__half*)de, heads);
  } else if (dtype == HG_F32 && pow2) {
    HG_SMB(float)
    if (n_long)
      k_softmax_bwd_long<float><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const float*)alpha, (const float*)grad, (float*)de, heads);
  } else if (dtype == HG_F16) {
    k_softmax_bwd<__half><<<g, 256, 0, st>>>(offsets, n_rows, (const __half*)alpha,
                                             (const __half*)grad, (__half*)de, heads, long_thresh);
    if (n_long)
      k_softmax_bwd_long<__half><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const __half*)alpha, (const __half*)grad, (__half*)de, heads);
  } else {
    k_softmax_bwd<float><<<g, 256, 0, st>>>(offsets, n_rows, (const float*)alpha,
                                            (const float*)grad, (float*)de, heads, long_thresh);
    if (n_long)
      k_softmax_bwd_long<float><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const float*)alpha, (const float*)grad, (float*)de, heads);
  }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_edge_rowsum(const int64_t* offsets, int64_t n_rows, int64_t num_edges,
                              const void* vals, const int32_t* perm, int32_t heads, void* out,
                              const int32_t* long_rows, int64_t n_long, int64_t long_thresh,
                              int dtype, void* stream) {
  (void)num_edges;
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1, "heads must be positive");
  HG_REQUIRE(n_long == 0 || long_rows, "long rows listed without an index array");
  if (n_rows == 0) return HG_OK;
  if (n_long == 0) long_thresh = INT64_MAX;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(n_rows, 8, 148 * 64);
  const bool pow2 = heads <= 16 && (heads & (heads - 1)) == 0;
#define HG_RS(TT)                                                                           \
  switch (heads) {                                                                          \
    case 1: k_edge_rowsum_h<TT, 1><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)vals, perm, (TT*)out, long_thresh); break; \
    case 2: k_edge_rowsum_h<TT, 2><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)vals, perm, (TT*)out, long_thresh); break; \
    case 4: k_edge_rowsum_h<TT, 4><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)vals, perm, (TT*)out, long_thresh); break; \
    case 8: k_edge_rowsum_h<TT, 8><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)vals, perm, (TT*)out, long_thresh); break; \
    default: k_edge_rowsum_h<TT, 16><<<g, 256, 0, st>>>(offsets, n_rows, (const TT*)vals, perm, (TT*)out, long_thresh); \
  }
  if (dtype == HG_F16 && pow2) {
    HG_RS(__half)
    if (n_long)
      k_edge_rowsum_long<__half><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const __half*)vals, perm, heads, (__half*)out);
  } else if (dtype == HG_F32 && pow2) {
    HG_RS(float)
    if (n_long)
      k_edge_rowsum_long<float><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const float*)vals, perm, heads, (float*)out);
  } else if (dtype == HG_F16) {
    k_edge_rowsum<__half><<<g, 256, 0, st>>>(offsets, n_rows, (const __half*)vals, perm, heads,
                                             (__half*)out, long_thresh);
    if (n_long)
      k_edge_rowsum_long<__half><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const __half*)vals, perm, heads, (__half*)out);
  } else {
    k_edge_rowsum<float><<<g, 256, 0, st>>>(offsets, n_rows, (const float*)vals, perm, heads,
                                            (float*)out, long_thresh);
    if (n_long)
      k_edge_rowsum_long<float><<<(unsigned)n_long, 1024, 0, st>>>(
          offsets, long_rows, (const float*)vals, perm, heads, (float*)out);
  }
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_scale_f64(const void* x, double s, void* out, int64_t count, int dtype,
                            void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  if (count == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(count, 256, 148 * 16);
  if (dtype == HG_F16)
    k_scale_f64<__half><<<g, 256, 0, st>>>((const __half*)x, s, (__half*)out, count);
  else
    k_scale_f64<float><<<g, 256, 0, st>>>((const float*)x, s, (float*)out, count);
  HG_LAUNCHED();
  return HG_OK;
}

// ------------------------------------------------------------ cross entropy

namespace hg {

// A team of TEAM lanes per row; lane t holds classes t, t+TEAM, ... (K per
// lane in registers, one fp64 exp per class; several rows per warp keep the
// fp64 latency chains overlapped).  fp64 like the reference; logits are read
// in their storage type (fp16 widens exactly, as models.convert does) and the
// gradient is rounded to fp32 first (the reference's float32 grad), scaled by
// an exact power of two, then to the gradient type (convert's backward).
template <typename L, typename G, int TEAM, int K>
__global__ void __launch_bounds__(256)
k_softmax_xent(const L* __restrict__ logits, int64_t ld, const int64_t* __restrict__ labels,
               int64_t n, int c_active, double denom, float scale, G* __restrict__ grad,
               double* __restrict__ nll) {
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TEAM - 1);
  const unsigned tmask = TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << (lane & ~(TEAM - 1)));
  const int64_t teams = (int64_t)gridDim.x * (blockDim.x / TEAM);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM; r < n; r += teams) {
    const L* z = logits + r * ld;
    double zv[K];
    double m = -INFINITY;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = tl + TEAM * k;
      zv[k] = j < c_active ? (double)Num<L>::to_f(z[j]) : -INFINITY;
      m = fmax(m, zv[k]);
    }
#pragma unroll
    for (int o = TEAM / 2; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(tmask, m, o, TEAM));
    double se = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      zv[k] = tl + TEAM * k < c_active ? exp(zv[k] - m) : 0.0;
      se += zv[k];
    }
#pragma unroll
    for (int o = TEAM / 2; o >= 1; o >>= 1) se += __shfl_xor_sync(tmask, se, o, TEAM);
    const int64_t lab = labels[r];
    G* g = grad + r * ld;
    // reciprocals instead of the reference's two divisions: the fp64 results
    // differ in the last bit at most, below the fp32 rounding that follows
    const double rse = 1.0 / se, rden = 1.0 / denom;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = tl + TEAM * k;
      if (j < ld) {
        float v = 0.0f;
        if (j < c_active) v = (float)((zv[k] * rse - (j == lab ? 1.0 : 0.0)) * rden) * scale;
        g[j] = Num<G>::from_f(v);
      }
    }
    if (tl == 0) nll[r] = log(se) - ((double)Num<L>::to_f(z[lab]) - m);
  }
}

// Classes beyond 32*K: recompute the exponentials (same operations).
template <typename L, typename G>
__global__ void __launch_bounds__(256)
k_softmax_xent_wide(const L* __restrict__ logits, int64_t ld, const int64_t* __restrict__ labels,
                    int64_t n, int c_active, double denom, float scale, G* __restrict__ grad,
                    double* __restrict__ nll) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
       r += nwarps) {
    const L* z = logits + r * ld;
    double m = -INFINITY;
    for (int j = lane; j < c_active; j += 32) m = fmax(m, (double)Num<L>::to_f(z[j]));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double se = 0.0;
    for (int j = lane; j < c_active; j += 32) se += exp((double)Num<L>::to_f(z[j]) - m);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int64_t lab = labels[r];
    G* g = grad + r * ld;
    for (int j = lane; j < ld; j += 32) {
      float v = 0.0f;
      if (j < c_active) {
        const double p = exp((double)Num<L>::to_f(z[j]) - m) / se;
        v = (float)((p - (j == lab ? 1.0 : 0.0)) / denom) * scale;
      }
      g[j] = Num<G>::from_f(v);
    }
    if (lane == 0) nll[r] = log(se) - ((double)Num<L>::to_f(z[lab]) - m);
  }
}

template <typename L, typename G>
static void launch_xent(const void* logits, int64_t ld, const int64_t* labels, int64_t n,
                        int c, double denom, float scale, void* grad, double* nll,
                        cudaStream_t st) {
  const L* lp = (const L*)logits;
  G* gp = (G*)grad;
  const int64_t w = ld > c ? ld : c;
#define HG_XENT(TEAM, K)                                                             \
  k_softmax_xent<L, G, TEAM, K><<<grid_for(n, 256 / TEAM, 148 * 32), 256, 0, st>>>( \
      lp, ld, labels, n, c, denom, scale, gp, nll)
  if (w <= 8) HG_XENT(8, 1);
  else if (w <= 16) HG_XENT(8, 2);
  else if (w <= 32) HG_XENT(8, 4);
  else if (w <= 48) HG_XENT(8, 6);
  else if (w <= 64) HG_XENT(8, 8);
  else if (w <= 128) HG_XENT(16, 8);
  else if (w <= 256) HG_XENT(32, 8);
  else k_softmax_xent_wide<L, G><<<grid_for(n, 8, 148 * 64), 256, 0, st>>>(lp, ld, labels, n, c, denom, scale, gp, nll);
#undef HG_XENT
}

}  // namespace hg

extern "C" int hg_softmax_xent(const void* logits, int logits_dtype, int64_t ld,
                               const int64_t* labels, int64_t n, int32_t c_active, double denom,
                               float grad_scale, void* grad, int grad_dtype, double* nll,
                               void* stream) {
  HG_REQUIRE(c_active >= 1 && c_active <= ld, "hg_softmax_xent: bad class counts");
  HG_REQUIRE((logits_dtype == HG_F16 || logits_dtype == HG_F32) &&
             (grad_dtype == HG_F16 || grad_dtype == HG_F32), "hg_softmax_xent: unknown dtype");
  if (n == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  if (logits_dtype == HG_F16) {
    if (grad_dtype == HG_F16) launch_xent<__half, __half>(logits, ld, labels, n, c_active, denom, grad_scale, grad, nll, st);
    else launch_xent<__half, float>(logits, ld, labels, n, c_active, denom, grad_scale, grad, nll, st);
  } else {
    if (grad_dtype == HG_F16) launch_xent<float, __half>(logits, ld, labels, n, c_active, denom, grad_scale, grad, nll, st);
    else launch_xent<float, float>(logits, ld, labels, n, c_active, denom, grad_scale, grad, nll, st);
  }
  HG_LAUNCHED();
  return HG_OK;
}

// --------------------------------------------------- GAT projections, Adam

namespace hg {

// Team of fh/V lanes per (node, head); lane chunk of V elements of z, a_l, a_r.
template <typename T, int V, int TEAM>
__global__ void __launch_bounds__(256)
k_head_dots(const T* __restrict__ z, const T* __restrict__ al, const T* __restrict__ ar,
            int64_t n, int heads, int fh, T* __restrict__ sl, T* __restrict__ sr) {
  using Raw = typename RawV<V * sizeof(T)>::type;
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TEAM - 1);
  const unsigned tmask =
      TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << (lane & ~(TEAM - 1)));
  const int64_t items = n * heads;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / TEAM);
  const int nchunk = fh / V;
  // grid-stride, IU (node, head) items in flight per team
  constexpr int IU = 4;
  for (int64_t it0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM; it0 < items;
       it0 += IU * stride) {
    float pl[IU], pr[IU];
#pragma unroll
    for (int u = 0; u < IU; ++u) pl[u] = pr[u] = 0.0f;
    for (int c = tl; c < nchunk; c += TEAM) {
      Raw zr[IU];
#pragma unroll
      for (int u = 0; u < IU; ++u) {
        const int64_t item = it0 + u * stride;
        if (item < items) {
          const int64_t node = item / heads;
          const int h = (int)(item - node * heads);
          zr[u] = *reinterpret_cast<const Raw*>(z + node * (int64_t)heads * fh + h * fh + c * V);
        }
      }
#pragma unroll
      for (int u = 0; u < IU; ++u) {
        const int64_t item = it0 + u * stride;
        if (item >= items) continue;
        const int h = (int)(item % heads);
        const int f = h * fh + c * V;
        const Raw lr_ = *reinterpret_cast<const Raw*>(al + f);
        const Raw rr_ = *reinterpret_cast<const Raw*>(ar + f);
        const T* za = reinterpret_cast<const T*>(&zr[u]);
        const T* la = reinterpret_cast<const T*>(&lr_);
        const T* ra = reinterpret_cast<const T*>(&rr_);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float zf = Num<T>::to_f(za[i]);
          pl[u] = fmaf(zf, Num<T>::to_f(la[i]), pl[u]);
          pr[u] = fmaf(zf, Num<T>::to_f(ra[i]), pr[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < IU; ++u) {
#pragma unroll
      for (int o = TEAM / 2; o >= 1; o >>= 1) {
        pl[u] += __shfl_xor_sync(tmask, pl[u], o, TEAM);
        pr[u] += __shfl_xor_sync(tmask, pr[u], o, TEAM);
      }
      const int64_t item = it0 + u * stride;
      if (tl == 0 && item < items) {
        sl[item] = Num<T>::from_f(pl[u]);
        sr[item] = Num<T>::from_f(pr[u]);
      }
    }
  }
}

// Head-dot backward, pass 1: blocks stride over rows; thread (rr, f) owns
// column f of row slot rr; writes gz and fp32 partial column sums.
constexpr int kHdbBlocks = 148 * 4;

template <typename T>
__global__ void __launch_bounds__(256)
k_head_dots_bwd(const T* __restrict__ z, const T* __restrict__ al, const T* __restrict__ ar,
                const T* __restrict__ gl, const T* __restrict__ gr, int64_t n, int heads, int fh,
                T* gz, const T* gz_in, float* __restrict__ part) {
  using N = Num<T>;
  const int F = heads * fh;
  const int rpi = F >= 256 ? 1 : 256 / F;
  const int rr = threadIdx.x / (F >= 256 ? 256 : F);
  for (int f0 = 0; f0 < F; f0 += 256) {
    const int f = f0 + (F >= 256 ? (int)threadIdx.x : (int)(threadIdx.x % F));
    const bool act = f < F && rr < rpi;
    const int h = act ? f / fh : 0;
    const T a1 = act ? al[f] : N::zero(), a2 = act ? ar[f] : N::zero();
    float sl = 0.0f, sr = 0.0f;
    if (act) {
      for (int64_t r = (int64_t)blockIdx.x * rpi + rr; r < n; r += (int64_t)gridDim.x * rpi) {
        const T g1 = gl[r * heads + h], g2 = gr[r * heads + h];
        const float zf = N::to_f(z[r * F + f]);
        const T v = N::add(N::mul(g1, a1), N::mul(g2, a2));
        if (gz) gz[r * F + f] = gz_in ? N::add(gz_in[r * F + f], v) : v;
        sl = fmaf(zf, N::to_f(g1), sl);
        sr = fmaf(zf, N::to_f(g2), sr);
      }
    }
    // fold the rpi row slots of the block in slot order (deterministic)
    __shared__ float bl[256], br[256];
    bl[threadIdx.x] = sl;
    br[threadIdx.x] = sr;
    __syncthreads();
    if (act && rr == 0) {
      float tl = 0.0f, tr = 0.0f;
      for (int q = 0; q < rpi; ++q) {
        tl += bl[q * (F >= 256 ? 256 : F) + (threadIdx.x)];
        tr += br[q * (F >= 256 ? 256 : F) + (threadIdx.x)];
      }
      part[((int64_t)blockIdx.x * 2 + 0) * F + f] = tl;
      part[((int64_t)blockIdx.x * 2 + 1) * F + f] = tr;
    }
    __syncthreads();
  }
}

// Vectorised pass 1 for binary16 with fh % 8 == 0: thread (rr, c) owns the
// 8-feature chunk c of row slot rr (one head), 16-byte loads / stores, fp32
// partials per feature folded over the row slots in slot order.  DZ = false
// (gz NULL: da only): no gz traffic, so <= 64 registers and all kHdbBlocks
// blocks resident at once -- the same rows in the same order, the same da bits.
template <bool DZ>
__global__ void __launch_bounds__(256, DZ ? 2 : 4)
k_head_dots_bwd_v8(const __half* __restrict__ z, const __half* __restrict__ al,
                   const __half* __restrict__ ar, const __half* __restrict__ gl,
                   const __half* __restrict__ gr, int64_t n, int heads, int fh,
                   __half* gz, const __half* gz_in, float* __restrict__ part) {
  extern __shared__ float hdb_sh[];  // [2][rpi][F]
  const int F = heads * fh, C = F / 8;
  const int rpi = 256 / C;
  const int rr = threadIdx.x / C, c = threadIdx.x - (threadIdx.x / C) * C;
  const bool act = rr < rpi;
  const int h = (c * 8) / fh;
  __align__(16) __half a1[8], a2[8];
  float sl[8], sr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) sl[i] = sr[i] = 0.0f;
  if (act) {
    *reinterpret_cast<uint4*>(a1) = *reinterpret_cast<const uint4*>(al + c * 8);
    *reinterpret_cast<uint4*>(a2) = *reinterpret_cast<const uint4*>(ar + c * 8);
    // RU rows per step, all their loads issued before any use (the row loop
    // was latency-bound with one 16-byte load in flight); rows still fold
    // into sl / sr in the same order, so the result is unchanged.
    constexpr int RU = 4;
    const int64_t stride = (int64_t)gridDim.x * rpi;
    for (int64_t r0 = (int64_t)blockIdx.x * rpi + rr; r0 < n; r0 += stride * RU) {
      __half g1[RU], g2[RU];
      uint4 zv[RU], prev[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int64_t r = r0 + u * stride;
        prev[u] = make_uint4(0, 0, 0, 0);
        if (r < n) {
          g1[u] = gl[r * heads + h];
          g2[u] = gr[r * heads + h];
          zv[u] = *reinterpret_cast<const uint4*>(z + r * F + c * 8);
          if (DZ && gz_in) prev[u] = *reinterpret_cast<const uint4*>(gz_in + r * F + c * 8);
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int64_t r = r0 + u * stride;
        if (r >= n) break;
        const float g1f = __half2float(g1[u]), g2f = __half2float(g2[u]);
        const __half* ze = reinterpret_cast<const __half*>(&zv[u]);
        const __half* pe = reinterpret_cast<const __half*>(&prev[u]);
        __align__(16) __half o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o[i] = __hadd_rn(__hmul_rn(g1[u], a1[i]), __hmul_rn(g2[u], a2[i]));
          if (gz_in) o[i] = __hadd_rn(pe[i], o[i]);
          const float zf = __half2float(ze[i]);
          sl[i] = fmaf(zf, g1f, sl[i]);
          sr[i] = fmaf(zf, g2f, sr[i]);
        }
        // gz NULL: the dz term went into the aggregation's store (hg_spmm head dots)
        if (DZ) *reinterpret_cast<uint4*>(gz + r * F + c * 8) = *reinterpret_cast<const uint4*>(o);
      }
    }
  }
  float* bl = hdb_sh;
  float* br = hdb_sh + rpi * F;
  if (act) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bl[rr * F + c * 8 + i] = sl[i];
      br[rr * F + c * 8 + i] = sr[i];
    }
  }
  __syncthreads();
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    float tl = 0.0f, tr = 0.0f;
    for (int q = 0; q < rpi; ++q) {
      tl += bl[q * F + f];
      tr += br[q * F + f];
    }
    part[((int64_t)blockIdx.x * 2 + 0) * F + f] = tl;
    part[((int64_t)blockIdx.x * 2 + 1) * F + f] = tr;
  }
}

// Pass 2: fold the per-block partials in block order, round once.
template <typename T>
__global__ void k_head_dots_bwd_fold(const float* __restrict__ part, int nblk, int F,
                                     T* __restrict__ gal, T* __restrict__ gar) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    float tl = 0.0f, tr = 0.0f;
    for (int b = 0; b < nblk; ++b) {
      tl += part[((int64_t)b * 2 + 0) * F + f];
      tr += part[((int64_t)b * 2 + 1) * F + f];
    }
    gal[f] = Num<T>::from_f(tl);
    gar[f] = Num<T>::from_f(tr);
  }
}

// Extras of the fused Adam step: the next step's published copy (and the
// transposed copies of up to kAdamMaxT 2-D weights, the forward GEMMs' B^T
// operands), the cleared gradient, and the step counter advanced in-kernel.
constexpr int kAdamMaxT = 8;
template <typename PT>
struct AdamExtra {
  PT* pub;
  PT* gzero;
  PT* pub_t;
  int* done;                 // non-null: t = *step + 1, written back by the last block
  int nt;
  int64_t t_off[kAdamMaxT], t_rows[kAdamMaxT], t_cols[kAdamMaxT], t_dst[kAdamMaxT];
};

template <typename G, typename PT>
__global__ void k_adam(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                       const G* __restrict__ grad, int64_t count, float lr, float omb1,
                       float omb2, double b1, double b2, float eps,
                       double* __restrict__ step, float unscale, const AdamExtra<PT> ex) {
  const double t = ex.done ? *step + 1.0 : *step;
  const float c1 = (float)(1.0 - pow(b1, t)), c2 = (float)(1.0 - pow(b2, t));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float g = __fmul_rn(Num<G>::to_f(grad[i]), unscale);
    float mi = m[i], vi = v[i];
    mi = __fadd_rn(mi, __fmul_rn(omb1, __fsub_rn(g, mi)));
    vi = __fadd_rn(vi, __fmul_rn(omb2, __fsub_rn(__fmul_rn(g, g), vi)));
    m[i] = mi;
    v[i] = vi;
    const float num = __fmul_rn(lr, __fdiv_rn(mi, c1));
    const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, c2)), eps);
    const float pn = __fsub_rn(p[i], __fdiv_rn(num, den));
    p[i] = pn;
    // the next step's published copy (ParamGroup.publish: RN cast of the
    // master), its transposed copy for 2-D weights, and the zeroed gradient,
    // fused here instead of separate passes
    if (ex.pub) {
      const PT h = Num<PT>::from_f(pn);
      ex.pub[i] = h;
      for (int j = 0; j < ex.nt; ++j) {
        const int64_t o = i - ex.t_off[j];
        if (o >= 0 && o < ex.t_rows[j] * ex.t_cols[j]) {
          const int64_t r = o / ex.t_cols[j], c = o - r * ex.t_cols[j];
          ex.pub_t[ex.t_dst[j] + c * ex.t_rows[j] + r] = h;
        }
      }
    }
    if (ex.gzero) ex.gzero[i] = Num<PT>::zero();
  }
  if (ex.done) {  // the last block to finish advances the device step count
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(ex.done, 1) == (int)gridDim.x - 1) {
        *step = t;
        *ex.done = 0;
      }
    }
  }
}

// loss = fp32(sum(nll) / denom): kLossBlocks blocks each sum a contiguous
// chunk (strided over the block's threads, then a fixed tree), the last block
// to finish (arrival counter, re-armed) adds the block partials in block order.
constexpr int kLossBlocks = 148;
__global__ void __launch_bounds__(512) k_loss_mean(const double* __restrict__ nll, int64_t n,
                                                   double denom, float* __restrict__ out,
                                                   double* __restrict__ part, int* __restrict__ done) {
  __shared__ double sh[512];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += nll[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sh[0];
    __threadfence();
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      __threadfence();
      double t = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(part + b);
      *out = (float)(t / denom);
      *done = 0;
    }
  }
}

}  // namespace hg

extern "C" int hg_head_dots(const void* z, const void* a_l, const void* a_r, int64_t n,
                            int32_t heads, int32_t fh, void* s_l, void* s_r, int dtype,
                            void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1 && fh >= 1, "hg_head_dots: bad shape");
  if (n == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t items = n * heads;
  const bool aligned = (reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(a_l) |
                        reinterpret_cast<uintptr_t>(a_r)) % 16 == 0;
#define HG_HD(TT, VV, TM)                                                                   \
  k_head_dots<TT, VV, TM><<<grid_for(items * TM, 256, 148 * 16), 256, 0, st>>>(            \
      (const TT*)z, (const TT*)a_l, (const TT*)a_r, n, heads, fh, (TT*)s_l, (TT*)s_r)
  if (dtype == HG_F16) {
    if (aligned && fh % 8 == 0) {
      const int nc = fh / 8;
      if (nc <= 1) HG_HD(__half, 8, 1);
      else if (nc <= 2) HG_HD(__half, 8, 2);
      else if (nc <= 4) HG_HD(__half, 8, 4);
      else if (nc <= 8) HG_HD(__half, 8, 8);
      else HG_HD(__half, 8, 16);
    } else {
      HG_HD(__half, 2, 8);
    }
  } else {
    if (aligned && fh % 4 == 0) HG_HD(float, 4, 8);
    else HG_HD(float, 1, 8);
  }
#undef HG_HD
  HG_LAUNCHED();
  return HG_OK;
}

template <typename PT>
static AdamExtra<PT> adam_extra(void* pub_out, void* grad_zero, int* step_done,
                                const int64_t* t_desc, int nt, void* pub_t) {
  AdamExtra<PT> ex{};
  ex.pub = (PT*)pub_out;
  ex.gzero = (PT*)grad_zero;
  ex.pub_t = (PT*)pub_t;
  ex.done = step_done;
  ex.nt = pub_t ? nt : 0;
  for (int j = 0; j < ex.nt; ++j) {
    ex.t_off[j] = t_desc[4 * j];
    ex.t_rows[j] = t_desc[4 * j + 1];
    ex.t_cols[j] = t_desc[4 * j + 2];
    ex.t_dst[j] = t_desc[4 * j + 3];
  }
  return ex;
}

extern "C" int hg_adam_step(float* master, float* m, float* v, const void* grad, int grad_dtype,
                            int64_t count, float lr, float omb1, float omb2, double b1, double b2,
                            float eps, double* step, float grad_unscale, void* pub_out,
                            void* grad_zero, int pub_dtype, int32_t* step_done,
                            const int64_t* t_desc, int32_t nt, void* pub_t, void* stream) {
  HG_REQUIRE(grad_dtype == HG_F16 || grad_dtype == HG_F32, "unknown dtype %d", grad_dtype);
  HG_REQUIRE(pub_dtype == HG_F16 || pub_dtype == HG_F32, "unknown dtype %d", pub_dtype);
  HG_REQUIRE(!(grad_zero == grad && grad_dtype != pub_dtype), "hg_adam_step: grad_zero aliases grad of another dtype");
  HG_REQUIRE(nt >= 0 && nt <= kAdamMaxT && (nt == 0 || (t_desc && pub_t && pub_out)),
             "hg_adam_step: at most %d transposed copies, with their descriptors", kAdamMaxT);
  if (count == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(count, 256, 148 * 8);
  if (grad_dtype == HG_F16 && pub_dtype == HG_F16)
    k_adam<__half, __half><<<g, 256, 0, st>>>(master, m, v, (const __half*)grad, count, lr, omb1,
                                              omb2, b1, b2, eps, step, grad_unscale,
                                              adam_extra<__half>(pub_out, grad_zero, step_done, t_desc, nt, pub_t));
  else if (grad_dtype == HG_F32 && pub_dtype == HG_F16)
    k_adam<float, __half><<<g, 256, 0, st>>>(master, m, v, (const float*)grad, count, lr, omb1,
                                             omb2, b1, b2, eps, step, grad_unscale,
                                             adam_extra<__half>(pub_out, grad_zero, step_done, t_desc, nt, pub_t));
  else if (grad_dtype == HG_F32)
    k_adam<float, float><<<g, 256, 0, st>>>(master, m, v, (const float*)grad, count, lr, omb1,
                                            omb2, b1, b2, eps, step, grad_unscale,
                                            adam_extra<float>(pub_out, grad_zero, step_done, t_desc, nt, pub_t));
  else
    HG_REQUIRE(false, "hg_adam_step: fp16 gradients with an fp32 published copy");
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_loss_mean_workspace(size_t* bytes) {
  HG_REQUIRE(bytes, "hg_loss_mean_workspace: null output");
  *bytes = kLossBlocks * sizeof(double) + 16;
  return HG_OK;
}

extern "C" int hg_loss_mean(const double* nll, int64_t n, double denom, float* loss_out,
                            void* ws, size_t ws_bytes, void* stream) {
  HG_REQUIRE(n >= 0 && loss_out && (n == 0 || nll), "hg_loss_mean: bad arguments");
  HG_REQUIRE(ws && ws_bytes >= kLossBlocks * sizeof(double) + 16 &&
                 (reinterpret_cast<uintptr_t>(ws) & 7) == 0,
             "hg_loss_mean: workspace too small");
  double* part = static_cast<double*>(ws);
  int* done = reinterpret_cast<int*>(part + kLossBlocks);
  k_loss_mean<<<kLossBlocks, 512, 0, as_stream(stream)>>>(nll, n, denom, loss_out, part, done);
  HG_LAUNCHED();
  return HG_OK;
}

extern "C" int hg_head_dots_bwd_workspace(int32_t heads, int32_t fh, size_t* bytes) {
  HG_REQUIRE(bytes && heads >= 1 && fh >= 1, "hg_head_dots_bwd_workspace: bad arguments");
  *bytes = (size_t)kHdbBlocks * 2 * heads * fh * sizeof(float);
  return HG_OK;
}

extern "C" int hg_head_dots_bwd(const void* z, const void* a_l, const void* a_r, const void* g_l,
                                const void* g_r, int64_t n, int32_t heads, int32_t fh, void* gz,
                                void* ga_l, void* ga_r, const void* gz_in, int dtype, void* ws,
                                size_t ws_bytes, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1 && fh >= 1, "hg_head_dots_bwd: bad shape");
  const int F = heads * fh;
  HG_REQUIRE(ws_bytes >= (size_t)kHdbBlocks * 2 * F * sizeof(float), "hg_head_dots_bwd: workspace too small");
  cudaStream_t st = as_stream(stream);
  float* part = (float*)ws;
  if (dtype == HG_F16) {
    const bool vec = fh % 8 == 0 && F / 8 <= 256 &&
                     ((reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(a_l) |
                       reinterpret_cast<uintptr_t>(a_r) | reinterpret_cast<uintptr_t>(gz)) & 15) == 0;
    if (vec) {
      const size_t sh = (size_t)2 * (256 / (F / 8)) * F * sizeof(float);
      if (sh > 48 * 1024)
        HG_CUDA(cudaFuncSetAttribute(gz ? k_head_dots_bwd_v8<true> : k_head_dots_bwd_v8<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
      (gz ? k_head_dots_bwd_v8<true> : k_head_dots_bwd_v8<false>)<<<kHdbBlocks, 256, sh, st>>>(
          (const __half*)z, (const __half*)a_l, (const __half*)a_r, (const __half*)g_l,
          (const __half*)g_r, n, heads, fh, (__half*)gz, (const __half*)gz_in, part);
    } else {
      k_head_dots_bwd<__half><<<kHdbBlocks, 256, 0, st>>>(
          (const __half*)z, (const __half*)a_l, (const __half*)a_r, (const __half*)g_l,
          (const __half*)g_r, n, heads, fh, (__half*)gz, (const __half*)gz_in, part);
    }
    k_head_dots_bwd_fold<__half><<<(F + 255) / 256, 256, 0, st>>>(part, kHdbBlocks, F,
                                                                (__half*)ga_l, (__half*)ga_r);
  } else {
    k_head_dots_bwd<float><<<kHdbBlocks, 256, 0, st>>>(
        (const float*)z, (const float*)a_l, (const float*)a_r, (const float*)g_l,
        (const float*)g_r, n, heads, fh, (float*)gz, (const float*)gz_in, part);
    k_head_dots_bwd_fold<float><<<(F + 255) / 256, 256, 0, st>>>(part, kHdbBlocks, F,
                                                               (float*)ga_l, (float*)ga_r);
  }
  HG_LAUNCHED();
  return HG_OK;
}
