// SpMM family for sm_100a.
//
//  * k_spmm_fast       fp32-guarded, row-owned: one lane team per work unit
//                      (hg_schedule_build), 128-bit gathers of neighbour rows,
//                      fp32 accumulation, one rounding at the row; heavy rows
//                      split into units whose fp32 carries are merged by
//                      k_spmm_fast_followup in slot order (no atomics).
//  * k_spmm_edge_ref   bit-exact replica of halfsparse's edge-parallel order
//                      (kernels.py:328-391 / _ref_spmm_edge 603-688).
//  * k_spmm_vertex_ref bit-exact replica of spmm_vertex_grouped (463-559).
#include <cstdlib>

#include "hg_common.cuh"

namespace hg {

template <int BYTES> struct RawVec;
// 32 bytes per lane: one LDG.256 (ld.global.nc.v8.b32, sm_100) per neighbour
// chunk -- half the load instructions of 16-byte lanes for the same bytes
struct alignas(32) U32x8 { uint32_t a[8]; };
template <> struct RawVec<32> { using type = U32x8; };
template <> struct RawVec<16> { using type = uint4; };
template <> struct RawVec<8> { using type = uint2; };
template <> struct RawVec<4> { using type = uint32_t; };

// Read-only gather of one lane chunk.
template <typename R>
__device__ __forceinline__ R ldg_raw(const R* p) {
  if constexpr (sizeof(R) == 32) {
    R v;
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]),
                   "=r"(v.a[5]), "=r"(v.a[6]), "=r"(v.a[7])
                 : "l"(p));
    return v;
  } else {
    return __ldg(p);
  }
}

// Convert a raw 16/8/4-byte vector of V elements of T to floats.
template <typename T, int V>
__device__ __forceinline__ void raw_to_float(const typename RawVec<V * sizeof(T)>::type& r,
                                             float (&f)[V]) {
  if constexpr (sizeof(T) == 2) {
    const __half2* h = reinterpret_cast<const __half2*>(&r);
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
      float2 t = __half22float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  } else {
    const float* p = reinterpret_cast<const float*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) f[i] = p[i];
  }
}

// fmode & 3: 0 -> rnd(S); 1 -> post: rnd(rnd(S) * f) for f > 0; 2 -> rnd(S * f);
// fmode & 4: then ReLU (models.relu: x > 0 ? x : 0, models.py:176-185).
template <typename T>
__device__ __forceinline__ T finalize_mode(float s, int fmode, T fo) {
  if ((fmode & 3) == 0) return Num<T>::from_f(s);
  if ((fmode & 3) == 1) {
    T h = Num<T>::from_f(s);
    return Num<T>::gt0(fo) ? Num<T>::mul(h, fo) : h;
  }
  return Num<T>::from_f(s * Num<T>::to_f(fo));
}

template <typename T>
__device__ __forceinline__ T finalize(float s, int fmode, T fo) {
  const T h = finalize_mode<T>(s, fmode, fo);
  return (fmode & 4) && !Num<T>::gt0(h) ? Num<T>::zero() : h;
}

template <typename T, int V>
__device__ __forceinline__ void store_out(T* dst, const float (&acc)[V], int fmode, T fo) {
  using Raw = typename RawVec<V * sizeof(T)>::type;
  Raw r;
  T* p = reinterpret_cast<T*>(&r);
#pragma unroll
  for (int i = 0; i < V; ++i) p[i] = finalize<T>(acc[i], fmode, fo);
  *reinterpret_cast<Raw*>(dst) = r;
}

// GIN's combine in the epilogue (models.py:220-240, scale_combine; hg_scale_combine):
// out = rnd(rnd(res * o) + rnd(h * lam)), h = the finished aggregate, products
// in fp64 -- the same roundings as the separate pass; o = lam = 1 is a plain
// rounded add (a residual gradient accumulated in the same store).
struct Combine {
  const void* res;   // NULL: off
  int64_t ldr;
  const void* ope;   // device scalar of the element type (NULL: 1)
  double lam;
  // GAT head-dot backward in the store (hg_head_dots_bwd's dz term): with
  // hgl set, out = rnd(h + rnd(rnd(gl[row, hd] al[c]) + rnd(gr[row, hd] ar[c]))),
  // hd = c / hfh -- the transposed aggregation's dz and the head dots' in one store
  const void* hgl;
  const void* hgr;
  const void* hal;
  const void* har;
  int hheads, hfh;
  int hcol0;  // the column slab's first column
};

template <typename T, int V>
__device__ __forceinline__ void store_out_comb(T* dst, const float (&acc)[V], int fmode, T fo,
                                               const T* res, double o, double lam) {
  using Raw = typename RawVec<V * sizeof(T)>::type;
  const Raw rr = *reinterpret_cast<const Raw*>(res);
  const T* re = reinterpret_cast<const T*>(&rr);
  Raw r;
  T* p = reinterpret_cast<T*>(&r);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const T h = finalize<T>(acc[i], fmode, fo);
    const T u = Num<T>::from_d(Num<T>::to_d(re[i]) * o);
    const T v = Num<T>::from_d(Num<T>::to_d(h) * lam);
    p[i] = Num<T>::add(u, v);
  }
  *reinterpret_cast<Raw*>(dst) = r;
}

template <typename T, int V>
__device__ __forceinline__ void store_out_hdots(T* dst, const float (&acc)[V], int fmode, T fo,
                                                const Combine& cb, int64_t row, int64_t col) {
  using Raw = typename RawVec<V * sizeof(T)>::type;
  const T* gl = static_cast<const T*>(cb.hgl) + row * cb.hheads;
  const T* gr = static_cast<const T*>(cb.hgr) + row * cb.hheads;
  const T* al = static_cast<const T*>(cb.hal);
  const T* ar = static_cast<const T*>(cb.har);
  Raw r;
  T* p = reinterpret_cast<T*>(&r);
  const int c0 = (int)col + cb.hcol0;
  int hd = c0 / cb.hfh, next = (hd + 1) * cb.hfh;
  T g1 = gl[hd], g2 = gr[hd];
  if constexpr (V % 2 == 0) {
    // the lane's columns inside one head (fh a multiple of V) and the head
    // vectors Raw-aligned: vector loads of a_l / a_r, paired math (the same
    // per-element IEEE roundings as the scalar path)
    if (c0 + V <= next && ((reinterpret_cast<uintptr_t>(al + c0) |
                            reinterpret_cast<uintptr_t>(ar + c0)) % sizeof(Raw)) == 0) {
      using T2 = typename Num<T>::T2;
      const Raw ra = *reinterpret_cast<const Raw*>(al + c0);
      const Raw rb = *reinterpret_cast<const Raw*>(ar + c0);
      const T2* a2 = reinterpret_cast<const T2*>(&ra);
      const T2* b2 = reinterpret_cast<const T2*>(&rb);
      const T2 g12 = Num<T>::bcast(g1), g22 = Num<T>::bcast(g2);
      T2* p2 = reinterpret_cast<T2*>(&r);
#pragma unroll
      for (int i = 0; i < V / 2; ++i) {
        const T2 hh = Num<T>::pack2(finalize<T>(acc[2 * i], fmode, fo),
                                    finalize<T>(acc[2 * i + 1], fmode, fo));
        p2[i] = Num<T>::add2(hh, Num<T>::add2(Num<T>::mul2(g12, a2[i]), Num<T>::mul2(g22, b2[i])));
      }
      *reinterpret_cast<Raw*>(dst) = r;
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = c0 + i;
    if (c == next) {  // the lane's columns cross into the next head
      ++hd;
      next += cb.hfh;
      g1 = gl[hd];
      g2 = gr[hd];
    }
    const T h = finalize<T>(acc[i], fmode, fo);
    p[i] = Num<T>::add(h, Num<T>::add(Num<T>::mul(g1, al[c]), Num<T>::mul(g2, ar[c])));
  }
  *reinterpret_cast<Raw*>(dst) = r;
}

template <typename T, int V>
__device__ __forceinline__ void store_fin(T* dst, const float (&acc)[V], int fmode, T fo,
                                          const Combine& cb, int64_t row, int64_t col) {
  if (cb.hgl) store_out_hdots<T, V>(dst, acc, fmode, fo, cb, row, col);
  else if (cb.res) store_out_comb<T, V>(dst, acc, fmode, fo,
                                   static_cast<const T*>(cb.res) + row * cb.ldr + col,
                                   cb.ope ? Num<T>::to_d(*static_cast<const T*>(cb.ope)) : 1.0, cb.lam);
  else store_out<T, V>(dst, acc, fmode, fo);
}

template <int V>
__device__ __forceinline__ void load_carry(const float* src, float (&acc)[V]) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int i = 0; i < V; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + i);
      acc[i] = v.x; acc[i + 1] = v.y; acc[i + 2] = v.z; acc[i + 3] = v.w;
    }
  } else if constexpr (V == 2) {
    const float2 v = *reinterpret_cast<const float2*>(src);
    acc[0] = v.x; acc[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = src[i];
  }
}

template <int V>
__device__ __forceinline__ void store_carry(float* dst, const float (&acc)[V]) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int i = 0; i < V; i += 4)
      *reinterpret_cast<float4*>(dst + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(dst) = make_float2(acc[0], acc[1]);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) dst[i] = acc[i];
  }
}

// Load CPL consecutive int32 starting at element index lo (possibly partially
// outside [0, limit)); out-of-range entries become 0.
template <int CPL>
__device__ __forceinline__ void load_idx(const int32_t* __restrict__ base, int64_t lo, int64_t limit,
                                         int (&out)[CPL]) {
  if (lo >= 0 && lo + CPL <= limit) {
    const int32_t* p = base + lo;
    if constexpr (CPL == 1) {
      out[0] = __ldcs(p);
    } else if constexpr (CPL == 2) {
      int2 v = __ldcs(reinterpret_cast<const int2*>(p));
      out[0] = v.x; out[1] = v.y;
    } else {
#pragma unroll
      for (int q = 0; q < CPL; q += 4) {
        int4 v = __ldcs(reinterpret_cast<const int4*>(p + q));
        out[q] = v.x; out[q + 1] = v.y; out[q + 2] = v.z; out[q + 3] = v.w;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      int64_t i = lo + q;
      out[q] = (i >= 0 && i < limit) ? __ldcs(base + i) : 0;
    }
  }
}

// ------------------------------------------------------------- fast kernel

// acc[i] += x[i] (f16 or f32 element), one fp32 rounding.  For binary16 inputs
// sm_100a fuses the widening into the add (FHADD / FHFMA: add.rn.f32.f16,
// fma.rn.f32.f16), halving the ALU work of the gather loop.
template <typename T, int V>
__device__ __forceinline__ void acc_add(float (&acc)[V],
                                        const typename RawVec<V * sizeof(T)>::type& r) {
  if constexpr (sizeof(T) == 2) {
    const unsigned short* h = reinterpret_cast<const unsigned short*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i)
      asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(acc[i]) : "h"(h[i]));
  } else {
    const float* p = reinterpret_cast<const float*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] += p[i];
  }
}

// acc[i] += w * x[i]; w in the element type.
template <typename T, int V>
__device__ __forceinline__ void acc_fma(float (&acc)[V], T w,
                                        const typename RawVec<V * sizeof(T)>::type& r) {
  if constexpr (sizeof(T) == 2) {
    const unsigned short* h = reinterpret_cast<const unsigned short*>(&r);
    const unsigned short wb = __half_as_ushort(w);
#pragma unroll
    for (int i = 0; i < V; ++i)
      asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i]) : "h"(wb), "h"(h[i]));
  } else {
    const float* p = reinterpret_cast<const float*>(&r);
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = fmaf(w, p[i], acc[i]);
  }
}

// Minimum resident blocks per SM: caps registers so that 256-thread blocks of
// single-chunk teams run 3-4 deep (24-32 warps/SM) for memory-level
// parallelism, without spilling (ptxas -v: 64 regs unweighted TEAM >= 8).
#ifndef HG_SPMM_EB32
#define HG_SPMM_EB32 4   // edges per batch of 32-byte-lane unit teams
#endif
#ifndef HG_SPMM_OCC32
#define HG_SPMM_OCC32 3  // 32-byte-lane unweighted teams (A/B builds: tools/exp/variants)
#endif
template <int TEAM, int NCH, bool WT, int VB = 16>
struct FastOcc {
  static constexpr int value =
      NCH == 1 ? ((!WT && VB == 16 && TEAM >= 8 && TEAM <= 16) ? 4
                  : (!WT && VB == 32) ? HG_SPMM_OCC32 : 3)
               : (NCH == 2 ? 2 : 1);
};

// Column ids of one batch for a non-power-of-two team: lane tl holds the ids
// of edges base + tl + q*TEAM (q < CPL, within the batch of EB).
template <int CPL, int TEAM, int EB, bool FULL>
__device__ __forceinline__ void load_batch_ids_strided(const int32_t* __restrict__ base_ptr,
                                                       int base, int tl, int limit,
                                                       int (&out)[CPL]) {
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int j = tl + q * TEAM;
    const int e = base + j;
    out[q] = (j < EB && (FULL || (e >= 0 && e < limit))) ? __ldcs(base_ptr + e) : 0;
  }
}

// Column ids of one batch: lane tl holds ids [base + tl*CPL, +CPL).  FULL
// batches lie inside [0, num_edges) and use unguarded vector loads.
template <int CPL, bool FULL>
__device__ __forceinline__ void load_batch_ids(const int32_t* __restrict__ base_ptr, int lo,
                                               int limit, int (&out)[CPL]) {
  if constexpr (FULL) {
    const int32_t* p = base_ptr + lo;
    if constexpr (CPL == 1) {
      out[0] = __ldcs(p);
    } else if constexpr (CPL == 2) {
      int2 v = __ldcs(reinterpret_cast<const int2*>(p));
      out[0] = v.x; out[1] = v.y;
    } else {
#pragma unroll
      for (int q = 0; q < CPL; q += 4) {
        int4 v = __ldcs(reinterpret_cast<const int4*>(p + q));
        out[q] = v.x; out[q + 1] = v.y; out[q + 2] = v.z; out[q + 3] = v.w;
      }
    }
  } else {
    load_idx<CPL>(base_ptr, lo, limit, out);
  }
}

// Per-team state of k_spmm_fast: lane column offsets, accumulators, unit range.
// Teams of TEAM lanes; TEAM need not be a power of two (e.g. 6 lanes for F=48:
// five teams per warp, 30 of 32 lanes busy).  Power-of-two teams load
// column ids as vectors (lane tl holds edges tl*CPL+q); other teams load
// scalars (lane tl holds edges tl + q*TEAM).
template <int TEAM>
struct TeamShape {
  static constexpr bool P2 = (TEAM & (TEAM - 1)) == 0;
  static constexpr int TPW = 32 / TEAM;  // teams per warp
};

// ATT: the edge weight is the GAT attention coefficient, computed in the
// gather loop from the column's s_r (loaded through the weight path with the
// column id as index) and the row's (s_l, m, 1/sum) -- bit for bit the alpha
// hg_gat_attention_fwd writes -- and stored by one lane per head.
constexpr float kAttLog2e = 1.4426950408889634f;  // = gat_fast.cu kLog2e

template <typename T, int V, int TEAM, int NCH, bool WEIGHTED, bool SUMW = false,
          bool PK = false, bool ATT = false>
struct FastTeam {
  static constexpr bool P2 = TeamShape<TEAM>::P2;
  // edges gathered per batch (packed teams: 4, the rolled accumulate shifts
  // the batch registers once per edge)
  static constexpr int EB = V * sizeof(T) == 32 ? (PK ? 4 : HG_SPMM_EB32) : (NCH >= 4 || PK) ? 4 : 8;
  static constexpr int CPL = P2 ? (TEAM >= EB ? 1 : EB / TEAM) : (EB + TEAM - 1) / TEAM;
  using Raw = typename RawVec<V * sizeof(T)>::type;

  const T* xl[NCH];
  bool cval[NCH];
  int chead[NCH];
  float acc[NCH][V];
  unsigned tmask;
  int tbase;  // lane id of the team's first lane
  int beg, end, ldx, heads;
  const T* w;
  bool use_widx;
  int wld, w2off;   // weight row stride; SUMW: offset of the summed second value block
  float acc2;       // SUMW: this lane's head sum of w[idx(e), w2off + head]

  // Packed unit (an aligned run of short rows walked as one edge stream):
  // each edge's row id comes with its column id; when it changes, the
  // finished row is stored and the accumulators cleared.  Each lane still
  // accumulates a row's edges one by one in edge order, so a packed row rounds
  // exactly like the same row processed as its own unit.  Empty rows of the
  // pack are written before the stream (write_empty_rows).
  int prow;      // row being accumulated (-1 before the first edge)
  T pfo;         // its output factor
  const T* px;
  T* py;
  const T* pfout;
  T* pout2;
  int pldy, pfmode;
  bool plead;
  Combine comb;   // GIN combine / residual add in the row store
  // fp32 partial-output mode (column-blocked aggregation, partition.py):
  // rows start from acc_in[r] and end in acc_out[r] unrounded (NULL: 0 / rnd)
  const float* accin;
  float* accout;
  int accld;

  __device__ __forceinline__ void load_acc(int r) {
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (cval[k]) load_carry<V>(accin + (int64_t)r * accld + (xl[k] - px), acc[k]);
  }

  // ATT state: the row's log2-domain s_l, running max and 1/sum per chunk
  const T* asl;
  const float2* astats;
  T* aout;
  float aslope;
  float aa[NCH], am[NCH], ainv[NCH];
  bool alead[NCH];

  __device__ __forceinline__ void load_att(int r) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      if (cval[k]) {
        const int64_t i = (int64_t)r * heads + chead[k];
        aa[k] = Num<T>::to_f(asl[i]) * kAttLog2e;
        const float2 st = astats[i];
        am[k] = st.x;
        ainv[k] = st.y;
      }
    }
  }

  // alpha of edge e for chunk k from its column's s_r (gat_fast.cu fwd_pass2)
  __device__ __forceinline__ T att_weight(int k, T srv, int e) const {
    float v = fmaf(Num<T>::to_f(srv), kAttLog2e, aa[k]);
    v = v > 0.0f ? v : v * aslope;
    const T a = Num<T>::from_f(ex2_neg(v - am[k]) * ainv[k]);
    if (alead[k]) aout[(int64_t)e * heads + chead[k]] = a;
    return a;
  }

  __device__ __forceinline__ void store_row() {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      if (cval[k]) {
        if (accout) store_carry<V>(accout + (int64_t)prow * accld + (xl[k] - px), acc[k]);
        else store_fin<T, V>(py + (int64_t)prow * pldy + (xl[k] - px), acc[k], pfmode, pfo, comb,
                             prow, xl[k] - px);
      }
#pragma unroll
      for (int i = 0; i < V; ++i) acc[k][i] = 0.0f;
    }
    if (SUMW) {
      if (plead) pout2[(int64_t)prow * heads + chead[0]] = Num<T>::from_f(acc2);
      acc2 = 0.0f;
    }
  }

  // Edge of row r arrives: close the previous row if r starts a new one.
  __device__ __forceinline__ void enter_row(int r) {
    if (r != prow) {
      if (prow >= 0) store_row();
      prow = r;
      pfo = pfout ? pfout[r] : Num<T>::zero();
      if (ATT) load_att(r);
      if (accin) load_acc(r);
    }
  }

  // Fetch the ids of batch [base, base+EB) into this lane's slots.
  template <bool FULL>
  __device__ __forceinline__ void load_ids_impl(const int32_t* __restrict__ p, int base, int tl,
                                                int limit, int (&out)[CPL]) const {
    if constexpr (P2) {
      if (tl * CPL < EB) load_batch_ids<CPL, FULL>(p, base + tl * CPL, limit, out);
    } else {
      load_batch_ids_strided<CPL, TEAM, EB, FULL>(p, base, tl, limit, out);
    }
  }

  __device__ __forceinline__ int shfl_id(const int (&ids)[CPL], int j) const {
    if constexpr (P2) return __shfl_sync(tmask, ids[j % CPL], j / CPL, TEAM);
    else return __shfl_sync(tmask, ids[j / TEAM], tbase + j % TEAM);
  }

  // One batch of EB edges [b, b+EB): issue every gather, then accumulate.
  template <bool FULL, bool PACKED = false>
  __device__ __forceinline__ void batch(int b, const int (&ids)[CPL], const int (&wids)[CPL],
                                        const int (&rids)[CPL]) {
    Raw raw[EB][NCH];
    T wv[EB][NCH];
    T w2v[EB];
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      const bool ok = FULL || (b + j >= beg && b + j < end);
      const int c = shfl_id(ids, j);
      int wi = b + j;
      if (WEIGHTED && use_widx) wi = shfl_id(wids, j);
      if (ATT) wi = c;  // s_r[c, head]
      const size_t roff = (size_t)(unsigned)c * (unsigned)ldx;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if (ok && cval[k]) {
          raw[j][k] = ldg_raw(reinterpret_cast<const Raw*>(xl[k] + roff));
          if (WEIGHTED) wv[j][k] = w[(size_t)(unsigned)wi * wld + chead[k]];
        }
      }
      if (SUMW) w2v[j] = (ok && cval[0]) ? w[(size_t)(unsigned)wi * wld + w2off + chead[0]] : Num<T>::zero();
    }
    if constexpr (PACKED) {
      // Rolled over the batch (one copy of the row-store path, so the kernel
      // stays inside the instruction cache): edge j is always in slot 0 and
      // the batch registers shift down one slot per step.
      int rj[EB];
#pragma unroll
      for (int j = 0; j < EB; ++j) rj[j] = shfl_id(rids, j);
#pragma unroll 1
      for (int j = 0; j < EB; ++j) {
        if (b + j >= beg && b + j < end) {
          enter_row(rj[0]);
          if (SUMW) acc2 += Num<T>::to_f(w2v[0]);
#pragma unroll
          for (int k = 0; k < NCH; ++k) {
            if (cval[k]) {
              if (WEIGHTED) acc_fma<T, V>(acc[k], ATT ? att_weight(k, wv[0][k], b + j) : wv[0][k], raw[0][k]);
              else acc_add<T, V>(acc[k], raw[0][k]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q + 1 < EB; ++q) {
          rj[q] = rj[q + 1];
          if (SUMW) w2v[q] = w2v[q + 1];
#pragma unroll
          for (int k = 0; k < NCH; ++k) {
            raw[q][k] = raw[q + 1][k];
            if (WEIGHTED) wv[q][k] = wv[q + 1][k];
          }
        }
      }
      return;
    }
    if (SUMW) {
#pragma unroll
      for (int j = 0; j < EB; ++j) acc2 += Num<T>::to_f(w2v[j]);
    }
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      const bool ok = FULL || (b + j >= beg && b + j < end);
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if (ok && cval[k]) {
          if (WEIGHTED) acc_fma<T, V>(acc[k], ATT ? att_weight(k, wv[j][k], b + j) : wv[j][k], raw[j][k]);
          else acc_add<T, V>(acc[k], raw[j][k]);
        }
      }
    }
  }
};

// PACKED = false: units {row, begin, end, slot} (slot -1 = whole row, else the
// row's fp32 carry slot).  PACKED = true: packs {first_row, begin, end, rows}
// of consecutive short rows (hg_schedule_build), each row stored as the edge
// stream crosses its end.
template <typename T, int V, int TEAM, int NCH, bool WEIGHTED, bool SUMW = false,
          bool PACKED = false, bool ATT = false>
__global__ void __launch_bounds__(256, (PACKED && NCH == 1 && V * sizeof(T) <= 16)
                                           ? 4
                                           : FastOcc<TEAM, NCH, WEIGHTED, V * sizeof(T)>::value)
k_spmm_fast(const int4* __restrict__ units, int64_t num_units, const int32_t* __restrict__ cols,
            int64_t num_edges, const T* __restrict__ w, const int32_t* __restrict__ widx,
            int heads, int fh, const T* __restrict__ x, T* __restrict__ y,
            float* __restrict__ carry, int F, int ldx, int ldy, int fmode,
            const T* __restrict__ fout, int wld, int w2off, T* __restrict__ out2,
            float* __restrict__ carry2, const int64_t* __restrict__ offsets,
            const int32_t* __restrict__ rowid, const T* __restrict__ att_sl,
            const float2* __restrict__ att_stats, T* __restrict__ att_out, float att_slope,
            const float* __restrict__ acc_in, float* __restrict__ acc_out, int acc_ld,
            int* __restrict__ split_cnt, const int32_t* __restrict__ slot_split,
            const int4* __restrict__ split_info, const Combine comb) {
  using Team = FastTeam<T, V, TEAM, NCH, WEIGHTED, SUMW, PACKED, ATT>;
  constexpr int EB = Team::EB;
  constexpr int CPL = Team::CPL;
  constexpr bool P2 = Team::P2;
  constexpr int TPW = TeamShape<TEAM>::TPW;

  const int lane = threadIdx.x & 31;
  const int tidx = lane / TEAM;
  if (tidx >= TPW) return;  // spare lanes of a non-power-of-two split
  const int tl = lane - tidx * TEAM;
  const int64_t team_id = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TPW + tidx;
  if (team_id >= num_units) return;

  const int4 un = units[team_id];
  const int row = un.x, slot = un.w;
  const int nvec = F / V;
  const int limit = (int)num_edges;
  const bool loader = P2 ? tl * CPL < EB : tl < EB;  // lanes that fetch column ids

  Team t;
  t.tbase = tidx * TEAM;
  t.tmask = TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << t.tbase);
  t.beg = un.y;
  t.end = un.z;
  t.ldx = ldx;
  t.heads = heads;
  t.w = w;
  t.use_widx = WEIGHTED && widx != nullptr;
  t.wld = wld;
  t.w2off = w2off;
  t.acc2 = 0.0f;
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int c = tl + k * TEAM;
    t.cval[k] = c < nvec;
    t.xl[k] = x + c * V;
    t.chead[k] = WEIGHTED ? (c * V) / fh : 0;
#pragma unroll
    for (int i = 0; i < V; ++i) t.acc[k][i] = 0.0f;
  }
  const bool lead = t.cval[0] && (tl * V) % fh == 0;  // SUMW: first lane of its head
  t.accin = acc_in;
  t.accout = acc_out;
  t.accld = acc_ld;
  t.comb = comb;
  t.px = x;
  if constexpr (ATT) {
    t.asl = att_sl;
    t.astats = att_stats;
    t.aout = att_out;
    t.aslope = att_slope;
#pragma unroll
    for (int k = 0; k < NCH; ++k) t.alead[k] = t.cval[k] && ((tl + k * TEAM) * V) % fh == 0;
    if (!PACKED) t.load_att(row);
  }
  if constexpr (PACKED) {
    t.prow = -1;
    t.pfo = Num<T>::zero();
    t.px = x;
    t.py = y;
    t.pfout = fout;
    t.pout2 = out2;
    t.pldy = ldy;
    t.pfmode = fmode;
    t.plead = lead;
    // empty rows of the pack (degrees read lane-parallel): finalize(0) with the
    // row's factor, as their own units would store
    constexpr unsigned kTeamBits = TEAM == 32 ? 0xffffffffu : ((1u << TEAM) - 1u);
    unsigned empty = 0;
#pragma unroll
    for (int q = 0; q < (kPackRows + TEAM - 1) / TEAM; ++q) {
      const int i = q * TEAM + tl;
      const bool e = i < slot && __ldg(offsets + row + i) == __ldg(offsets + row + i + 1);
      empty |= ((__ballot_sync(t.tmask, e) >> t.tbase) & kTeamBits) << (q * TEAM);
    }
    while (empty) {
      const int i = __ffs(empty) - 1;
      empty &= empty - 1;
      t.prow = row + i;
      t.pfo = fout ? fout[row + i] : Num<T>::zero();
      if (acc_in) t.load_acc(row + i);
      t.store_row();
    }
    t.prow = -1;
  }
  const int beg = t.beg, end = t.end;
  // fp32 partial mode: the row's first unit starts from acc_in
  if (!PACKED && acc_in && (slot < 0 || (int64_t)beg == __ldg(offsets + row))) t.load_acc(row);

  // Batches aligned to the absolute address of cols (vector id loads).
  const int mis = (int)((reinterpret_cast<uintptr_t>(cols) >> 2) & (EB - 1));
  int b = beg - ((beg + mis) & (EB - 1));
  if constexpr (PACKED) {  // one (guarded) batch site, ids prefetched one batch ahead
    int ids[CPL] = {}, wids[CPL] = {}, rids[CPL] = {};
    if (b < end && loader) {
      t.template load_ids_impl<false>(cols, b, tl, limit, ids);
      if (t.use_widx) t.template load_ids_impl<false>(widx, b, tl, limit, wids);
      t.template load_ids_impl<false>(rowid, b, tl, limit, rids);
    }
    for (; b < end; b += EB) {
      int nids[CPL] = {}, nwids[CPL] = {}, nrids[CPL] = {};
      if (b + EB < end && loader) {
        t.template load_ids_impl<false>(cols, b + EB, tl, limit, nids);
        if (t.use_widx) t.template load_ids_impl<false>(widx, b + EB, tl, limit, nwids);
        t.template load_ids_impl<false>(rowid, b + EB, tl, limit, nrids);
      }
      t.template batch<false, true>(b, ids, wids, rids);
#pragma unroll
      for (int q = 0; q < CPL; ++q) { ids[q] = nids[q]; wids[q] = nwids[q]; rids[q] = nrids[q]; }
    }
    if (t.prow >= 0) t.store_row();  // the pack's last non-empty row
    return;
  }
  if (b < beg) {  // partial head batch
    int ids[CPL] = {}, wids[CPL] = {}, rids[CPL] = {};
    if (loader) t.template load_ids_impl<false>(cols, b, tl, limit, ids);
    if (t.use_widx && loader) t.template load_ids_impl<false>(widx, b, tl, limit, wids);
    t.template batch<false>(b, ids, wids, rids);
    b += EB;
  }
  if (b + EB <= end) {  // full batches, column ids prefetched one batch ahead
    int ids[CPL] = {}, wids[CPL] = {}, rids[CPL] = {};
    if (loader) t.template load_ids_impl<true>(cols, b, tl, limit, ids);
    if (t.use_widx && loader) t.template load_ids_impl<true>(widx, b, tl, limit, wids);
    for (;;) {
      const int nb = b + EB;
      const bool more = nb + EB <= end;
      int nids[CPL] = {}, nwids[CPL] = {};
      if (more && loader) t.template load_ids_impl<true>(cols, nb, tl, limit, nids);
      if (more && t.use_widx && loader) t.template load_ids_impl<true>(widx, nb, tl, limit, nwids);
      t.template batch<true>(b, ids, wids, rids);
      b = nb;
      if (!more) break;
#pragma unroll
      for (int q = 0; q < CPL; ++q) { ids[q] = nids[q]; wids[q] = nwids[q]; }
    }
  }
  if (b < end) {  // partial tail batch
    int ids[CPL] = {}, wids[CPL] = {}, rids[CPL] = {};
    if (loader) t.template load_ids_impl<false>(cols, b, tl, limit, ids);
    if (t.use_widx && loader) t.template load_ids_impl<false>(widx, b, tl, limit, wids);
    t.template batch<false>(b, ids, wids, rids);
  }

  if (slot < 0 && acc_out) {
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (t.cval[k]) store_carry<V>(acc_out + (int64_t)row * acc_ld + (t.xl[k] - x), t.acc[k]);
  } else if (slot < 0) {
    const T fo = fout ? fout[row] : Num<T>::zero();
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (t.cval[k]) store_fin<T, V>(y + (int64_t)row * ldy + (t.xl[k] - x), t.acc[k], fmode, fo, comb,
                                     row, t.xl[k] - x);
  } else {
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (t.cval[k]) store_carry<V>(carry + (int64_t)slot * F + (t.xl[k] - x), t.acc[k]);
  }
  if (SUMW && lead) {  // first lane of each head
    if (slot < 0) out2[(int64_t)row * heads + t.chead[0]] = Num<T>::from_f(t.acc2);
    else carry2[(int64_t)slot * heads + t.chead[0]] = t.acc2;
  }
  if (slot >= 0 && split_cnt != nullptr) {
    // Fused follow-up: the split row's last unit to finish (a per-row arrival
    // counter) folds the fp32 carries in slot order -- the arithmetic of
    // k_spmm_fast_followup, so bitwise the same -- and re-arms the counter.
    __threadfence();
    __syncwarp(t.tmask);
    int si = 0, last = 0;
    if (tl == 0) {
      si = __ldg(slot_split + slot);
      last = atomicAdd(split_cnt + si, 1) == __ldg(&split_info[si].z) - 1;
    }
    si = __shfl_sync(t.tmask, si, t.tbase);
    last = __shfl_sync(t.tmask, last, t.tbase);
    if (last) {
      __threadfence();
      const int4 sr = split_info[si];
      const T fo = fout ? fout[sr.x] : Num<T>::zero();
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if (!t.cval[k]) continue;
        const int64_t col = t.xl[k] - x;
        float a2[V];
#pragma unroll
        for (int i = 0; i < V; ++i) a2[i] = 0.0f;
        for (int q = 0; q < sr.z; ++q) {
          const float* src = carry + (int64_t)(sr.y + q) * F + col;
          float b2[V];
          if constexpr (V % 4 == 0) {
#pragma unroll
            for (int i = 0; i < V; i += 4) {
              const float4 v = __ldcg(reinterpret_cast<const float4*>(src + i));
              b2[i] = v.x; b2[i + 1] = v.y; b2[i + 2] = v.z; b2[i + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < V; ++i) b2[i] = __ldcg(src + i);
          }
#pragma unroll
          for (int i = 0; i < V; ++i) a2[i] += b2[i];
        }
        if (acc_out) store_carry<V>(acc_out + (int64_t)sr.x * acc_ld + col, a2);
        else store_fin<T, V>(y + (int64_t)sr.x * ldy + col, a2, fmode, fo, comb, sr.x, col);
      }
      if (SUMW) {
        for (int hh = tl; hh < heads; hh += TEAM) {
          float sum = 0.0f;
          for (int q = 0; q < sr.z; ++q) sum += __ldcg(carry2 + (int64_t)(sr.y + q) * heads + hh);
          out2[(int64_t)sr.x * heads + hh] = Num<T>::from_f(sum);
        }
      }
      if (tl == 0) split_cnt[si] = 0;
    }
  }
}

// One team per split row: fp32 carries folded in slot (edge) order.
template <typename T, int V, int TEAM, int NCH>
__global__ void __launch_bounds__(256)
k_spmm_fast_followup(const int4* __restrict__ split_rows, int64_t num_split,
                     const float* __restrict__ carry, T* __restrict__ y, int F, int ldy,
                     int fmode, const T* __restrict__ fout, int heads2,
                     const float* __restrict__ carry2, T* __restrict__ out2,
                     float* __restrict__ acc_out, int acc_ld, const Combine comb) {
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TEAM - 1);
  const int64_t team = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
  if (team >= num_split) return;
  const int4 sr = split_rows[team];
  if (out2) {  // second-value head sums of the split row, folded in slot order
    for (int hh = tl; hh < heads2; hh += TEAM) {
      float s = 0.0f;
      for (int p = 0; p < sr.z; ++p) s += carry2[(int64_t)(sr.y + p) * heads2 + hh];
      out2[(int64_t)sr.x * heads2 + hh] = Num<T>::from_f(s);
    }
  }
  const int nvec = F / V;
  const T fo = fout ? fout[sr.x] : Num<T>::zero();
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int c = tl + k * TEAM;
    if (c >= nvec) continue;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.0f;
    // slots fetched 4 at a time (independent loads in flight), added in slot order
    constexpr int PF = 4;
    for (int p = 0; p < sr.z; p += PF) {
      float buf[PF][V];
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        if (p + q < sr.z) {
          const float* src = carry + (int64_t)(sr.y + p + q) * F + c * V;
#pragma unroll
          for (int i = 0; i < V; ++i) buf[q][i] = src[i];
        }
      }
#pragma unroll
      for (int q = 0; q < PF; ++q)
        if (p + q < sr.z) {
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] += buf[q][i];
        }
    }
    if (acc_out) store_carry<V>(acc_out + (int64_t)sr.x * acc_ld + c * V, acc);
    else store_fin<T, V>(y + (int64_t)sr.x * ldy + c * V, acc, fmode, fo, comb, sr.x, c * V);
  }
}

struct FastArgs {
  const int64_t* offsets;
  const int32_t* cols;
  int64_t n_rows, n_cols, num_edges;
  const int4* units;
  int64_t num_units;
  const int4* split_rows;
  int64_t num_split;
  const int4* packs;
  int64_t num_packs;
  const int32_t* rowid;
  const void* w;
  const int32_t* widx;
  int heads, fh;
  const void* x;
  void* y;
  float* carry;
  int F, ldx, ldy, fmode;
  const void* fout;
  int wld, w2off;
  void* out2;
  float* carry2;
  const void* att_sl;      // ATT (hg_gat_aggregate): s_l, per-row (m, 1/sum), alpha out
  const float2* att_stats;
  void* att_out;
  float att_slope;
  const float* acc_in;     // fp32 partial mode (hg_spmm_acc)
  float* acc_out;
  int acc_ld;
  int* split_cnt;          // fused follow-up (hg_spmm split_counters / slot_split)
  const int32_t* slot_split;
  Combine comb;            // GIN combine / residual add in the store (res NULL: off)
  cudaStream_t st;
};

template <int X> struct Pow2Up { static constexpr int value = X <= 1 ? 1 : 2 * Pow2Up<(X + 1) / 2>::value; };
template <> struct Pow2Up<1> { static constexpr int value = 1; };

template <typename T, int V, int TEAM, int NCH, bool WT, bool SUMW = false, bool ATT = false>
static int launch_fast(const FastArgs& a) {
  constexpr int kThreads = 256;
  constexpr int teams_per_block = (kThreads / 32) * TeamShape<TEAM>::TPW;
  constexpr int TEAMF = Pow2Up<TEAM>::value;  // follow-up pass: power-of-two teams
  if (a.num_units > 0) {
    int64_t blocks = (a.num_units + teams_per_block - 1) / teams_per_block;
    k_spmm_fast<T, V, TEAM, NCH, WT, SUMW, false, ATT><<<(unsigned)blocks, kThreads, 0, a.st>>>(
        a.units, a.num_units, a.cols, a.num_edges, (const T*)a.w, a.widx, a.heads, a.fh,
        (const T*)a.x, (T*)a.y, a.carry, a.F, a.ldx, a.ldy, a.fmode, (const T*)a.fout,
        a.wld, a.w2off, (T*)a.out2, a.carry2, a.offsets, nullptr, (const T*)a.att_sl,
        a.att_stats, (T*)a.att_out, a.att_slope, a.acc_in, a.acc_out, a.acc_ld, a.split_cnt,
        a.slot_split, a.split_rows, a.comb);
    HG_LAUNCHED();
  }
  if (a.num_packs > 0) {
    int64_t blocks = (a.num_packs + teams_per_block - 1) / teams_per_block;
    k_spmm_fast<T, V, TEAM, NCH, WT, SUMW, true, ATT><<<(unsigned)blocks, kThreads, 0, a.st>>>(
        a.packs, a.num_packs, a.cols, a.num_edges, (const T*)a.w, a.widx, a.heads, a.fh,
        (const T*)a.x, (T*)a.y, nullptr, a.F, a.ldx, a.ldy, a.fmode, (const T*)a.fout,
        a.wld, a.w2off, (T*)a.out2, nullptr, a.offsets, a.rowid, (const T*)a.att_sl,
        a.att_stats, (T*)a.att_out, a.att_slope, a.acc_in, a.acc_out, a.acc_ld, nullptr,
        nullptr, nullptr, a.comb);
    HG_LAUNCHED();
  }
  if (a.num_split > 0 && a.split_cnt == nullptr) {
    int64_t blocks = (a.num_split + kThreads / TEAMF - 1) / (kThreads / TEAMF);
    k_spmm_fast_followup<T, V, TEAMF, NCH><<<(unsigned)blocks, kThreads, 0, a.st>>>(
        a.split_rows, a.num_split, a.carry, (T*)a.y, a.F, a.ldy, a.fmode, (const T*)a.fout,
        SUMW ? a.heads : 0, a.carry2, SUMW ? (T*)a.out2 : nullptr, a.acc_out, a.acc_ld, a.comb);
    HG_LAUNCHED();
  }
  return HG_OK;
}

// Weighted aggregation that also sums a second per-edge value block (w2off)
// per head: one team size per power-of-two chunk count, single chunk per lane.
// 32-byte lanes for binary16 rows of 48..512 elements, multiples of 16 (C3
// sweep: F=64 1.11 -> 1.07 ms, 128: 2.12 -> 2.03, 256: 4.57 -> 4.27, 512: 9.18 ->
// 8.60; F=16/32 got slower with 1-2 lane teams).  A/B switch for measurement:
// HG_SPMM_LANE32=0 in the environment of the first call.
static const bool kLane32 = [] {
  const char* e = getenv("HG_SPMM_LANE32");
  return !(e && e[0] == '0');
}();

template <typename T, int V>
static int dispatch_sumw(const FastArgs& a) {
  const int nvec = a.F / V;
  HG_REQUIRE(nvec <= 32 && a.fh % V == 0, "hg_spmm: summed weights need F/V <= 32 and heads of whole vectors");
  if (nvec <= 1) return launch_fast<T, V, 1, 1, true, true>(a);
  if (nvec <= 2) return launch_fast<T, V, 2, 1, true, true>(a);
  if (nvec <= 4) return launch_fast<T, V, 4, 1, true, true>(a);
  if (nvec <= 8) return launch_fast<T, V, 8, 1, true, true>(a);
  if (nvec <= 16) return launch_fast<T, V, 16, 1, true, true>(a);
  return launch_fast<T, V, 32, 1, true, true>(a);
}

template <typename T, int V, bool WT, bool ATT = false>
static int dispatch_layout(const FastArgs& a) {
  const int nvec = a.F / V;
  // Teams stay power-of-two lane groups even when some lanes idle (F=48: 6 of
  // 8): a 16-byte-per-lane warp load is served in quarter-warp (8-lane)
  // wavefronts, and a team straddling two quarters doubles the L1 data-pipe
  // wavefronts (ncu, profiles/r01: 7-lane teams ran 27% slower than 8-lane
  // teams at the same L2 sector count).
  if (nvec <= 1) return launch_fast<T, V, 1, 1, WT, false, ATT>(a);
  if (nvec <= 2) return launch_fast<T, V, 2, 1, WT, false, ATT>(a);
  if (nvec <= 4) return launch_fast<T, V, 4, 1, WT, false, ATT>(a);
  if (nvec <= 8) return launch_fast<T, V, 8, 1, WT, false, ATT>(a);
  if (nvec <= 16) return launch_fast<T, V, 16, 1, WT, false, ATT>(a);
  if (nvec <= 32) return launch_fast<T, V, 32, 1, WT, false, ATT>(a);
  if (nvec <= 64) return launch_fast<T, V, 32, 2, WT, false, ATT>(a);
  if (nvec <= 128) return launch_fast<T, V, 32, 4, WT, false, ATT>(a);
  if (nvec <= 256) return launch_fast<T, V, 32, 8, WT, false, ATT>(a);
  HG_REQUIRE(false, "hg_spmm: feature length %d too large", a.F);
}

// 32-byte lanes (binary16 x 16), single chunk per lane: F <= 512.
template <typename T, bool WT, bool ATT = false>
static int dispatch_layout32(const FastArgs& a) {
  const int nvec = a.F / 16;
  if (nvec <= 1) return launch_fast<T, 16, 1, 1, WT, false, ATT>(a);
  if (nvec <= 2) return launch_fast<T, 16, 2, 1, WT, false, ATT>(a);
  if (nvec <= 4) return launch_fast<T, 16, 4, 1, WT, false, ATT>(a);
  if (nvec <= 8) return launch_fast<T, 16, 8, 1, WT, false, ATT>(a);
  if (nvec <= 16) return launch_fast<T, 16, 16, 1, WT, false, ATT>(a);
  return launch_fast<T, 16, 32, 1, WT, false, ATT>(a);
}

template <typename T>
static int dispatch_fast(const FastArgs& a) {
  constexpr int VB = 16 / sizeof(T);
  const bool aligned = (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(a.y) % 16 == 0);
  const bool big = aligned && (a.fh % VB == 0) && a.ldx % VB == 0 && a.ldy % VB == 0;
  const bool att = a.att_stats != nullptr;
  if constexpr (sizeof(T) == 2) {
    const bool a32 = (reinterpret_cast<uintptr_t>(a.x) % 32 == 0) &&
                     (reinterpret_cast<uintptr_t>(a.y) % 32 == 0) && a.fh % 16 == 0 &&
                     a.ldx % 16 == 0 && a.ldy % 16 == 0 && a.F >= 48 && a.F <= 512;
    if (a32 && kLane32) {
      if (att) return dispatch_layout32<T, true, true>(a);
      if (a.out2) return dispatch_sumw<T, 16>(a);
      return a.w ? dispatch_layout32<T, true>(a) : dispatch_layout32<T, false>(a);
    }
  }
  if (att) return big ? dispatch_layout<T, VB, true, true>(a) : dispatch_layout<T, 2, true, true>(a);
  if (a.out2) return big ? dispatch_sumw<T, VB>(a) : dispatch_sumw<T, 2>(a);
  if (a.w) return big ? dispatch_layout<T, VB, true>(a) : dispatch_layout<T, 2, true>(a);
  return big ? dispatch_layout<T, VB, false>(a) : dispatch_layout<T, 2, false>(a);
}

static size_t elem_size(int dtype) { return dtype == HG_F16 ? 2 : 4; }

// Half the device's L2 (per-device attribute cache), the working-set budget of
// one aggregation pass's gathered feature slab.
static size_t l2_budget() {
  static size_t cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return (size_t)48 << 20;
  if (!cache[dev]) {
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    cache[dev] = l2 > 0 ? (size_t)l2 / 2 : (size_t)48 << 20;
  }
  return cache[dev];
}

// Slab width (columns) for hg_spmm: F itself unless X exceeds the L2 budget and
// a multiple of 32 columns >= 32 fits it.
static int slab_width(int64_t n_cols, int F, size_t es, bool sliceable) {
  if (!sliceable || n_cols <= 0) return F;
  const size_t budget = l2_budget();
  if ((size_t)F * n_cols * es <= budget) return F;
  const int64_t cand = (int64_t)(budget / ((size_t)n_cols * es)) / 32 * 32;
  return (cand >= 32 && cand < F) ? (int)cand : F;
}

// X' = rnd(X * s[:, None]): the vectorised row-scale pass of dense.cu.
static int scale_rows(const void* x, const void* s, int64_t rows, int F, void* out, int dtype,
                      cudaStream_t st) {
  return hg_bias_scale_rows(x, nullptr, s, rows, F, out, dtype, st);
}

}  // namespace hg

using namespace hg;

extern "C" int hg_spmm_workspace(int64_t n_cols, int32_t F, int64_t num_slots, int has_in_scale,
                                 int32_t sum_heads, int dtype, size_t* bytes) {
  HG_REQUIRE(bytes && F > 0 && n_cols >= 0 && num_slots >= 0 && sum_heads >= 0,
             "hg_spmm_workspace: bad arguments");
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  Carver cv(nullptr, 0);
  cv.take<float>((size_t)num_slots * F);
  if (has_in_scale) cv.take<char>((size_t)n_cols * F * elem_size(dtype));
  if (sum_heads) cv.take<float>((size_t)num_slots * sum_heads);
  *bytes = cv.used;
  return HG_OK;
}

static int spmm_impl(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                     int64_t n_cols, int64_t num_edges, const int32_t* units, int64_t num_units,
                     const int32_t* split_rows, int64_t num_split_rows, int64_t num_slots,
                     const int32_t* packs, int64_t num_packs, const int32_t* pack_rowid,
                     const void* w, const int32_t* w_index, int32_t heads, const void* x,
                     void* y, int32_t F, int64_t ldx, int64_t ldy, int32_t scaling,
                     int32_t relu, const void* in_scale, const void* out_factor,
                     int64_t w_ld, int32_t w2_off, void* out2, int dtype, void* ws,
                     size_t ws_bytes, void* stream, const float* acc_in, float* acc_out,
                     int32_t* split_counters = nullptr, const int32_t* slot_split = nullptr,
                     Combine comb = Combine{}) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(F > 0 && F % 2 == 0, "feature length %d must be even and positive", F);
  HG_REQUIRE(heads >= 1 && F % heads == 0 && (F / heads) % 2 == 0,
             "feature length %d does not split into %d even heads", F, heads);
  HG_REQUIRE(scaling >= HG_SCALING_POST && scaling <= HG_SCALING_DISCRETIZED,
             "unknown scaling %d", scaling);
  HG_REQUIRE(n_rows >= 0 && n_cols >= 0 && num_edges >= 0, "hg_spmm: bad sizes");
  HG_REQUIRE(num_edges <= (int64_t)INT32_MAX, "hg_spmm: edge count exceeds int32 units");
  if (ldx == 0) ldx = F;
  if (ldy == 0) ldy = F;
  HG_REQUIRE(ldx >= F && ldy >= F && ldx <= INT32_MAX && ldy <= INT32_MAX,
             "hg_spmm: row strides (%lld, %lld) must be >= F=%d", (long long)ldx, (long long)ldy, F);
  HG_REQUIRE(!in_scale || ldx == F, "hg_spmm: in_scale needs a dense x (ldx == F)");
  if (w_ld == 0) w_ld = heads;
  HG_REQUIRE(!w || (w_ld >= heads && w_ld <= INT32_MAX), "hg_spmm: weight row stride %lld < heads %d",
             (long long)w_ld, heads);
  HG_REQUIRE(!out2 || (w && w2_off >= heads && w2_off + heads <= w_ld),
             "hg_spmm: summed second weight block needs w and heads <= w2_off <= w_ld - heads");
  // id batches are aligned to the address of cols and loaded as vectors from
  // cols, w_index and pack_rowid alike: the three must share their 16-byte phase
  HG_REQUIRE(reinterpret_cast<uintptr_t>(cols) % 4 == 0 &&
                 (!w_index || ((reinterpret_cast<uintptr_t>(cols) ^
                                reinterpret_cast<uintptr_t>(w_index)) & 15) == 0) &&
                 (!pack_rowid || ((reinterpret_cast<uintptr_t>(cols) ^
                                   reinterpret_cast<uintptr_t>(pack_rowid)) & 15) == 0),
             "hg_spmm: cols, w_index and pack_rowid must have the same address modulo 16");
  cudaStream_t st = as_stream(stream);
  if (n_rows == 0) return HG_OK;
  Carver cv(ws, ws_bytes);
  float* carry = cv.take<float>((size_t)num_slots * F);
  void* xs = in_scale ? cv.take<char>((size_t)n_cols * F * elem_size(dtype)) : nullptr;
  float* carry2 = out2 ? cv.take<float>((size_t)num_slots * heads) : nullptr;
  HG_REQUIRE(cv.fits(), "hg_spmm: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  HG_REQUIRE(num_slots == 0 || carry != nullptr, "hg_spmm: carry workspace missing");
  if (in_scale) {
    int rc = scale_rows(x, in_scale, n_cols, F, xs, dtype, st);
    if (rc) return rc;
    x = xs;
  }
  FastArgs a{};
  a.offsets = offsets; a.cols = cols; a.n_rows = n_rows; a.n_cols = n_cols;
  a.num_edges = num_edges;
  a.units = reinterpret_cast<const int4*>(units); a.num_units = num_units;
  a.split_rows = reinterpret_cast<const int4*>(split_rows); a.num_split = num_split_rows;
  a.packs = reinterpret_cast<const int4*>(packs); a.num_packs = packs ? num_packs : 0;
  a.rowid = pack_rowid;
  HG_REQUIRE(a.num_packs == 0 || num_edges == 0 || pack_rowid, "hg_spmm: packs need pack_rowid");
  a.w = w; a.widx = w_index; a.heads = heads; a.fh = F / heads;
  a.x = x; a.y = y; a.carry = carry; a.F = F; a.ldx = (int)ldx; a.ldy = (int)ldy;
  a.fmode = (out_factor == nullptr ? 0 : (scaling == HG_SCALING_POST ? 1 : 2)) | (relu ? 4 : 0);
  a.fout = out_factor; a.st = st;
  a.wld = (int)w_ld; a.w2off = w2_off; a.out2 = out2; a.carry2 = carry2;
  a.acc_in = acc_in; a.acc_out = acc_out; a.acc_ld = F;
  HG_REQUIRE(!comb.res || (!acc_out && !(relu) && comb.ldr >= F &&
                           ((reinterpret_cast<uintptr_t>(comb.res) | (uintptr_t)(comb.ldr * elem_size(dtype))) & 15) == 0),
             "hg_spmm: combine needs a 16-byte aligned residual with rows >= F, no ReLU, no fp32 output");
  a.comb = comb;
  if (split_counters && slot_split && num_split_rows > 0) {
    a.split_cnt = split_counters;
    a.slot_split = slot_split;
  }
  // Column slabs: when X (n_cols x F) overflows the L2 budget but a slab of
  // >= 32 columns fits, aggregate slab by slab so the random row gathers of
  // each pass hit L2 (the column stream is re-read once per slab, sequentially).
  const int W = out2 ? F : slab_width(n_cols, F, elem_size(dtype), w == nullptr || heads == 1);
  for (int j = 0; j < F; j += W) {
    FastArgs s = a;
    s.F = F - j < W ? F - j : W;
    if (heads == 1) s.fh = s.F;
    s.x = static_cast<const char*>(x) + (size_t)j * elem_size(dtype);
    s.y = static_cast<char*>(y) + (size_t)j * elem_size(dtype);
    if (acc_in) s.acc_in = acc_in + j;
    if (acc_out) s.acc_out = acc_out + j;
    if (comb.res) s.comb.res = static_cast<const char*>(comb.res) + (size_t)j * elem_size(dtype);
    s.comb.hcol0 = j;
    const int rc = dtype == HG_F16 ? dispatch_fast<__half>(s) : dispatch_fast<float>(s);
    if (rc) return rc;
  }
  return HG_OK;
}

extern "C" int hg_spmm(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                       int64_t n_cols, int64_t num_edges, const int32_t* units, int64_t num_units,
                       const int32_t* split_rows, int64_t num_split_rows, int64_t num_slots,
                       const int32_t* packs, int64_t num_packs, const int32_t* pack_rowid,
                       const void* w, const int32_t* w_index, int32_t heads, const void* x,
                       void* y, int32_t F, int64_t ldx, int64_t ldy, int32_t scaling,
                       int32_t relu, const void* in_scale, const void* out_factor,
                       int64_t w_ld, int32_t w2_off, void* out2, int dtype, void* ws,
                       size_t ws_bytes, void* stream, int32_t* split_counters,
                       const int32_t* slot_split, const void* comb_res, int64_t comb_ldr,
                       const void* comb_ope, double comb_lam, const void* hd_gl,
                       const void* hd_gr, const void* hd_al, const void* hd_ar) {
  HG_REQUIRE(!hd_gl || (hd_gr && hd_al && hd_ar && !comb_res && heads >= 1 && F % heads == 0 &&
                        !out2 && !relu),
             "hg_spmm: the head-dot store needs g_l, g_r, a_l, a_r, F = heads x fh, no residual "
             "combine, second output or ReLU");
  return spmm_impl(offsets, cols, n_rows, n_cols, num_edges, units, num_units, split_rows,
                   num_split_rows, num_slots, packs, num_packs, pack_rowid, w, w_index, heads, x, y,
                   F, ldx, ldy, scaling, relu, in_scale, out_factor, w_ld, w2_off, out2, dtype, ws,
                   ws_bytes, stream, nullptr, nullptr, split_counters, slot_split,
                   Combine{comb_res, comb_ldr, comb_ope, comb_lam, hd_gl, hd_gr, hd_al, hd_ar,
                           heads, hd_gl ? F / heads : 1, 0});
}

extern "C" int hg_spmm_acc(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                           int64_t n_cols, int64_t num_edges, const int32_t* units,
                           int64_t num_units, const int32_t* split_rows, int64_t num_split_rows,
                           int64_t num_slots, const int32_t* packs, int64_t num_packs,
                           const int32_t* pack_rowid, const void* w, const int32_t* w_index,
                           int32_t heads, int64_t w_ld, const void* x, void* y, int32_t F,
                           int64_t ldx, int64_t ldy, int32_t scaling, int32_t relu,
                           const void* out_factor, const float* acc_in, float* acc_out, int dtype,
                           void* ws, size_t ws_bytes, void* stream) {
  HG_REQUIRE(F % 4 == 0, "hg_spmm_acc: F=%d must be a multiple of 4 (fp32 row vectors)", F);
  HG_REQUIRE(((reinterpret_cast<uintptr_t>(acc_in) | reinterpret_cast<uintptr_t>(acc_out)) & 15) == 0,
             "hg_spmm_acc: accumulators must be 16-byte aligned");
  HG_REQUIRE(acc_out || y, "hg_spmm_acc: no output");
  return spmm_impl(offsets, cols, n_rows, n_cols, num_edges, units, num_units, split_rows,
                   num_split_rows, num_slots, packs, num_packs, pack_rowid, w, w_index, heads, x,
                   acc_out ? nullptr : y, F, ldx, ldy, scaling, relu, nullptr, out_factor, w_ld, 0,
                   nullptr, dtype, ws, ws_bytes, stream, acc_in, acc_out);
}

// Fused GAT layer core, forward (fast numerics): the weighted aggregation of
// hg_spmm with each edge's attention coefficient computed in the gather loop
// from s_l, s_r and the per-row softmax statistics of hg_gat_attention_stats,
// and written to alpha_out (needed by the backward) by one lane per head.
extern "C" int hg_gat_aggregate(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                                int64_t n_cols, int64_t num_edges, const int32_t* units,
                                int64_t num_units, const int32_t* split_rows,
                                int64_t num_split_rows, int64_t num_slots, const int32_t* packs,
                                int64_t num_packs, const int32_t* pack_rowid, const void* s_l,
                                const void* s_r, const float* stats, float slope,
                                void* alpha_out, int32_t heads, const void* x, void* y, int32_t F,
                                int64_t ldx, int64_t ldy, int32_t relu, int dtype, void* ws,
                                size_t ws_bytes, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "hg_gat_aggregate: unknown dtype %d", dtype);
  HG_REQUIRE(heads >= 1 && F >= 2 && F % heads == 0 && (F / heads) % 2 == 0,
             "hg_gat_aggregate: F=%d must split into %d heads of even width", F, heads);
  HG_REQUIRE(n_rows >= 0 && n_cols >= 0 && num_edges >= 0 && num_edges <= (int64_t)INT32_MAX,
             "hg_gat_aggregate: bad sizes");
  if (ldx == 0) ldx = F;
  if (ldy == 0) ldy = F;
  HG_REQUIRE(ldx >= F && ldy >= F && ldx <= INT32_MAX && ldy <= INT32_MAX,
             "hg_gat_aggregate: row strides must be >= F");
  HG_REQUIRE(reinterpret_cast<uintptr_t>(cols) % 4 == 0 &&
                 (!pack_rowid || ((reinterpret_cast<uintptr_t>(cols) ^
                                   reinterpret_cast<uintptr_t>(pack_rowid)) & 15) == 0),
             "hg_gat_aggregate: cols and pack_rowid must have the same address modulo 16");
  if (n_rows == 0) return HG_OK;
  HG_REQUIRE(s_l && s_r && stats && alpha_out && x && y, "hg_gat_aggregate: null operand");
  Carver cv(ws, ws_bytes);
  float* carry = cv.take<float>((size_t)num_slots * F);
  HG_REQUIRE(cv.fits(), "hg_gat_aggregate: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  FastArgs a{};
  a.offsets = offsets; a.cols = cols; a.n_rows = n_rows; a.n_cols = n_cols;
  a.num_edges = num_edges;
  a.units = reinterpret_cast<const int4*>(units); a.num_units = num_units;
  a.split_rows = reinterpret_cast<const int4*>(split_rows); a.num_split = num_split_rows;
  a.packs = reinterpret_cast<const int4*>(packs); a.num_packs = packs ? num_packs : 0;
  a.rowid = pack_rowid;
  HG_REQUIRE(a.num_packs == 0 || num_edges == 0 || pack_rowid, "hg_gat_aggregate: packs need pack_rowid");
  a.w = s_r; a.widx = nullptr; a.heads = heads; a.fh = F / heads; a.wld = heads;
  a.x = x; a.y = y; a.carry = carry; a.F = F; a.ldx = (int)ldx; a.ldy = (int)ldy;
  a.fmode = relu ? 4 : 0;
  a.att_sl = s_l; a.att_stats = reinterpret_cast<const float2*>(stats); a.att_out = alpha_out;
  a.att_slope = slope;
  a.st = as_stream(stream);
  return dtype == HG_F16 ? dispatch_fast<__half>(a) : dispatch_fast<float>(a);
}

// ------------------------------------------------------ reference edge order

namespace hg {

// shared-memory header of k_spmm_edge_ref: brow int64[2W], nseg int[W], ent int[2W]
__host__ __device__ inline size_t edge_ref_hdr(int W) { return ((size_t)28 * W + 15) / 16 * 16; }

template <typename T, bool WEIGHTED>
__global__ void k_spmm_edge_ref(const int64_t* __restrict__ offsets,
                                const int32_t* __restrict__ cols, int64_t n_rows,
                                int64_t num_edges, int C, int W, const T* __restrict__ w,
                                const T* __restrict__ x, T* __restrict__ y, int F, int scaling,
                                const T* __restrict__ fout, int kb, T* __restrict__ carry_vals,
                                int64_t* __restrict__ carry_rows) {
  using N = Num<T>;
  using T2 = typename N::T2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = F / 2;
  int64_t* brow = reinterpret_cast<int64_t*>(smem_raw);   // [W][2]
  int* nseg = reinterpret_cast<int*>(brow + 2 * W);       // [W]
  int* ent = nseg + W;                                    // [2W] entry -> (warp*2+slot)
  T2* bval = reinterpret_cast<T2*>(smem_raw + edge_ref_hdr(W));  // [W][2][P]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cta = blockIdx.x;
  const int64_t cta_e0 = cta * (int64_t)W * C;
  const int64_t e0 = (cta * W + warp) * (int64_t)C;
  const int64_t e1 = e0 + C < num_edges ? e0 + C : num_edges;
  const bool post = scaling == HG_SCALING_POST;
  const bool pre = scaling == HG_SCALING_PRE;
  const bool disc = scaling == HG_SCALING_DISCRETIZED;
  const T2* x2 = reinterpret_cast<const T2*>(x);
  T2* y2 = reinterpret_cast<T2*>(y);
  const T one = N::from_f(1.0f);

  int ns = 0;
  if (e0 < num_edges) {
    int64_t r = row_of_edge(offsets, n_rows, e0);
    int64_t e = e0;
    while (e < e1) {
      while (offsets[r + 1] <= e) ++r;
      const int64_t s = e;
      const int64_t t = offsets[r + 1] < e1 ? offsets[r + 1] : e1;
      const bool is_first = ns == 0;
      const bool is_last = t == e1;
      const T fo = fout ? fout[r] : N::zero();
      const T2 fo2 = N::bcast(fo);
      for (int p = lane; p < P; p += 32) {
        T2 acc = N::zero2();
        if (disc) {
          T2 raw = N::zero2();
          int cnt = 0;
          for (int64_t q = s; q < t; ++q) {
            const T2 xv = x2[(int64_t)cols[q] * P + p];
            raw = WEIGHTED ? N::fma2(N::bcast(w[q]), xv, raw) : N::add2(xv, raw);
            if (++cnt == kb || q + 1 == t) {
              acc = fout ? N::fma2(raw, fo2, acc) : N::add2(raw, acc);
              raw = N::zero2();
              cnt = 0;
            }
          }
        } else {
          for (int64_t q = s; q < t; ++q) {
            const T2 xv = x2[(int64_t)cols[q] * P + p];
            if (pre && fout) {
              const T m = WEIGHTED ? N::mul(w[q], fo) : fo;
              acc = N::fma2(N::bcast(m), xv, acc);
            } else if (WEIGHTED) {
              acc = N::fma2(N::bcast(w[q]), xv, acc);
            } else {
              acc = N::fma2(N::bcast(one), xv, acc);
            }
          }
        }
        if (is_first) {
          bval[(warp * 2 + 0) * P + p] = acc;
        } else if (is_last) {
          bval[(warp * 2 + 1) * P + p] = acc;
        } else {  // interior segment: a complete row that began in this warp
          y2[r * P + p] = (post && fout && N::gt0(fo)) ? N::mul2(acc, fo2) : acc;
        }
      }
      if (lane == 0) {
        if (is_first) brow[warp * 2] = r;
        else if (is_last) brow[warp * 2 + 1] = r;
      }
      ++ns;
      e = t;
    }
  }
  if (lane == 0) nseg[warp] = ns;
  __syncthreads();
  if (warp != 0) return;

  // Boundary segments of the CTA in edge order; chains = runs of equal rows.
  int total = 0;
  for (int v = 0; v < W; ++v) {
    const int k = nseg[v];
    if (k >= 1) { if (lane == 0) ent[total] = v * 2; ++total; }
    if (k >= 2) { if (lane == 0) ent[total] = v * 2 + 1; ++total; }
  }
  __syncwarp();
  int i = 0;
  while (i < total) {
    const int64_t r = brow[ent[i]];
    int j = i + 1;
    while (j < total && brow[ent[j]] == r) ++j;
    const int cnt = j - i;
    const bool carry = j == total;
    const T fo = fout ? fout[r] : N::zero();
    const bool scale_now = !carry && post && fout && N::gt0(fo) && offsets[r] >= cta_e0;
    for (int p = lane; p < P; p += 32) {
      for (int stride = 1; stride < cnt; stride <<= 1)
        for (int q = 0; q + stride < cnt; q += 2 * stride)
          bval[ent[i + q] * P + p] = N::add2(bval[ent[i + q] * P + p], bval[ent[i + q + stride] * P + p]);
      const T2 v = bval[ent[i] * P + p];
      if (carry) reinterpret_cast<T2*>(carry_vals)[cta * P + p] = v;
      else y2[r * P + p] = scale_now ? N::mul2(v, N::bcast(fo)) : v;
    }
    if (carry && lane == 0) carry_rows[cta] = r;
    i = j;
  }
}

// Fold each CTA's carry into its row in ascending CTA order, then post-scale.
template <typename T>
__global__ void k_spmm_edge_ref_followup(const typename Num<T>::T2* __restrict__ carry_vals,
                                         const int64_t* __restrict__ carry_rows, int64_t num_ctas,
                                         T* __restrict__ y, int F, int scaling,
                                         const T* __restrict__ fout) {
  using N = Num<T>;
  using T2 = typename N::T2;
  const int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= num_ctas) return;
  const int64_t r = carry_rows[c];
  if (c > 0 && carry_rows[c - 1] == r) return;  // not the leader of this row's run
  const int P = F / 2;
  T2* y2 = reinterpret_cast<T2*>(y);
  const T fo = fout ? fout[r] : N::zero();
  const bool scale = scaling == HG_SCALING_POST && fout && N::gt0(fo);
  for (int p = lane; p < P; p += 32) {
    T2 v = y2[r * P + p];
    for (int64_t j = c; j < num_ctas && carry_rows[j] == r; ++j) v = N::add2(v, carry_vals[j * P + p]);
    y2[r * P + p] = scale ? N::mul2(v, N::bcast(fo)) : v;
  }
}

}  // namespace hg

static size_t edge_ref_smem(int W, int F, int dtype) {
  return hg::edge_ref_hdr(W) + (size_t)W * 2 * F * hg::elem_size(dtype);
}

extern "C" int hg_spmm_edge_ref_workspace(int64_t n_cols, int64_t num_edges, int32_t F,
                                          int32_t warp_chunk, int32_t warps_per_cta,
                                          int has_in_scale, int dtype, size_t* bytes) {
  HG_REQUIRE(bytes && F > 0 && warp_chunk > 0 && warps_per_cta > 0,
             "hg_spmm_edge_ref_workspace: bad arguments");
  int64_t nw = (num_edges + warp_chunk - 1) / warp_chunk;
  int64_t nc = (nw + warps_per_cta - 1) / warps_per_cta;
  Carver cv(nullptr, 0);
  cv.take<char>((size_t)nc * F * elem_size(dtype));
  cv.take<int64_t>(nc);
  if (has_in_scale) cv.take<char>((size_t)n_cols * F * elem_size(dtype));
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_spmm_edge_ref(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                                int64_t n_cols, int64_t num_edges, int32_t C, int32_t W,
                                const void* w, const void* x, void* y, int32_t F,
                                int32_t scaling, const void* in_scale, const void* out_factor,
                                void* staging_partials, int64_t* staging_rows, int dtype,
                                void* ws, size_t ws_bytes, void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(F > 0 && F % 2 == 0, "feature length %d must be even and positive", F);
  HG_REQUIRE(C >= 64 && C % 2 == 0, "warp_chunk must be >= 64 and even, got %d", C);
  HG_REQUIRE(W >= 1 && W <= 32, "warps_per_cta must be in [1, 32], got %d", W);
  HG_REQUIRE(scaling >= HG_SCALING_POST && scaling <= HG_SCALING_DISCRETIZED,
             "unknown scaling %d", scaling);
  cudaStream_t st = as_stream(stream);
  const size_t es = elem_size(dtype);
  if (n_rows > 0) HG_CUDA(cudaMemsetAsync(y, 0, (size_t)n_rows * F * es, st));
  if (num_edges == 0 || n_rows == 0) return HG_OK;
  const int64_t nw = (num_edges + C - 1) / C;
  const int64_t nc = (nw + W - 1) / W;
  Carver cv(ws, ws_bytes);
  void* cvals = cv.take<char>((size_t)nc * F * es);
  int64_t* crows = cv.take<int64_t>(nc);
  void* xs = in_scale ? cv.take<char>((size_t)n_cols * F * es) : nullptr;
  HG_REQUIRE(cv.fits(), "hg_spmm_edge_ref: workspace too small");
  if (staging_partials) cvals = staging_partials;
  if (staging_rows) crows = staging_rows;
  if (in_scale) {
    int rc = scale_rows(x, in_scale, n_cols, F, xs, dtype, st);
    if (rc) return rc;
    x = xs;
  }
  // discretization batch k = simt.subwarp_layout(F).subwarps (simt.py:86-98)
  const int kb = F > 64 ? 1 : 32 / (F / 2);
  const size_t smem = edge_ref_smem(W, F, dtype);
  HG_REQUIRE(smem <= 227 * 1024, "hg_spmm_edge_ref: F=%d too large for %d warps per CTA", F, W);
  const dim3 grid((unsigned)nc), block(32 * W);
  if (dtype == HG_F16) {
    auto kfn = w ? k_spmm_edge_ref<__half, true> : k_spmm_edge_ref<__half, false>;
    HG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kfn<<<grid, block, smem, st>>>(offsets, cols, n_rows, num_edges, C, W, (const __half*)w,
                                   (const __half*)x, (__half*)y, F, scaling,
                                   (const __half*)out_factor, kb, (__half*)cvals, crows);
    HG_LAUNCHED();
    k_spmm_edge_ref_followup<__half><<<grid_for(nc, 8), 256, 0, st>>>(
        (const __half2*)cvals, crows, nc, (__half*)y, F, scaling, (const __half*)out_factor);
  } else {
    auto kfn = w ? k_spmm_edge_ref<float, true> : k_spmm_edge_ref<float, false>;
    HG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kfn<<<grid, block, smem, st>>>(offsets, cols, n_rows, num_edges, C, W, (const float*)w,
                                   (const float*)x, (float*)y, F, scaling,
                                   (const float*)out_factor, kb, (float*)cvals, crows);
    HG_LAUNCHED();
    k_spmm_edge_ref_followup<float><<<grid_for(nc, 8), 256, 0, st>>>(
        (const float2*)cvals, crows, nc, (float*)y, F, scaling, (const float*)out_factor);
  }
  HG_LAUNCHED();
  return HG_OK;
}

// -------------------------------------------------- reference vertex groups

namespace hg {

template <typename T>
__global__ void k_spmm_vertex_ref(const int64_t* __restrict__ offsets,
                                  const int32_t* __restrict__ cols, int64_t n_rows,
                                  const T* __restrict__ x, T* __restrict__ y, int F, int scaling,
                                  const T* __restrict__ fout, const int64_t* __restrict__ gbase,
                                  T* __restrict__ stage, int64_t* __restrict__ stage_rows) {
  using N = Num<T>;
  using T2 = typename N::T2;
  const int lane = threadIdx.x & 31;
  const int P = F / 2;
  const T2* x2 = reinterpret_cast<const T2*>(x);
  T2* y2 = reinterpret_cast<T2*>(y);
  T2* s2 = reinterpret_cast<T2*>(stage);
  const bool pre = scaling == HG_SCALING_PRE, disc = scaling == HG_SCALING_DISCRETIZED;
  const bool post = scaling == HG_SCALING_POST;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += nwarps) {
    const int64_t beg = offsets[r], end = offsets[r + 1];
    const int64_t ng = (end - beg + 31) / 32;
    const T fo = fout ? fout[r] : N::zero();
    const T2 fo2 = N::bcast(fo);
    const T2 m2 = (pre && fout) ? fo2 : N::bcast(N::from_f(1.0f));
    if (stage && ng > 1 && lane < ng) {
      for (int64_t g = lane; g < ng; g += 32) stage_rows[gbase[r] + g] = r;
    }
    for (int p = lane; p < P; p += 32) {
      T2 yv = N::zero2();
      for (int64_t g = 0; g < ng; ++g) {
        const int64_t gb = beg + g * 32;
        const int64_t ge = gb + 32 < end ? gb + 32 : end;
        T2 acc = N::zero2();
        for (int64_t q = gb; q < ge; ++q) acc = N::fma2(m2, x2[(int64_t)cols[q] * P + p], acc);
        const T2 part = (disc && fout) ? N::mul2(acc, fo2) : acc;
        if (stage && ng > 1) s2[(gbase[r] + g) * P + p] = part;
        yv = g == 0 ? part : N::add2(yv, part);
      }
      if (post && fout && N::gt0(fo)) yv = N::mul2(yv, fo2);
      y2[r * P + p] = yv;
    }
  }
}

}  // namespace hg

extern "C" int hg_spmm_vertex_ref_workspace(int64_t n_cols, int32_t F, int has_in_scale,
                                            int dtype, size_t* bytes) {
  HG_REQUIRE(bytes && F > 0, "hg_spmm_vertex_ref_workspace: bad arguments");
  Carver cv(nullptr, 0);
  if (has_in_scale) cv.take<char>((size_t)n_cols * F * elem_size(dtype));
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_spmm_vertex_ref(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                                  int64_t n_cols, const void* x, void* y, int32_t F,
                                  int32_t scaling, const void* in_scale, const void* out_factor,
                                  const int64_t* group_base, void* staging_partials,
                                  int64_t* staging_rows, int dtype, void* ws, size_t ws_bytes,
                                  void* stream) {
  HG_REQUIRE(dtype == HG_F16 || dtype == HG_F32, "unknown dtype %d", dtype);
  HG_REQUIRE(F > 0 && F % 2 == 0, "feature length %d must be even and positive", F);
  HG_REQUIRE(scaling >= HG_SCALING_POST && scaling <= HG_SCALING_DISCRETIZED,
             "unknown scaling %d", scaling);
  HG_REQUIRE(!staging_partials || (group_base && staging_rows),
             "hg_spmm_vertex_ref: staging needs group_base and staging_rows");
  cudaStream_t st = as_stream(stream);
  if (n_rows == 0) return HG_OK;
  Carver cv(ws, ws_bytes);
  void* xs = in_scale ? cv.take<char>((size_t)n_cols * F * elem_size(dtype)) : nullptr;
  HG_REQUIRE(cv.fits(), "hg_spmm_vertex_ref: workspace too small");
  if (in_scale) {
    int rc = scale_rows(x, in_scale, n_cols, F, xs, dtype, st);
    if (rc) return rc;
    x = xs;
  }
  const int g = grid_for(n_rows, 8, 148 * 64);
  if (dtype == HG_F16)
    k_spmm_vertex_ref<__half><<<g, 256, 0, st>>>(offsets, cols, n_rows, (const __half*)x,
                                                 (__half*)y, F, scaling,
                                                 (const __half*)out_factor, group_base,
                                                 (__half*)staging_partials, staging_rows);
  else
    k_spmm_vertex_ref<float><<<g, 256, 0, st>>>(offsets, cols, n_rows, (const float*)x,
                                                (float*)y, F, scaling, (const float*)out_factor,
                                                group_base, (float*)staging_partials,
                                                staging_rows);
  HG_LAUNCHED();
  return HG_OK;
}

// ── Gather ceiling probe (measurement only) ───────────────────────────────────
// The memory access of one SpMM with all arithmetic, scheduling and output
// removed: the column ids streamed once in edge order, and for every edge the
// row_bytes of X at its column fetched with 16-byte loads by a power-of-two lane
// team (the k_spmm_fast team shape).  Its time is the floor any gather SpMM on
// that graph and width can reach; bench.py reports hg_spmm's time against it.
namespace hg {
template <int TEAM, typename R = uint4>
__global__ void __launch_bounds__(256) k_gather_probe(const int* __restrict__ cols, int64_t E,
                                                      const R* __restrict__ x, int64_t ldv,
                                                      int lanes, unsigned* __restrict__ out) {
  constexpr int RPL = 32 / TEAM;  // rows fetched per warp load
  const int lane = threadIdx.x & 31;
  const int sub = lane % TEAM, slot = lane / TEAM;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned acc = 0;
  for (int64_t base = warp * 32; base < E; base += nwarps * 32) {
    const int c = base + lane < E ? __ldg(cols + base + lane) : -1;
    R v[TEAM];
#pragma unroll
    for (int k = 0; k < TEAM; ++k) {
      const int r = __shfl_sync(0xffffffffu, c, k * RPL + slot);
      if (r >= 0 && sub < lanes) v[k] = ldg_raw(x + (int64_t)r * ldv + sub);
      else memset(&v[k], 0, sizeof(R));
    }
#pragma unroll
    for (int k = 0; k < TEAM; ++k) {
      const unsigned* w = reinterpret_cast<const unsigned*>(&v[k]);
#pragma unroll
      for (int i = 0; i < (int)(sizeof(R) / 4); ++i) acc ^= w[i];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc == 0x9e3779b9u) atomicXor(out, acc);  // keeps the loads live
}
}  // namespace hg

extern "C" int hg_gather_probe(const int32_t* cols, int64_t num_edges, const void* x,
                               int32_t row_bytes, int64_t ld_bytes, uint32_t* out, void* stream) {
  HG_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0 && row_bytes <= 1024,
             "hg_gather_probe: row_bytes %d must be a multiple of 16 in [16, 1024]", row_bytes);
  HG_REQUIRE(row_bytes <= 512 || (row_bytes % 32 == 0 && ld_bytes % 32 == 0 && kLane32),
             "hg_gather_probe: rows over 512 bytes need 32-byte lanes");
  HG_REQUIRE(ld_bytes % 16 == 0 && ld_bytes >= row_bytes && num_edges >= 0,
             "hg_gather_probe: bad row stride");
  HG_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0, "hg_gather_probe: x must be 16-byte aligned");
  if (num_edges == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  // the SpMM's lane width: 32 bytes for rows of 96..1024 bytes that are whole
  // 32-byte chunks (k_spmm_fast's binary16 rule), else 16
  if (kLane32 && row_bytes % 32 == 0 && ld_bytes % 32 == 0 && row_bytes >= 96 &&
      reinterpret_cast<uintptr_t>(x) % 32 == 0) {
    const int lanes = row_bytes / 32;
    const int64_t ldv = ld_bytes / 32;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = (unsigned)sms * 8;
    const U32x8* xv = (const U32x8*)x;
    unsigned* o = (unsigned*)out;
    if (lanes <= 4) k_gather_probe<4, U32x8><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
    else if (lanes <= 8) k_gather_probe<8, U32x8><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
    else k_gather_probe<16, U32x8><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
    HG_LAUNCHED();
    return HG_OK;
  }
  const int lanes = row_bytes / 16;
  const int64_t ldv = ld_bytes / 16;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned g = (unsigned)sms * 8;
  const int4* xv = (const int4*)x;
  unsigned* o = (unsigned*)out;
  if (lanes <= 1) k_gather_probe<1><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
  else if (lanes <= 2) k_gather_probe<2><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
  else if (lanes <= 4) k_gather_probe<4><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
  else if (lanes <= 8) k_gather_probe<8><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
  else if (lanes <= 16) k_gather_probe<16><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
  else k_gather_probe<32><<<g, 256, 0, st>>>(cols, num_edges, xv, ldv, lanes, o);
  HG_LAUNCHED();
  return HG_OK;
}
