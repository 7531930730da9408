// Graph construction on the GPU: canonical CSR (sort + dedup), the transposed
// CSC with its stable permutation, degree-factor tables and the
// degree-bucketed work-unit scheduler.  Integer work, bit-exact with the
// reference's numpy definitions (sparse.py:56-125, kernels.py:118-140).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cstdarg>
#include <cstdio>

#include "hg_common.cuh"

namespace hg {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

// ------------------------------------------------------------------ CSR build

__global__ void k_make_keys(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                            int64_t m, int64_t n, uint64_t* __restrict__ keys,
                            int* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = rows[i], c = cols[i];
    if (r < 0 || c < 0) atomicOr(flags, 1);
    else if (r >= n || c >= n) atomicOr(flags, 2);
    keys[i] = (uint64_t)r * (uint64_t)n + (uint64_t)c;
  }
}

__global__ void k_split_keys(const uint64_t* __restrict__ keys, int64_t m, int64_t n,
                             int32_t* __restrict__ cols_out, int64_t* __restrict__ rows_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    uint64_t r = k / (uint64_t)n;
    cols_out[i] = (int32_t)(k - r * (uint64_t)n);
    if (rows_out) rows_out[i] = (int64_t)r;
  }
}

// offsets[r] = first i with keys[i] >= r*n (lower bound), r in [0, n].
__global__ void k_offsets_from_keys(const uint64_t* __restrict__ keys, int64_t m, int64_t n,
                                    int64_t* __restrict__ offsets) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t target = (uint64_t)r * (uint64_t)n;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    offsets[r] = lo;
  }
}

struct CsrBuildPlan {
  uint64_t* keys;
  uint64_t* keys_alt;
  uint64_t* uniq;
  int* flags;
  int64_t* nsel;
  void* cub_tmp;
  size_t cub_bytes;
};

static int plan_build_csr(Carver& cv, int64_t m, int64_t n, CsrBuildPlan& p) {
  p.keys = cv.take<uint64_t>(m > 0 ? m : 1);
  p.keys_alt = cv.take<uint64_t>(m > 0 ? m : 1);
  p.uniq = cv.take<uint64_t>(m > 0 ? m : 1);
  p.flags = cv.take<int>(1);
  p.nsel = cv.take<int64_t>(1);
  size_t sort_bytes = 0, uniq_bytes = 0;
  cub::DoubleBuffer<uint64_t> db(nullptr, nullptr);
  HG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, db, (int64_t)m, 0, 64));
  HG_CUDA(cub::DeviceSelect::Unique(nullptr, uniq_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (int64_t*)nullptr, (int64_t)m));
  p.cub_bytes = sort_bytes > uniq_bytes ? sort_bytes : uniq_bytes;
  p.cub_tmp = cv.take<char>(p.cub_bytes);
  return HG_OK;
}

}  // namespace hg

using namespace hg;

extern "C" const char* hg_last_error(void) { return hg::g_err; }
extern "C" int hg_abi_version(void) { return HG_ABI_VERSION; }

extern "C" int hg_build_csr_workspace(int64_t num_edges_in, int64_t n, size_t* bytes) {
  HG_REQUIRE(bytes && num_edges_in >= 0 && n > 0, "hg_build_csr_workspace: bad arguments");
  Carver cv(nullptr, 0);
  CsrBuildPlan p;
  int rc = plan_build_csr(cv, num_edges_in, n, p);
  if (rc) return rc;
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_build_csr(const int64_t* rows_in, const int64_t* cols_in, int64_t m, int64_t n,
                            int64_t* offsets_out, int32_t* cols_out, int64_t* rows_out,
                            int64_t* num_edges_out, void* ws, size_t ws_bytes, void* stream) {
  HG_REQUIRE(n > 0, "vertex count must be positive");
  HG_REQUIRE(m >= 0 && num_edges_out && offsets_out, "hg_build_csr: bad arguments");
  HG_REQUIRE(n <= (int64_t)INT32_MAX, "hg_build_csr: vertex count exceeds int32 column ids");
  cudaStream_t st = as_stream(stream);
  Carver cv(ws, ws_bytes);
  CsrBuildPlan p;
  int rc = plan_build_csr(cv, m, n, p);
  if (rc) return rc;
  HG_REQUIRE(cv.fits(), "hg_build_csr: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  if (m == 0) {
    HG_CUDA(cudaMemsetAsync(offsets_out, 0, sizeof(int64_t) * (n + 1), st));
    HG_CUDA(cudaStreamSynchronize(st));
    *num_edges_out = 0;
    return HG_OK;
  }
  HG_CUDA(cudaMemsetAsync(p.flags, 0, sizeof(int), st));
  k_make_keys<<<grid_for(m, 256, 148 * 32), 256, 0, st>>>(rows_in, cols_in, m, n, p.keys, p.flags);
  HG_LAUNCHED();
  int end_bit = bits_for((uint64_t)n * (uint64_t)n - 1);
  cub::DoubleBuffer<uint64_t> db(p.keys, p.keys_alt);
  size_t tb = p.cub_bytes;
  HG_CUDA(cub::DeviceRadixSort::SortKeys(p.cub_tmp, tb, db, (int64_t)m, 0, end_bit, st));
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceSelect::Unique(p.cub_tmp, tb, db.Current(), p.uniq, p.nsel, (int64_t)m, st));
  int flags = 0;
  int64_t e = 0;
  HG_CUDA(cudaMemcpyAsync(&flags, p.flags, sizeof(int), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaMemcpyAsync(&e, p.nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaStreamSynchronize(st));
  HG_REQUIRE(!(flags & 1), "negative vertex id");
  HG_REQUIRE(!(flags & 2), "vertex id out of range");
  k_split_keys<<<grid_for(e, 256, 148 * 32), 256, 0, st>>>(p.uniq, e, n, cols_out, rows_out);
  HG_LAUNCHED();
  k_offsets_from_keys<<<grid_for(n + 1, 256, 148 * 32), 256, 0, st>>>(p.uniq, e, n, offsets_out);
  HG_LAUNCHED();
  HG_CUDA(cudaStreamSynchronize(st));
  *num_edges_out = e;
  return HG_OK;
}

// ------------------------------------------------------------------ transpose

namespace hg {

__global__ void k_edge_rows_iota(const int64_t* __restrict__ offsets, int64_t n, int64_t m,
                                 int32_t* __restrict__ rows, int32_t* __restrict__ iota) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    rows[e] = (int32_t)row_of_edge(offsets, n, e);
    iota[e] = (int32_t)e;
  }
}

__global__ void k_gather_rows(const int32_t* __restrict__ perm, const int32_t* __restrict__ rows,
                              int64_t m, int32_t* __restrict__ t_cols) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    t_cols[i] = rows[perm[i]];
}

__global__ void k_offsets_from_sorted(const uint32_t* __restrict__ sorted, int64_t m, int64_t n,
                                      int64_t* __restrict__ offsets) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)sorted[mid] < r) lo = mid + 1; else hi = mid;
    }
    offsets[r] = lo;
  }
}

struct TransposePlan {
  int32_t* rows;
  uint32_t* keys_alt;
  int32_t* iota;
  uint32_t* keys_sorted;
  void* cub_tmp;
  size_t cub_bytes;
};

static int plan_transpose(Carver& cv, int64_t m, TransposePlan& p) {
  int64_t mm = m > 0 ? m : 1;
  p.rows = cv.take<int32_t>(mm);
  p.keys_alt = cv.take<uint32_t>(mm);
  p.iota = cv.take<int32_t>(mm);
  p.keys_sorted = cv.take<uint32_t>(mm);
  size_t b = 0;
  HG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                          (const int32_t*)nullptr, (int32_t*)nullptr, (int64_t)m,
                                          0, 32));
  p.cub_bytes = b;
  p.cub_tmp = cv.take<char>(b);
  return HG_OK;
}

}  // namespace hg

extern "C" int hg_transpose_workspace(int64_t n, int64_t m, size_t* bytes) {
  HG_REQUIRE(bytes && m >= 0 && n > 0, "hg_transpose_workspace: bad arguments");
  Carver cv(nullptr, 0);
  TransposePlan p;
  int rc = plan_transpose(cv, m, p);
  if (rc) return rc;
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_transpose(const int64_t* offsets, const int32_t* cols, int64_t n, int64_t m,
                            int64_t* t_offsets, int32_t* t_cols, int32_t* perm, void* ws,
                            size_t ws_bytes, void* stream) {
  HG_REQUIRE(n > 0 && m >= 0, "hg_transpose: bad sizes");
  HG_REQUIRE(m <= (int64_t)INT32_MAX, "hg_transpose: edge count exceeds int32 permutation");
  cudaStream_t st = as_stream(stream);
  Carver cv(ws, ws_bytes);
  TransposePlan p;
  int rc = plan_transpose(cv, m, p);
  if (rc) return rc;
  HG_REQUIRE(cv.fits(), "hg_transpose: workspace too small");
  if (m == 0) {
    HG_CUDA(cudaMemsetAsync(t_offsets, 0, sizeof(int64_t) * (n + 1), st));
    return HG_OK;
  }
  k_edge_rows_iota<<<grid_for(m, 256, 148 * 32), 256, 0, st>>>(offsets, n, m, p.rows, p.iota);
  HG_LAUNCHED();
  // LSD radix sort is stable: equal columns keep ascending (row) order, which is
  // exactly np.argsort(col*n + row, kind="stable") on a canonical edge list.
  size_t tb = p.cub_bytes;
  int end_bit = bits_for((uint64_t)(n - 1));
  HG_CUDA(cub::DeviceRadixSort::SortPairs(p.cub_tmp, tb, (const uint32_t*)cols, p.keys_sorted,
                                          p.iota, perm, (int64_t)m, 0, end_bit, st));
  k_gather_rows<<<grid_for(m, 256, 148 * 32), 256, 0, st>>>(perm, p.rows, m, t_cols);
  HG_LAUNCHED();
  k_offsets_from_sorted<<<grid_for(n + 1, 256, 148 * 32), 256, 0, st>>>(p.keys_sorted, m, n,
                                                                         t_offsets);
  HG_LAUNCHED();
  return HG_OK;
}

// ------------------------------------------------------------- degree factors

namespace hg {

template <typename T>
__global__ void k_degree_factors(const int64_t* __restrict__ offsets, int64_t n, int kind,
                                 T* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = offsets[v + 1] - offsets[v];
    float f = 0.0f;
    if (d > 0) {
      float df = __ll2float_rn(d);  // numpy .astype(np.float32)
      f = (kind == HG_FACTOR_INV) ? __fdiv_rn(1.0f, df) : __fdiv_rn(1.0f, __fsqrt_rn(df));
    }
    out[v] = Num<T>::from_f(f);
  }
}

}  // namespace hg

extern "C" int hg_degree_factors(const int64_t* offsets, int64_t n, int kind, int dtype,
                                 void* out, void* stream) {
  HG_REQUIRE(n > 0, "hg_degree_factors: vertex count must be positive");
  HG_REQUIRE(kind == HG_FACTOR_INV || kind == HG_FACTOR_INV_SQRT, "unknown factor kind %d", kind);
  cudaStream_t st = as_stream(stream);
  int g = grid_for(n, 256, 148 * 16);
  if (dtype == HG_F16)
    k_degree_factors<__half><<<g, 256, 0, st>>>(offsets, n, kind, (__half*)out);
  else if (dtype == HG_F32)
    k_degree_factors<float><<<g, 256, 0, st>>>(offsets, n, kind, (float*)out);
  else
    HG_REQUIRE(false, "unknown dtype %d", dtype);
  HG_LAUNCHED();
  return HG_OK;
}

// ------------------------------------------------------------------ scheduler

namespace hg {

static constexpr int kNumClasses = 33;  // len 0 -> class 0, else floor(log2(len)) + 1

// Per row: unit count, carry slots, split flag; with packing (pack_rows > 0, a
// power of two <= 32) a row inside an aligned block of pack_rows rows holding
// at most pack_edges edges in total gets no unit -- the block becomes one pack,
// flagged at its first row.  Blocks are whole half/quarter warps
// (blockDim % 32 == 0).
__global__ void k_unit_counts(const int64_t* __restrict__ offsets, int64_t n, int64_t cap,
                              int pack_rows, int64_t pack_edges,
                              int64_t* __restrict__ nparts, int64_t* __restrict__ split_parts,
                              int64_t* __restrict__ split_flag, int64_t* __restrict__ pack_flag) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = base + threadIdx.x;
    const bool in = r < n;
    const int64_t d = in ? offsets[r + 1] - offsets[r] : 0;
    bool packed = false;
    if (pack_rows > 0 && in) {
      const int64_t r0 = r & ~(int64_t)(pack_rows - 1);
      const int64_t r1 = r0 + pack_rows < n ? r0 + pack_rows : n;
      packed = offsets[r1] - offsets[r0] <= pack_edges;
    }
    if (in) {
      const int64_t p = packed ? 0 : (d == 0 ? 1 : (d + cap - 1) / cap);
      nparts[r] = p;
      split_parts[r] = p > 1 ? p : 0;
      split_flag[r] = p > 1 ? 1 : 0;
      pack_flag[r] = packed && (r & (pack_rows - 1)) == 0 ? 1 : 0;
    }
  }
}

__global__ void k_emit_units(const int64_t* __restrict__ offsets, int64_t n, int64_t cap,
                             const int64_t* __restrict__ nparts,
                             const int64_t* __restrict__ unit_base,
                             const int64_t* __restrict__ slot_base,
                             const int64_t* __restrict__ split_idx, int4* __restrict__ units,
                             uint32_t* __restrict__ keys, int32_t* __restrict__ iota,
                             int4* __restrict__ split_rows, int pack_rows,
                             const int64_t* __restrict__ pack_flag,
                             const int64_t* __restrict__ pack_idx, int4* __restrict__ packs) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t beg = offsets[r], end = offsets[r + 1];
    if (pack_rows > 0 && pack_flag[r]) {
      const int64_t cnt = n - r < pack_rows ? n - r : pack_rows;
      packs[pack_idx[r]] = make_int4((int)r, (int)beg, (int)offsets[r + cnt], (int)cnt);
    }
    int64_t p = nparts[r];
    int64_t ub = unit_base[r];
    for (int64_t j = 0; j < p; ++j) {
      int64_t b = beg + j * cap;
      int64_t e = b + cap < end ? b + cap : end;
      int64_t len = e - b;
      int cls = len == 0 ? 0 : 64 - __clzll((unsigned long long)len);
      units[ub + j] = make_int4((int)r, (int)b, (int)e, p > 1 ? (int)(slot_base[r] + j) : -1);
      keys[ub + j] = (uint32_t)(kNumClasses - 1 - cls);  // descending length class
      iota[ub + j] = (int32_t)(ub + j);
    }
    if (p > 1) split_rows[split_idx[r]] = make_int4((int)r, (int)slot_base[r], (int)p, 0);
  }
}

__global__ void k_gather_units(const int4* __restrict__ src, const int32_t* __restrict__ order,
                               int64_t m, int4* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[order[i]];
}

struct SchedPlan {
  int64_t *nparts, *split_parts, *split_flag, *unit_base, *slot_base, *split_idx;
  int64_t *pack_flag, *pack_idx;
  int4* units_tmp;
  uint32_t *keys, *keys_alt;
  int32_t *iota, *order;
  int64_t* totals;
  void* cub_tmp;
  size_t cub_bytes;
};

static int64_t max_units_for(int64_t n, int64_t m, int64_t cap) { return n + (m + cap - 1) / cap; }

static int plan_schedule(Carver& cv, int64_t n, int64_t max_units, SchedPlan& p) {
  p.nparts = cv.take<int64_t>(n);
  p.split_parts = cv.take<int64_t>(n);
  p.split_flag = cv.take<int64_t>(n);
  p.unit_base = cv.take<int64_t>(n + 1);
  p.slot_base = cv.take<int64_t>(n + 1);
  p.split_idx = cv.take<int64_t>(n + 1);
  p.pack_flag = cv.take<int64_t>(n);
  p.pack_idx = cv.take<int64_t>(n + 1);
  p.units_tmp = cv.take<int4>(max_units);
  p.keys = cv.take<uint32_t>(max_units);
  p.keys_alt = cv.take<uint32_t>(max_units);
  p.iota = cv.take<int32_t>(max_units);
  p.order = cv.take<int32_t>(max_units);
  p.totals = cv.take<int64_t>(4);
  size_t b1 = 0, b2 = 0;
  HG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b1, (int64_t*)nullptr, (int64_t*)nullptr,
                                        (int64_t)n));
  HG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, (const uint32_t*)nullptr,
                                          (uint32_t*)nullptr, (const int32_t*)nullptr,
                                          (int32_t*)nullptr, (int64_t)max_units, 0, 6));
  p.cub_bytes = b1 > b2 ? b1 : b2;
  p.cub_tmp = cv.take<char>(p.cub_bytes);
  return HG_OK;
}

}  // namespace hg

extern "C" int hg_schedule_workspace(int64_t n, int64_t m, int32_t cap, size_t* bytes) {
  HG_REQUIRE(bytes && n > 0 && m >= 0 && cap > 0, "hg_schedule_workspace: bad arguments");
  Carver cv(nullptr, 0);
  SchedPlan p;
  int rc = plan_schedule(cv, n, max_units_for(n, m, cap), p);
  if (rc) return rc;
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_schedule_build(const int64_t* offsets, int64_t n, int32_t cap,
                                 int32_t pack_rows, int32_t pack_edges, int32_t* units,
                                 int64_t max_units, int32_t* split_rows, int64_t max_split,
                                 int32_t* packs, int64_t max_packs, int64_t* counts_out, void* ws,
                                 size_t ws_bytes, void* stream) {
  HG_REQUIRE(n > 0 && cap > 0 && counts_out, "hg_schedule_build: bad arguments");
  HG_REQUIRE(pack_rows == 0 || (pack_rows >= 2 && pack_rows <= kPackRows &&
                                (pack_rows & (pack_rows - 1)) == 0 && pack_edges >= 0 &&
                                pack_edges <= cap && packs &&
                                max_packs >= (n + pack_rows - 1) / pack_rows),
             "hg_schedule_build: pack_rows must be a power of two in [2, %d] with "
             "0 <= pack_edges <= split_cap and room for ceil(n / pack_rows) packs",
             kPackRows);
  HG_REQUIRE(n <= (int64_t)INT32_MAX, "hg_schedule_build: too many rows");
  cudaStream_t st = as_stream(stream);
  int64_t m = 0;
  HG_CUDA(cudaMemcpyAsync(&m, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaStreamSynchronize(st));
  HG_REQUIRE(m <= (int64_t)INT32_MAX, "hg_schedule_build: edge count exceeds int32 units");
  int64_t need_units = max_units_for(n, m, cap);
  HG_REQUIRE(max_units >= need_units, "hg_schedule_build: max_units %lld < %lld",
             (long long)max_units, (long long)need_units);
  HG_REQUIRE(max_split >= (m + cap - 1) / cap, "hg_schedule_build: max_split too small");
  Carver cv(ws, ws_bytes);
  SchedPlan p;
  int rc = plan_schedule(cv, n, need_units, p);
  if (rc) return rc;
  HG_REQUIRE(cv.fits(), "hg_schedule_build: workspace too small");

  int g = grid_for(n, 256, 148 * 16);
  k_unit_counts<<<g, 256, 0, st>>>(offsets, n, cap, pack_rows, pack_edges, p.nparts,
                                   p.split_parts, p.split_flag, p.pack_flag);
  HG_LAUNCHED();
  // exclusive scans as inclusive scans shifted by one slot (base[0] = 0)
  HG_CUDA(cudaMemsetAsync(p.unit_base, 0, sizeof(int64_t), st));
  HG_CUDA(cudaMemsetAsync(p.slot_base, 0, sizeof(int64_t), st));
  HG_CUDA(cudaMemsetAsync(p.split_idx, 0, sizeof(int64_t), st));
  size_t tb = p.cub_bytes;
  HG_CUDA(cub::DeviceScan::InclusiveSum(p.cub_tmp, tb, p.nparts, p.unit_base + 1, (int64_t)n, st));
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceScan::InclusiveSum(p.cub_tmp, tb, p.split_parts, p.slot_base + 1, (int64_t)n,
                                        st));
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceScan::InclusiveSum(p.cub_tmp, tb, p.split_flag, p.split_idx + 1, (int64_t)n,
                                        st));
  HG_CUDA(cudaMemsetAsync(p.pack_idx, 0, sizeof(int64_t), st));
  if (pack_rows > 0) {
    tb = p.cub_bytes;
    HG_CUDA(cub::DeviceScan::InclusiveSum(p.cub_tmp, tb, p.pack_flag, p.pack_idx + 1, (int64_t)n,
                                          st));
  }
  int64_t totals[4] = {0, 0, 0, 0};
  HG_CUDA(cudaMemcpyAsync(&totals[0], p.unit_base + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaMemcpyAsync(&totals[1], p.split_idx + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaMemcpyAsync(&totals[2], p.slot_base + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (pack_rows > 0)
    HG_CUDA(cudaMemcpyAsync(&totals[3], p.pack_idx + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            st));
  k_emit_units<<<g, 256, 0, st>>>(offsets, n, cap, p.nparts, p.unit_base, p.slot_base,
                                  p.split_idx, p.units_tmp, p.keys, p.iota, (int4*)split_rows,
                                  pack_rows, p.pack_flag, p.pack_idx, (int4*)packs);
  HG_LAUNCHED();
  HG_CUDA(cudaStreamSynchronize(st));
  int64_t nu = totals[0];
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceRadixSort::SortPairs(p.cub_tmp, tb, p.keys, p.keys_alt, p.iota, p.order,
                                          (int64_t)nu, 0, 6, st));
  k_gather_units<<<grid_for(nu, 256, 148 * 16), 256, 0, st>>>(p.units_tmp, p.order, nu,
                                                              (int4*)units);
  HG_LAUNCHED();
  HG_CUDA(cudaStreamSynchronize(st));
  counts_out[0] = totals[0];
  counts_out[1] = totals[1];
  counts_out[2] = totals[2];
  counts_out[3] = totals[3];
  return HG_OK;
}
