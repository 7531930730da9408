// GPU ingest of the reference's whitespace edge-list text (sparse.load_edge_list,
// sparse.py:143-177): the file bytes are copied to HBM once and parsed here.
//
//   1. line terminators: '\n', or '\r' not followed by '\n' (Python universal
//      newlines, so line numbers match the reference's enumerate(fh, 1));
//      found with 16-byte loads, per-block counts, a scan, and a write pass.
//   2. one thread per line: str.strip/str.split semantics on ASCII whitespace
//      (' ', \t, \n, \r, \v, \f, \x1c-\x1f); empty and '#'/'%' lines skipped;
//      fewer than two fields -> "expected 'src dst'"; int() syntax ([+-]digits
//      with single '_' between digits) else "non-integer vertex id"; then
//      "negative vertex id".  The first failing line wins (atomicMin).
//   3. edge lines compacted in file order (cub::DeviceSelect::Flagged), max id
//      reduced -- the (rows, cols) arrays the reference hands to from_edges.
#include <cub/cub.cuh>

#include "hg_common.cuh"

namespace hg {

enum : uint32_t { kLineSkip = 0, kLineEdge = 1, kErrFields = 2, kErrInt = 3, kErrNeg = 4, kErrBig = 5 };


// Line terminators in one pass over the text: block b owns bytes
// [b*kTermChunk, (b+1)*kTermChunk), thread t a 64-byte run of it read as four
// 16-byte vectors (the byte after a '\r' decides whether it ends a line).
// Pass 1 counts per block; pass 2 re-reads, block-scans the per-thread counts
// and writes the terminator positions in file order.
constexpr int kTermThreads = 256;
constexpr int kTermPerThread = 64;
constexpr int64_t kTermChunk = (int64_t)kTermThreads * kTermPerThread;

__device__ __forceinline__ unsigned term_mask64(const unsigned char* __restrict__ t, int64_t n,
                                                int64_t p0, uint64_t& mask) {
  __align__(16) unsigned char b[kTermPerThread + 1];
  if (p0 + kTermPerThread < n && ((reinterpret_cast<uintptr_t>(t) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(b + 16 * q) = *reinterpret_cast<const uint4*>(t + p0 + 16 * q);
    b[kTermPerThread] = t[p0 + kTermPerThread];
  } else {
    for (int i = 0; i <= kTermPerThread; ++i) b[i] = p0 + i < n ? t[p0 + i] : 0;
  }
  mask = 0;
#pragma unroll
  for (int i = 0; i < kTermPerThread; ++i) {
    const bool in = p0 + i < n;
    const bool term = b[i] == '\n' || (b[i] == '\r' && (p0 + i + 1 == n || b[i + 1] != '\n'));
    if (in && term) mask |= 1ull << i;
  }
  return __popcll(mask);
}

__global__ void __launch_bounds__(kTermThreads)
k_count_terms(const unsigned char* __restrict__ t, int64_t n, int64_t* __restrict__ counts) {
  using BR = cub::BlockReduce<unsigned, kTermThreads>;
  __shared__ typename BR::TempStorage tmp;
  uint64_t mask;
  const int64_t p0 = (int64_t)blockIdx.x * kTermChunk + (int64_t)threadIdx.x * kTermPerThread;
  const unsigned c = p0 < n ? term_mask64(t, n, p0, mask) : 0u;
  const unsigned total = BR(tmp).Sum(c);
  if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kTermThreads)
k_write_terms(const unsigned char* __restrict__ t, int64_t n, const int64_t* __restrict__ base,
              int64_t* __restrict__ terms) {
  using BS = cub::BlockScan<unsigned, kTermThreads>;
  __shared__ typename BS::TempStorage tmp;
  uint64_t mask = 0;
  const int64_t p0 = (int64_t)blockIdx.x * kTermChunk + (int64_t)threadIdx.x * kTermPerThread;
  const unsigned c = p0 < n ? term_mask64(t, n, p0, mask) : 0u;
  unsigned off;
  BS(tmp).ExclusiveSum(c, off);
  int64_t o = base[blockIdx.x] + off;
  while (mask) {
    const int i = __ffsll((long long)mask) - 1;
    terms[o++] = p0 + i;
    mask &= mask - 1;
  }
}

__device__ __forceinline__ bool is_ws(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

// Python int() of one field [a, b): 0 ok, kErrInt syntax, kErrBig > int64.
__device__ __forceinline__ uint32_t parse_int(const unsigned char* t, int64_t a, int64_t b,
                                              int64_t& out) {
  bool neg = false;
  if (t[a] == '+' || t[a] == '-') {
    neg = t[a] == '-';
    ++a;
  }
  if (a >= b) return kErrInt;
  unsigned long long v = 0;
  bool big = false, prev_digit = false;
  for (int64_t i = a; i < b; ++i) {
    const unsigned char c = t[i];
    if (c >= '0' && c <= '9') {
      const unsigned d = c - '0';
      if (v > (0x7fffffffffffffffULL - d) / 10ULL) big = true;
      else v = v * 10ULL + d;
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return kErrInt;
    }
  }
  if (!prev_digit) return kErrInt;
  if (big) return neg ? kErrNeg : kErrBig;
  out = neg ? -(int64_t)v : (int64_t)v;
  return 0;
}

__global__ void k_parse_lines(const unsigned char* __restrict__ text, int64_t nbytes,
                              const int64_t* __restrict__ terms, int64_t n_terms, int64_t n_lines,
                              int64_t* __restrict__ src, int64_t* __restrict__ dst,
                              uint8_t* __restrict__ is_edge, int64_t* __restrict__ line_max,
                              unsigned long long* __restrict__ first_err) {
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < n_lines;
       ln += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = ln == 0 ? 0 : terms[ln - 1] + 1;
    const int64_t end = ln < n_terms ? terms[ln] : nbytes;
    uint32_t status = kLineSkip;
    int64_t a = 0, b = 0;
    while (i < end && is_ws(text[i])) ++i;
    if (i < end && text[i] != '#' && text[i] != '%') {
      // fields 1 and 2
      const int64_t a0 = i;
      while (i < end && !is_ws(text[i])) ++i;
      const int64_t b0 = i;
      while (i < end && is_ws(text[i])) ++i;
      const int64_t a1 = i;
      while (i < end && !is_ws(text[i])) ++i;
      const int64_t b1 = i;
      if (a1 == b1) {
        status = kErrFields;
      } else {
        const uint32_t e0 = parse_int(text, a0, b0, a);
        const uint32_t e1 = parse_int(text, a1, b1, b);
        if (e0 == kErrInt || e1 == kErrInt) status = kErrInt;
        else if (e0 == kErrNeg || e1 == kErrNeg || a < 0 || b < 0) status = kErrNeg;
        else if (e0 == kErrBig || e1 == kErrBig) status = kErrBig;
        else status = kLineEdge;
      }
    }
    is_edge[ln] = status == kLineEdge;
    src[ln] = a;
    dst[ln] = b;
    line_max[ln] = status == kLineEdge ? (a > b ? a : b) : -1;
    // ids beyond int64 only fail after every line parsed (the reference's
    // np.asarray overflow), so they rank behind all line errors
    if (status >= kErrFields)
      atomicMin(first_err, ((unsigned long long)(ln + 1 + (status == kErrBig ? n_lines : 0)) << 4) | status);
  }
}

struct IngestPlan {
  int64_t* terms;
  int64_t* n_sel;
  int64_t* src;
  int64_t* dst;
  uint8_t* is_edge;
  int64_t* line_max;
  int64_t* max_id;
  unsigned long long* first_err;
  int64_t nblk;
  int64_t* blk;   // per-block terminator counts (+ a zero)
  int64_t* blkx;  // their exclusive scan: first terminator slot per block, total last
  void* cub_tmp;
  size_t cub_bytes;
};

static int plan_ingest(Carver& cv, int64_t nbytes, int64_t n_lines, IngestPlan& p) {
  const int64_t L = n_lines > 0 ? n_lines : 1;
  p.terms = cv.take<int64_t>(L);
  p.n_sel = cv.take<int64_t>(2);
  p.src = cv.take<int64_t>(L);
  p.dst = cv.take<int64_t>(L);
  p.is_edge = cv.take<uint8_t>(L);
  p.line_max = cv.take<int64_t>(L);
  p.max_id = cv.take<int64_t>(1);
  p.first_err = cv.take<unsigned long long>(1);
  p.nblk = (nbytes + kTermChunk - 1) / kTermChunk;
  p.blk = cv.take<int64_t>(p.nblk + 1);
  p.blkx = cv.take<int64_t>(p.nblk + 1);
  size_t b1 = 0, b2 = 0, b3 = 0;
  HG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b1, (int64_t*)nullptr, (int64_t*)nullptr,
                                        p.nblk + 1));
  HG_CUDA(cub::DeviceSelect::Flagged(nullptr, b2, (int64_t*)nullptr, (uint8_t*)nullptr,
                                     (int64_t*)nullptr, (int64_t*)nullptr, L));
  HG_CUDA(cub::DeviceReduce::Max(nullptr, b3, (int64_t*)nullptr, (int64_t*)nullptr, L));
  p.cub_bytes = b1 > b2 ? b1 : b2;
  if (b3 > p.cub_bytes) p.cub_bytes = b3;
  p.cub_tmp = cv.take<char>(p.cub_bytes);
  return HG_OK;
}

}  // namespace hg

using namespace hg;

extern "C" int hg_count_lines_workspace(int64_t nbytes, size_t* bytes) {
  HG_REQUIRE(bytes && nbytes >= 0, "hg_count_lines_workspace: bad arguments");
  const int64_t nblk = (nbytes + kTermChunk - 1) / kTermChunk;
  size_t b = 0;
  HG_CUDA(cub::DeviceReduce::Sum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr,
                                 nblk > 0 ? nblk : 1));
  Carver cv(nullptr, 0);
  cv.take<int64_t>(nblk > 0 ? nblk : 1);
  cv.take<int64_t>(1);
  cv.take<char>(b);
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_count_lines(const void* text, int64_t nbytes, int64_t* n_lines_out, void* ws,
                              size_t ws_bytes, void* stream) {
  HG_REQUIRE(nbytes >= 0 && n_lines_out, "hg_count_lines: bad arguments");
  if (nbytes == 0) {
    *n_lines_out = 0;
    return HG_OK;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t nblk = (nbytes + kTermChunk - 1) / kTermChunk;
  Carver cv(ws, ws_bytes);
  int64_t* counts = cv.take<int64_t>(nblk);
  int64_t* cnt = cv.take<int64_t>(1);
  size_t b = 0;
  HG_CUDA(cub::DeviceReduce::Sum(nullptr, b, counts, cnt, nblk));
  void* tmp = cv.take<char>(b);
  HG_REQUIRE(cv.fits(), "hg_count_lines: workspace too small");
  k_count_terms<<<(unsigned)nblk, kTermThreads, 0, st>>>((const unsigned char*)text, nbytes,
                                                        counts);
  HG_LAUNCHED();
  HG_CUDA(cub::DeviceReduce::Sum(tmp, b, counts, cnt, nblk, st));
  int64_t terms = 0;
  unsigned char last = 0;
  HG_CUDA(cudaMemcpyAsync(&terms, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaMemcpyAsync(&last, (const unsigned char*)text + nbytes - 1, 1,
                          cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaStreamSynchronize(st));
  // a final line without a terminator still counts
  *n_lines_out = terms + ((last == '\n' || last == '\r') ? 0 : 1);
  return HG_OK;
}

extern "C" int hg_parse_edges_workspace(int64_t nbytes, int64_t n_lines, size_t* bytes) {
  HG_REQUIRE(bytes && nbytes >= 0 && n_lines >= 0, "hg_parse_edges_workspace: bad arguments");
  Carver cv(nullptr, 0);
  IngestPlan p;
  int rc = plan_ingest(cv, nbytes, n_lines, p);
  if (rc) return rc;
  *bytes = cv.used;
  return HG_OK;
}

extern "C" int hg_parse_edges(const void* text, int64_t nbytes, int64_t n_lines, int64_t* rows_out,
                              int64_t* cols_out, int64_t* result /* host int64[4] */, void* ws,
                              size_t ws_bytes, void* stream) {
  HG_REQUIRE(nbytes >= 0 && n_lines >= 0 && result, "hg_parse_edges: bad arguments");
  result[0] = 0;
  result[1] = -1;
  result[2] = 0;
  result[3] = 0;
  if (n_lines == 0) return HG_OK;
  cudaStream_t st = as_stream(stream);
  Carver cv(ws, ws_bytes);
  IngestPlan p;
  int rc = plan_ingest(cv, nbytes, n_lines, p);
  if (rc) return rc;
  HG_REQUIRE(cv.fits(), "hg_parse_edges: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  const unsigned char* t = (const unsigned char*)text;
  size_t tb = p.cub_bytes;
  HG_CUDA(cudaMemsetAsync(p.blk + p.nblk, 0, sizeof(int64_t), st));
  k_count_terms<<<(unsigned)p.nblk, kTermThreads, 0, st>>>(t, nbytes, p.blk);
  HG_LAUNCHED();
  HG_CUDA(cub::DeviceScan::ExclusiveSum(p.cub_tmp, tb, p.blk, p.blkx, p.nblk + 1, st));
  k_write_terms<<<(unsigned)p.nblk, kTermThreads, 0, st>>>(t, nbytes, p.blkx, p.terms);
  HG_LAUNCHED();
  int64_t n_terms = 0;
  HG_CUDA(cudaMemcpyAsync(&n_terms, p.blkx + p.nblk, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaStreamSynchronize(st));
  HG_REQUIRE(n_terms <= n_lines && n_lines <= n_terms + 1,
             "hg_parse_edges: n_lines %lld does not match the text (%lld terminators)",
             (long long)n_lines, (long long)n_terms);
  HG_CUDA(cudaMemsetAsync(p.first_err, 0xff, sizeof(unsigned long long), st));
  k_parse_lines<<<grid_for(n_lines, 256, 148 * 64), 256, 0, st>>>(
      t, nbytes, p.terms, n_terms, n_lines, p.src, p.dst, p.is_edge, p.line_max, p.first_err);
  HG_LAUNCHED();
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceSelect::Flagged(p.cub_tmp, tb, p.src, p.is_edge, rows_out, p.n_sel, n_lines, st));
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceSelect::Flagged(p.cub_tmp, tb, p.dst, p.is_edge, cols_out, p.n_sel + 1, n_lines, st));
  tb = p.cub_bytes;
  HG_CUDA(cub::DeviceReduce::Max(p.cub_tmp, tb, p.line_max, p.max_id, n_lines, st));
  int64_t counts[2] = {0, 0};
  int64_t mx = -1;
  unsigned long long err = 0;
  HG_CUDA(cudaMemcpyAsync(counts, p.n_sel, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaMemcpyAsync(&mx, p.max_id, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaMemcpyAsync(&err, p.first_err, sizeof(err), cudaMemcpyDeviceToHost, st));
  HG_CUDA(cudaStreamSynchronize(st));
  result[0] = counts[0];
  result[1] = mx;
  if (err != ~0ULL) {
    result[3] = (int64_t)(err & 15);
    result[2] = (int64_t)(err >> 4) - (result[3] == kErrBig ? n_lines : 0);
  }
  return HG_OK;
}
