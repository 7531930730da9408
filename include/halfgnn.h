/*
 * halfgnn.h -- C ABI of the B200 (sm_100a) half-precision GNN hot path.
 *
 * One shared library (libhalfgnn.so).  Every entry point:
 *   - returns int: HG_OK (0), HG_EINVAL (1, bad argument; text in hg_last_error()),
 *     HG_ECUDA (2, CUDA failure);
 *   - takes only device pointers, POD sizes and a cudaStream_t (passed as void*);
 *   - never allocates device memory: scratch is sized by the matching *_workspace
 *     query and supplied by the caller;
 *   - is stream-ordered and reentrant (no global mutable state besides the
 *     thread-local error text).  Graph-construction calls (hg_build_csr,
 *     hg_schedule_build) synchronise their stream once, because their output
 *     size is data dependent; the compute calls never synchronise.
 *
 * Element types: "half" buffers hold IEEE binary16 bit patterns (uint16_t),
 * "float" buffers IEEE binary32.  A `dtype` argument selects HG_F16 / HG_F32
 * for the operators that exist in both precision modes of the reference
 * (halfsparse DenseTensor modes "half" / "float32").
 *
 * Each function cites the reference operator (path:line under the halfsparse
 * package, pkg/src/halfsparse/) whose behaviour it replaces.
 */
#ifndef HALFGNN_H
#define HALFGNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_ABI_VERSION 6

enum { HG_OK = 0, HG_EINVAL = 1, HG_ECUDA = 2 };
enum { HG_F16 = 0, HG_F32 = 1 };
/* kernels.py:50 SCALINGS */
enum { HG_SCALING_POST = 0, HG_SCALING_PRE = 1, HG_SCALING_DISCRETIZED = 2 };
/* degree-factor kinds, kernels.py:118-140 ("left"/"right" use 1/d, "both" 1/sqrt(d)) */
enum { HG_FACTOR_INV = 1, HG_FACTOR_INV_SQRT = 2 };

/* Thread-local text of the last HG_EINVAL / HG_ECUDA. */
const char* hg_last_error(void);
int hg_abi_version(void);

/* ---------------------------------------------------------------- graph build */

/* CooGraph.from_edges + coo_to_csr (sparse.py:56-69, 97-101): canonicalise an
 * unsorted int64 edge list (sort by (row, col), drop duplicates) and emit CSR.
 * Errors (HG_EINVAL): "negative vertex id", "vertex id out of range".
 * cols_out / rows_out need capacity num_edges_in; rows_out may be NULL.
 * *num_edges_out (HOST pointer) receives the deduplicated edge count.
 * Synchronises `stream`. */
int hg_build_csr_workspace(int64_t num_edges_in, int64_t n, size_t* bytes);
int hg_build_csr(const int64_t* rows_in, const int64_t* cols_in, int64_t num_edges_in,
                 int64_t n, int64_t* offsets_out, int32_t* cols_out, int64_t* rows_out,
                 int64_t* num_edges_out, void* ws, size_t ws_bytes, void* stream);

/* transpose(g, return_perm=True) + col_degrees (sparse.py:109-125): CSC of a
 * canonical CSR and the stable permutation perm[new] = old edge id
 * (np.argsort(col*n+row, kind="stable")). */
int hg_transpose_workspace(int64_t n, int64_t num_edges, size_t* bytes);
int hg_transpose(const int64_t* offsets, const int32_t* cols, int64_t n, int64_t num_edges,
                 int64_t* t_offsets, int32_t* t_cols, int32_t* perm, void* ws,
                 size_t ws_bytes, void* stream);

/* _degree_factors / _ref_factors (kernels.py:118-140, 583-600): per vertex
 * rnd(fp32(1)/fp32(d)) or rnd(fp32(1)/sqrtf(fp32(d))), 0 for d == 0; degrees are
 * offsets[v+1]-offsets[v] (pass CSR offsets for row degrees, CSC for column). */
int hg_degree_factors(const int64_t* offsets, int64_t n, int kind, int dtype, void* out,
                      void* stream);

/* ------------------------------------------------------------------ scheduler */

/* Degree-bucketed work units replacing simt.plan_edge_parallel /
 * plan_vertex_grouped (simt.py:158-201) for the fp32-guarded kernels.
 * Every row becomes max(1, ceil(deg/split_cap)) units {row, begin, end, slot}
 * (int32 x4); slot = -1 for a whole row, else the row's fp32 carry slot.
 * Units are ordered by descending length class floor(log2(len))+1, rows
 * ascending inside a class (stable).  split_rows receives {row, first_slot,
 * nparts, 0} for every row with nparts > 1, rows ascending.
 * Packing (pack_rows > 0: a power of two in [2, 16], 0 <= pack_edges <=
 * split_cap): every aligned block of pack_rows rows [k*pack_rows, ...) holding
 * at most pack_edges edges in total becomes one pack {first_row, begin, end,
 * rows} (int32 x4, rows ascending) instead of per-row units -- short rows
 * walked as one edge stream by hg_spmm, so a run of near-empty rows costs one
 * team, not one dependent load chain per row.  pack_rows = 0: no packs.
 * Capacities: max_units >= n + ceil(E/split_cap), max_split >= ceil(E/split_cap),
 * max_packs >= ceil(n/pack_rows).
 * counts_out (HOST int64[4]) = {num_units, num_split_rows, num_slots, num_packs}.
 * Synchronises `stream`. */
int hg_schedule_workspace(int64_t n, int64_t num_edges, int32_t split_cap, size_t* bytes);
int hg_schedule_build(const int64_t* offsets, int64_t n, int32_t split_cap, int32_t pack_rows,
                      int32_t pack_edges, int32_t* units, int64_t max_units, int32_t* split_rows,
                      int64_t max_split, int32_t* packs, int64_t max_packs,
                      int64_t* counts_out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------- SpMM */

/* fp32-guarded row-owned SpMM (the B200 hot kernel for spmm_v / spmm_ve,
 * kernels.py:394-401; models.spmm_agg / spmm_weighted, models.py:274-314).
 *   S[r] = sum_{e in row r} m_e * X'[cols[e]]   (fp32 accumulation),
 *   X'   = rnd(X * in_scale[:, None])          (in_scale may be NULL),
 *   m_e  = 1, or w[(w_index ? w_index[e] : e) * heads + head(f)] when w != NULL,
 *   head(f) = f / (F / heads).
 *   post:               y = rnd(rnd(S) * out_factor)   (keeps fp16 overflow of raw sums)
 *   pre / discretized:  y = rnd(S * out_factor)        (one rounding)
 *   out_factor NULL:    y = rnd(S)
 * Rows are local (n_rows, offsets rebased to 0); cols index X's n_cols rows, so
 * a row partition runs unchanged on all-gathered features.  Heavy rows are
 * split into units with fp32 carry slots merged in slot order by a follow-up
 * pass: no atomics, bitwise deterministic.  x / y rows are ldx / ldy elements
 * apart (0 = F): a narrower F can run over wider (padded) storage, e.g. 48
 * classes in 64-wide rows whose 128-byte lines never straddle; in_scale needs
 * ldx == F.  relu != 0 applies models.relu to each output (the next layer's
 * activation fused into the aggregation's epilogue).  Edge e's weights are
 * w[idx(e) * w_ld + head] (w_ld 0 = heads).  out2 != NULL additionally writes
 * out2[r, h] = rnd(sum_e w[idx(e) * w_ld + w2_off + h]) (fp32 sum, same row
 * ownership): the GAT backward's column sums of d_e read from the same
 * interleaved (alpha, d_e) rows as the transposed aggregation's weights
 * (models.py:309-311, 335-337); needs F/8 <= 32 lanes of whole-vector heads.
 * packs / num_packs: the hg_schedule_build packs of the same CSR (NULL / 0 when
 * the schedule was built without packing), pack_rowid: int32 row id per edge
 * (needed with packs); a packed row's result is bitwise the one it gets as its
 * own unit.
 * split_counters / slot_split (both NULL: a separate follow-up launch folds
 * the split rows' carries): int32 [num_split_rows] arrival counters, all zero
 * (and left zero), and int32 [num_slots] = the split_rows index owning each
 * slot; then the last unit of each split row to finish folds its carries in
 * slot order inside the same launch (bitwise the follow-up's result).  Calls
 * sharing the counters must be stream-ordered.
 * comb_res (NULL: off; [n_rows, F] pitch comb_ldr, 16-byte aligned rows): the
 * GIN combine in the row store, y = rnd(rnd(res * ope) + rnd(h * lam)) with h
 * the finished aggregate, fp64 products (models.py:220-240 scale_combine);
 * comb_ope: device scalar of the element type (NULL: 1); with ope = NULL and
 * lam = 1 a rounded residual add (a gradient accumulated into the output).
 * Not with relu.
 * hd_gl (NULL: off) with hd_gr, hd_al, hd_ar: the GAT head-dot backward's dz
 * term in the same store (GATLayer, models.py:492-509; hg_head_dots_bwd with
 * gz_in): y[r, c] = rnd(h + rnd(rnd(hd_gl[r, c / fh] * hd_al[c]) +
 * rnd(hd_gr[r, c / fh] * hd_ar[c]))), fh = F / heads; hd_gl / hd_gr:
 * [n_rows, heads], hd_al / hd_ar: [F].  Not with comb_res, out2 or relu. */
int hg_spmm_workspace(int64_t n_cols, int32_t F, int64_t num_slots, int has_in_scale,
                      int32_t sum_heads, int dtype, size_t* bytes);
int hg_spmm(const int64_t* offsets, const int32_t* cols, int64_t n_rows, int64_t n_cols,
            int64_t num_edges, const int32_t* units, int64_t num_units,
            const int32_t* split_rows, int64_t num_split_rows, int64_t num_slots,
            const int32_t* packs, int64_t num_packs, const int32_t* pack_rowid,
            const void* w, const int32_t* w_index, int32_t heads, const void* x, void* y,
            int32_t F, int64_t ldx, int64_t ldy, int32_t scaling, int32_t relu,
            const void* in_scale, const void* out_factor, int64_t w_ld, int32_t w2_off,
            void* out2, int dtype, void* ws, size_t ws_bytes, void* stream,
            int32_t* split_counters, const int32_t* slot_split, const void* comb_res,
            int64_t comb_ldr, const void* comb_ope, double comb_lam, const void* hd_gl,
            const void* hd_gr, const void* hd_al, const void* hd_ar);

/* hg_spmm in fp32 partial mode, for column-blocked aggregation
 * (a row's edges split by the rank owning their column, block q run as soon as
 * rank q's feature rows have landed; partition.py): each row starts from
 * acc_in[r] (NULL: 0) and, with acc_out != NULL, ends unrounded in acc_out[r]
 * ([n_rows, F] fp32, 16-byte aligned, may alias acc_in); with acc_out NULL the
 * row is finished into y like hg_spmm (scaling / out_factor / relu).  Chaining
 * the blocks in ascending column order reproduces hg_spmm's fp32 sum bit for
 * bit on every row that is one unit in each block; split rows regroup their
 * carries.  Weights as hg_spmm (w / w_index / heads / w_ld; a block's
 * w_index maps its edges back to the unblocked edge order).  F: a multiple of 4. */
int hg_spmm_acc(const int64_t* offsets, const int32_t* cols, int64_t n_rows, int64_t n_cols,
                int64_t num_edges, const int32_t* units, int64_t num_units,
                const int32_t* split_rows, int64_t num_split_rows, int64_t num_slots,
                const int32_t* packs, int64_t num_packs, const int32_t* pack_rowid,
                const void* w, const int32_t* w_index, int32_t heads, int64_t w_ld,
                const void* x, void* y, int32_t F, int64_t ldx, int64_t ldy, int32_t scaling,
                int32_t relu, const void* out_factor, const float* acc_in, float* acc_out,
                int dtype, void* ws, size_t ws_bytes, void* stream);

/* Reference-order SpMM, bit-exact with halfsparse _spmm_edge_parallel
 * (kernels.py:328-391; order spelled out in _ref_spmm_edge, kernels.py:603-688):
 * warp w owns edges [w*warp_chunk, ...), CTA c owns warps [c*warps_per_cta, ...);
 * per-segment fused folds (discretized batches of k = subwarp_layout(F).subwarps),
 * adjacent-pair chain trees inside a CTA, one carry per CTA folded in CTA
 * order by a follow-up pass, then post scaling.  staging_partials
 * ([num_ctas*F], dtype) / staging_rows ([num_ctas] int64) receive the carry-out
 * slots (StagingBuffer, kernels.py:70-87); both may be NULL. */
int hg_spmm_edge_ref_workspace(int64_t n_cols, int64_t num_edges, int32_t F,
                               int32_t warp_chunk, int32_t warps_per_cta, int has_in_scale,
                               int dtype, size_t* bytes);
int hg_spmm_edge_ref(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                     int64_t n_cols, int64_t num_edges, int32_t warp_chunk,
                     int32_t warps_per_cta, const void* w, const void* x, void* y, int32_t F,
                     int32_t scaling, const void* in_scale, const void* out_factor,
                     void* staging_partials, int64_t* staging_rows, int dtype, void* ws,
                     size_t ws_bytes, void* stream);

/* Vertex-grouped SpMMv, bit-exact with spmm_vertex_grouped (kernels.py:463-559):
 * <=32-slot neighbour groups folded sequentially, discretized partial
 * rnd(acc*f_r), ascending merge, post scaling.  If staging_partials != NULL,
 * group_base[r] (int64, exclusive scan of the group counts of rows with more
 * than one group) places row r's partials at staging_partials[group_base[r]+g]. */
int hg_spmm_vertex_ref_workspace(int64_t n_cols, int32_t F, int has_in_scale, int dtype,
                                 size_t* bytes);
int hg_spmm_vertex_ref(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                       int64_t n_cols, const void* x, void* y, int32_t F, int32_t scaling,
                       const void* in_scale, const void* out_factor,
                       const int64_t* group_base, void* staging_partials,
                       int64_t* staging_rows, int dtype, void* ws, size_t ws_bytes,
                       void* stream);

/* Measurement only (no reference counterpart): the gather pattern of one SpMM
 * with the arithmetic removed -- cols[0..num_edges) streamed once and, per
 * edge, row_bytes (multiple of 16, <= 512; <= 1024 for whole 32-byte chunks)
 * of x at cols[e] * ld_bytes fetched with the k_spmm_fast team shape and lane
 * width (32-byte lanes for rows of >= 96 bytes in whole 32-byte chunks).  Its time is the floor of any gather SpMM of
 * that graph and width; bench.py reports hg_spmm against it.  *out is written
 * only on a hash collision (keeps the loads live). */
int hg_gather_probe(const int32_t* cols, int64_t num_edges, const void* x, int32_t row_bytes,
                    int64_t ld_bytes, uint32_t* out, void* stream);

/* --------------------------------------------------------------- SDDMM & GAT */

/* sddmm (kernels.py:407-455), per head: out[e*heads+h] = tree-dot of
 * X[row(e), h*fh:(h+1)*fh] and Y[cols[e], ...], fh = F/heads: products rounded
 * one by one, adjacent pairs summed, adjacent-pair tree with pass-through.
 * Bit-exact.  Uses the hg_schedule_build units (slots ignored). */
int hg_sddmm(const int64_t* offsets, const int32_t* cols, int64_t n_rows, int64_t num_edges,
             const int32_t* units, int64_t num_units, const void* x, const void* y,
             void* out, int32_t F, int32_t heads, int dtype, void* stream);

/* attention_scores + leaky_relu (models.py:317-326, 188-200), per head:
 * e = rnd(s_l[row] + s_r[col]); out = e > 0 ? e : rnd(e * slope) (slope in fp64). */
int hg_attn_scores(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                   int64_t num_edges, const void* s_l, const void* s_r, int32_t heads,
                   double slope, void* out, int dtype, void* stream);

/* Rows longer than long_thresh (listed in long_rows, n_long of them; pass
 * n_long = 0 to disable) are processed by one 1024-thread CTA each, with the
 * identical reduction tree, so power-law hubs do not serialise on one warp. */

/* edge_softmax forward (models.py:382-402): per row and head, m = max,
 * s = rnd(e-m), ex = rnd(exp(s)), den = adjacent-pair tree of ex in CSR order,
 * alpha = rnd(ex/den).  Bit-exact. */
int hg_edge_softmax_fwd(const int64_t* offsets, int64_t n_rows, int64_t num_edges,
                        const void* e, void* alpha, int32_t heads, const int32_t* long_rows,
                        int64_t n_long, int64_t long_thresh, int dtype, void* stream);
/* edge_softmax backward (models.py:403-410): prod = rnd(alpha*g),
 * s = tree-sum(prod), de = rnd(alpha*rnd(g - s)).  Bit-exact. */
int hg_edge_softmax_bwd(const int64_t* offsets, int64_t n_rows, int64_t num_edges,
                        const void* alpha, const void* grad, void* de, int32_t heads,
                        const int32_t* long_rows, int64_t n_long, int64_t long_thresh,
                        int dtype, void* stream);

/* Row sums of per-edge values (attention_scores backward, models.py:329-337),
 * fp32 accumulation, one rounding: out[r*heads+h] = rnd(sum_e v[idx(e)*heads+h]),
 * idx(e) = perm ? perm[e] : e (perm turns a CSC walk into column sums). */
int hg_edge_rowsum(const int64_t* offsets, int64_t n_rows, int64_t num_edges,
                   const void* vals, const int32_t* perm, int32_t heads, void* out,
                   const int32_t* long_rows, int64_t n_long, int64_t long_thresh, int dtype,
                   void* stream);

/* ------------------------------------------------------------------- loss */

/* convert(logits, "float32") + cross_entropy forward + backward + convert's
 * backward in one pass (models.py:203-217, 552-572), fp64 math: per row i,
 * z = logits[i, :c_active] - max (logits widened exactly from logits_dtype),
 * nll[i] = log(sum exp z) - z[label], and
 * grad[i, j] = rnd_g(fp32((softmax(z)_j - [j == label]) / denom) * grad_scale)
 * for j < c_active, 0 for c_active <= j < ld (storage padding); rnd_g rounds to
 * grad_dtype (fp16 = convert's backward).  grad_scale: 1, or a power of two (a
 * static loss scale, exact).  Loss = sum(nll) / denom. */
int hg_softmax_xent(const void* logits, int logits_dtype, int64_t ld, const int64_t* labels,
                    int64_t n, int32_t c_active, double denom, float grad_scale, void* grad,
                    int grad_dtype, double* nll, void* stream);

/* fp32-guarded SDDMM (numerics="fast"): out[e*heads+h] = rnd(sum over the head's
 * fh features of X[row(e)] * Y[cols[e]]), exact f16 products accumulated in
 * fp32, one rounding; arguments as hg_sddmm plus optional packs (the
 * hg_schedule_build packs of the same CSR, with pack_rowid = int32 row id per
 * edge; NULL / 0 / NULL for none).  Packed rows give bitwise the unit result.
 * Packs need a butterfly layout (F / V <= 32, power-of-two head widths in
 * V-element vectors); other layouts fall back to the exact kernel and reject
 * packs. */
int hg_sddmm_fast(const int64_t* offsets, const int32_t* cols, int64_t n_rows, int64_t num_edges,
                  const int32_t* units, int64_t num_units, const int32_t* packs,
                  int64_t num_packs, const int32_t* pack_rowid, const void* x, const void* y,
                  void* out, int32_t F, int32_t heads, int dtype, void* stream);

/* GAT attention projections (models.py:503-506, s_l = z a_l, s_r = z a_r) for all
 * heads at once: s_l[n*H+h] = rnd(sum_f z[n, h*fh+f] * a_l[h*fh+f]) (fp32
 * accumulation of exact products, one rounding), same for s_r. */
int hg_head_dots(const void* z, const void* a_l, const void* a_r, int64_t n, int32_t heads,
                 int32_t fh, void* s_l, void* s_r, int dtype, void* stream);
/* Its backward (the N x 1 by 1 x F matmul gradients of models.py:151-155):
 * gz[n, h*fh+f] = rnd(rnd(g_l[n,h] a_l[h,f]) + rnd(g_r[n,h] a_r[h,f])) and
 * ga_{l,r}[h, f] = rnd(sum_n z[n, h*fh+f] g_{l,r}[n, h]) with a deterministic
 * two-pass fp32 reduction (workspace: hg_head_dots_bwd_workspace).  With gz_in
 * (may alias gz) the result is accumulated: gz = rnd(gz_in + that value) -- the
 * two gradient contributions z receives in a GAT layer, summed in one pass.
 * gz NULL: only ga_l / ga_r (the dz term already folded into the transposed
 * aggregation's store, hg_spmm hd_gl). */
int hg_head_dots_bwd_workspace(int32_t heads, int32_t fh, size_t* bytes);
int hg_head_dots_bwd(const void* z, const void* a_l, const void* a_r, const void* g_l,
                     const void* g_r, int64_t n, int32_t heads, int32_t fh, void* gz,
                     void* ga_l, void* ga_r, const void* gz_in, int dtype, void* ws,
                     size_t ws_bytes, void* stream);

/* models.Adam step (models.py:583-592) over flat fp32 arrays, the reference's
 * operation order with one fp32 rounding per op:
 *   m += omb1*(g-m); v += omb2*(g*g-v); p -= lr*(m/c1) / (sqrt(v/c2) + eps),
 *   c1 = fp32(1 - b1^t), c2 = fp32(1 - b2^t) with t = *step (device fp64).
 * omb1/omb2 are fp32(1 - b1) / fp32(1 - b2) formed in double by the caller.
 * g is read from `grad` (dtype), widened and multiplied by grad_unscale (1 for
 * the reference; 2^-k undoes a static power-of-two loss scale exactly).
 * pub_out (may be NULL): the next step's published copy, rnd(p) in pub_dtype
 * (Param.publish, models.py:418-433); grad_zero (may be NULL): a pub_dtype
 * gradient buffer zeroed after use (the next step's accumulation target).
 * step_done (may be NULL): an int32 counter, zero, left zero; then the step
 * used is *step + 1 and is written back to *step by the kernel (the device step
 * count advances with no extra launch).  t_desc (HOST int64[4 * nt], nt <= 8,
 * needs pub_out and pub_t): {flat offset, rows K, cols N, offset in pub_t} of
 * 2-D weights whose transposed published copy [N, K] is also written. */
int hg_adam_step(float* master, float* m, float* v, const void* grad, int grad_dtype,
                 int64_t count, float lr, float omb1, float omb2, double b1, double b2,
                 float eps, double* step, float grad_unscale, void* pub_out,
                 void* grad_zero, int pub_dtype, int32_t* step_done, const int64_t* t_desc,
                 int32_t nt, void* pub_t, void* stream);

/* cross_entropy's mean (models.py:552-572): *loss_out = fp32(sum(nll) / denom),
 * fp64 sums in a fixed order (block chunks, then the block partials in block
 * order by the last block).  ws: hg_loss_mean_workspace bytes, 8-byte aligned,
 * its trailing counter zero (left zero) -- a dedicated buffer per stream. */
int hg_loss_mean_workspace(size_t* bytes);
int hg_loss_mean(const double* nll, int64_t n, double denom, float* loss_out, void* ws,
                 size_t ws_bytes, void* stream);

/* ------------------------------------------------------ dense GEMM (tcgen05) */

/* models.matmul -> add_bias -> left-norm input scaling (models.py:141-166,
 * kernels.py:358-361) as one tensor-core GEMM with a fused epilogue:
 *   out[m, n] = rnd(rnd(rnd(sum_k a[m, k] * bt[n, k]) + bias[n]) * row_scale[m]),
 * then max(out, 0) when relu != 0 (models.relu, 176-185)
 * binary16 operands, fp32 accumulation in TMEM (tcgen05.mma kind::f16, M=128
 * tiles, TMA-fed 4-stage ring), one rounding per step; bias / row_scale may be
 * NULL.  a: [m, k] pitch lda; bt: [n, k] pitch ldb (B transposed, K-major);
 * out: [m, n] pitch ldo.  n: multiple of 8 in [8, 256] (8 mod 16 runs as the
 * next multiple of 16, the padding neither read from bt nor stored); pitches
 * multiples of 8 elements; 16-byte aligned pointers.  Also the backward's
 * dx = g W^T (matmul backward, models.py:151-153): a = g, bt = W. */
int hg_gemm_tc(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt, int32_t n,
               int64_t ldb, const void* bias, const void* row_scale, int32_t relu, void* out,
               int64_t ldo, void* stream);

/* The GAT projection with its head dots in one pass (GATLayer, models.py:492-509: z =
 * matmul(x, W), then s_l = matmul(z_h, a_l[h]), s_r likewise, per head):
 * out = rnd(a @ bt^T) as hg_gemm_tc (no bias / row_scale / relu), and
 * dot_out_a[m, h] = rnd(sum_f out[m, h*fh + f] * dot_a[h*fh + f]) (dot_out_b
 * from dot_b) -- exact products of the rounded z, fp32 sums, one rounding --
 * formed from the TMEM accumulator tile in the epilogue instead of a second
 * read of z (hg_head_dots); each epilogue thread owns whole heads, so no
 * cross-thread sum.  heads <= 8, fh = n / heads a multiple of 16, heads even
 * unless fh == 16;
 * dot_a / dot_b: [heads * fh] binary16; dot_out_*: [m, heads]. */
int hg_gemm_tc_dots(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt, int32_t n,
                    int64_t ldb, void* out, int64_t ldo, const void* dot_a, const void* dot_b,
                    int32_t heads, void* dot_out_a, void* dot_out_b, void* stream);

/* The ReLU backward folded into the next layer's dX GEMM (models.relu
 * backward, models.py:176-185, on matmul's dx, 151-153): out = rnd(a @ bt^T)
 * where mask > 0, else +0 (NaN mask -> 0) -- mask = the ReLU's output, [m, n]
 * binary16 pitch ldm, read one tile ahead in the epilogue.  n % 16 == 0; the
 * caller guarantees the dX is that ReLU's only gradient contribution. */
int hg_gemm_tc_masked(const void* a, int64_t m, int64_t k, int64_t lda, const void* bt, int32_t n,
                      int64_t ldb, void* out, int64_t ldo, const void* mask, int64_t ldm,
                      void* stream);

/* matmul backward's weight gradient (models.py:154-155, b._accumulate(mm(a.T,
 * g))): out[m, n] = rnd(sum_k a[k, m] b[k, n]) -- fp32 accumulation, one
 * rounding -- with accumulate != 0: out = rnd(out + that) (Tensor._accumulate,
 * models.py:107-109).  a: [k, m] pitch lda (the layer input x), b: [k, n] pitch
 * ldb (the output gradient); the contraction over the k vertices is split
 * across the SMs (tcgen05, fp32 TMEM partials), partials summed in a fixed
 * order.  bias_out (may be NULL): [n] = rnd(sum_k b[k, n]), the bias gradient
 * (add_bias backward, models.py:168-170), same accumulate rule, computed from
 * the same read of b.  m, n: multiples of 8, n <= 256; 16-byte aligned a / b. */
int hg_gemm_wgrad_workspace(int64_t k, int64_t m, int32_t n, size_t* bytes);
int hg_gemm_wgrad(const void* a, int64_t k, int64_t m, int64_t lda, const void* b, int32_t n,
                  int64_t ldb, void* out, int64_t ldo, void* bias_out, int32_t accumulate,
                  void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------- multi-GPU exchange */

/* The row-partitioned feature exchange (SURVEY 8(b) hg_allgather_features,
 * 8(e); Python: partition.Exchange over torch.distributed) for callers that
 * hold their own NCCL communicator.  libnccl.so.2 is bound at run time
 * (hg_nccl_available() = 0 when it cannot be loaded).  comm is an ncclComm_t.
 *   hg_nccl_unique_id:     128-byte ncclUniqueId (rank 0 shares it out of band)
 *   hg_nccl_comm_init:     ncclCommInitRank (the CUDA device current at the call)
 *   hg_allgather_features: x_full[s_q .. s_{q+1}) = rank q's x_local for every q
 *     (row_bytes bytes per row; splits: HOST int64[parts + 1], s_0 = 0, the
 *     nnz-balanced split points); one NCCL group of exact-count broadcasts on
 *     `stream`, no padding to the largest partition. */
int hg_nccl_available(void);
int hg_nccl_unique_id(void* id_out);
int hg_nccl_comm_init(void** comm_out, int32_t nranks, const void* id, int32_t rank);
int hg_nccl_comm_destroy(void* comm);
int hg_allgather_features(void* comm, const void* x_local, void* x_full, const int64_t* splits,
                          int32_t parts, int32_t rank, int64_t row_bytes, void* stream);

/* ----------------------------------------------------------------- ingest */

/* sparse.load_edge_list (sparse.py:143-177) on the GPU.  `text` is the file's
 * bytes in device memory.  hg_count_lines -> *n_lines_out (HOST) = number of
 * lines under Python universal newlines ('\n', '\r\n', lone '\r'); then
 * hg_parse_edges writes the edge lines' (src, dst) in file order to rows_out /
 * cols_out (capacity n_lines each) and result (HOST int64[4]) = {num_edges,
 * max id (-1 if none), first bad line (1-based, 0 if none), code}: code 2 =
 * "expected 'src dst'", 3 = "non-integer vertex id", 4 = "negative vertex id",
 * 5 = id beyond int64 (reported after every line error, like the reference's
 * np.asarray overflow).  Whitespace is ASCII (str.split on ' ', \t-\r,
 * \x1c-\x1f); fields follow int() syntax ([+-]digits, single '_' between digits). */
int hg_count_lines_workspace(int64_t nbytes, size_t* bytes);
int hg_count_lines(const void* text, int64_t nbytes, int64_t* n_lines_out, void* ws,
                   size_t ws_bytes, void* stream);
int hg_parse_edges_workspace(int64_t nbytes, int64_t n_lines, size_t* bytes);
int hg_parse_edges(const void* text, int64_t nbytes, int64_t n_lines, int64_t* rows_out,
                   int64_t* cols_out, int64_t* result, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------- fp32-guarded GAT ("fast" numerics) */

/* Row classes for the row-owned fast kernels: rows with <= short_max edges run
 * one thread per (row, head); medium_rows (int32 ids, short_max < deg <=
 * long threshold) one warp per row; long_rows one 256-thread CTA per row.
 * Every row must fall in exactly one class.  heads: power of two <= 16. */

/* attention_scores + leaky_relu + edge_softmax (models.py:188-200, 317-326,
 * 382-401) in one pass: alpha[e, h] = rnd(exp(l_e - m) / sum exp(l - m)) with
 * l_e = leaky(s_l[r, h] + s_r[c, h]) in fp32 (slope), fp32 online max/sum.
 * alpha rows are alpha_ld elements apart (0 = heads; 2*heads for interleaved
 * (alpha | d_e) rows that the fused transposed aggregation reads). */
int hg_gat_attention_fwd(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                         const void* s_l, const void* s_r, int32_t heads, float slope,
                         void* alpha, int64_t alpha_ld, const int32_t* medium_rows,
                         int64_t n_medium, const int32_t* long_rows, int64_t n_long,
                         int32_t short_max, int dtype, void* stream);

/* The first pass of hg_gat_attention_fwd alone: stats[(r, h)] = (m, 1/s), the
 * log2-domain row max and reciprocal exp-sum of leaky(s_l[r] + s_r[c]) (float
 * pairs, 8-byte aligned, [n_rows, heads]) -- what hg_gat_aggregate needs to
 * form alpha = rnd(exp2(l - m) * (1/s)) bit for bit as hg_gat_attention_fwd. */
int hg_gat_attention_stats(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                           const void* s_l, const void* s_r, int32_t heads, float slope,
                           float* stats, const int32_t* medium_rows, int64_t n_medium,
                           const int32_t* long_rows, int64_t n_long, int32_t short_max,
                           int dtype, void* stream);

/* Fused GAT layer core, forward (attention_scores -> leaky_relu -> edge_softmax
 * -> spmm_weighted, models.py:317-412 + 293-314, in one row-owned pass over
 * the hg_spmm schedule): y[r] = sum_e alpha_e * x[c_e] per head (fp32,
 * [relu]), alpha_e computed in the gather loop from s_l[r], s_r[c_e] and
 * stats (hg_gat_attention_stats) and written to alpha_out [E, heads] for the
 * backward.  Bit-identical to hg_gat_attention_fwd + hg_spmm(w = alpha) on
 * the same schedule; no E x heads array is read.  Workspace: as hg_spmm with
 * in_scale = 0 and no second values. */
int hg_gat_aggregate(const int64_t* offsets, const int32_t* cols, int64_t n_rows, int64_t n_cols,
                     int64_t num_edges, const int32_t* units, int64_t num_units,
                     const int32_t* split_rows, int64_t num_split_rows, int64_t num_slots,
                     const int32_t* packs, int64_t num_packs, const int32_t* pack_rowid,
                     const void* s_l, const void* s_r, const float* stats, float slope,
                     void* alpha_out, int32_t heads, const void* x, void* y, int32_t F,
                     int64_t ldx, int64_t ldy, int32_t relu, int dtype, void* ws,
                     size_t ws_bytes, void* stream);

/* Backward of the above (models.py:188-200, 329-333, 403-410): per row,
 * D = sum alpha*dalpha (fp32); de[e, h] = rnd(alpha (dalpha - D) * leaky'(l_e));
 * ds_l[r, h] = rnd(sum_e of the unrounded de).  alpha and de rows are ae_ld
 * elements apart (0 = heads), dalpha is dense.  The column sums (ds_r) follow
 * with hg_edge_sums_fast over the CSC and perm, or inside hg_spmm (out2). */
int hg_gat_attention_bwd(const int64_t* offsets, const int32_t* cols, int64_t n_rows,
                         const void* s_l, const void* s_r, int32_t heads, float slope,
                         const void* alpha, const void* dalpha, void* de, int64_t ae_ld,
                         void* ds_l, const int32_t* medium_rows, int64_t n_medium,
                         const int32_t* long_rows, int64_t n_long, int32_t short_max,
                         int dtype, void* stream);

/* out[r, h] = rnd(sum_{e in row r} vals[(perm ? perm[e] : e), h]) with fp32
 * accumulation (row / column sums of per-edge values, models.py:329-337). */
int hg_edge_sums_fast(const int64_t* offsets, int64_t n_rows, const void* vals,
                      const int32_t* perm, int32_t heads, void* out,
                      const int32_t* medium_rows, int64_t n_medium, const int32_t* long_rows,
                      int64_t n_long, int32_t short_max, int dtype, void* stream);

/* Mean over concatenated heads: out[n, f] = rnd(sum_h y[n, h*f + f'] / heads) in
 * fp64 (exact sum); backward gin[n, h*f + f'] = rnd(g[n, f'] / heads). */
int hg_head_mean(const void* y, int64_t n, int32_t heads, int32_t f, void* out, int dtype,
                 void* stream);
int hg_head_mean_bwd(const void* g, int64_t n, int32_t heads, int32_t f, void* gin, int dtype,
                     void* stream);

/* ---------------------------------------------------------------- elementwise */

/* out = rnd(x * s) with the product formed in fp64 (the reference multiplies
 * fp16/fp32 values by Python floats in float64: leaky_relu slope,
 * scale_combine lam, models.py:188-240). */
int hg_scale_f64(const void* x, double s, void* out, int64_t count, int dtype, void* stream);

/* models.add_bias (models.py:161-166) fused with the SpMM's left-norm input
 * scaling (kernels.py:358-361): out[r, f] = rnd(rnd(x[r, f] + bias[f]) * row_scale[r]).
 * bias and row_scale may each be NULL (step skipped).  x, out: [rows, F]. */
int hg_bias_scale_rows(const void* x, const void* bias, const void* row_scale, int64_t rows,
                       int32_t F, void* out, int dtype, void* stream);

/* GIN combine, scale_combine (models.py:220-240):
 *   out = rnd(rnd(x * one_plus_eps) + rnd(a * lam)) (products in fp64);
 * backward: gx = rnd(g * one_plus_eps), ga = rnd(g * lam), and
 * gope = rnd(sum x * g) with an fp64, fixed-order sum.  gx / ga / gope may be
 * NULL (not needed); one_plus_eps / gope are device scalars. */
int hg_scale_combine(const void* x, const void* a, const void* one_plus_eps, double lam,
                     int64_t count, void* out, int dtype, void* stream);
int hg_scale_combine_bwd_workspace(size_t* bytes);
int hg_scale_combine_bwd(const void* x, const void* g, const void* one_plus_eps, double lam,
                         int64_t count, void* gx, void* ga, void* gope, int dtype, void* ws,
                         size_t ws_bytes, void* stream);

/* dst[i, :] = src[idx[i], :] for rows of row_bytes bytes (e.g. per-edge values
 * [E, H] re-ordered into CSC order through perm, w[perm] of models.py:309). */
int hg_gather_rows(const void* src, const int32_t* idx, int64_t rows, int32_t row_bytes,
                   void* dst, void* stream);

/* relu backward (models.py:176-185) from the ReLU output y: out = y > 0 ? g : 0. */
int hg_relu_grad(const void* y, const void* g, int64_t count, void* out, int dtype, void* stream);

/* add_bias backward (models.py:168-170): out[f] = rnd(sum_r x[r, f]), fp32
 * accumulation in a fixed (deterministic) order. */
int hg_col_sums_workspace(int64_t rows, int32_t F, size_t* bytes);
int hg_col_sums(const void* x, int64_t rows, int32_t F, void* out, int dtype, void* ws,
                size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HALFGNN_H */
