/*
 * misa_b200 — C ABI of the B200-native (sm_100a) MISA / DSA indexer.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void*), is stream-ordered (no host synchronisation inside), keeps
 * no device allocations across calls, and returns 0 on success or a negative
 * error code; misa_last_error() holds a thread-local message.  The caller owns
 * all memory (inputs, outputs, workspace).  Nothing here falls back to the CPU.
 *
 * Layouts (row-major, contiguous unless an ld is given):
 *   keys      bf16 [n_keys][D]            D = head_dim padded to 64 or 128 (zero pad is exact)
 *   queries   bf16 [n_rows][Hp][D]        Hp = n_heads padded to a power of two (>= 8)
 *   weights   f32  [n_rows][Hp]           padded heads carry weight 0
 *   prefix_len i32 [n_rows]               n_t: row t scores keys [0, n_t)
 *   heads     i32 [n_rows][hq]            routed heads, ascending, -1 padded
 *   topk      i32 [n_rows][topk_ld]       selected key indices, ascending, -1 padded
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/misa):
 *   misa_pool_keys        pooling.py:57-84   build_block_summary (+ per-token in-block prefix sums)
 *   misa_pool_append      pooling.py:87-115  incremental_append (decode)
 *   misa_route_scores     routing.py:38-64   route_head_importance, block_attention GEMM part
 *   misa_route_select     routing.py:38-75   route_head_importance epilogue + route_topk_heads
 *   misa_score_materialize dsa.py:37-61, routing.py:78-99  gated_relu_scores / dsa_score / misa_score
 *   misa_score_materialize_split  the same, key-axis split (decode)
 *   misa_score_materialize_paged  the same over a paged key cache (decode)
 *   misa_score_filter     dsa.py:37-76 fused with the candidate pass of topk_tokens
 *   misa_score_filter_split  the same over key-split items (decode)
 *   misa_select_threshold (no reference counterpart: sampled threshold for the fused top-k)
 *   misa_select_topk      dsa.py:64-76       topk_tokens over the filtered candidates
 *   misa_select_topk_runs routing.py:157-159 the coarse top-k' set of misa_hier_select (unordered runs)
 *   misa_select_dense_runs dsa.py:79-92      topk_within over those runs (re-rank selection)
 *   misa_select_dense     dsa.py:64-92       topk_tokens / topk_within over a dense score row
 *   misa_select_dense_long dsa.py:64-76      topk_tokens over long dense rows (decode), all SMs
 *   misa_refine_scores    dsa.py:95-115      dsa_rescore (MISA-dagger fine stage), routing.py:144-174
 *   misa_refine_candidates dsa.py:95-115     the same, scores packed as misa_select_topk candidate lists
 *   misa_merge_topk       (no reference counterpart: key-sharded multi-GPU merge)
 *   misa_shard_map_indices (no reference counterpart: local -> global key index of a shard)
 *   misa_list_kth / misa_list_prune (no reference counterpart: pruned key-shard exchange)
 *   misa_*_varlen         several independent key sequences / workloads in one call
 *                         (workload.py:40-110 per workload; the reference loops over them)
 *   misa_relevance_dots   dsa.py:18-34       relevance_dots (raw per-query dot products)
 *   misa_pack_rows_f64    workload.py:202-254 load_workload payload (f64) -> device bf16 layouts
 *   misa_sparse_attention (no reference counterpart: PAPER.md Eq. 3, the selection's consumer)
 *   misa_quant_rows_fp8   (no reference counterpart: FP8 upstream indexer projections)
 */
#ifndef MISA_B200_H_
#define MISA_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MISA_OK 0
#define MISA_EINVAL (-1)       /* invalid argument / shape (the reference raises ValueError) */
#define MISA_ECUDA (-2)        /* CUDA runtime / driver error */
#define MISA_EUNSUPPORTED (-3) /* shape outside the compiled kernel set */

/* router score kinds (config.py:14-17) */
#define MISA_ROUTER_BLOCK_ATTENTION 0
#define MISA_ROUTER_GATE_ONLY 1
#define MISA_ROUTER_QUERY_NORM 2

/* select flags (bit set per row in flags[]) */
#define MISA_FLAG_OVERFLOW 1  /* more candidates than capacity: row must be re-selected densely */
#define MISA_FLAG_UNDERFLOW 2 /* fewer candidates than min(k, n): threshold too high */

int misa_abi_version(void);
const char* misa_last_error(void);
int misa_sm_count(void);

/* K1: in-block inclusive prefix sums of the keys (f32 [n_keys][D]), full-block means
 * (f32 [n_keys / B][D]) and their exact hi/mid/lo bf16 split (bf16 [3][planes_rows][D],
 * rows >= n_keys / B zero-filled).  Any of the outputs may be NULL. */
int misa_pool_keys(const void* keys, int64_t n_keys, int head_dim, int block_size, float* prefix_sums,
                   float* pooled, void* pooled_planes, int64_t planes_rows, void* stream);

/* Decode: append one key row.  prefix_sums row n_keys_before is written from row
 * n_keys_before-1 (or started fresh at a block boundary); when the append closes a
 * block its mean and planes row are written. */
int misa_pool_append(const void* keys, int64_t n_keys_before, int head_dim, int block_size, float* prefix_sums,
                     float* pooled, void* pooled_planes, int64_t planes_rows, void* stream);

/* K2a: router partial sums.  partial[c][t][j] = sum over full blocks b in chunk c
 * (128 blocks per chunk, b < n_t / B) of ReLU(q_tj . pooled_b), computed on tcgen05 with
 * the pooled keys split into three bf16 planes (f32-grade); chunk 0 also adds
 * ReLU(q_tj . partial-block mean) when n_t % B != 0.  Work list: item i covers the 128
 * flattened (t, j) rows of tile it_tile[i] against block chunk it_chunk[i] with
 * it_ncols[i] (multiple of 16, <= 128; 0 = partial-block term only) pooled columns;
 * items are grouped by chunk.  Rows whose chunk c has no item are not written.
 * n_heads_pad: a power of two in [8, 128]. */
int misa_route_scores(const void* queries, int64_t n_rows, int n_heads_pad, int head_dim, const void* pooled_planes,
                      int64_t planes_rows, const float* prefix_sums, const int32_t* prefix_len, int block_size,
                      const int32_t* it_tile, const int32_t* it_chunk, const int32_t* it_ncols, int n_items,
                      float* partial, void* stream);

/* misa_route_scores over several key sequences packed with every sequence starting at a
 * pooled-block boundary: row t's pooled blocks start at block row_boff[t] (its keys at key
 * row_boff[t] * block_size); item i serves the rows of its tile with row_boff == it_boff[i],
 * its chunk counted from that block. */
int misa_route_scores_varlen(const void* queries, int64_t n_rows, int n_heads_pad, int head_dim,
                             const void* pooled_planes, int64_t planes_rows, const float* prefix_sums,
                             const int32_t* prefix_len, int block_size, const int32_t* it_tile,
                             const int32_t* it_chunk, const int32_t* it_ncols, const int32_t* it_boff,
                             const int32_t* row_boff, int n_items, float* partial, void* stream);

/* K2b: importance E_tj = |w_tj| * sum_c partial / ceil(n_t/B) (block_attention), w_tj
 * (gate_only) or ||q_tj|| (query_norm); top-h heads (ties -> smaller head) ascending into
 * heads[t][0..h), -1 padded to heads_ld.  importance may be NULL. */
int misa_route_select(const float* partial, int n_chunks, const float* weights, const void* queries,
                      const int32_t* prefix_len, int64_t n_rows, int n_heads, int n_heads_pad, int head_dim,
                      int block_size, int h, int kind, int32_t* heads, int heads_ld, float* importance,
                      void* stream);

/* K3/K6 scoring on tcgen05.  Row t uses heads_per_query query vectors: heads[t][j]
 * (MISA, -1 = empty slot) or head j < n_heads (DSA, heads == NULL).  Key s of row t is
 * key row s*key_stride and valid for s < ceil(n_t / key_stride).  Work is given as
 * groups of 256/heads_per_query consecutive rows (items[i] = group id, item_tiles[i]
 * = number of 128-key tiles), scheduled longest first.
 * materialize: out[t*out_ld + s] = score for valid s. */
int misa_score_materialize(const void* keys, int64_t n_keys, int64_t key_stride, int head_dim,
                           const void* queries, const float* weights, int n_heads, int n_heads_pad,
                           const int32_t* heads, int heads_per_query, const int32_t* prefix_len, int64_t n_rows,
                           const int32_t* items, const int32_t* item_tiles, int n_items, float* out,
                           int64_t out_ld, void* stream);

/* materialize with a key-axis split of the work (decode: few row groups, long prefixes):
 * item i scans tiles [item_tile0[i], item_tile0[i] + item_tiles[i]) of group items[i]. */
int misa_score_materialize_split(const void* keys, int64_t n_keys, int64_t key_stride, int head_dim,
                                 const void* queries, const float* weights, int n_heads, int n_heads_pad,
                                 const int32_t* heads, int heads_per_query, const int32_t* prefix_len,
                                 int64_t n_rows, const int32_t* items, const int32_t* item_tiles,
                                 const int32_t* item_tile0, int n_items, float* out, int64_t out_ld, void* stream);

/* materialize over a paged key cache (decode): logical key s of every row lives at pool row
 * page_table[s / page_size] * page_size + s % page_size (page_size a multiple of 128). */
int misa_score_materialize_paged(const void* key_pool, int64_t n_pool_keys, int head_dim, const void* queries,
                                 const float* weights, int n_heads, int n_heads_pad, const int32_t* heads,
                                 int heads_per_query, const int32_t* prefix_len, int64_t n_rows,
                                 const int32_t* items, const int32_t* item_tiles, const int32_t* item_tile0,
                                 int n_items, const int32_t* page_table, int page_size, float* out, int64_t out_ld,
                                 void* stream);

/* filter: append (score, s) with score >= tau[t] to cand[(t*4 + w)*cap + i] (w = TMEM lane
 * quadrant of the key within its tile); cand_count[t*4 + w] = total seen (may exceed cap). */
int misa_score_filter(const void* keys, int64_t n_keys, int head_dim, const void* queries, const float* weights,
                      int n_heads, int n_heads_pad, const int32_t* heads, int heads_per_query,
                      const int32_t* prefix_len, int64_t n_rows, const int32_t* items, const int32_t* item_tiles,
                      int n_items, const float* tau, uint64_t* cand, int cap, int32_t* cand_count, void* stream);

/* Several key sequences in one call (the reference's independent workloads / prefixes,
 * workload.py:91-110, batched): work item i covers rows [item_row0[i], item_row0[i] +
 * item_nrows[i]) (<= 256/heads_per_query rows, all of one sequence) whose keys start at key
 * row item_key0[i] (for materialize: in units of key_stride rows); key indices in the
 * output stay relative to the sequence.  Otherwise as misa_score_materialize / _filter. */
int misa_score_materialize_varlen(const void* keys, int64_t n_keys, int64_t key_stride, int head_dim,
                                  const void* queries, const float* weights, int n_heads, int n_heads_pad,
                                  const int32_t* heads, int heads_per_query, const int32_t* prefix_len,
                                  int64_t n_rows, const int32_t* item_row0, const int32_t* item_nrows,
                                  const int32_t* item_key0, const int32_t* item_tiles, int n_items, float* out,
                                  int64_t out_ld, void* stream);
int misa_score_filter_varlen(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                             const float* weights, int n_heads, int n_heads_pad, const int32_t* heads,
                             int heads_per_query, const int32_t* prefix_len, int64_t n_rows,
                             const int32_t* item_row0, const int32_t* item_nrows, const int32_t* item_key0,
                             const int32_t* item_tiles, int n_items, const float* tau, uint64_t* cand, int cap,
                             int32_t* cand_count, void* stream);

/* Per-row threshold: tau[t] = j-th largest sampled score, j = ceil(beta*k*m/n), m = ceil(n/stride);
 * tau[t] = -inf when n <= append_all_len (every key is kept). */
int misa_select_threshold(const float* sample_scores, int64_t ld, const int32_t* prefix_len, int64_t n_rows,
                          int key_stride, int k, float beta, int64_t append_all_len, float* tau, void* stream);

/* Exact top-k (score desc, index asc) from filtered candidates; output ascending indices.
 * Rows with n_t <= k select [0, n_t) (without scores; when topk_scores is requested such
 * rows are selected from their candidates instead, which must then hold every key).
 * topk_scores (optional) holds the scores aligned with topk.  flags[t] gets MISA_FLAG_*
 * on overflow / underflow (row left -1).  max_prefix_len (an upper bound of prefix_len, or 0
 * when unknown) lets the merge-free chunk-ordered selector size its staging. */
int misa_select_topk(const uint64_t* cand, const int32_t* cand_count, int cap, const int32_t* prefix_len,
                     int64_t n_rows, int k, int64_t max_prefix_len, int32_t* topk, int64_t topk_ld,
                     float* topk_scores, int32_t* flags, void* stream);

/* Exact top-k over dense rows: value scores[r*ld + i] for i < row_len[r] with index
 * idx[r*idx_ld + i] (or i when idx == NULL); rows listed in rows[] (or all when NULL). */
int misa_select_dense(const float* scores, int64_t ld, const int32_t* idx, int64_t idx_ld, const int32_t* row_len,
                      const int32_t* rows, int64_t n_rows, int k, int32_t* topk, int64_t topk_ld,
                      float* topk_scores, void* stream);

/* Exact top-k over long dense rows (decode: few rows x up to millions of keys) using all
 * SMs: tau[t] from a 1/32-strided sample (j = beta*k/32), per-4096-key segment counts
 * (seg_cnt: n_rows x ceil(max_len/4096)), index-ordered compaction of scores >= tau into
 * cand_scores / cand_idx (n_rows x cap, cand_count[t] = total), the register selector on the
 * candidates, and an on-device exact re-selection of rows whose count fell outside
 * [min(k, n), cap].  Same output contract as misa_select_dense. */
int misa_select_dense_long(const float* scores, int64_t ld, const int32_t* row_len, int64_t n_rows, int k,
                           int64_t max_len, float beta, float* tau, int32_t* seg_cnt, float* cand_scores,
                           int32_t* cand_idx, int32_t* cand_count, int cap, int32_t* topk, int64_t topk_ld,
                           float* topk_scores, void* stream);

/* misa_select_topk with an unordered result (MISA-dagger's coarse candidates): the selected
 * set of each row is written as kQuadrants = 4 consecutive runs, each ascending (the selected
 * keys of quadrant list q), with their lengths in runs[t*4 + q] (16-byte aligned); padded with
 * -1 past min(k, n).  Skips the ordering passes of the ascending output.  Flags as
 * misa_select_topk (flagged rows: runs 0). */
int misa_select_topk_runs(const uint64_t* cand, const int32_t* cand_count, int cap, const int32_t* prefix_len,
                          int64_t n_rows, int k, int64_t max_prefix_len, int32_t* topk, int64_t topk_ld,
                          int32_t* runs, int32_t* flags, void* stream);

/* Ascending sort, in place, of each row's first min(k, prefix_len[t]) entries (k <= 16384):
 * the ordering step after an unordered selection. */
int misa_sort_rows(int32_t* rows, int64_t ld, const int32_t* prefix_len, int64_t n_rows, int k, void* stream);

/* misa_select_dense over rows made of 4 ascending runs (runs[t*4 + q] lengths, summing to
 * row_len[t]) with explicit indices idx: the top-k (score desc, index asc), ascending. */
int misa_select_dense_runs(const float* scores, int64_t ld, const int32_t* idx, int64_t idx_ld,
                           const int32_t* row_len, const int32_t* runs, int64_t n_rows, int k, int32_t* topk,
                           int64_t topk_ld, void* stream);

/* MISA-dagger fine stage: out[t*out_ld + i] = sum_j w_tj ReLU(q_tj . key[cand[t][i]]) over all
 * heads, for i < n_cand[t] (cand ascending, -1 padded), for the rows listed in rows[0..n_items)
 * (longest first); with row_key0 (several key sequences, else null) row t's candidate i is key
 * row_key0[t] + cand[t][i].  Gathered-key tcgen05 contraction (16-byte cp.async row gathers into the
 * 128-B-swizzled operand layout; completion on the stage mbarrier). */
int misa_refine_scores(const void* keys, int64_t n_keys, int head_dim, const void* queries, const float* weights,
                       int n_heads, int n_heads_pad, const int32_t* cand, int64_t cand_ld, const int32_t* n_cand,
                       const int32_t* rows, int n_items, int64_t n_rows, const int32_t* row_key0, float* out,
                       int64_t out_ld, void* stream);

/* Raw query.key dot products (dsa.py:18-34 relevance_dots): out[i*out_ld + j] = q_j . key[i]
 * for keys i < n_keys and query rows j < n_queries (<= 128; queries bf16 [n_queries_pad][D],
 * n_queries_pad a power of two in [8, 128], pad rows zero).  The refine kernel's tcgen05
 * contraction over contiguous key tiles, with an epilogue that stores the accumulator. */
int misa_relevance_dots(const void* keys, int64_t n_keys, int head_dim, const void* queries, int n_queries,
                        int n_queries_pad, float* out, int64_t out_ld, void* stream);

/* Archived workloads (MISAWKLD, workload.py:202-254) -> device layouts: src (n_rows, d) f64 rows
 * are rounded to bf16 into dst [.][D] (columns d..D-1 zeroed), src row r landing on row
 * dst_row0 + (r / group) * dst_group_stride + r % group; *n_inexact (optional, accumulated)
 * counts elements bf16 does not represent exactly. */
int misa_pack_rows_f64(const double* src, int64_t n_rows, int d, int64_t group, int64_t dst_group_stride, void* dst,
                       int D, int64_t dst_row0, unsigned long long* n_inexact, void* stream);

/* misa_refine_scores with the scores packed for misa_select_topk: lists[t][i] = cand[t][i] << 32 |
 * f32 bits of the score, i < n_cand[t] <= 4 * list_cap, viewed as 4 lists of list_cap slots
 * (list_count[t][q] = the filled slots of list q).  When cand holds a coarse selection whose
 * 32-key chunks are contiguous (misa_select_topk / _runs output), misa_select_topk over these
 * lists with prefix_len = the rows' prefix lengths is the re-rank's top-k (dsa.py:79-92), the
 * ascending order coming from its chunk scan. */
int misa_refine_candidates(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                           const float* weights, int n_heads, int n_heads_pad, const int32_t* cand, int64_t cand_ld,
                           const int32_t* n_cand, const int32_t* rows, int n_items, int64_t n_rows,
                           const int32_t* row_key0, uint64_t* lists, int list_cap, int32_t* list_count,
                           void* stream);

/* misa_score_filter over key-split work items (decode: a few rows against long prefixes, every
 * SM busy): item i scores rows group items[i] over key tiles [item_tile0[i], +item_tiles[i]).
 * cand_count must be zeroed: each warp reserves its 32-key chunk's slots of a (row, quadrant)
 * list with one atomicAdd, so chunks are contiguous and ascending inside a list (chunk order
 * within a list is arbitrary; misa_select_topk's ordering needs no more). */
int misa_score_filter_split(const void* keys, int64_t n_keys, int head_dim, const void* queries, const float* weights,
                            int n_heads, int n_heads_pad, const int32_t* heads, int heads_per_query,
                            const int32_t* prefix_len, int64_t n_rows, const int32_t* items,
                            const int32_t* item_tiles, const int32_t* item_tile0, int n_items, const float* tau,
                            uint64_t* cand, int cap, int32_t* cand_count, void* stream);

/* The indexer's consumer (Eq. 3, Sparse MLA in MQA mode; outside the reference):
 * out[t][h][0:dv] = sum_{s in topk[t]} softmax_s(scale * q[t][h] . kv[s]) * kv[s][0:dv], one
 * latent row per token shared by all heads.  queries bf16 [n_rows][128][dqk] (heads padded
 * to 128 rows), kv bf16 [n_keys][dqk], topk [n_rows][topk_ld] (each row's k slots: tokens
 * first, -1 after), out f32 [n_rows][n_heads][dv].  dqk 128 (dv 64/128) or 256 (dv
 * 128/256). */
int misa_sparse_attention(const void* queries, int64_t n_rows, int n_heads, int head_dim_qk, const void* kv,
                          int64_t n_keys, const int32_t* topk, int64_t topk_ld, int k, int head_dim_v, float scale,
                          float* out, void* stream);

/* Multi-GPU merge: n_parts local (score, index) top-k lists per row (parts[p][t][i], scores
 * aligned, -1 padded) -> global top-k ascending.  Same tie rule (score desc, index asc).
 * topk_scores (optional) receives the selected scores aligned with topk (-inf padded), so
 * merges can be chained when n_parts * k_in exceeds one CTA's register capacity (16384). */
int misa_merge_topk(const float* part_scores, const int32_t* part_idx, int n_parts, int64_t part_stride,
                    int64_t n_rows, int k_in, int k, int32_t* topk, int64_t topk_ld, float* topk_scores,
                    void* stream);

/* Key-shard exchange pruning (no reference counterpart).  tau[t] = the m-th
 * largest score of row t's list (scores[t][0..n_cols), -inf entries are padding), or -inf when
 * the row holds fewer than m entries.  With m_g entries per shard summing to k, the global k-th
 * score is >= min over shards of their tau: entries below it cannot be selected. */
int misa_list_kth(const float* scores, int64_t ld, int64_t n_rows, int n_cols, int m, float* tau, void* stream);

/* Order-preserving compaction of the entries with score >= tau[t] (and index >= 0) of each
 * row into out (n_rows x cap, -1 / -inf padded); count[t] = the number kept (a row with
 * count > cap was truncated and must be exchanged unpruned). */
int misa_list_prune(const float* scores, const int32_t* idx, int64_t ld, int64_t n_rows, int n_cols,
                    const float* tau, int cap, float* out_scores, int32_t* out_idx, int32_t* count, void* stream);

/* Block-cyclic key sharding: in place, local key index i of shard `shard` (of n_shards,
 * blocks of `block` keys) -> global index ((i / block) * n_shards + shard) * block + i % block;
 * -1 entries are kept. */
int misa_shard_map_indices(int32_t* idx, int64_t n, int block, int n_shards, int shard, void* stream);

/* Row-wise FP8 e4m3 quantization (the upstream indexer projections' activations / weights):
 * x (n_rows, cols) bf16 -> out (n_rows, cols) e4m3 bytes with scales[r] = amax_r / 448, so that
 * x[r][c] ~= e4m3(out[r][c]) * scales[r] (round to nearest, saturating; a zero row gets scale 1).
 * cols % 8 == 0; x 16-byte and out 8-byte aligned. */
int misa_quant_rows_fp8(const void* x, int64_t n_rows, int cols, void* out, float* scales, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MISA_B200_H_ */
