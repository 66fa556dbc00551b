/* knnjoin.h -- C ABI of libknnjoin.so, the B200 (sm_100a) hot path of the sparse KNN join of
 * Wang et al., "Efficient K-Nearest Neighbor Join Algorithms for High Dimensional Sparse Data"
 * (arxiv 1011.2807; /root/reference/PAPER.md).  SURVEY.md §8(b) is the contract.
 *
 * Operation (§3): for every sparse r in R return the k vectors s of S with the largest
 * dot(r, s) = sum_i r[i]*s[i] (Eq. 1), ties broken toward the LOWER S id, zero scores never
 * returned, rows with fewer than k positive scores padded with (id -1, score 0).  Scores are accumulated
 * through the inverted lists I_d of S (Alg. 3), built here as an S-tiled,
 * feature-major CSC ("tiled inverted index").
 *
 * Conventions for every entry point
 *  - Every data pointer is a CUDA DEVICE pointer unless stated otherwise; every call is stream-ordered on
 *    `stream` (a cudaStream_t passed as void*; NULL = legacy default stream) and returns without
 *    synchronising, except knnjoin_validate_csr, which synchronises.
 *  - The library allocates no device memory: the caller owns inputs, outputs, index storage and
 *    workspaces, sized by the *_bytes queries (host-only computations, no device access).
 *  - No exception or abort crosses the ABI.  Failures return a knnjoin_status; knnjoin_last_error()
 *    returns a thread-local message for the last failing call on the calling thread.
 *  - Sparse vectors are CSR rows of (feature d, weight w) pairs, features 0-based (PAPER.md:51 uses
 *    1..D; reading c5) and strictly ascending, weights w > 0.  Structural validity
 *    is checked only by knnjoin_validate_csr, never on the hot path; on the hot path R features >= d are
 *    ignored (S has no such nonzero, so they add 0 to Eq. 1) and nothing is read out of bounds.
 */
#ifndef KNNJOIN_H
#define KNNJOIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KNNJOIN_OK = 0,
  KNNJOIN_ERR_ARG = 1,          /* null pointer, k out of range, bad option, negative size */
  KNNJOIN_ERR_DIM = 2,          /* dimensionality mismatch / d <= 0 */
  KNNJOIN_ERR_CSR = 3,          /* knnjoin_validate_csr found a structurally invalid row */
  KNNJOIN_ERR_UNSUPPORTED = 4,  /* dtype combination or size outside the supported range */
  KNNJOIN_ERR_WORKSPACE = 5,    /* storage / workspace smaller than the matching *_bytes query */
  KNNJOIN_ERR_CUDA = 6          /* a CUDA runtime call failed; message carries cudaGetErrorString */
} knnjoin_status;

typedef enum {
  KNNJOIN_BINARY = 0,  /* no values array: every stored feature has weight 1 */
  KNNJOIN_INT8 = 1,    /* int8_t values, 1..127 */
  KNNJOIN_FP32 = 2     /* float values, finite and > 0 */
} knnjoin_dtype;

/* A CSR matrix.  indptr: int64[n_rows+1], indptr[0] == 0, indptr[n_rows] == nnz, non-decreasing.
 * indices: int32[nnz], strictly ascending within each row.  values: NULL for BINARY, int8_t[nnz] or
 * float[nnz] otherwise.  All three are device pointers. */
typedef struct {
  int64_t n_rows;
  int64_t nnz;
  const int64_t* indptr;
  const int32_t* indices;
  const void* values;
  knnjoin_dtype dtype;
} knnjoin_csr;

/* Build options.  tile: S ids per tile (the S-block of Alg. 1 mapped to a shared-memory score array);
 * 0 = default 8192; must be a multiple of 2048 and <= 14336 (posting ids are stored as 16-bit byte offsets of
 * their score column, 4 * local id).
 * prune / alpha: prune = 1 builds the index for the threshold-pruned query mode (the
 *   r-side form of IIIB's threshold refinement, PAPER.md:161-173 and Alg. 4): the storage
 *   additionally keeps S's forward rows (indptr, features, int8 weights) and, for INT8 S, the largest weight
 *   of every feature, and head features are off.  alpha in (0, 1] is the default pruning aggressiveness of
 *   queries on this index (0 = 0.25).  A pruned query, per row r and S tile, orders r's features by
 *   c_d = q_r[d] * maxweight(d) (descending, ties by feature), takes as non-essential the longest suffix N
 *   with sum_{d in N} c_d <= min(alpha * theta, theta - 1) (theta = the score of r's running k-th key),
 *   skips the tile's posting slices of N, and completes exactly -- from the forward row of s against N --
 *   every s whose partial score plus sum_{d in N, slice non-empty} c_d reaches theta.  An s that the
 *   skipped slices alone could reach has score < theta and cannot enter.  Results are identical to the
 *   unpruned query; only the work changes.  prune = 0: alpha must be 0.
 * forward: NULL, or (prune = 1) a CSR with S's row count whose rows are kept as the forward rows instead of
 *   S's own (f1, IIIB-literal: the residual rows s' of knnjoin_iiib_split, completed by residual queries).
 * head_density / head_max: "head features" (BINARY S only).  Up to head_max (0 = 32, at most 32) of the
 *   most frequent features with df >= head_density * |S| (0 = default 1/8, negative = no head features) are
 *   not stored as id lists: each S row gets one 32-bit word of head-feature bits.  During the top-k scan the
 *   query bounds their contribution to a score by the sum of the row's largest head weights (popcount of
 *   the shared head bits) and adds it exactly, from per-batch 16-entry lookup tables, only where that bound
 *   can beat the running k-th score (the threshold refinement of IIIB, applied to the
 *   head features).  Results are identical; only the work changes. */
typedef struct {
  int32_t tile;
  int32_t prune;
  float alpha;
  float head_density;
  int32_t head_max;
  const knnjoin_csr* forward;
} knnjoin_options;

/* Query options (all optional; pass NULL for defaults).
 *  batch_rows: R rows per CTA batch (0 = auto).
 *  cta_warps:  warps per CTA of the accumulation kernel, 4, 8 or 16.  Auto (batch_rows and cta_warps both
 *              0): an index without head features gets 4-warp one-row CTAs, six per SM; one with head features
 *              gets 8-warp CTAs, three (or two) per SM, with the largest batch whose score arrays fit.  The head
 *              count is known on the device only, so for a BINARY-S index with head features enabled both
 *              candidate shapes are launched and each returns at entry unless it matches the count: the call
 *              never synchronises and is always capturable in a CUDA graph.
 *  tiles_per_pass: S tiles swept by all batches before any batch moves on (0 = auto: about a third of the
 *              L2 cache worth of index per pass; the whole index when it fits).  Top-k state is carried
 *              between passes in the workspace; results do not depend on it.  Auto also splits the tiles
 *              into independent groups when R has fewer batches than two waves of resident CTAs (small R,
 *              serving): each group's lists are merged by rank after the kernel (K4), same result.
 *  Graph capture: knnjoin_query issues only stream-ordered work and may be captured into a CUDA graph.
 *  counters:   NULL, or a device int64_t[4] that the query ADDS into: [0] postings visited (Eq. 4 second
 *              term; head postings are counted whether or not their completion is skipped),
 *              [1] candidate inserts into the top-k lists, [2] head postings whose exact addition was skipped
 *              because the score bound could not reach the running k-th score, [3] exact head completions
 *              ((row, S row) pairs).
 *  ev_begin / ev_end: NULL, or cudaEvent_t (as void*) recorded on `stream` immediately before and after
 *              the score-accumulation + top-k kernel, so callers can time that kernel alone.
 *  phase_cycles: NULL, or a device int64_t[8] that the query ADDS SM clock cycles into, summed over CTAs
 *              (thread 0 of each CTA): [0] staging, [1] sparse atomics, [2] (unused), [3] scan + top-k,
 *              [4] list merge + output, [5] batch fetch / setup + head tables.  Profiling aid; off when NULL.
 *  row_order:  0 (default) = rows are batched in descending order of their work estimate
 *              w_r = sum_{d in r} |I_d| (the row's share of Eq. 4's second term),
 *              so the heaviest batches are handed out first; 1 = input order.  Outputs are always in input
 *              row order and identical either way.
 *  tile_begin / tile_end: restrict the query to the S tiles [tile_begin, tile_end) of the index (S ids
 *              [tile_begin*tile, tile_end*tile)); 0 / 0 = every tile.  Out of range -> KNNJOIN_ERR_ARG.
 *  resume_keys: NULL, or a device uint64_t[n_rows*k] of ordering keys (the out_keys of an earlier query of the
 *              same R and k over DISJOINT S ids -- other tiles of this index, or another index with a disjoint
 *              s_id_base range; input row order): the query continues those lists, so two queries over [0, a)
 *              and [a, n_tiles) give the one-query result, and S blocks streamed from host memory one index at
 *              a time give the one-index result (f4, Alg. 1's block nested loop).
 *  theta_in:   NULL, or a device uint64_t[n_rows] of per-row key floors (input row order): candidates of this
 *              query's tiles with key < theta_in[r] are not kept (0 = no floor).  S-sharded multi-GPU (f2,
 *              SURVEY.md §8(f)): the k-th key a row reached on ANY shard bounds the global k-th key from
 *              below, so a shard may drop its candidates below the maximum over shards -- the merged result
 *              is unchanged, and the floor tightens the pruning of head-feature completions (the threshold
 *              carried from previous computation).  Keys equal to the floor are kept.
 *  prune_alpha: threshold pruning on an index built with prune = 1 (see knnjoin_options): 0 = the index's
 *              alpha, in (0, 1] = this alpha, < 0 = off.  On an index built without prune it must be 0 or
 *              negative.  Pruned queries run the one-row 4-warp shape (batch_rows / cta_warps must be 0 or
 *              1 / 4).  counters [2] then counts the 16-byte posting units (8 postings, padding included) whose
 *              loads were skipped, and [3] the exact completions ((row, S row) pairs).
 *  residual:   1 = f1 (IIIB-literal, Alg. 4 lines 15-24): the index holds only the indexed
 *              parts s'' of its S rows and its forward rows are the residual parts s' (knnjoin_iiib_split):
 *              every s with a non-zero partial score is completed with dot(r, s') (line 21) before the
 *              candidate test.  Needs an index built with prune = 1; not combinable with prune_alpha > 0.
 *              counters [3] counts the completions.
 *  precision:  score arithmetic.  0 (auto, default): FP32-R queries accumulate in 32-bit per-row
 *              fixed point; every row's final list is then certified -- with E_r = smax * sum_d |q_d - r_d sigma_r|
 *              the bound on any pair's absolute error and y_min the smallest positive score of the list, the list
 *              meets the tolerance rule of DESIGN.md reading c15 when E_r (2 + tol) <= (tol - 2^-23) y_min -- and
 *              the rows that fail are recomputed at 64-bit fixed point (wide.cu), which holds the rule at any
 *              dynamic range of practical inputs (weights spanning many decades).  Auto skips the
 *              recomputation in a partial query (tile range, resume_keys, theta_in, or a residual query): the
 *              caller certifies the complete lists with knnjoin_certify.  A query whose keys a later query resumes
 *              must use precision 1, so that every resumed list keeps the 32-bit key encoding.  1: 32-bit only (with `uncertified`, the failing rows are
 *              reported, not recomputed).  2: 64-bit for every row.  Integer R with integer S is exact at 32 bits
 *              (precision is ignored); FP32 S always runs at 64 bits (1 -> KNNJOIN_ERR_UNSUPPORTED).
 *              KEY ENCODING: 32-bit results key the fixed-point score (score field = the row's fixed-point sum,
 *              decoded with the row's scale); 64-bit results key the fp32 score itself (score field = fp32 bits of
 *              the score; candidates within fp32 rounding tie and go to the lower id).  Rows recomputed by auto
 *              mode therefore carry fp32-keyed out_keys; they are the rows listed in `uncertified`.
 *  row_list / row_count: 64-bit queries only: NULL, or device int32 rows of R to process (input row numbers) and
 *              a device int32 count; other rows' outputs are left untouched.
 *  uncertified: NULL, or device int32[1 + R.n_rows]: [0] = number of rows whose 32-bit list fails the
 *              certification (auto: the rows recomputed at 64 bits), followed by those rows in no particular order.
 *              Written by every query (count 0 when nothing was certified: integer inputs, 64-bit queries).
 *  tolerance:  relative tolerance of the certification (0 = 1e-5, BASELINE.json north_star). */
typedef struct {
  int32_t batch_rows;
  int64_t* counters;
  void* ev_begin;
  void* ev_end;
  int64_t* phase_cycles;
  int32_t cta_warps;
  int32_t tiles_per_pass;
  int32_t row_order;
  int64_t tile_begin;
  int64_t tile_end;
  const uint64_t* resume_keys;
  const uint64_t* theta_in;
  float prune_alpha;
  int32_t residual;
  int32_t precision;
  const int32_t* row_list;
  const int32_t* row_count;
  int32_t* uncertified;
  float tolerance;
} knnjoin_query_options;

typedef struct knnjoin_index knnjoin_index; /* opaque HOST handle; borrows the caller's index storage */

typedef struct {
  int64_t n_s;          /* rows of S indexed */
  int64_t s_id_base;    /* global id of S row 0 (S-sharded multi-GPU: the shard's first id) */
  int32_t d;            /* dimensionality */
  int32_t tile;         /* S ids per tile */
  int64_t n_tiles;      /* ceil(n_s / tile) */
  int64_t offsets;      /* entries of the offset table: d*(n_tiles+1)+1 */
  int64_t unit_capacity;/* 16-byte posting units reserved in the storage (upper bound) */
  int64_t storage_bytes;/* bytes of index storage the handle uses */
  knnjoin_dtype s_dtype;
  int64_t head_min_df;  /* df from which a feature may be a head feature (-1: head features off) */
  int32_t head_max;     /* cap on the number of head features (their count is known on the device only) */
  int32_t prune;        /* 1: built for pruned queries (forward rows kept) */
  float alpha;          /* default pruning alpha of queries on this index (prune = 1) */
} knnjoin_index_info;

/* ---- index build: Create_Inverted_List_IIB (Alg. 3 lines 5-8) on the device ------ */

/* Bytes of device storage the index of S needs (an upper bound computed on the host from n_rows, nnz, d
 * and the tile width).  Returns 0 and sets knnjoin_last_error on invalid arguments. */
size_t knnjoin_index_bytes(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt);

/* Bytes of device scratch knnjoin_build_index needs (sort buffers and scan temporaries). */
size_t knnjoin_build_workspace_bytes(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt);

/* Build the tiled inverted index of S (BINARY, INT8 or FP32 weights) into `index_storage` (>= knnjoin_index_bytes bytes, 256-byte
 * aligned) using `workspace` (>= knnjoin_build_workspace_bytes bytes).  Layout:
 * for tile t (S ids [t*tile, (t+1)*tile)) and feature f, the postings of I_f restricted to the tile are a
 * contiguous, 16-byte aligned slice of local ids stored as byte offsets 4 * (s - tile base) (+ uint8 / fp32 values
 * for INT8 / FP32 S), padded with dummy ids 4 * (tile + (0..31)); inside each full 256-posting block postings are ordered by shared-memory bank, the last
 * partial block is transposed so a warp's lanes touch consecutive ids; head features (see head_density)
 * are stored as one 32-bit word per S row instead of id lists.
 * s_id_base: global id of S row 0 (ids returned by queries are s_id_base + local row).
 * S may be freed after the call's work completes on `stream`; the storage must outlive every query.
 * FP32 S stores its weights as fp32 (6 bytes per posting) and is queried at 64-bit fixed point (precision);
 * prune = 1 needs BINARY or INT8 S.  *out receives a host handle to release with knnjoin_free_index. */
knnjoin_status knnjoin_build_index(const knnjoin_csr* S, int32_t d, int64_t s_id_base, const knnjoin_options* opt,
                                   void* index_storage, size_t storage_bytes, void* workspace, size_t workspace_bytes,
                                   void* stream, knnjoin_index** out);

knnjoin_status knnjoin_index_stats(const knnjoin_index* idx, knnjoin_index_info* out); /* host only */
void knnjoin_free_index(knnjoin_index* idx); /* frees the HOST handle only; storage stays the caller's */

/* ---- query: Find_Matches_IIB (Alg. 3 lines 9-17) for every r, fused with top-k ---- */

/* Bytes of device scratch knnjoin_query needs for R and k. */
size_t knnjoin_query_workspace_bytes(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k,
                                     const knnjoin_query_options* qopt);

/* For every row r of R (1 <= k <= 256) write, in rank order (score desc, id asc):
 *   out_ids[r*k + i]    int32  global S id, or -1 for padding;
 *   out_scores[r*k + i] float  dot(r, s): exact for BINARY/INT8 R and S; otherwise the fixed-point sum / scale,
 *                              within the certified tolerance (see precision);
 *   out_keys[r*k + i]   uint64 (optional, may be NULL) the packed ordering key
 *                              (score_u32 << 32) | (0xFFFFFFFF - global_id), 0 for padding, as consumed by
 *                              knnjoin_merge (S-sharded multi-GPU); score_u32 per `precision`'s key encoding.
 * out_ids / out_scores may be NULL when out_keys is given.  R dtype: BINARY, INT8 or FP32.
 * Integer (BINARY/INT8 x BINARY/INT8) scores must fit in 32 bits: d * 127 * 127 < 2^32, else UNSUPPORTED.
 * Empty R: nothing is written.  Empty S: every row is padding. */
knnjoin_status knnjoin_query(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k,
                             const knnjoin_query_options* qopt, uint64_t* out_keys, int32_t* out_ids,
                             float* out_scores, void* workspace, size_t workspace_bytes, void* stream);

/* ---- S-sharded merge: P partial top-k lists per row -> global top-k ---------------- */

size_t knnjoin_merge_workspace_bytes(const knnjoin_csr* R);

/* Merge options (NULL = defaults).  float_keys: 1 = the keys carry fp32 scores (64-bit queries; implied for FP32
 * S), 0 = 32-bit fixed-point scores decoded with R's per-row scale.  row_list / row_count: NULL, or device int32
 * rows and a device count: only the listed rows are merged and written (the 64-bit re-run of uncertified rows in
 * a sharded join); their lists sit at their own row positions of the [P][n_rows][k] slabs. */
typedef struct {
  int32_t float_keys;
  const int32_t* row_list;
  const int32_t* row_count;
} knnjoin_merge_options;

/* keys: uint64[P][n_rows][k] (each [n_rows][k] slab is one shard's out_keys, e.g. gathered by an NCCL
 * all-gather): every row of every slab sorted descending with its 0 padding last, and the P slabs from
 * disjoint S id ranges (distinct keys), as knnjoin_query writes them.  Each merged key is placed by rank
 * (its position plus the larger keys of the other slabs, binary searches).  Writes the global top-k per row into out_keys / out_ids / out_scores (any may be NULL
 * but not all), using R, d (the index dimensionality) and s_dtype (the dtype of S) only to recover the
 * per-row score scale, exactly as knnjoin_query computed it.
 * The merge is exact: keys encode (score, lower-id-wins) as one unsigned integer. */
knnjoin_status knnjoin_merge(const uint64_t* keys, int32_t P, const knnjoin_csr* R, int32_t d,
                             knnjoin_dtype s_dtype, int32_t k, const knnjoin_merge_options* mopt, uint64_t* out_keys,
                             int32_t* out_ids, float* out_scores, void* workspace, size_t workspace_bytes, void* stream);

/* ---- certification of 32-bit fixed-point lists -------------------------------------------
 * keys: uint64[n_rows][k], complete 32-bit lists of FP32 R (e.g. knnjoin_merge's output of a sharded join, or
 * the last of a chain of resumed queries), s_dtype BINARY or INT8 (the scale knnjoin_query used).  Writes to
 * out_list (device int32[1 + n_rows]) the count and the rows whose lists fail the tolerance rule (see
 * knnjoin_query_options.precision); integer R: count 0.  The caller then recomputes those rows with a 64-bit
 * query (precision 2, row_list = out_list + 1, row_count = out_list) and merges with float_keys = 1. */
size_t knnjoin_certify_workspace_bytes(const knnjoin_csr* R);
knnjoin_status knnjoin_certify(const uint64_t* keys, const knnjoin_csr* R, int32_t d, knnjoin_dtype s_dtype, int32_t k,
                               float tolerance, int32_t* out_list, void* workspace, size_t workspace_bytes, void* stream);

/* ---- f1: IIIB-literal (Alg. 4) building blocks --------------------------------------
 * The paper's improved algorithm per (R block, S block): dimensions reordered by their non-zero count in the
 * R block (descending; ties by dimension; dimensions absent from the block last), maxWeight_d = the largest
 * weight of dimension d in the R block, MinPruneScore = min over the block's rows of pruneScore(r) (the k-th
 * score so far, 0 while fewer than k are held).  Each s of the S block is walked in that order with
 * t += maxWeight_d * w; from the first feature at which t > MinPruneScore on, its features are indexed (s''),
 * the others stay in s'.  The S block is then indexed from s'' (prune = 1, forward = s') and queried with
 * residual = 1, which adds dot(r, s') to every touched s (Theorem 1: an s sharing no indexed
 * feature with r has dot(r, s) <= MinPruneScore <= pruneScore(r) and cannot enter).  R is one block here. */

/* Bytes of the device profile of R (maxWeight, dimension order, sort scratch). */
size_t knnjoin_iiib_profile_bytes(const knnjoin_csr* R, int32_t d);

/* Alg. 4 lines 6-7 over all of R: writes the profile into `profile` (device, >= knnjoin_iiib_profile_bytes). */
knnjoin_status knnjoin_iiib_profile(const knnjoin_csr* R, int32_t d, void* profile, size_t profile_bytes, void* stream);

/* MinPruneScore of R from the keys of the S blocks done so far (keys: [n_rows][k] as knnjoin_query writes them,
 * or NULL before the first block -> 0), written to out2 (device double[2]) as {min_r kth_score(r) (real
 * units), max_r 1/sigma_r}.  For FP32 R (per-row fixed-point scores) knnjoin_iiib_split lowers the threshold
 * of an s by (sum of its weights + 1) * out2[1] so that rounding can never let an unindexed-only s enter. */
knnjoin_status knnjoin_iiib_threshold(const uint64_t* keys, const knnjoin_csr* R, int32_t d, knnjoin_dtype s_dtype,
                                      int32_t k, double* out2, void* workspace, size_t workspace_bytes, void* stream);
size_t knnjoin_iiib_threshold_workspace_bytes(const knnjoin_csr* R);

/* Alg. 4 lines 8-14 on the S block: split every row of S into the indexed part (out_idx) and the residual
 * part (out_res), both CSRs with S's row count, features ascending, INT8 values carried (out_*_values NULL
 * for BINARY S); the arrays of each need room for nnz(S) entries and n_rows + 1 indptr entries.  Their nnz
 * are known on the device only (indptr[n_rows]).  threshold: device double[2] from knnjoin_iiib_threshold;
 * r_integer: 1 when R is BINARY/INT8 (exact scores: no rounding margin). */
knnjoin_status knnjoin_iiib_split(const knnjoin_csr* S, int32_t d, const void* profile, const double* threshold,
                                  int32_t r_integer, int64_t* idx_indptr, int32_t* idx_indices, int8_t* idx_values,
                                  int64_t* res_indptr, int32_t* res_indices, int8_t* res_values, void* workspace,
                                  size_t workspace_bytes, void* stream);
size_t knnjoin_iiib_split_workspace_bytes(const knnjoin_csr* S);

/* ---- validation (not on the hot path) ------------------------------------------------------------- */

/* Checks, on the device, that `m` is a valid CSR for dimensionality d: indptr[0]==0, non-decreasing,
 * indptr[n_rows]==nnz; indices strictly ascending within each row and in [0, d); values > 0 (and finite
 * for FP32).  SYNCHRONISES `stream`.  Returns KNNJOIN_OK, or KNNJOIN_ERR_CSR with *bad_row (host
 * pointer, may be NULL) set to the first offending row (-1 for a global indptr problem). */
knnjoin_status knnjoin_validate_csr(const knnjoin_csr* m, int32_t d, void* stream, int64_t* bad_row);

const char* knnjoin_last_error(void);
const char* knnjoin_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KNNJOIN_H */
