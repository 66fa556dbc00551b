// query.cu -- K2 (query prep) and the host side of K3 (score accumulation fused with per-tile top-k; the kernel
// itself is in accumulate.cuh) of the KNN join.
//
// What is computed: for every r in R, Find_Matches_IIB (Alg. 3 lines 9-17):
//   A[s] += r[d] * s[d] for every posting (s, s[d]) of I_d, for every feature (d, r[d]) of r  (a4)
//   then every s with A[s] > pruneScore(r) enters r's candidate set                          (a5)
// with S split into tiles (the S blocks of Alg. 1) and pruneScore carried across tiles.
//
// GPU mapping:
//  * k_row_scale  (a3) per-row fixed-point scale sigma_r = 2^30 / (sum_d r_d * smax) for FP32 R, 1 otherwise.
//  * k_row_work + CUB sort (a3) rows ordered by their work w_r = sum_{d in r} |I_d|, heaviest batches first.
//  * k_build_runs (a3) one CTA per batch of B rows: block radix sort of the rows' (feature, row) entries into
//    "runs" (feature f, mask of batch rows that contain f, q_b = r_b[f] quantised).  A run's posting slice
//    is loaded once and applied to every row in its mask (cross-row reuse).
//  * k_prune_prep (a6, pruned queries) per-row suffix bounds of the c-descending feature order.
//  * knnjoin_query: workspace layout, the CTA shape (pick_shape: 8-warp CTAs with B = 2 rows for indexes with
//    head features, 4-warp one-row CTAs otherwise), pass slabs sized for L2 or the small-R tile-group split,
//    and the launch of k_accumulate_topk (accumulate.cuh: per tile, stage the runs' slice bounds, accumulate
//    with shared-memory atomics over contiguous per-warp window ranges, scan + top-k per warp column strip;
//    per batch, merge the warps' lists by rank and write ids / scores / keys).
#include <cub/cub.cuh>

#include "accumulate.cuh"

namespace kj {
namespace {


// ------------------------------------------------------------------------------------------- a3 prep
__global__ void k_row_scale_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                   const float* __restrict__ values, int64_t n, int32_t d, int32_t smax,
                                   double* __restrict__ sigma, double* __restrict__ inv_sigma,
                                   double* __restrict__ err) {
  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  if (values) {
    for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32)
      if (indices[j] < d) s += (double)values[j];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  double sg = 1.0;
  if (values && s > 0.0) sg = kFixedOne / (s * (double)smax);
  if (lane == 0) {
    if (sigma) sigma[row] = sg;
    if (inv_sigma) inv_sigma[row] = 1.0 / sg;
  }
  if (err) {  // E_r = smax * sum_d |q_d - r_d sigma_r|, q_d exactly as quantize() rounds it (0 for integer R)
    double e = 0.0;
    if (values) {
      for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32)
        if (indices[j] < d) {
          const double x = (double)values[j] * sg;
          int32_t q = (int32_t)rint(x);
          q = q < 1 ? 1 : q;
          e += fabs((double)q - x);
        }
#pragma unroll
      for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    if (lane == 0) err[row] = e * (double)smax;
  }
}

__device__ __forceinline__ int32_t quantize(const void* __restrict__ values, knnjoin_dtype rdt, int64_t j, double sg) {
  if (rdt == KNNJOIN_FP32) {
    int32_t q = (int32_t)rint((double)((const float*)values)[j] * sg);
    return q < 1 ? 1 : q;
  }
  if (rdt == KNNJOIN_INT8) return (int32_t)((const int8_t*)values)[j];
  return 1;
}

// One warp merges the B rows of `batch` (lane b < B walks row b): one run per distinct feature, in ascending
// feature order.  Fallback for batches with more entries than the block sort below holds.
__device__ void warp_merge_runs(int64_t batch, int lane, const int64_t* __restrict__ indptr,
                                const int32_t* __restrict__ indices, const void* __restrict__ values,
                                knnjoin_dtype rdt, int64_t n_r, int32_t d, int B, const double* __restrict__ sigma,
                                const int32_t* __restrict__ perm, const int64_t* __restrict__ rbase,
                                uint32_t* __restrict__ runs_f, int32_t* __restrict__ runs_q,
                                uint32_t* __restrict__ batch_nruns) {
  const int64_t pos = batch * B + lane;  // position in the (work-sorted) row order
  bool mine = lane < B && pos < n_r;
  int64_t ptr = 0, end = 0;
  double sg = 1.0;
  if (mine) {
    const int64_t row = perm ? perm[pos] : pos;
    ptr = indptr[row];
    end = indptr[row + 1];
    sg = sigma[row];
  }
  int64_t base = rbase ? rbase[batch * B] : indptr[batch * B];
  uint32_t nruns = 0;
  for (;;) {
    int32_t f = 0x7FFFFFFF;
    if (ptr < end) {
      f = indices[ptr];
      if (f >= d) { ptr = end; f = 0x7FFFFFFF; }  // ascending: every later feature is >= d too
    }
    int32_t fmin = f;
#pragma unroll
    for (int o = 16; o; o >>= 1) fmin = min(fmin, __shfl_xor_sync(0xffffffffu, fmin, o));
    if (fmin == 0x7FFFFFFF) break;
    bool has = mine && f == fmin;
    uint32_t mask = __ballot_sync(0xffffffffu, has);
    size_t run = (size_t)(base + nruns);
    if (lane < B) {
      int32_t q = 0;
      if (has) {
        q = quantize(values, rdt, ptr, sg);
        ++ptr;
      }
      runs_q[run * B + lane] = q;
    }
    if (lane == 0) runs_f[run] = (uint32_t)fmin | (mask << 24);
    ++nruns;
  }
  if (lane == 0) batch_nruns[batch] = nruns;
}

constexpr int kRunThreads = 128;  // block sort: kRunThreads x ITEMS (row, feature) entries per batch

// One CTA per batch: the batch's (feature, row) entries are block-radix-sorted in shared memory, equal
// features collapse into one run (row mask + per-row q), runs are written in ascending feature order.
// Batches with more entries than the capacity fall back to warp_merge_runs.
template <int kRunItems>
__global__ void __launch_bounds__(kRunThreads) k_build_runs(const int64_t* __restrict__ indptr,
                                                            const int32_t* __restrict__ indices,
                                                            const void* __restrict__ values, knnjoin_dtype rdt,
                                                            int64_t n_r, int32_t d, int B, int64_t n_batches,
                                                            const double* __restrict__ sigma,
                                                            const int32_t* __restrict__ perm,
                                                            const int64_t* __restrict__ rbase,
                                                            uint32_t* __restrict__ runs_f, int32_t* __restrict__ runs_q,
                                                            uint32_t* __restrict__ batch_nruns, int key_bits,
                                                            const int32_t* __restrict__ gate, int gate_heads) {
  if (gate && ((*gate > 0) != (gate_heads != 0))) return;  // device-side shape choice (knnjoin_query)
  using BRS = cub::BlockRadixSort<uint32_t, kRunThreads, kRunItems, int32_t>;
  using BScan = cub::BlockScan<int, kRunThreads>;
  __shared__ union {
    typename BRS::TempStorage sort;
    typename BScan::TempStorage scan;
    uint32_t keys[kRunThreads * kRunItems];
  } sm;
  __shared__ int32_t s_q[kRunThreads * kRunItems];
  const int64_t batch = blockIdx.x;
  if (batch >= n_batches) return;
  const int tid = threadIdx.x;
  const int64_t pos0 = batch * B;  // batch rows are positions pos0.. of the (work-sorted) row order
  const int nb = (int)min((int64_t)B, n_r - pos0);
  // entry j of the batch (rows concatenated in batch order) lives at CSR position rs[b] + (j - pre[b])
  int64_t rs[8], pre[9];
  pre[0] = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    rs[b] = 0;
    int64_t len = 0;
    if (b < nb) {
      const int64_t row = perm ? perm[pos0 + b] : pos0 + b;
      rs[b] = indptr[row];
      len = indptr[row + 1] - rs[b];
    }
    pre[b + 1] = pre[b] + len;
  }
  const int64_t ne = pre[8];
  if (ne > kRunThreads * kRunItems) {
    if (tid < 32)
      warp_merge_runs(batch, tid, indptr, indices, values, rdt, n_r, d, B, sigma, perm, rbase, runs_f, runs_q,
                      batch_nruns);
    return;
  }
  // key = feature << 3 | row-in-batch (entries with feature >= d sort last and are dropped)
  uint32_t key[kRunItems];
  int32_t q[kRunItems];
#pragma unroll
  for (int it = 0; it < kRunItems; ++it) {
    const int64_t j = tid * kRunItems + it;
    key[it] = 0xFFFFFFFFu;
    q[it] = 0;
    if (j < ne) {
      // row of entry j and its CSR position (unrolled selects keep rs / pre in registers)
      int b = 0;
#pragma unroll
      for (int i = 1; i < 8; ++i) b += (j >= pre[i]) ? 1 : 0;
      int64_t rsb = rs[0], preb = 0;
#pragma unroll
      for (int i = 1; i < 8; ++i)
        if (b == i) { rsb = rs[i]; preb = pre[i]; }
      const int64_t e = rsb + (j - preb);
      const int32_t f = indices[e];
      if (f < d) {
        key[it] = ((uint32_t)f << 3) | (uint32_t)b;
        q[it] = quantize(values, rdt, e, sigma[perm ? perm[pos0 + b] : pos0 + b]);
      }
    }
  }
  BRS(sm.sort).Sort(key, q, 0, key_bits);
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kRunItems; ++it) {
    sm.keys[tid * kRunItems + it] = key[it];
    s_q[tid * kRunItems + it] = q[it];
  }
  __syncthreads();
  int starts = 0;
  bool is_start[kRunItems];
#pragma unroll
  for (int it = 0; it < kRunItems; ++it) {
    const int i = tid * kRunItems + it;
    const uint32_t k = key[it];
    is_start[it] = k != 0xFFFFFFFFu && (i == 0 || (sm.keys[i - 1] >> 3) != (k >> 3));
    starts += is_start[it];
  }
  __syncthreads();  // sm.keys is overwritten by the scan temp storage
  uint32_t keys_local[kRunItems];
#pragma unroll
  for (int it = 0; it < kRunItems; ++it) keys_local[it] = key[it];
  int run_idx, total;
  BScan(sm.scan).ExclusiveSum(starts, run_idx, total);
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kRunItems; ++it) sm.keys[tid * kRunItems + it] = keys_local[it];
  __syncthreads();
  const size_t base = (size_t)(rbase ? rbase[pos0] : indptr[pos0]);
#pragma unroll
  for (int it = 0; it < kRunItems; ++it) {
    if (is_start[it]) {
      const int i = tid * kRunItems + it;
      const uint32_t f = keys_local[it] >> 3;
      uint32_t mask = 0;
      int32_t qb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int j = i; j < kRunThreads * kRunItems && j < i + 8; ++j) {
        const uint32_t kj = sm.keys[j];
        if (kj == 0xFFFFFFFFu || (kj >> 3) != f) break;
        mask |= 1u << (kj & 7u);
        const int32_t qj = s_q[j];
#pragma unroll
        for (int bb = 0; bb < 8; ++bb)
          if ((int)(kj & 7u) == bb) qb[bb] = qj;
      }
      const size_t run = base + run_idx;
      runs_f[run] = f | (mask << 24);
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (b < B) runs_q[run * B + b] = qb[b];
      ++run_idx;
    }
  }
  if (tid == 0) batch_nruns[batch] = (uint32_t)total;
}


// ------------------------------------------------------------------------------------ host dispatch
struct QueryWs {
  size_t sigma_at, inv_at, runs_f_at, runs_q_at, nruns_at, counter_at, state_at, done_at, wkey_at, wkey2_at,
      perm_at, perm2_at, rlen_at, rbase_at, cub_at, cub_bytes, part_at, part_bytes, prune_at,
      // certification + 64-bit fallback (wide.cu): E_r, the final fixed keys, the failing-row list, sigma64,
      // 1/sigma64, the wide item counter and the tile-group lists of the first kWideCapRows listed rows
      err_at, keys_at, cert_at, sig64_at, inv64_at, wctr_at, wpart_at, wpart_bytes, done_bytes, total;
  int32_t wide_G;
};

// a6 (pruned queries, one row per batch): per run i of a row, prune_suf[i] = the sum of c_j = q_j * maxweight(f_j)
// over the runs j at or after i in the order (c descending, run index ascending) -- the row's features sorted
// by their bound, suffix sums.  The non-essential set of a tile is {i : prune_suf[i] <= budget}: a suffix of
// that order whose bounds sum to at most the budget.  One CTA per row: block radix sort of (c, -i) ascending,
// whose inclusive prefix sums are exactly those suffix sums.  Rows with more runs than the sort holds keep every
// feature essential (prune_suf = max).
constexpr int kPruneThreads = 128, kPruneItems = 16;
__global__ void __launch_bounds__(kPruneThreads) k_prune_prep(const int64_t* __restrict__ indptr,
                                                              const int64_t* __restrict__ rbase,
                                                              const uint32_t* __restrict__ runs_f,
                                                              const int32_t* __restrict__ runs_q,
                                                              const uint32_t* __restrict__ batch_nruns,
                                                              const uint32_t* __restrict__ fmax,
                                                              uint2* __restrict__ prune_suf) {
  using BRS = cub::BlockRadixSort<uint64_t, kPruneThreads, kPruneItems, int32_t>;
  using BScan = cub::BlockScan<uint64_t, kPruneThreads>;
  __shared__ union {
    typename BRS::TempStorage sort;
    typename BScan::TempStorage scan;
  } sm;
  constexpr int kCapRuns = kPruneThreads * kPruneItems;  // 2048 = 2^11: the run index fits 11 key bits
  const int64_t batch = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t base = rbase ? rbase[batch] : indptr[batch];
  const int n = (int)batch_nruns[batch];
  if (n > kCapRuns) {
    for (int i = tid; i < n; i += kPruneThreads) prune_suf[base + i] = make_uint2(0xFFFFFFFFu, 0u);
    return;
  }
  constexpr uint64_t kInvalid = ~0ull;
  uint64_t key[kPruneItems];
  int32_t idx[kPruneItems];
#pragma unroll
  for (int it = 0; it < kPruneItems; ++it) {
    const int i = tid * kPruneItems + it;
    key[it] = kInvalid;
    idx[it] = i;
    if (i < n) {
      const uint32_t f = runs_f[base + i] & 0xFFFFFFu;
      uint64_t c = (uint64_t)(uint32_t)runs_q[base + i] * (fmax ? (uint64_t)fmax[f] : 1ull);
      if (c > 0xFFFFFFFFull) c = 0xFFFFFFFFull;
      key[it] = (c << 11) | (uint64_t)(kCapRuns - 1 - i);  // ascending (c, -i) = reverse of (c desc, i asc)
    }
  }
  BRS(sm.sort).Sort(key, idx, 0, 44);
  __syncthreads();
  uint64_t c[kPruneItems];
#pragma unroll
  for (int it = 0; it < kPruneItems; ++it) c[it] = key[it] == kInvalid ? 0ull : key[it] >> 11;
  BScan(sm.scan).InclusiveSum(c, c);
#pragma unroll
  for (int it = 0; it < kPruneItems; ++it)
    if (key[it] != kInvalid)
      prune_suf[base + idx[it]] = make_uint2(c[it] > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c[it],
                                             (uint32_t)(key[it] >> 11));
}

bool shape_supported(int B, int NW, int KS) {
  if (B * KS > 24 || B > NW) return false;
  if (NW == 4) return B == 1 || B == 2;
  if (NW == 8) return B == 1 || B == 2 || B == 3 || B == 4;
  if (NW == 16) return B == 1 || B == 2 || B == 4 || B == 6 || B == 8;
  return false;
}

// pick (B rows per batch, NW warps per CTA): an explicit request must fit; auto prefers 8-warp CTAs with
// three (then two) resident per SM -- barrier and latency stalls of one overlap the others -- then one
// 16-warp CTA, largest B first.
// heads: the index has head features (-1 unknown).  Without them there is little cross-row reuse and short
// slices, so small CTAs (4 warps, one row, 4-6 per SM) that barrier rarely and overlap well win; with them
// (Zipf-like S) batches of rows share slices and head tables, and three 8-warp CTAs per SM win.
bool pick_shape(int T, int k, int req_B, int req_NW, int heads, Shape* out) {
  const int KS = ks_for_k(k);
  const size_t max_smem = 227 * 1024;
  const size_t per_sm = 228 * 1024;
  auto fits = [&](int B, int NW, int ctas) {
    if (!shape_supported(B, NW, KS)) return false;
    if (T % (NW * 128) != 0) return false;
    size_t b = smem_bytes(B, T, k, NW, heads != 0);
    return b <= max_smem && ctas * (b + 1024) <= per_sm;
  };
  const int Bs[] = {8, 6, 4, 3, 2, 1};
  if (req_B || req_NW) {
    for (int NW : {8, 16, 4}) {
      if (req_NW && NW != req_NW) continue;
      for (int B : Bs) {
        if (req_B && B != req_B) continue;
        if (fits(B, NW, 1)) { *out = {B, NW}; return true; }
      }
    }
    return false;
  }
  if (heads == 0)
    for (int ctas : {6, 5, 4, 3})
      if (fits(1, 4, ctas)) { *out = {1, 4}; return true; }
  for (int B : Bs)
    if (B >= 2 && fits(B, 8, 3)) { *out = {B, 8}; return true; }
  for (int B : Bs)
    if (B >= 3 && fits(B, 8, 2)) { *out = {B, 8}; return true; }
  for (int B : Bs)
    if (fits(B, 16, 1)) { *out = {B, 16}; return true; }
  for (int B : Bs)
    if (fits(B, 8, 1)) { *out = {B, 8}; return true; }
  return false;
}

// CTAs a shape keeps resident (launch bounds / shared memory of pick_shape): bounds the split-mode lists
int ctas_per_sm(int NW) { return NW == 4 ? 6 : (NW == 8 ? 3 : 1); }
// a query with fewer batches than kSplitWaves waves of resident CTAs splits its tiles into groups:
// G = ceil(ctas / n_batches) below one wave, 2 between one and two waves (measured on C2-shaped serving
// batches: more, smaller groups lose to their per-item setup and merge)
constexpr int64_t kSplitWaves = 2;
int64_t split_groups(int64_t n_batches, int64_t ctas) {
  if (n_batches >= kSplitWaves * ctas) return 1;
  return n_batches < ctas ? (ctas + n_batches - 1) / n_batches : 2;
}

// shapes: the candidate CTA shapes of the query (one, or the two the device chooses between); every region is
// sized for the largest need over them
bool query_ws_layout(int64_t n_r, int64_t nnz_r, const Shape* shapes, int n_shapes, int k, int sms, int64_t n_tiles,
                     QueryWs* W) {
  int Bmax = 1, Bmin = 8;
  size_t part = 0;
  for (int i = 0; i < n_shapes; ++i) {
    const int B = shapes[i].B;
    Bmax = B > Bmax ? B : Bmax;
    Bmin = B < Bmin ? B : Bmin;
    // split mode (fewer than kSplitWaves x resident CTAs batches): G tile groups x n_r rows x k keys, with
    // G <= max(ceil(ctas / n_batches), 2) => G * n_r <= (kSplitWaves * ctas + n_batches) * B
    const int64_t nb = (n_r + B - 1) / B;
    const int64_t ctas = (int64_t)sms * ctas_per_sm(shapes[i].NW);
    const size_t pb = nb < kSplitWaves * ctas ? 8 * (size_t)k * (size_t)((kSplitWaves * ctas + nb) * B) : 0;
    part = pb > part ? pb : part;
  }
  const int64_t n_batches = (n_r + Bmin - 1) / Bmin;
  const int B = Bmax;
  size_t at = 0;
  W->sigma_at = at;   at = align_up(at + 8 * (size_t)n_r, 256);
  W->inv_at = at;     at = align_up(at + 8 * (size_t)n_r, 256);
  W->runs_f_at = at;  at = align_up(at + 4 * (size_t)nnz_r, 256);
  W->runs_q_at = at;  at = align_up(at + 4 * (size_t)nnz_r * B, 256);
  W->nruns_at = at;   at = align_up(at + 4 * (size_t)n_batches, 256);
  W->counter_at = at; at = align_up(at + 16, 256);
  W->state_at = at;   at = align_up(at + 8 * (size_t)n_r * k, 256);
  W->done_at = at;    at = align_up(at + 4 * (size_t)n_batches, 256);
  // a3 row order: work keys, permutation (double-buffered for the radix sort), row lengths, run bases
  size_t sort_bytes = 0, scan_bytes = 0;
  if (cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                (const int32_t*)nullptr, (int32_t*)nullptr, (int)n_r) != cudaSuccess)
    return false;
  if (cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)n_r) !=
      cudaSuccess)
    return false;
  W->cub_bytes = sort_bytes > scan_bytes ? sort_bytes : scan_bytes;
  W->wkey_at = at;    at = align_up(at + 4 * (size_t)n_r, 256);
  W->wkey2_at = at;   at = align_up(at + 4 * (size_t)n_r, 256);
  W->perm_at = at;    at = align_up(at + 4 * (size_t)n_r, 256);
  W->perm2_at = at;   at = align_up(at + 4 * (size_t)n_r, 256);
  W->rlen_at = at;    at = align_up(at + 8 * (size_t)n_r, 256);
  W->rbase_at = at;   at = align_up(at + 8 * (size_t)n_r, 256);
  W->cub_at = at;     at = align_up(at + W->cub_bytes, 256);
  W->part_bytes = part;
  W->part_at = at;    at = align_up(at + W->part_bytes, 256);
  W->prune_at = at;   at = align_up(at + 8 * (size_t)nnz_r, 256);  // a6 {suffix bound, c} per run (pruned queries)
  W->err_at = at;     at = align_up(at + 8 * (size_t)n_r, 256);
  W->keys_at = at;    at = align_up(at + 8 * (size_t)n_r * k, 256);
  W->cert_at = at;    at = align_up(at + 4 * (size_t)(n_r + 1), 256);
  W->sig64_at = at;   at = align_up(at + 8 * (size_t)n_r, 256);
  W->inv64_at = at;   at = align_up(at + 8 * (size_t)n_r, 256);
  W->wctr_at = at;    at = align_up(at + 16, 256);
  W->wpart_bytes = wide_part_bytes(k, n_tiles, sms, &W->wide_G);
  W->done_bytes = 4 * (size_t)n_batches;
  W->wpart_at = at;   at = align_up(at + W->wpart_bytes, 256);
  W->total = at;
  return true;
}

// a3: per-row work estimate w_r = sum_{d in r} |I_d| (the row's share of Eq. 4's second term),
// saturated to 32 bits; warp per row.  Sorting rows by w_r (descending) hands the heaviest batches out first
// so the persistent CTAs finish together.
__global__ void k_row_work(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t n,
                           int32_t d, const int32_t* __restrict__ df, uint32_t* __restrict__ wkey,
                           int32_t* __restrict__ iota) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  unsigned long long w = 0;
  for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32) {
    const int32_t f = indices[j];
    if (f < d) w += (unsigned long long)df[f];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if (lane == 0) {
    // monotone 16-bit code of w (5-bit exponent, 11-bit mantissa): a coarse order needs two radix passes only
    const uint32_t w32 = w > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)w;
    uint32_t code = w32;
    if (w32 >= 2048u) {
      const uint32_t e = 31u - __clz(w32);  // >= 11
      code = ((e - 10u) << 11) | ((w32 >> (e - 11u)) & 0x7FFu);
    }
    wkey[row] = code;
    iota[row] = (int32_t)row;
  }
}

__global__ void k_sorted_len(const int64_t* __restrict__ indptr, const int32_t* __restrict__ perm, int64_t n,
                             int64_t* __restrict__ len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = perm[i];
  len[i] = indptr[r + 1] - indptr[r];
}

cudaError_t launch_shape(const Shape& sh, const QP& p, int sms, cudaStream_t st) {
  switch (ks_for_k(p.k)) {
    case 1: return launch_accumulate<1>(sh, p, sms, st);
    case 4: return launch_accumulate<4>(sh, p, sms, st);
    case 8: return launch_accumulate<8>(sh, p, sms, st);
  }
  return cudaErrorInvalidValue;
}


int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

bool check_query_args(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k) {
  if (!idx || !R) { set_error("index or R is NULL"); return false; }
  if (k < 1 || k > kMaxK) { set_error("k must be in [1, %d] (got %d)", kMaxK, k); return false; }
  if (R->n_rows < 0 || R->nnz < 0) { set_error("negative R size"); return false; }
  if (R->dtype != KNNJOIN_BINARY && R->dtype != KNNJOIN_INT8 && R->dtype != KNNJOIN_FP32) { set_error("bad R dtype"); return false; }
  return true;
}

}  // namespace

void launch_row_scale(const knnjoin_csr* R, int32_t d, int32_t smax, double* sigma, double* inv_sigma, double* err,
                      cudaStream_t st) {
  if (R->n_rows <= 0) return;
  int64_t threads = R->n_rows * 32;
  k_row_scale_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      R->indptr, R->indices, R->dtype == KNNJOIN_FP32 ? (const float*)R->values : nullptr, R->n_rows, d, smax, sigma,
      inv_sigma, err);
}

}  // namespace kj

using namespace kj;

KJ_API size_t knnjoin_query_workspace_bytes(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k,
                                            const knnjoin_query_options* qopt) {
  if (!check_query_args(idx, R, k)) return 0;
  // the auto shape may depend on the index's head count (known on the device): size for both candidates
  Shape shapes[2];
  for (int heads : {0, 1}) {
    if (!pick_shape(idx->tile, k, qopt ? qopt->batch_rows : 0, qopt ? qopt->cta_warps : 0, heads, &shapes[heads])) {
      set_error("no (batch_rows, cta_warps) shape fits shared memory for tile %d, k %d", idx->tile, k);
      return 0;
    }
  }
  QueryWs W;
  if (!query_ws_layout(R->n_rows, R->nnz, shapes, 2, k, device_sms(), idx->n_tiles, &W)) {
    set_error("workspace sizing failed (CUB temporary storage query)");
    return 0;
  }
  return W.total;
}

KJ_API knnjoin_status knnjoin_query(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k,
                                    const knnjoin_query_options* qopt, uint64_t* out_keys, int32_t* out_ids,
                                    float* out_scores, void* workspace, size_t workspace_bytes, void* stream) {
  KJ_NVTX("knnjoin_query");
  if (!check_query_args(idx, R, k)) return KNNJOIN_ERR_ARG;
  if (R->n_rows == 0) return KNNJOIN_OK;  // empty R: nothing to write
  if (!out_keys && (!out_ids || !out_scores)) { set_error("need out_keys or both out_ids and out_scores"); return KNNJOIN_ERR_ARG; }
  const bool s_fp32 = idx->s_dtype == KNNJOIN_FP32;
  const bool r_fp32 = R->dtype == KNNJOIN_FP32;
  const int precision = qopt ? qopt->precision : 0;
  if (precision < 0 || precision > 2) { set_error("precision must be 0 (auto), 1 (32-bit) or 2 (64-bit)"); return KNNJOIN_ERR_ARG; }
  if (s_fp32 && precision == 1) { set_error("FP32 S is queried at 64-bit fixed point only (precision 0 or 2)"); return KNNJOIN_ERR_UNSUPPORTED; }
  if (!r_fp32 && !s_fp32 && (double)idx->d * 127.0 * 127.0 >= 4294967296.0) {
    set_error("integer scores may overflow 32 bits for d = %d", idx->d);
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if (qopt && (qopt->row_list != nullptr) != (qopt->row_count != nullptr)) {
    set_error("row_list and row_count go together");
    return KNNJOIN_ERR_ARG;
  }
  if (qopt && !(qopt->tolerance >= 0.0f && qopt->tolerance < 1.0f)) { set_error("tolerance must be in [0, 1)"); return KNNJOIN_ERR_ARG; }
  const double tol = (qopt && qopt->tolerance > 0.0f) ? (double)qopt->tolerance : kDefaultTolerance;
  // 64-bit path for the whole query: FP32 S (no 32-bit path), or precision 2 with FP32 R (integer x integer
  // scores are exact at 32 bits, precision is ignored there)
  const bool wide_all = s_fp32 || (precision == 2 && r_fp32);
  // a6: effective pruning alpha (0 = not pruned)
  float alpha = 0.0f;
  if (qopt && qopt->prune_alpha != 0.0f && !idx->prune && qopt->prune_alpha > 0.0f) {
    set_error("prune_alpha > 0 needs an index built with options.prune = 1");
    return KNNJOIN_ERR_ARG;
  }
  if (qopt && (qopt->prune_alpha > 1.0f || qopt->prune_alpha != qopt->prune_alpha)) {
    set_error("prune_alpha must be <= 1");
    return KNNJOIN_ERR_ARG;
  }
  if (idx->prune) alpha = (qopt && qopt->prune_alpha != 0.0f) ? (qopt->prune_alpha > 0.0f ? qopt->prune_alpha : 0.0f) : idx->alpha;
  const bool residual = qopt && qopt->residual;
  if (residual) {
    if (!idx->prune) { set_error("residual queries need an index built with prune = 1 (forward rows = s')"); return KNNJOIN_ERR_ARG; }
    if (qopt->prune_alpha > 0.0f) { set_error("residual (f1) and prune_alpha > 0 (a6) are exclusive"); return KNNJOIN_ERR_ARG; }
    alpha = 0.0f;
  }
  if (wide_all && (alpha > 0.0f || residual)) {
    set_error("64-bit queries (FP32 S or precision 2) do not combine with pruning (a6) or residual (f1) queries");
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if (!wide_all && qopt && qopt->row_list) {
    set_error("row_list applies to 64-bit queries (FP32 S or precision 2)");
    return KNNJOIN_ERR_ARG;
  }
  if (qopt && (qopt->tile_begin < 0 || qopt->tile_end < 0 || qopt->tile_begin > idx->n_tiles ||
               qopt->tile_end > idx->n_tiles || (qopt->tile_end > 0 && qopt->tile_begin > qopt->tile_end))) {
    set_error("tile range [%lld, %lld) outside [0, %lld]", (long long)qopt->tile_begin, (long long)qopt->tile_end,
              (long long)idx->n_tiles);
    return KNNJOIN_ERR_ARG;
  }
  const bool auto_shape = !qopt || (qopt->batch_rows == 0 && qopt->cta_warps == 0);
  // Shapes: an index whose head-feature count may be non-zero (BINARY S with head features enabled) has two
  // candidate auto shapes, chosen on the DEVICE: both are launched and each gates itself on the index's head
  // count (the mismatched one returns at entry), so the call never waits for the host to learn the count.
  const bool may_have_heads = idx->head_max > 0;
  Shape sh_heads{0, 0}, sh_plain{0, 0};
  const int req_B = qopt ? qopt->batch_rows : 0, req_NW = qopt ? qopt->cta_warps : 0;
  if (!pick_shape(idx->tile, k, req_B, req_NW, 0, &sh_plain) ||
      (may_have_heads && !pick_shape(idx->tile, k, req_B, req_NW, 1, &sh_heads))) {
    set_error("batch_rows %d / cta_warps %d unsupported for tile %d, k %d", req_B, req_NW, idx->tile, k);
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if ((alpha > 0.0f || residual) && (size_t)((idx->d + 31) / 32) * 4 + smem_bytes(1, idx->tile, k, 4, false) > 200 * 1024) {
    set_error("pruned queries keep a d-bit map in shared memory: d = %d too large", idx->d);
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if ((alpha > 0.0f || residual) && !(sh_plain.B == 1 && sh_plain.NW == 4)) {
    set_error("pruned queries run one-row 4-warp CTAs (batch_rows 1, cta_warps 4); got %d / %d", sh_plain.B, sh_plain.NW);
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  // the workspace is laid out for the larger of the candidate shapes (only one of them runs)
  const int sms = device_sms();
  QueryWs W;
  {
    const Shape shapes[2] = {sh_plain, sh_heads};
    if (!query_ws_layout(R->n_rows, R->nnz, shapes, may_have_heads ? 2 : 1, k, sms, idx->n_tiles, &W)) {
      set_error("workspace sizing failed (CUB temporary storage query)");
      return KNNJOIN_ERR_CUDA;
    }
  }
  if (!workspace || workspace_bytes < W.total) { set_error("query workspace %zu < %zu bytes", workspace_bytes, W.total); return KNNJOIN_ERR_WORKSPACE; }
  if ((uintptr_t)workspace & 255) { set_error("workspace must be 256-byte aligned"); return KNNJOIN_ERR_ARG; }
  if (!R->indptr || (R->nnz > 0 && !R->indices) || (R->dtype != KNNJOIN_BINARY && R->nnz > 0 && !R->values)) {
    set_error("R pointers are NULL");
    return KNNJOIN_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* wb = (char*)workspace;
  cudaError_t e;
  const int64_t t0 = qopt ? qopt->tile_begin : 0;
  const int64_t t1 = (qopt && qopt->tile_end > 0) ? qopt->tile_end : idx->n_tiles;

  // ------------------------------------------------------------------ 64-bit fixed point for every row
  if (wide_all) {
    if (qopt && qopt->ev_begin) cudaEventRecord((cudaEvent_t)qopt->ev_begin, st);
    e = launch_wide(idx, R, k, t0, t1, qopt ? qopt->row_list : nullptr, qopt ? qopt->row_count : nullptr,
                    qopt ? qopt->resume_keys : nullptr, qopt ? qopt->theta_in : nullptr, (double*)(wb + W.sig64_at),
                    (double*)(wb + W.inv64_at), (uint32_t*)(wb + W.wctr_at), (uint64_t*)(wb + W.wpart_at), W.wide_G,
                    (unsigned long long*)(qopt ? qopt->counters : nullptr), out_keys, out_ids, out_scores, sms, st);
    if (qopt && qopt->ev_end) cudaEventRecord((cudaEvent_t)qopt->ev_end, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_accumulate_wide");
    if (qopt && qopt->uncertified && (e = cudaMemsetAsync(qopt->uncertified, 0, 4, st)) != cudaSuccess)
      return cuda_fail(e, "memset uncertified");
    return KNNJOIN_OK;
  }

  // ------------------------------------------------------------------ 32-bit fixed point (a3-a7)
  // certification of FP32-R lists (wide.cu): auto mode recomputes failing rows at 64 bits, unless the query is
  // part of a chained / sharded computation (tile range, resume_keys, theta_in), whose lists only the caller
  // sees whole (it certifies them with knnjoin_certify)
  // (a residual query's index holds only the indexed parts s'' of S: a 64-bit re-run over it would miss dot(r, s'),
  // so f1's caller certifies and recomputes at the end as well)
  const bool partial = qopt && (qopt->resume_keys || qopt->theta_in || t0 != 0 || t1 != idx->n_tiles || residual);
  const bool certify = r_fp32 && ((precision == 0 && !partial) || (qopt && qopt->uncertified));
  const bool fallback = certify && precision == 0 && !partial;
  uint64_t* keys_dst = out_keys ? out_keys : (certify ? (uint64_t*)(wb + W.keys_at) : nullptr);
  double* sigma = (double*)(wb + W.sigma_at);
  double* inv_sigma = (double*)(wb + W.inv_at);
  double* err = (double*)(wb + W.err_at);
  uint32_t* runs_f = (uint32_t*)(wb + W.runs_f_at);
  int32_t* runs_q = (int32_t*)(wb + W.runs_q_at);
  uint32_t* nruns = (uint32_t*)(wb + W.nruns_at);
  uint32_t* counter = (uint32_t*)(wb + W.counter_at);
  uint64_t* state_keys = (uint64_t*)(wb + W.state_at);
  uint32_t* pass_done = (uint32_t*)(wb + W.done_at);
  const int32_t smax = idx->s_dtype == KNNJOIN_INT8 ? 127 : 1;
  if ((e = cudaMemsetAsync(counter, 0, 16, st)) != cudaSuccess) return cuda_fail(e, "memset counter");
  if ((e = cudaMemsetAsync(pass_done, 0, W.done_bytes, st)) != cudaSuccess) return cuda_fail(e, "memset pass_done");
  launch_row_scale(R, idx->d, smax, sigma, inv_sigma, certify ? err : nullptr, st);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_row_scale");
  const int32_t* perm = nullptr;
  const int64_t* rbase = nullptr;
  if (!(qopt && qopt->row_order == 1) && R->n_rows > 1) {  // a3: rows by descending work
    uint32_t* wkey = (uint32_t*)(wb + W.wkey_at);
    uint32_t* wkey2 = (uint32_t*)(wb + W.wkey2_at);
    int32_t* iota = (int32_t*)(wb + W.perm_at);
    int32_t* pm = (int32_t*)(wb + W.perm2_at);
    int64_t* rlen = (int64_t*)(wb + W.rlen_at);
    int64_t* rb = (int64_t*)(wb + W.rbase_at);
    const int64_t n = R->n_rows;
    k_row_work<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(R->indptr, R->indices, n, idx->d, idx->df, wkey, iota);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_row_work");
    size_t cb = W.cub_bytes;
    if ((e = cub::DeviceRadixSort::SortPairsDescending(wb + W.cub_at, cb, wkey, wkey2, iota, pm, (int)n, 0, 16, st)) !=
        cudaSuccess)
      return cuda_fail(e, "row sort");
    k_sorted_len<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(R->indptr, pm, n, rlen);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_sorted_len");
    cb = W.cub_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(wb + W.cub_at, cb, rlen, rb, (int)n, st)) != cudaSuccess)
      return cuda_fail(e, "row base scan");
    perm = pm;
    rbase = rb;
  }
  int dev = 0, l2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  int kbits = 3;  // (feature << 3 | row) keys: bits for features < d, plus 3
  while (kbits < 32 && ((int64_t)1 << (kbits - 3)) <= (int64_t)idx->d) ++kbits;  // invalid keys sort last

  // one candidate shape: run building (a3) + K3.  gate: the index's head count (device); the launch runs only
  // when (count > 0) == want_heads.
  auto run_shape = [&](const Shape& sh, const int32_t* gate, int want_heads, bool first, bool last) -> knnjoin_status {
    const int B = sh.B;
    const int64_t n_batches = (R->n_rows + B - 1) / B;
    const double mean = (double)R->nnz / (double)n_batches * 1.5;
    // block-sort capacity from the mean entries per batch (x1.5 headroom); larger batches use the warp merge
    const int items = mean <= kRunThreads * 4 ? 4 : (mean <= kRunThreads * 8 ? 8 : (mean <= kRunThreads * 16 ? 16 : 32));
    auto runs = [&](auto kern) {
      kern<<<(unsigned)n_batches, kRunThreads, 0, st>>>(R->indptr, R->indices, R->values, R->dtype, R->n_rows, idx->d, B,
                                                       n_batches, sigma, perm, rbase, runs_f, runs_q, nruns, kbits,
                                                       gate, want_heads);
    };
    if (items == 4) runs(k_build_runs<4>);
    else if (items == 8) runs(k_build_runs<8>);
    else if (items == 16) runs(k_build_runs<16>);
    else runs(k_build_runs<32>);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_build_runs");
    uint2* prune_suf = nullptr;
    if (alpha > 0.0f) {
      prune_suf = (uint2*)(wb + W.prune_at);
      k_prune_prep<<<(unsigned)n_batches, kPruneThreads, 0, st>>>(R->indptr, rbase, runs_f, runs_q, nruns, idx->fmax,
                                                                 prune_suf);
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_prune_prep");
    }
    QP p;
    p.off = idx->off;
    p.unit_cap = idx->unit_cap;
    p.ids = idx->ids;
    p.vals = idx->vals;
    p.head_slot = idx->head_slot;
    p.head_feat = idx->head_feat;
    p.head_cols = idx->head_cols;
    p.gate = gate;
    p.gate_heads = want_heads;
    p.d = idx->d;
    p.T = idx->tile;
    p.NT = idx->n_tiles;
    p.t0 = t0;
    p.t1 = t1;
    p.theta_in = qopt ? qopt->theta_in : nullptr;
    p.resume = qopt ? qopt->resume_keys : nullptr;
    p.s_id_base = idx->s_id_base;
    p.head_smem = want_heads;
    p.n_r = R->n_rows;
    p.k = k;
    p.n_batches = n_batches;
    p.r_indptr = R->indptr;
    p.perm = perm;
    p.rbase = rbase;
    p.runs_f = runs_f;
    p.runs_q = runs_q;
    p.batch_nruns = nruns;
    p.inv_sigma = inv_sigma;
    p.batch_counter = counter;
    {
      // tiles per pass: a slab of the index small enough to stay in L2 while every batch sweeps it
      int64_t tpp = qopt ? qopt->tiles_per_pass : 0;
      if (tpp <= 0) {
        const double per_tile =
            (double)(idx->storage_bytes - idx->fwd_bytes) / (double)(idx->n_tiles > 0 ? idx->n_tiles : 1);
        tpp = (int64_t)((double)(l2 > 0 ? l2 : (96 << 20)) / 3.0 / (per_tile > 1.0 ? per_tile : 1.0));
        if (tpp < 1) tpp = 1;
      }
      const int64_t span = p.t1 - p.t0;
      if (tpp > span) tpp = span > 0 ? span : 1;
      // few batches (small R, serving): the tiles are split into G independent groups (split_groups) so that
      // the G x n_batches items fill the resident CTAs; each group's lists go to part_keys and are merged by
      // rank
      p.split = 0;
      p.part_keys = nullptr;
      const int64_t ctas = (int64_t)sms * ctas_per_sm(sh.NW);
      if (!(qopt && qopt->tiles_per_pass) && W.part_bytes && span > 1 && n_batches < kSplitWaves * ctas) {
        int64_t G = split_groups(n_batches, ctas);
        if (G > span) G = span;
        if (G > 1 && (size_t)G * (size_t)R->n_rows * (size_t)k * 8 <= W.part_bytes) {
          tpp = (span + G - 1) / G;
          p.split = 1;
          p.part_keys = (uint64_t*)(wb + W.part_at);
        }
      }
      p.tiles_per_pass = tpp;
      p.n_passes = span > 0 ? (span + tpp - 1) / tpp : 1;  // an empty range still runs one (tile-less) pass
    }
    p.alpha = alpha;
    p.prune_suf = prune_suf;
    p.fwd_ptr = idx->fwd_ptr;
    p.fwd_idx = idx->fwd_idx;
    p.fwd_val = idx->fwd_val;
    p.fmax = idx->fmax;
    p.prune_words = (idx->d + 31) / 32;
    p.residual = residual ? 1 : 0;
    p.state_keys = state_keys;
    p.pass_done = pass_done;
    p.counters = (unsigned long long*)(qopt ? qopt->counters : nullptr);
    p.phase = (unsigned long long*)(qopt ? qopt->phase_cycles : nullptr);
    p.out_keys = keys_dst;
    p.out_ids = out_ids;
    p.out_scores = out_scores;
    if (first && qopt && qopt->ev_begin) cudaEventRecord((cudaEvent_t)qopt->ev_begin, st);
    e = launch_shape(sh, p, sms, st);
    if (last && qopt && qopt->ev_end) cudaEventRecord((cudaEvent_t)qopt->ev_end, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_accumulate_topk");
    if (p.split) {  // the tile groups' lists hold disjoint S ids: K4's rank merge gives the one-pass result
      e = launch_merge_keys_gated(p.part_keys, (int32_t)p.n_passes, R->n_rows, k, inv_sigma, gate, want_heads, keys_dst,
                                  out_ids, out_scores, st);
      if (e != cudaSuccess) return cuda_fail(e, "split merge");
    }
    return KNNJOIN_OK;
  };
  knnjoin_status rc;
  if (!may_have_heads) {
    if ((rc = run_shape(sh_plain, nullptr, 0, true, true)) != KNNJOIN_OK) return rc;
  } else if (!auto_shape || (sh_plain.B == sh_heads.B && sh_plain.NW == sh_heads.NW)) {
    // one shape for both cases (requested explicitly): the instance with the head code handles a zero count
    if ((rc = run_shape(sh_heads, nullptr, 1, true, true)) != KNNJOIN_OK) return rc;
  } else {
    const int32_t* gate = idx->head_feat + kMaxHead;
    if ((rc = run_shape(sh_heads, gate, 1, true, false)) != KNNJOIN_OK) return rc;
    if ((rc = run_shape(sh_plain, gate, 0, false, true)) != KNNJOIN_OK) return rc;
  }

  // ------------------------------------------------------------------ certification + 64-bit fallback
  if (certify) {
    int32_t* list = (qopt && qopt->uncertified) ? qopt->uncertified : (int32_t*)(wb + W.cert_at);
    if ((e = launch_certify(keys_dst, err, R->n_rows, k, tol, list, st)) != cudaSuccess) return cuda_fail(e, "k_certify");
    if (fallback) {
      e = launch_wide(idx, R, k, t0, t1, list + 1, list, nullptr, nullptr, (double*)(wb + W.sig64_at),
                      (double*)(wb + W.inv64_at), (uint32_t*)(wb + W.wctr_at), (uint64_t*)(wb + W.wpart_at), W.wide_G,
                      nullptr, out_keys, out_ids, out_scores, sms, st);
      if (e != cudaSuccess) return cuda_fail(e, "k_accumulate_wide (fallback)");
    }
  } else if (qopt && qopt->uncertified) {
    if ((e = cudaMemsetAsync(qopt->uncertified, 0, 4, st)) != cudaSuccess) return cuda_fail(e, "memset uncertified");
  }
  return KNNJOIN_OK;
}
