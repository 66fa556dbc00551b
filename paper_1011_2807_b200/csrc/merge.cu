// merge.cu -- K4 (S-sharded merge of partial top-k lists), CSR validation, error plumbing.
//
// K4: with S split into P contiguous id ranges (one per GPU), every rank computes the
// top-k of every r against its shard (knnjoin_query -> out_keys); after an all-gather the P sorted lists
// of a row are merged here.  Keys pack (score, lower id wins) into one unsigned integer
// (topk.cuh), so the merge is exact and equals the single-index result bit for bit.  The fixed-point
// scale of a row depends only on r and the dtype of S, so all ranks produce comparable keys.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "topk.cuh"

namespace kj {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int64_t checked_grid_cap(int64_t grid) {
#ifdef KJ_CHECKS
  if (const char* s = getenv("KNNJOIN_MAX_CTAS")) {
    const long long cap = atoll(s);
    if (cap > 0 && grid > cap) return cap;
  }
#endif
  return grid;
}

knnjoin_status cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return KNNJOIN_ERR_CUDA;
}

int ks_for_k(int32_t k) { return k <= 32 ? 1 : (k <= 128 ? 4 : 8); }

__device__ unsigned long long g_bad;  // validation result word (module global, not an allocation)

namespace {

// Warp per row.  The P lists of a row are sorted (descending, zero padding last) and hold distinct keys
// (disjoint S id ranges), so the merged position of a key is its position in its own list plus the number of
// larger keys in the other P-1 lists (binary searches); positions past the row's positive keys are padding.
// float_keys: the score field is fp32 bits of the score (64-bit fixed-point queries, wide.cu), else a 32-bit
// fixed-point sum decoded with inv_sigma.  row_list / row_count: list position i holds output row row_list[i]
// (only the first *row_count positions are merged); nullptr: position i is row i.  n: slab stride (rows per
// slab); limit: positions merged (<= n).  keys_by_row: the lists of
// listed row r sit at slab position r (a [P][n][k] gather of whole-R outputs), else at list position i.
__global__ void k_merge(const uint64_t* __restrict__ keys, int32_t P, int64_t n, int64_t limit, int32_t k,
                        const double* __restrict__ inv_sigma, int float_keys, const int32_t* __restrict__ row_list,
                        const int32_t* __restrict__ row_count, int keys_by_row, const int32_t* __restrict__ gate,
                        int gate_heads, uint64_t* out_keys, int32_t* out_ids, float* out_scores) {
  if (gate && ((*gate > 0) != (gate_heads != 0))) return;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= limit || (row_count && i >= (int64_t)*row_count)) return;
  const int64_t r = row_list ? (int64_t)row_list[i] : i;
  const int64_t at = keys_by_row ? r : i;
  auto list = [&](int pr) { return keys + ((size_t)pr * n + at) * k; };
  auto count_gt = [&](const uint64_t* lst, uint64_t x) {
    int lo = 0, hi = k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg((const unsigned long long*)lst + mid) > x) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  auto emit = [&](int pos, uint64_t key) {
    const size_t o = (size_t)r * k + pos;
    const uint32_t score = (uint32_t)(key >> 32);
    if (score == 0) {
      if (out_keys) out_keys[o] = 0;
      if (out_ids) out_ids[o] = -1;
      if (out_scores) out_scores[o] = 0.0f;
    } else {
      if (out_keys) out_keys[o] = key;
      if (out_ids) out_ids[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)key);
      if (out_scores) out_scores[o] = float_keys ? __uint_as_float(score) : (float)((double)score * inv_sigma[r]);
    }
  };
  for (int e = lane; e < P * k; e += 32) {
    const int pr = e / k, pos = e % k;
    const uint64_t x = __ldg((const unsigned long long*)list(pr) + pos);
    if (x == 0) continue;
    int rank = pos;
    for (int q = 0; q < P && rank < k; ++q)
      if (q != pr) rank += count_gt(list(q), x);
    if (rank < k) emit(rank, x);
  }
  int npos = 0;  // positive keys over all lists (capped below by the loop)
  for (int q = 0; q < P && npos < k; ++q) npos += count_gt(list(q), 0);
  for (int pos = npos + lane; pos < k; pos += 32) emit(pos, 0);
}

}  // namespace

cudaError_t launch_merge_keys_ex(const uint64_t* keys, int32_t P, int64_t n, int64_t limit, int32_t k,
                                 const double* inv_sigma, int float_keys, const int32_t* row_list,
                                 const int32_t* row_count, int keys_by_row, uint64_t* out_keys, int32_t* out_ids,
                                 float* out_scores, cudaStream_t st) {
  if (limit <= 0) return cudaSuccess;
  const int64_t threads = limit * 32;
  k_merge<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(keys, P, n, limit, k, inv_sigma, float_keys, row_list, row_count,
                                                             keys_by_row, nullptr, 0, out_keys, out_ids, out_scores);
  return cudaGetLastError();
}

cudaError_t launch_merge_keys_gated(const uint64_t* keys, int32_t P, int64_t n, int32_t k, const double* inv_sigma,
                                    const int32_t* gate, int gate_heads, uint64_t* out_keys, int32_t* out_ids,
                                    float* out_scores, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t threads = n * 32;
  k_merge<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(keys, P, n, n, k, inv_sigma, 0, nullptr, nullptr, 0, gate,
                                                             gate_heads, out_keys, out_ids, out_scores);
  return cudaGetLastError();
}

cudaError_t launch_merge_keys(const uint64_t* keys, int32_t P, int64_t n, int32_t k, const double* inv_sigma,
                              uint64_t* out_keys, int32_t* out_ids, float* out_scores, cudaStream_t st) {
  return launch_merge_keys_ex(keys, P, n, n, k, inv_sigma, 0, nullptr, nullptr, 0, out_keys, out_ids, out_scores, st);
}

namespace {

// warp per row; records the smallest offending row in *bad (as unsigned long long)
__global__ void k_validate(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const void* __restrict__ values, knnjoin_dtype dt, int64_t n, int64_t nnz, int32_t d,
                           unsigned long long* bad) {
  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= n) return;
  int64_t a = indptr[row], b = indptr[row + 1];
  bool ok = (a <= b) && a >= 0 && b <= nnz;
  if (row == 0 && a != 0) ok = false;
  if (row == n - 1 && b != nnz) ok = false;
  if (ok) {
    for (int64_t j = a + lane; j < b; j += 32) {
      int32_t f = indices[j];
      if (f < 0 || f >= d) ok = false;
      if (j > a && indices[j - 1] >= f) ok = false;
      if (dt == KNNJOIN_INT8 && ((const int8_t*)values)[j] <= 0) ok = false;
      if (dt == KNNJOIN_FP32) {
        float v = ((const float*)values)[j];
        if (!(v > 0.0f) || !isfinite(v)) ok = false;
      }
    }
  }
  if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicMin(bad, (unsigned long long)row);
}

}  // namespace
}  // namespace kj

using namespace kj;

KJ_API const char* knnjoin_last_error(void) { return g_err; }
KJ_API const char* knnjoin_version(void) { return "knnjoin-b200 0.1 (sm_100a)"; }

KJ_API size_t knnjoin_merge_workspace_bytes(const knnjoin_csr* R) {
  if (!R || R->n_rows < 0) { set_error("bad R"); return 0; }
  return align_up(8 * (size_t)R->n_rows, 256) + 256;
}

KJ_API knnjoin_status knnjoin_merge(const uint64_t* keys, int32_t P, const knnjoin_csr* R, int32_t d,
                                    knnjoin_dtype s_dtype, int32_t k, const knnjoin_merge_options* mopt,
                                    uint64_t* out_keys, int32_t* out_ids, float* out_scores,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  KJ_NVTX("knnjoin_merge");
  if (!R || P < 1 || k < 1 || k > kMaxK) { set_error("bad merge arguments (P %d, k %d)", P, k); return KNNJOIN_ERR_ARG; }
  if (!out_keys && !out_ids && !out_scores) { set_error("no output"); return KNNJOIN_ERR_ARG; }
  if (s_dtype != KNNJOIN_BINARY && s_dtype != KNNJOIN_INT8 && s_dtype != KNNJOIN_FP32) { set_error("bad S dtype"); return KNNJOIN_ERR_ARG; }
  const int float_keys = (s_dtype == KNNJOIN_FP32 || (mopt && mopt->float_keys)) ? 1 : 0;
  if (mopt && (mopt->row_list != nullptr) != (mopt->row_count != nullptr)) {
    set_error("row_list and row_count go together");
    return KNNJOIN_ERR_ARG;
  }
  size_t need = knnjoin_merge_workspace_bytes(R);
  if (!workspace || workspace_bytes < need) { set_error("merge workspace %zu < %zu", workspace_bytes, need); return KNNJOIN_ERR_WORKSPACE; }
  if (R->n_rows == 0) return KNNJOIN_OK;
  if (!keys) { set_error("keys is NULL"); return KNNJOIN_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  double* inv = (double*)workspace;
  if (d <= 0) { set_error("d must be > 0"); return KNNJOIN_ERR_DIM; }
  if (!float_keys) launch_row_scale(R, d, s_dtype == KNNJOIN_INT8 ? 127 : 1, nullptr, inv, nullptr, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "row scale");
  if ((e = launch_merge_keys_ex(keys, P, R->n_rows, R->n_rows, k, inv, float_keys, mopt ? mopt->row_list : nullptr,
                                mopt ? mopt->row_count : nullptr, 1, out_keys, out_ids, out_scores, st)) != cudaSuccess)
    return cuda_fail(e, "k_merge");
  return KNNJOIN_OK;
}

static std::mutex g_validate_mu;

KJ_API knnjoin_status knnjoin_validate_csr(const knnjoin_csr* m, int32_t d, void* stream, int64_t* bad_row) {
  KJ_NVTX("knnjoin_validate_csr");
  if (bad_row) *bad_row = -1;
  if (!m) { set_error("NULL csr"); return KNNJOIN_ERR_ARG; }
  if (d <= 0) { set_error("d must be > 0"); return KNNJOIN_ERR_DIM; }
  if (m->n_rows < 0 || m->nnz < 0) { set_error("negative sizes"); return KNNJOIN_ERR_CSR; }
  if (m->n_rows == 0) {
    if (m->nnz != 0) { set_error("n_rows == 0 but nnz != 0"); return KNNJOIN_ERR_CSR; }
    return KNNJOIN_OK;
  }
  if (!m->indptr || (m->nnz > 0 && !m->indices)) { set_error("NULL pointers"); return KNNJOIN_ERR_ARG; }
  if (m->dtype != KNNJOIN_BINARY && m->nnz > 0 && !m->values) { set_error("values missing for dtype %d", (int)m->dtype); return KNNJOIN_ERR_ARG; }
  std::lock_guard<std::mutex> lock(g_validate_mu);  // g_bad is one module-global word
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long init = ~0ull, hbad = ~0ull;
  cudaError_t e = cudaMemcpyToSymbolAsync(g_bad, &init, sizeof(init), 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "validate init");
  unsigned long long* dbad = nullptr;
  if ((e = cudaGetSymbolAddress((void**)&dbad, g_bad)) != cudaSuccess) return cuda_fail(e, "validate symbol");
  int64_t threads = m->n_rows * 32;
  k_validate<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(m->indptr, m->indices, m->values, m->dtype, m->n_rows,
                                                             m->nnz, d, dbad);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_validate");
  if ((e = cudaMemcpyFromSymbolAsync(&hbad, g_bad, sizeof(hbad), 0, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "validate readback");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "validate sync");
  if (hbad != ~0ull) {
    if (bad_row) *bad_row = (int64_t)hbad;
    set_error("invalid CSR row %lld", (long long)hbad);
    return KNNJOIN_ERR_CSR;
  }
  return KNNJOIN_OK;
}
