// iiib.cu -- f1: the paper's improved inverted-index algorithm IIIB (Alg. 4) literally, as
// device building blocks for one R block (all of R) and a sequence of S blocks:
//   knnjoin_iiib_profile    Alg. 4 lines 6-7: dimension order by non-zero count in the R block, maxWeight_d
//   knnjoin_iiib_threshold  MinPruneScore = min over the block's rows of pruneScore(r)
//   knnjoin_iiib_split      Alg. 4 lines 8-14: per s, t += maxWeight_d * w in that order; from the first feature
//                           with t > MinPruneScore on the features are indexed (s''), the rest stay in s'
// The S block is then indexed from s'' (knnjoin_build_index, prune = 1, forward = s') and queried with
// residual = 1 (Find_Matches_IIIB, lines 15-24: accumulate over I_d, then add dot(r, s') for every touched s).
#include <cub/cub.cuh>

#include "common.cuh"

namespace kj {
namespace {

// weight of entry j of a CSR as a real number (BINARY: 1)
__device__ __forceinline__ double weight_of(const void* values, knnjoin_dtype dt, int64_t j) {
  if (dt == KNNJOIN_FP32) return (double)((const float*)values)[j];
  if (dt == KNNJOIN_INT8) return (double)((const int8_t*)values)[j];
  return 1.0;
}

struct ProfileLayout {
  size_t maxw_at, cnt_at, rank_at, key_at, key2_at, iota_at, order_at, cub_at, cub_bytes, total;
};

bool profile_layout(int32_t d, ProfileLayout* L) {
  size_t sort_bytes = 0;
  if (cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                      (const int32_t*)nullptr, (int32_t*)nullptr, (int)d) != cudaSuccess)
    return false;
  size_t at = 0;
  L->maxw_at = at;  at = align_up(at + 8 * (size_t)d, 256);
  L->cnt_at = at;   at = align_up(at + 4 * (size_t)d, 256);
  L->rank_at = at;  at = align_up(at + 4 * (size_t)d, 256);
  L->key_at = at;   at = align_up(at + 4 * (size_t)d, 256);
  L->key2_at = at;  at = align_up(at + 4 * (size_t)d, 256);
  L->iota_at = at;  at = align_up(at + 4 * (size_t)d, 256);
  L->order_at = at; at = align_up(at + 4 * (size_t)d, 256);
  L->cub_at = at;
  L->cub_bytes = sort_bytes;
  at = align_up(at + sort_bytes, 256);
  L->total = at;
  return true;
}

// line 7: maxWeight_d(B_r) (positive doubles order like their bit patterns) and the non-zero count per d
__global__ void k_r_profile(const int32_t* __restrict__ indices, const void* __restrict__ values, knnjoin_dtype dt,
                            int64_t nnz, int32_t d, unsigned long long* __restrict__ maxw_bits,
                            uint32_t* __restrict__ cnt) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nnz) return;
  const int32_t f = indices[j];
  if (f < 0 || f >= d) return;
  atomicAdd(&cnt[f], 1u);
  atomicMax(&maxw_bits[f], (unsigned long long)__double_as_longlong(weight_of(values, dt, j)));
}

// line 6: sort key of dimension f = count descending (stable radix sort keeps dimension ascending among ties;
// dimensions absent from the block have count 0 and come last, ascending -- reading c10)
__global__ void k_rank_keys(const uint32_t* __restrict__ cnt, int32_t d, uint32_t* __restrict__ key,
                            int32_t* __restrict__ iota) {
  const int32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= d) return;
  key[f] = ~cnt[f];
  iota[f] = f;
}

__global__ void k_rank_scatter(const int32_t* __restrict__ order, int32_t d, int32_t* __restrict__ rank) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) rank[order[i]] = i;
}

// MinPruneScore over all rows from their current k-th keys, in real units: {min_r kth(r)/sigma_r,
// max_r 1/sigma_r}.  One CTA.
__global__ void k_iiib_threshold(const uint64_t* __restrict__ keys, int64_t n, int32_t k,
                                 const double* __restrict__ inv_sigma, double* __restrict__ out2) {
  using BR = cub::BlockReduce<double, 1024>;
  __shared__ typename BR::TempStorage tmp;
  double mn = 1e300, mx = 0.0;
  for (int64_t r = threadIdx.x; r < n; r += 1024) {
    const double kth = keys ? (double)(uint32_t)(keys[r * k + (k - 1)] >> 32) : 0.0;  // 0: under-full (c3)
    mn = fmin(mn, kth * inv_sigma[r]);
    mx = fmax(mx, inv_sigma[r]);
  }
  const double a = BR(tmp).Reduce(mn, cub::Min());
  __syncthreads();
  const double b = BR(tmp).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) {
    out2[0] = n > 0 ? a : 0.0;
    out2[1] = b;
  }
}

// lines 8-13 for one s (warp per row): with c_j = maxWeight(d_j) * w_j and the row's features in rank order,
// the indexed features are those at or after the first position where the running sum t exceeds the
// threshold, i.e. rank_j >= rho where rho = the smallest rank with sum_{rank_i <= rho} c_i > M.  Found by a
// binary search over rho (each step one warp reduction); rho = d when t never exceeds M.
__global__ void k_iiib_cut(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const int8_t* __restrict__ values, int64_t n, int32_t d,
                           const unsigned long long* __restrict__ maxw_bits, const int32_t* __restrict__ rank,
                           const double* __restrict__ thr, int32_t r_integer, int32_t* __restrict__ rho_out,
                           int64_t* __restrict__ n_idx, int64_t* __restrict__ n_res) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int64_t b = indptr[row], e = indptr[row + 1];
  // M: MinPruneScore; for FP32 R lowered by (sum_s w + 1) * max 1/sigma so that the fixed-point score of an
  // s reached only through s' stays below every row's fixed-point k-th score (reading c23)
  double wsum = 0.0;
  for (int64_t j = b + lane; j < e; j += 32) wsum += values ? (double)values[j] : 1.0;
#pragma unroll
  for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  const double M = r_integer ? thr[0] : thr[0] - (wsum + 1.0) * thr[1];
  auto prefix = [&](int32_t rho) {  // sum of c over the row's features with rank <= rho
    double t = 0.0;
    for (int64_t j = b + lane; j < e; j += 32) {
      const int32_t f = indices[j];
      if (f >= 0 && f < d && rank[f] <= rho)
        t += __longlong_as_double((long long)maxw_bits[f]) * (values ? (double)values[j] : 1.0);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
  };
  int32_t lo = 0, hi = d;  // smallest rho in [0, d) with prefix(rho) > M, or d
  if (!(prefix(d - 1) > M)) {
    lo = d;
  } else {
    hi = d - 1;
    while (lo < hi) {
      const int32_t mid = lo + ((hi - lo) >> 1);
      if (prefix(mid) > M) hi = mid; else lo = mid + 1;
    }
  }
  int64_t ni = 0;
  for (int64_t j = b + lane; j < e; j += 32) {
    const int32_t f = indices[j];
    ni += (f >= 0 && f < d ? rank[f] : d) >= lo ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ni += __shfl_xor_sync(0xffffffffu, ni, o);
  if (lane == 0) {
    rho_out[row] = lo;
    n_idx[row] = ni;
    n_res[row] = (e - b) - ni;
  }
}

// line 13-14: scatter every feature of s to I (s'') or to s', keeping feature order (warp per row, ballots)
__global__ void k_iiib_scatter(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                               const int8_t* __restrict__ values, int64_t n, int32_t d, const int32_t* __restrict__ rank,
                               const int32_t* __restrict__ rho, const int64_t* __restrict__ idx_indptr,
                               int32_t* __restrict__ idx_indices, int8_t* __restrict__ idx_values,
                               const int64_t* __restrict__ res_indptr, int32_t* __restrict__ res_indices,
                               int8_t* __restrict__ res_values) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int64_t b = indptr[row], e = indptr[row + 1];
  const int32_t cut = rho[row];
  int64_t oi = idx_indptr[row], orr = res_indptr[row];
  for (int64_t j0 = b; j0 < e; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool v = j < e;
    int32_t f = 0;
    bool ind = false;
    if (v) {
      f = indices[j];
      ind = (f >= 0 && f < d ? rank[f] : d) >= cut;
    }
    const uint32_t mi = __ballot_sync(0xffffffffu, v && ind), mr = __ballot_sync(0xffffffffu, v && !ind);
    const uint32_t below = (1u << lane) - 1u;
    if (v && ind) {
      const int64_t o = oi + __popc(mi & below);
      idx_indices[o] = f;
      if (values) idx_values[o] = values[j];
    } else if (v) {
      const int64_t o = orr + __popc(mr & below);
      res_indices[o] = f;
      if (values) res_values[o] = values[j];
    }
    oi += __popc(mi);
    orr += __popc(mr);
  }
}

struct SplitWs {
  size_t rho_at, ni_at, nr_at, cub_at, cub_bytes, total;
};

bool split_ws_layout(int64_t n, SplitWs* W) {
  size_t scan_bytes = 0;
  if (cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr,
                                    (int)(n > 0 ? n : 1)) != cudaSuccess)
    return false;
  size_t at = 0;
  W->rho_at = at; at = align_up(at + 4 * (size_t)n, 256);
  W->ni_at = at;  at = align_up(at + 8 * (size_t)n, 256);
  W->nr_at = at;  at = align_up(at + 8 * (size_t)n, 256);
  W->cub_at = at;
  W->cub_bytes = scan_bytes;
  at = align_up(at + scan_bytes, 256);
  W->total = at;
  return true;
}

}  // namespace
}  // namespace kj

using namespace kj;

KJ_API size_t knnjoin_iiib_profile_bytes(const knnjoin_csr* R, int32_t d) {
  if (!R || d <= 0) { set_error("R is NULL or d <= 0"); return 0; }
  ProfileLayout L;
  if (!profile_layout(d, &L)) { set_error("profile sizing failed"); return 0; }
  return L.total;
}

KJ_API knnjoin_status knnjoin_iiib_profile(const knnjoin_csr* R, int32_t d, void* profile, size_t profile_bytes,
                                           void* stream) {
  KJ_NVTX("knnjoin_iiib_profile");
  if (!R || d <= 0 || !profile) { set_error("R / profile NULL or d <= 0"); return KNNJOIN_ERR_ARG; }
  ProfileLayout L;
  if (!profile_layout(d, &L)) { set_error("profile sizing failed"); return KNNJOIN_ERR_ARG; }
  if (profile_bytes < L.total) { set_error("profile %zu < %zu bytes", profile_bytes, L.total); return KNNJOIN_ERR_WORKSPACE; }
  if (R->nnz > 0 && (!R->indices || (R->dtype != KNNJOIN_BINARY && !R->values))) { set_error("R pointers are NULL"); return KNNJOIN_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  char* pb = (char*)profile;
  cudaError_t e;
  if ((e = cudaMemsetAsync(pb + L.maxw_at, 0, 8 * (size_t)d, st)) != cudaSuccess) return cuda_fail(e, "memset maxw");
  if ((e = cudaMemsetAsync(pb + L.cnt_at, 0, 4 * (size_t)d, st)) != cudaSuccess) return cuda_fail(e, "memset cnt");
  if (R->nnz > 0)
    k_r_profile<<<(unsigned)((R->nnz + 255) / 256), 256, 0, st>>>(R->indices, R->values, R->dtype, R->nnz, d,
                                                                  (unsigned long long*)(pb + L.maxw_at),
                                                                  (uint32_t*)(pb + L.cnt_at));
  k_rank_keys<<<(unsigned)((d + 255) / 256), 256, 0, st>>>((const uint32_t*)(pb + L.cnt_at), d,
                                                           (uint32_t*)(pb + L.key_at), (int32_t*)(pb + L.iota_at));
  size_t cb = L.cub_bytes;
  if ((e = cub::DeviceRadixSort::SortPairs(pb + L.cub_at, cb, (const uint32_t*)(pb + L.key_at),
                                           (uint32_t*)(pb + L.key2_at), (const int32_t*)(pb + L.iota_at),
                                           (int32_t*)(pb + L.order_at), (int)d, 0, 32, st)) != cudaSuccess)
    return cuda_fail(e, "dimension sort");
  k_rank_scatter<<<(unsigned)((d + 255) / 256), 256, 0, st>>>((const int32_t*)(pb + L.order_at), d,
                                                              (int32_t*)(pb + L.rank_at));
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "iiib profile");
  return KNNJOIN_OK;
}

KJ_API size_t knnjoin_iiib_threshold_workspace_bytes(const knnjoin_csr* R) {
  if (!R || R->n_rows < 0) { set_error("bad R"); return 0; }
  return align_up(16 * (size_t)(R->n_rows > 0 ? R->n_rows : 1), 256);
}

KJ_API knnjoin_status knnjoin_iiib_threshold(const uint64_t* keys, const knnjoin_csr* R, int32_t d,
                                             knnjoin_dtype s_dtype, int32_t k, double* out2, void* workspace,
                                             size_t workspace_bytes, void* stream) {
  KJ_NVTX("knnjoin_iiib_threshold");
  if (!R || !out2 || d <= 0 || k < 1 || k > kMaxK) { set_error("bad iiib_threshold arguments"); return KNNJOIN_ERR_ARG; }
  if (!workspace || workspace_bytes < knnjoin_iiib_threshold_workspace_bytes(R)) {
    set_error("iiib_threshold workspace too small");
    return KNNJOIN_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* sigma = (double*)workspace;
  double* inv = sigma + (R->n_rows > 0 ? R->n_rows : 1);
  // the per-row scale of knnjoin_query (smax = 127 for INT8 S, 1 for BINARY S)
  launch_row_scale(R, d, s_dtype == KNNJOIN_INT8 ? 127 : 1, sigma, inv, nullptr, st);
  k_iiib_threshold<<<1, 1024, 0, st>>>(keys, R->n_rows, k, inv, out2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "iiib threshold");
  return KNNJOIN_OK;
}

KJ_API size_t knnjoin_iiib_split_workspace_bytes(const knnjoin_csr* S) {
  if (!S || S->n_rows < 0) { set_error("bad S"); return 0; }
  SplitWs W;
  if (!split_ws_layout(S->n_rows, &W)) { set_error("split sizing failed"); return 0; }
  return W.total;
}

KJ_API knnjoin_status knnjoin_iiib_split(const knnjoin_csr* S, int32_t d, const void* profile, const double* threshold,
                                         int32_t r_integer, int64_t* idx_indptr, int32_t* idx_indices,
                                         int8_t* idx_values, int64_t* res_indptr, int32_t* res_indices,
                                         int8_t* res_values, void* workspace, size_t workspace_bytes, void* stream) {
  KJ_NVTX("knnjoin_iiib_split");
  if (!S || d <= 0 || !profile || !threshold || !idx_indptr || !res_indptr) { set_error("bad iiib_split arguments"); return KNNJOIN_ERR_ARG; }
  if (S->dtype != KNNJOIN_BINARY && S->dtype != KNNJOIN_INT8) { set_error("S must be BINARY or INT8"); return KNNJOIN_ERR_UNSUPPORTED; }
  if (S->nnz > 0 && (!S->indices || !idx_indices || !res_indices ||
                     (S->dtype == KNNJOIN_INT8 && (!S->values || !idx_values || !res_values)))) {
    set_error("S / output pointers are NULL");
    return KNNJOIN_ERR_ARG;
  }
  SplitWs W;
  if (!split_ws_layout(S->n_rows, &W)) { set_error("split sizing failed"); return KNNJOIN_ERR_ARG; }
  if (!workspace || workspace_bytes < W.total) { set_error("iiib_split workspace too small"); return KNNJOIN_ERR_WORKSPACE; }
  ProfileLayout L;
  profile_layout(d, &L);
  cudaStream_t st = (cudaStream_t)stream;
  const char* pb = (const char*)profile;
  char* wb = (char*)workspace;
  int32_t* rho = (int32_t*)(wb + W.rho_at);
  int64_t* ni = (int64_t*)(wb + W.ni_at);
  int64_t* nr = (int64_t*)(wb + W.nr_at);
  const int8_t* sv = S->dtype == KNNJOIN_INT8 ? (const int8_t*)S->values : nullptr;
  cudaError_t e;
  if ((e = cudaMemsetAsync(idx_indptr, 0, 8, st)) != cudaSuccess) return cuda_fail(e, "memset indptr");
  if ((e = cudaMemsetAsync(res_indptr, 0, 8, st)) != cudaSuccess) return cuda_fail(e, "memset indptr");
  if (S->n_rows == 0) return KNNJOIN_OK;
  const unsigned grid = (unsigned)((S->n_rows * 32 + 255) / 256);
  k_iiib_cut<<<grid, 256, 0, st>>>(S->indptr, S->indices, sv, S->n_rows, d,
                                   (const unsigned long long*)(pb + L.maxw_at), (const int32_t*)(pb + L.rank_at),
                                   threshold, r_integer, rho, ni, nr);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_iiib_cut");
  size_t cb = W.cub_bytes;
  if ((e = cub::DeviceScan::InclusiveSum(wb + W.cub_at, cb, ni, idx_indptr + 1, (int)S->n_rows, st)) != cudaSuccess)
    return cuda_fail(e, "scan indexed");
  cb = W.cub_bytes;
  if ((e = cub::DeviceScan::InclusiveSum(wb + W.cub_at, cb, nr, res_indptr + 1, (int)S->n_rows, st)) != cudaSuccess)
    return cuda_fail(e, "scan residual");
  k_iiib_scatter<<<grid, 256, 0, st>>>(S->indptr, S->indices, sv, S->n_rows, d, (const int32_t*)(pb + L.rank_at), rho,
                                       idx_indptr, idx_indices, idx_values, res_indptr, res_indices, res_values);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_iiib_scatter");
  return KNNJOIN_OK;
}
