// topk.cuh -- warp-held top-k lists of packed keys.
//
// A key packs the total order of reading c1 (score desc, lower S id first) into one unsigned compare:
//     key = (uint64(score_u32) << 32) | (0xFFFFFFFF - global_id)
// A list of capacity k lives in registers across the 32 lanes of one warp: position p = s*32 + lane
// (slot s < KS = ceil(k/32)), sorted descending.  Empty positions hold 0, which is below kKeyFloor
// (score 0) and therefore below every admissible key; zero scores are never admitted (reading c2).
// "pruneScore(r)" of Alg. 2 is the key at position k-1 (kth()), or kKeyFloor while under-full (c3).
#pragma once
#include "common.cuh"

namespace kj {

__device__ __forceinline__ uint64_t make_key(uint32_t score, uint32_t gid) {
  return ((uint64_t)score << 32) | (uint64_t)(0xFFFFFFFFu - gid);
}

template <int KS>
__device__ __forceinline__ uint64_t list_kth(const uint64_t (&L)[KS], int k) {
  const int p = k - 1;
  uint64_t v = 0;
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    uint64_t t = __shfl_sync(0xffffffffu, L[s], p & 31);
    if (s == (p >> 5)) v = t;
  }
  return v > kKeyFloor ? v : kKeyFloor;
}

// Insert the warp-uniform key x (caller guarantees x > list_kth).  Elements at positions >= k are
// ignored by every reader; shifting keeps positions < k sorted.
template <int KS>
__device__ __forceinline__ void list_insert(uint64_t (&L)[KS], uint64_t x, int lane) {
  int pos = 0;
#pragma unroll
  for (int s = 0; s < KS; ++s) pos += __popc(__ballot_sync(0xffffffffu, L[s] > x));
#pragma unroll
  for (int s = KS - 1; s >= 0; --s) {
    uint64_t up = __shfl_up_sync(0xffffffffu, L[s], 1);
    uint64_t carry = 0;
    if (s > 0) carry = __shfl_sync(0xffffffffu, L[s > 0 ? s - 1 : 0], 31);
    if (lane == 0) up = carry;
    const int p = s * 32 + lane;
    if (p > pos) L[s] = up;
    else if (p == pos) L[s] = x;
  }
}

// Offer every lane's candidate `c` (0 = none) to the warp list; returns the number inserted.  theta is the
// caller's admission threshold (>= the list's own k-th key); it only ever rises.
template <int KS>
__device__ __forceinline__ int list_offer_lanes(uint64_t (&L)[KS], uint64_t c, uint64_t& theta, int k, int lane) {
  int n = 0;
  uint32_t m = __ballot_sync(0xffffffffu, c > theta);
  while (m) {
    int src = __ffs(m) - 1;
    m &= m - 1;
    uint64_t x = __shfl_sync(0xffffffffu, c, src);
    if (x > theta) {
      list_insert<KS>(L, x, lane);
      const uint64_t kth = list_kth<KS>(L, k);
      if (kth > theta) theta = kth;
      ++n;
    }
  }
  return n;
}

// Write positions < k of the list as (ids, scores, keys) of output row r (rank order).
template <int KS>
__device__ __forceinline__ void list_finalize(const uint64_t (&L)[KS], int k, int64_t r, double inv_sigma,
                                              uint64_t* out_keys, int32_t* out_ids, float* out_scores, int lane) {
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    const int p = s * 32 + lane;
    if (p < k) {
      uint64_t key = L[s];
      uint32_t score = (uint32_t)(key >> 32);
      size_t o = (size_t)r * k + p;
      if (score == 0) {
        if (out_keys) out_keys[o] = 0;
        if (out_ids) out_ids[o] = -1;
        if (out_scores) out_scores[o] = 0.0f;
      } else {
        if (out_keys) out_keys[o] = key;
        if (out_ids) out_ids[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)key);
        if (out_scores) out_scores[o] = (float)((double)score * inv_sigma);
      }
    }
  }
}

}  // namespace kj
