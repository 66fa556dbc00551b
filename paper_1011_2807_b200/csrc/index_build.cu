// index_build.cu -- K1: the tiled inverted index of S, built on the device.
//
// This is Create_Inverted_List_IIB (Alg. 3 lines 5-8: "for every feature (d, w) of
// every s insert (s, w) into I_d") re-shaped for the GPU.  The lists are partitioned into S-id tiles of
// `tile` ids (the analogue of Alg. 1's S blocks, sized so one tile's score array fits in shared memory)
// and laid out feature-major so that slice (f, t) = I_f ∩ tile t is contiguous:
//
//   off[f*(n_tiles+1) + t] .. off[f*(n_tiles+1) + t + 1]   16-byte posting units of slice (f, t)
//   ids[8*u .. 8*u+8)                                        8 local ids per unit, as byte offsets 4*(s - t*tile);
//                                                            padding entries hold 4*(tile + (u mod 32)), dummy columns
//   vals[8*u .. 8*u+8)                                       INT8 S weights (same positions)
//
// Head features.  For BINARY S, the (up to 32) most frequent features with df >= head_density * |S| are
// not stored as id lists at all: every S row s gets a 32-bit word head_cols[s] whose bit i says "s has
// head feature head_feat[i]".  The query bounds their contribution by a popcount and adds it exactly from
// per-batch lookup tables (4 features per table) only where the bound can beat the running k-th score
// (DESIGN.md "Head features").
//
// Steps (all stream-ordered, integer, deterministic, no contended atomics -- Zipf head features put every
// row of a tile on the same key, so a global-atomic histogram would serialise):
//   1. k_keys      key(s, f) = f*(n_tiles+1) + t(s) for every nonzero, value = (local id, weight)
//   2. CUB stable radix sort of (key, value) pairs -- CSR order is ascending s, so each key's postings come
//      out in ascending s (Alg. 3 inserts "in B_s scan order")
//   3. k_seg_first / k_seg_count: run-length of equal keys -> first[key], counts[key]; k_df: df[f] = |I_f|
//   4. head selection (k_head_select, one CTA): features with df >= min_df ranked by (df desc, f asc)
//   5. k_units: units(key) = ceil(count/8) (0 for head features); CUB exclusive scan: off = scan(units)
//   6. k_fill_pads, k_scatter (posting of sorted rank rho at position rho of its slice), k_block_layout:
//      in slices of at least 32 units every block (256 postings, or the final partial one) is ordered by
//      shared-memory bank (id mod 32), so slot j of the units holds postings of ~distinct banks; a slice of
//      m < 32 units is transposed (unit i holds sorted postings i, i+m, ..., i+7m) so the lanes of a warp
//      hit consecutive ids
//   7. k_head_cols: one 32-bit head word per S row.
// The paper counts this as Eq. 4's first term, sum |s_i| postings.
#include <cub/cub.cuh>

#include "common.cuh"

namespace kj {

int32_t resolve_tile(const knnjoin_options* opt) {
  int32_t t = (opt && opt->tile) ? opt->tile : kDefaultTile;
  if (t <= 0 || t > kMaxTile || t % kTileQuantum != 0) return -1;
  return t;
}

bool index_layout(const knnjoin_csr* S, int32_t d, int32_t tile, bool prune, IndexLayout* L, const knnjoin_csr* F) {
  if (!F) F = S;
  if (!S || d <= 0 || tile <= 0 || S->n_rows < 0 || S->nnz < 0) return false;
  L->n_tiles = (S->n_rows + tile - 1) / tile;
  L->n_off = (int64_t)d * (L->n_tiles + 1) + 1;
  int64_t slices = (int64_t)d * L->n_tiles;
  int64_t nonempty = S->nnz < slices ? S->nnz : slices;
  L->unit_cap = S->nnz / 8 + nonempty + 1;  // sum ceil(c/8) <= nnz/8 + 7/8 * #non-empty slices
  size_t at = 0;
  L->off_at = at;
  at = align_up(at + sizeof(uint32_t) * (size_t)L->n_off, 256);
  L->df_at = at;
  at = align_up(at + sizeof(int32_t) * (size_t)d, 256);
  L->head_slot_at = at;
  at = align_up(at + sizeof(int32_t) * (size_t)d, 256);
  L->head_feat_at = at;
  at = align_up(at + sizeof(int32_t) * (kMaxHead + 1), 256);  // [kMaxHead] features + n_head
  L->head_cols_at = at;
  at = align_up(at + sizeof(uint32_t) * (size_t)L->n_tiles * tile, 256);
  L->ids_at = at;
  at = align_up(at + 16 * (size_t)L->unit_cap, 256);
  L->vals_at = at;
  if (S->dtype == KNNJOIN_INT8) at = align_up(at + 8 * (size_t)L->unit_cap, 256);
  if (S->dtype == KNNJOIN_FP32) at = align_up(at + 32 * (size_t)L->unit_cap, 256);  // fp32 weights, 8 per unit
  L->wmax_at = at;  // largest S weight (u32 for BINARY / INT8, float bits for FP32)
  at = align_up(at + 4, 256);
  L->fwd_ptr_at = L->fwd_idx_at = L->fwd_val_at = L->fmax_at = at;
  if (prune) {
    L->fwd_ptr_at = at;
    at = align_up(at + sizeof(int64_t) * (size_t)(S->n_rows + 1), 256);
    L->fwd_idx_at = at;
    at = align_up(at + sizeof(int32_t) * (size_t)F->nnz, 256);
    L->fwd_val_at = at;
    if (S->dtype == KNNJOIN_INT8) at = align_up(at + (size_t)F->nnz, 256);
    L->fmax_at = at;
    if (S->dtype == KNNJOIN_INT8) at = align_up(at + sizeof(uint32_t) * (size_t)d, 256);
  }
  L->total = at;
  return true;
}

namespace {

struct BuildWs {
  size_t counts_at, units_at, first_at, endp_at, ka_at, kb_at, va_at, vb_at, cub_at,
      cub_bytes, total;
};

// the feature-key build applies (see k_keys_f)
bool use_fkey(const knnjoin_csr* S) {
  return S->dtype == KNNJOIN_BINARY || (S->dtype == KNNJOIN_INT8 && S->n_rows < ((int64_t)1 << 24));
}

int end_bit_for(int64_t max_key) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) <= max_key) ++b;
  return b;
}

bool build_ws_layout(const knnjoin_csr* S, int32_t d, const IndexLayout& L, BuildWs* W) {
  size_t nnz = (size_t)S->nnz, n_off = (size_t)L.n_off;
  size_t sort_bytes = 0, scan_bytes = 0;
  cudaError_t e = S->dtype == KNNJOIN_FP32
                      ? cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                        (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)nnz, 0,
                                                        end_bit_for(L.n_off - 1))
                      : cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                        (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)nnz, 0,
                                                        end_bit_for(L.n_off - 1));
  if (e != cudaSuccess) return false;
  e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n_off);
  if (e != cudaSuccess) return false;
  size_t at = 0;
  W->counts_at = at; at = align_up(at + 4 * n_off, 256);
  W->units_at = at;  at = align_up(at + 4 * n_off, 256);
  W->first_at = at;  at = align_up(at + 4 * n_off, 256);
  W->endp_at = at;   at = align_up(at + 4 * n_off, 256);
  W->ka_at = at;     at = align_up(at + 4 * nnz, 256);
  W->kb_at = at;     at = align_up(at + 4 * nnz, 256);
  // sort values: (local id | int8 weight << 16) as u32, or (local id | fp32 weight bits << 32) as u64 (FP32 S)
  const size_t vb = S->dtype == KNNJOIN_FP32 ? 8 : 4;
  W->va_at = at;     at = align_up(at + vb * nnz, 256);
  W->vb_at = at;     at = align_up(at + vb * nnz, 256);
  W->cub_at = at;
  W->cub_bytes = sort_bytes;
  if (scan_bytes > W->cub_bytes) W->cub_bytes = scan_bytes;
  at = align_up(at + W->cub_bytes, 256);
  W->total = at;
  return true;
}

bool check_build_args(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt, int32_t* tile) {
  if (!S) { set_error("S is NULL"); return false; }
  if (d <= 0) { set_error("d must be > 0 (got %d)", d); return false; }
  if (d >= (1 << 24)) { set_error("d must be < 2^24 (feature ids share a word with an 8-row mask)"); return false; }
  if (S->n_rows < 0 || S->nnz < 0) { set_error("negative S size"); return false; }
  if (S->dtype != KNNJOIN_BINARY && S->dtype != KNNJOIN_INT8 && S->dtype != KNNJOIN_FP32) {
    set_error("bad S dtype %d", (int)S->dtype);
    return false;
  }
  if (S->dtype == KNNJOIN_FP32 && opt && opt->prune) {
    set_error("FP32 S is queried at 64-bit fixed point only: prune = 1 (a6 / f1) needs BINARY or INT8 S");
    return false;
  }
  if (S->nnz >= ((int64_t)1 << 31)) { set_error("nnz(S) must be < 2^31 per index (shard S)"); return false; }
  *tile = resolve_tile(opt);
  if (*tile < 0) { set_error("tile must be a multiple of %d in [%d, %d]", kTileQuantum, kTileQuantum, kMaxTile); return false; }
  if (opt && opt->prune != 0 && opt->prune != 1) { set_error("options.prune must be 0 or 1"); return false; }
  if (opt && (!(opt->alpha >= 0.0f && opt->alpha <= 1.0f) || (opt->prune == 0 && opt->alpha != 0.0f))) {
    set_error("options.alpha must be in [0, 1] (0 = default), and 0 when prune = 0");
    return false;
  }
  if (opt && opt->head_max > kMaxHead) { set_error("head_max must be <= %d", kMaxHead); return false; }
  if (opt && opt->forward) {
    const knnjoin_csr* F = opt->forward;
    if (!opt->prune) { set_error("options.forward needs prune = 1"); return false; }
    if (F->n_rows != S->n_rows || F->dtype != S->dtype || F->nnz < 0) {
      set_error("options.forward must have S's row count and dtype");
      return false;
    }
  }
  if ((int64_t)d * ((S->n_rows + *tile - 1) / *tile + 1) + 1 >= ((int64_t)1 << 31)) {
    set_error("d * (n_tiles+1) too large for 32-bit slice keys; shard S or raise the tile width");
    return false;
  }
  return true;
}

// warp per S row.  Sort value: local id | weight << 16 (VT = u32: BINARY / INT8) or | fp32 bits << 32 (VT = u64)
template <typename VT>
__global__ void k_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                       const void* __restrict__ values, int64_t n_s, int32_t d, int32_t tile, int64_t n_tiles,
                       uint32_t* __restrict__ keys, VT* __restrict__ vals, uint32_t sentinel_key) {
  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= n_s) return;
  int64_t t = row / tile;
  uint32_t local = (uint32_t)(row - t * tile);
  for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32) {
    int32_t f = indices[j];
    if (f >= 0 && f < d) {
      keys[j] = (uint32_t)((int64_t)f * (n_tiles + 1) + t);
      if constexpr (sizeof(VT) == 8)
        vals[j] = (VT)local | ((VT)__float_as_uint(((const float*)values)[j]) << 32);
      else
        vals[j] = local | ((values ? (uint32_t)(uint8_t)((const int8_t*)values)[j] : 0u) << 16);
    } else {
      keys[j] = sentinel_key;
      vals[j] = 0;
    }
  }
}

// first sorted position of every present key
__global__ void k_seg_first(const uint32_t* __restrict__ keys, int64_t nnz, uint32_t sentinel_key,
                            uint32_t* __restrict__ first) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  uint32_t k = keys[i];
  if (k < sentinel_key && (i == 0 || keys[i - 1] != k)) first[k] = (uint32_t)i;
}

// posting count of every present key (absent keys keep the memset 0)
__global__ void k_seg_count(const uint32_t* __restrict__ keys, int64_t nnz, uint32_t sentinel_key,
                            const uint32_t* __restrict__ first, uint32_t* __restrict__ counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  uint32_t k = keys[i];
  if (k < sentinel_key && (i == nnz - 1 || keys[i + 1] != k)) counts[k] = (uint32_t)(i + 1) - first[k];
}

// ---- feature-key build (BINARY S, INT8 S with < 2^24 rows): the CSR is in row order, so a STABLE sort by the
// feature alone yields (feature, row) order -- the (feature, tile, row) order of the slice keys -- with
// ceil(log2(d + 1)) key bits instead of those of f * (n_tiles + 1) + t (one radix pass fewer at C4's sizes).
// Sort value: the row s (BINARY) or s << 8 | weight (INT8); the slice key is recomputed from (f, s / tile).
__global__ void k_keys_f(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                         const void* __restrict__ values, int64_t n_s, int32_t d, uint32_t* __restrict__ keys,
                         uint32_t* __restrict__ vals) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_s) return;
  for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32) {
    const int32_t f = indices[j];
    keys[j] = (f >= 0 && f < d) ? (uint32_t)f : (uint32_t)d;  // invalid features sort last (key d)
    vals[j] = values ? ((uint32_t)row << 8) | (uint32_t)(uint8_t)((const int8_t*)values)[j] : (uint32_t)row;
  }
}

__device__ __forceinline__ uint32_t fkey_slice(uint32_t f, uint32_t v, int wshift, uint32_t tile, int64_t n_tiles) {
  return (uint32_t)((int64_t)f * (n_tiles + 1) + (v >> wshift) / tile);
}

// segment bounds of every present slice key: first[key] = first sorted position, endp[key] = one past the last
// (both memset 0, so absent keys have count endp - first = 0)
__global__ void k_seg_f(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t nnz, int32_t d,
                        int wshift, uint32_t tile, int64_t n_tiles, uint32_t* __restrict__ first,
                        uint32_t* __restrict__ endp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const uint32_t f = keys[i];
  if (f >= (uint32_t)d) return;
  const uint32_t k = fkey_slice(f, vals[i], wshift, tile, n_tiles);
  if (i == 0 || keys[i - 1] != f || fkey_slice(f, vals[i - 1], wshift, tile, n_tiles) != k) first[k] = (uint32_t)i;
  if (i == nnz - 1 || keys[i + 1] != f || fkey_slice(f, vals[i + 1], wshift, tile, n_tiles) != k) endp[k] = (uint32_t)(i + 1);
}

__global__ void k_counts_f(const uint32_t* __restrict__ first, const uint32_t* __restrict__ endp, int64_t n,
                           uint32_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) counts[i] = endp[i] - first[i];
}

// posting of sorted rank rho goes to position rho of its slice (k_block_layout permutes inside blocks)
__global__ void k_scatter_f(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t nnz,
                            int32_t d, int wshift, uint32_t tile, int64_t n_tiles, const uint32_t* __restrict__ off,
                            const uint32_t* __restrict__ first, const uint32_t* __restrict__ units,
                            uint16_t* __restrict__ ids, uint8_t* __restrict__ wvals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const uint32_t f = keys[i];
  if (f >= (uint32_t)d) return;
  const uint32_t v = vals[i], srow = v >> wshift, t = srow / tile;
  const uint32_t k = (uint32_t)((int64_t)f * (n_tiles + 1) + t);
  if (units[k] == 0) return;  // head feature
  const uint32_t dst = (uint32_t)i - first[k];
  KJ_CHECK(dst < 8 * units[k]);
  const size_t pos = (size_t)off[k] * 8 + dst;
  ids[pos] = (uint16_t)((srow - t * tile) << 2);  // byte offset of the score column
  if (wvals) wvals[pos] = (uint8_t)(v & 0xFFu);
}

// warp per feature: df[f] = sum over tiles of counts[f][t]; also the (df, f) pairs for head selection
__global__ void k_df(const uint32_t* __restrict__ counts, int32_t d, int64_t n_tiles, int32_t* __restrict__ df) {
  int64_t f = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (f >= d) return;
  uint32_t s = 0;
  for (int64_t t = lane; t < n_tiles; t += 32) s += counts[f * (n_tiles + 1) + t];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) df[f] = (int32_t)s;
}

// one CTA: the first head_max features of the (df desc, f asc) order with df >= min_df become heads.  The
// features with df >= min_df are few (at most nnz / min_df, i.e. 8x the mean row length at the default density),
// so they are compacted into shared memory and each is placed by its rank among them; if more than kTopCap
// qualify, head_max rounds of "largest pair below the previous one" (block argmax) select them instead.
constexpr int kTopThreads = 1024;
constexpr int kTopCap = 4096;
__global__ void __launch_bounds__(kTopThreads) k_head_select(const int32_t* __restrict__ df, int32_t d,
                                                              uint32_t min_df, int32_t head_max,
                                                              int32_t* __restrict__ head_slot,
                                                              int32_t* __restrict__ head_feat) {
  __shared__ uint32_t c_df[kTopCap];
  __shared__ int32_t c_f[kTopCap];
  __shared__ int s_cnt;
  __shared__ unsigned long long s_best;
  const int tid = threadIdx.x;
  if (tid == 0) s_cnt = 0;
  for (int i = tid; i < kMaxHead; i += kTopThreads) head_feat[i] = -1;
  __syncthreads();
  if (head_max > 0 && min_df != 0xFFFFFFFFu) {
    const uint32_t lo = min_df > 0 ? min_df : 1u;
    for (int f = tid; f < d; f += kTopThreads) {
      const uint32_t v = (uint32_t)df[f];
      if (v >= lo) {
        const int at = atomicAdd(&s_cnt, 1);
        if (at < kTopCap) { c_df[at] = v; c_f[at] = f; }
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt <= kTopCap) {
      for (int i = tid; i < cnt; i += kTopThreads) {
        const uint32_t vi = c_df[i];
        const int32_t fi = c_f[i];
        int rank = 0;
        for (int j = 0; j < cnt; ++j) rank += (c_df[j] > vi || (c_df[j] == vi && c_f[j] < fi)) ? 1 : 0;
        if (rank < head_max) {
          head_feat[rank] = fi;
          head_slot[fi] = rank;
        }
      }
    } else {
      // packed order key: (df << 32) | (~f) -- larger key = earlier in (df desc, f asc)
      unsigned long long prev = ~0ull;
      for (int r = 0; r < head_max; ++r) {
        unsigned long long best = 0;
        for (int f = tid; f < d; f += kTopThreads) {
          const uint32_t v = (uint32_t)df[f];
          const unsigned long long key = ((unsigned long long)v << 32) | (unsigned long long)(~(uint32_t)f);
          if (v >= lo && key < prev && key > best) best = key;
        }
        if (tid == 0) s_best = 0;
        __syncthreads();
        if (best) atomicMax(&s_best, best);
        __syncthreads();
        prev = s_best;
        __syncthreads();
        if (prev == 0) break;
        if (tid == 0) {
          const int32_t f = (int32_t)(~(uint32_t)prev);
          head_feat[r] = f;
          head_slot[f] = r;
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int n = 0;
    if (head_max > 0 && min_df != 0xFFFFFFFFu) n = min(s_cnt, head_max);
    head_feat[kMaxHead] = n;  // n_head (heads are a prefix of the (df desc, f asc) order)
  }
}

__global__ void k_units(const uint32_t* __restrict__ counts, uint32_t* __restrict__ units, int64_t n,
                        int64_t n_tiles, const int32_t* __restrict__ head_slot) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = counts[i];
  uint32_t u = (c + 7u) >> 3;
  if (c && head_slot[i / (n_tiles + 1)] >= 0) u = 0;  // head features live in head_cols, not in id lists
  units[i] = u;
}

// padding entries point at one of 32 dummy score columns [tile, tile+32) (spread over banks by unit index),
// so the accumulation kernel issues its shared-memory atomics without a per-posting predicate
__global__ void k_fill_pads(uint4* __restrict__ ids, int64_t units, uint32_t tile) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= units) return;
  uint32_t pad = (tile + (uint32_t)(u & 31)) << 2;  // byte offset of a dummy column
  pad |= pad << 16;
  ids[u] = make_uint4(pad, pad, pad, pad);
}

// posting of sorted rank rho goes to position rho of its slice (k_block_layout permutes inside full blocks)
template <typename VT, typename WT>
__global__ void k_scatter(const uint32_t* __restrict__ keys, const VT* __restrict__ vals, int64_t nnz,
                          const uint32_t* __restrict__ off, const uint32_t* __restrict__ first,
                          const uint32_t* __restrict__ units, uint32_t sentinel_key, uint16_t* __restrict__ ids,
                          WT* __restrict__ wvals) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  uint32_t key = keys[i];
  if (key >= sentinel_key || units[key] == 0) return;  // invalid feature or head feature
  // rank rho inside the slice: a slice of fewer than 32 units (one partial block of m units) is transposed here
  // (position p -> unit p % m, slot p / m); longer slices keep rho and k_block_layout orders their blocks by
  // bank
  const uint32_t rho = (uint32_t)i - first[key];
  const uint32_t U = units[key], nfull = U / 32, m = U - 32 * nfull;
  uint32_t dst = rho;
  if (nfull == 0) dst = (rho % m) * 8 + rho / m;  // short slice (one partial block): transpose here
  const size_t pos = (size_t)off[key] * 8 + dst;
  KJ_CHECK(dst < 8 * U && key < sentinel_key);
  const VT v = vals[i];
  ids[pos] = (uint16_t)((v & 0xFFFFu) << 2);  // byte offset of the score column
  if (wvals) wvals[pos] = sizeof(VT) == 8 ? (WT)(v >> 32) : (WT)(v >> 16);
}

// Warp per slice of at least 32 units (grid-stride over keys; shorter slices were transposed by k_scatter):
// every block of m <= 32 units, stable counting sort by bank (id mod 32; padding last): rank r -> position r
// (unit r/8, slot r%8).  Deterministic: ranks come from slot-ordered
// match_any passes, not from the order of atomics.
template <typename WT>
__global__ void k_block_layout(const uint32_t* __restrict__ off, const uint32_t* __restrict__ units, int64_t n_keys,
                               uint32_t tile, uint16_t* __restrict__ ids, WT* __restrict__ wvals) {
  __shared__ uint32_t s_cnt[8][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* cnt = s_cnt[wib];
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t key = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; key < n_keys; key += nwarps) {
    const uint32_t U = units[key];
    if (U == 0) continue;
    const size_t base = (size_t)off[key] * 8;
    if (U < 32) continue;  // short slice: transposed by k_scatter
    const uint32_t nblk = (U + 31) / 32;
    for (uint32_t blk = 0; blk < nblk; ++blk) {
      const uint32_t m = min(32u, U - 32u * blk);
      const size_t b0 = base + (size_t)blk * 256;
      uint16_t id[8];
      WT w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) { id[j] = 0xFFFF; w[j] = 0; }
      if (lane < (int)m) {
        const uint4 x = *(const uint4*)(ids + b0 + 8 * lane);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) id[j] = (uint16_t)(xs[j >> 1] >> (16 * (j & 1)));
        if (wvals) {
#pragma unroll
          for (int j = 0; j < 8; ++j) w[j] = wvals[b0 + 8 * lane + j];
        }
      }
      // stable counting sort by bank (bucket 32 = padding, after every real posting; bucket 33 = lanes past
      // a partial block's m units, not counted): rank r -> unit r / 8, slot r % 8, so slot j of the units
      // holds ranks j, 8 + j, ...: postings spread across the bank order
      uint32_t dst[8];
      {
        cnt[lane] = 0;
        if (lane == 0) cnt[32] = 0;
        __syncwarp();
        const bool live = lane < (int)m;
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // bucket sizes
          const uint32_t bk = !live ? 33u : (id[j] >= 4 * tile ? 32u : ((id[j] >> 2) & 31u));
          const uint32_t peers = __match_any_sync(0xffffffffu, bk);
          if (bk < 33u && (peers & lt) == 0) cnt[bk] += __popc(peers);
          __syncwarp();
        }
        const uint32_t c = cnt[lane];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        __syncwarp();
        cnt[lane] = incl - c;
        if (lane == 31) cnt[32] = incl;  // padding after every real posting
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // ranks in (slot, lane) order within each bucket
          const uint32_t bk = !live ? 33u : (id[j] >= 4 * tile ? 32u : ((id[j] >> 2) & 31u));
          const uint32_t peers = __match_any_sync(0xffffffffu, bk);
          const uint32_t start = bk < 33u ? cnt[bk] : 0u;
          dst[j] = start + __popc(peers & lt);
          __syncwarp();
          if (bk < 33u && (peers & lt) == 0) cnt[bk] = start + __popc(peers);
          __syncwarp();
        }
      }
      __syncwarp();
      if (lane < (int)m) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          ids[b0 + dst[j]] = id[j];
          if (wvals) wvals[b0 + dst[j]] = w[j];
        }
      }
      __syncwarp();
    }
  }
}

// warp per S row: bit i of head_cols[row] <=> row has head feature head_feat[i]; tail columns of the last
// tile stay 0 (memset)
__global__ void k_head_cols(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t n_s,
                            int32_t d, const int32_t* __restrict__ head_slot, uint32_t* __restrict__ cols) {
  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= n_s) return;
  uint32_t w = 0;
  for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32) {
    const int32_t f = indices[j];
    if (f >= 0 && f < d) {
      const int32_t sl = head_slot[f];
      if (sl >= 0) w |= 1u << sl;
    }
  }
  w = __reduce_or_sync(0xffffffffu, w);
  if (lane == 0) cols[row] = w;
}

// pruned mode, INT8 S: the largest weight of every feature (an upper bound of s[d] for the pruning bound
// c_d = q_r[d] * maxweight(d))
__global__ void k_fmax(const int32_t* __restrict__ indices, const int8_t* __restrict__ values, int64_t nnz, int32_t d,
                       uint32_t* __restrict__ fmax) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const int32_t f = indices[i];
  if (f >= 0 && f < d) atomicMax(&fmax[f], (uint32_t)(uint8_t)values[i]);
}

// the largest weight of S (u32 for INT8; float bits for FP32 -- positive floats order like their bits): the
// 64-bit fixed-point scale of wide queries (wide.cu) keeps every partial score below 2^62 with it
// (grid-stride, one atomic per CTA: a per-warp atomic on the one word serialises at L2 -- 7.7 ms on C5's 375 M
// weights, measured)
__global__ void __launch_bounds__(256) k_wmax(const void* __restrict__ values, knnjoin_dtype dt, int64_t nnz,
                                              uint32_t* __restrict__ wmax) {
  __shared__ uint32_t s_max[8];
  uint32_t v = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (dt == KNNJOIN_FP32) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
      v = max(v, __float_as_uint(((const float*)values)[i]));
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
      v = max(v, (uint32_t)(uint8_t)((const int8_t*)values)[i]);
  }
  v = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? s_max[threadIdx.x] : 0u;
    v = __reduce_max_sync(0xffffffffu, v);
    if (threadIdx.x == 0 && v) atomicMax(wmax, v);
  }
}

}  // namespace

// minimum df of a head feature (0xFFFFFFFF = no heads); BINARY S only
uint32_t head_min_df(const knnjoin_csr* S, const knnjoin_options* opt) {
  if (S->dtype != KNNJOIN_BINARY || S->n_rows == 0) return 0xFFFFFFFFu;
  if (opt && opt->prune) return 0xFFFFFFFFu;  // pruned mode runs the head-free one-row kernel
  float dens = opt ? opt->head_density : 0.0f;
  if (dens < 0.0f) return 0xFFFFFFFFu;
  if (dens == 0.0f) dens = kDefaultHeadDensity;
  double m = ceil((double)dens * (double)S->n_rows);
  if (m < 1.0) m = 1.0;
  return m > 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)m;
}

}  // namespace kj

using namespace kj;

KJ_API size_t knnjoin_index_bytes(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt) {
  int32_t tile;
  if (!check_build_args(S, d, opt, &tile)) return 0;
  IndexLayout L;
  if (!index_layout(S, d, tile, opt && opt->prune, &L, opt ? opt->forward : nullptr)) { set_error("bad index layout arguments"); return 0; }
  return L.total;
}

KJ_API size_t knnjoin_build_workspace_bytes(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt) {
  int32_t tile;
  if (!check_build_args(S, d, opt, &tile)) return 0;
  IndexLayout L;
  BuildWs W;
  if (!index_layout(S, d, tile, opt && opt->prune, &L, opt ? opt->forward : nullptr) || !build_ws_layout(S, d, L, &W)) { set_error("workspace sizing failed"); return 0; }
  return W.total;
}

KJ_API knnjoin_status knnjoin_build_index(const knnjoin_csr* S, int32_t d, int64_t s_id_base,
                                          const knnjoin_options* opt, void* storage, size_t storage_bytes,
                                          void* workspace, size_t workspace_bytes, void* stream,
                                          knnjoin_index** out) {
  KJ_NVTX("knnjoin_build_index");
  if (!out) { set_error("out is NULL"); return KNNJOIN_ERR_ARG; }
  *out = nullptr;
  int32_t tile;
  if (!check_build_args(S, d, opt, &tile)) return (S && d <= 0) ? KNNJOIN_ERR_DIM : KNNJOIN_ERR_ARG;
  if (s_id_base < 0 || s_id_base + S->n_rows > (int64_t)0x7FFFFFFF) {
    set_error("global S ids must fit in int32 (s_id_base + n_rows < 2^31)");
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if (S->n_rows > 0 && (!S->indptr || (S->nnz > 0 && !S->indices))) { set_error("S pointers are NULL"); return KNNJOIN_ERR_ARG; }
  if (S->dtype != KNNJOIN_BINARY && S->nnz > 0 && !S->values) { set_error("INT8 / FP32 S needs values"); return KNNJOIN_ERR_ARG; }
  IndexLayout L;
  BuildWs W;
  if (!index_layout(S, d, tile, opt && opt->prune, &L, opt ? opt->forward : nullptr) || !build_ws_layout(S, d, L, &W)) { set_error("layout failed"); return KNNJOIN_ERR_ARG; }
  if (!storage || storage_bytes < L.total) { set_error("index storage %zu < %zu bytes", storage_bytes, L.total); return KNNJOIN_ERR_WORKSPACE; }
  if (!workspace || workspace_bytes < W.total) { set_error("build workspace %zu < %zu bytes", workspace_bytes, W.total); return KNNJOIN_ERR_WORKSPACE; }
  if (((uintptr_t)storage & 255) || ((uintptr_t)workspace & 255)) { set_error("storage and workspace must be 256-byte aligned"); return KNNJOIN_ERR_ARG; }

  cudaStream_t st = (cudaStream_t)stream;
  char* sb = (char*)storage;
  char* wb = (char*)workspace;
  uint32_t* off = (uint32_t*)(sb + L.off_at);
  int32_t* df = (int32_t*)(sb + L.df_at);
  int32_t* head_slot = (int32_t*)(sb + L.head_slot_at);
  int32_t* head_feat = (int32_t*)(sb + L.head_feat_at);
  uint32_t* head_cols = (uint32_t*)(sb + L.head_cols_at);
  uint16_t* ids = (uint16_t*)(sb + L.ids_at);
  uint8_t* vals = S->dtype == KNNJOIN_INT8 ? (uint8_t*)(sb + L.vals_at) : nullptr;
  uint32_t* vals32 = S->dtype == KNNJOIN_FP32 ? (uint32_t*)(sb + L.vals_at) : nullptr;  // fp32 weight bits
  uint32_t* wmax = (uint32_t*)(sb + L.wmax_at);
  const bool f32 = S->dtype == KNNJOIN_FP32;
  uint32_t* counts = (uint32_t*)(wb + W.counts_at);
  uint32_t* units = (uint32_t*)(wb + W.units_at);
  uint32_t* first = (uint32_t*)(wb + W.first_at);
  uint32_t* ka = (uint32_t*)(wb + W.ka_at);
  uint32_t* kb = (uint32_t*)(wb + W.kb_at);
  uint32_t* va = (uint32_t*)(wb + W.va_at);
  uint32_t* vb = (uint32_t*)(wb + W.vb_at);
  uint64_t* va64 = (uint64_t*)va;
  uint64_t* vb64 = (uint64_t*)vb;
  void* cubtmp = wb + W.cub_at;
  const uint32_t sentinel_key = (uint32_t)(L.n_off - 1);
  const uint32_t min_df = head_min_df(S, opt);
  int32_t head_max = (opt && opt->head_max > 0) ? opt->head_max : kMaxHead;
  if (min_df == 0xFFFFFFFFu) head_max = 0;

  cudaError_t e;
  if ((e = cudaMemsetAsync(counts, 0, 4 * (size_t)L.n_off, st)) != cudaSuccess) return cuda_fail(e, "memset counts");
  if ((e = cudaMemsetAsync(head_slot, 0xFF, 4 * (size_t)d, st)) != cudaSuccess) return cuda_fail(e, "memset head_slot");
  if ((e = cudaMemsetAsync(head_cols, 0, 4 * (size_t)L.n_tiles * tile, st)) != cudaSuccess) return cuda_fail(e, "memset head_cols");
  if (vals && (e = cudaMemsetAsync(vals, 0, 8 * (size_t)L.unit_cap, st)) != cudaSuccess) return cuda_fail(e, "memset vals");
  if (vals32 && (e = cudaMemsetAsync(vals32, 0, 32 * (size_t)L.unit_cap, st)) != cudaSuccess) return cuda_fail(e, "memset vals");
  if ((e = cudaMemsetAsync(wmax, 0, 4, st)) != cudaSuccess) return cuda_fail(e, "memset wmax");
  if (S->dtype == KNNJOIN_BINARY) {
    if ((e = cudaMemsetAsync(wmax, 0x01, 1, st)) != cudaSuccess) return cuda_fail(e, "wmax");  // weight 1
  } else if (S->nnz > 0) {
    {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t want = (S->nnz + 255) / 256, cap = (int64_t)sms * 8;
      k_wmax<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(S->values, S->dtype, S->nnz, wmax);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_wmax");
  }
  const unsigned gnnz = (unsigned)((S->nnz + 255) / 256);
  const bool fkey = use_fkey(S);
  const int wshift = S->dtype == KNNJOIN_INT8 ? 8 : 0;
  uint32_t* endp = (uint32_t*)(wb + W.endp_at);
  if (fkey && S->nnz > 0) {
    if ((e = cudaMemsetAsync(first, 0, 4 * (size_t)L.n_off, st)) != cudaSuccess) return cuda_fail(e, "memset first");
    if ((e = cudaMemsetAsync(endp, 0, 4 * (size_t)L.n_off, st)) != cudaSuccess) return cuda_fail(e, "memset endp");
    const int64_t threads = S->n_rows * 32;
    k_keys_f<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(S->indptr, S->indices, wshift ? S->values : nullptr,
                                                                S->n_rows, d, ka, va);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_keys_f");
    size_t tb = W.cub_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(cubtmp, tb, ka, kb, va, vb, (int)S->nnz, 0, end_bit_for(d), st)) != cudaSuccess)
      return cuda_fail(e, "radix sort");
    k_seg_f<<<gnnz, 256, 0, st>>>(kb, vb, S->nnz, d, wshift, (uint32_t)tile, L.n_tiles, first, endp);
    k_counts_f<<<(unsigned)((L.n_off + 255) / 256), 256, 0, st>>>(first, endp, L.n_off, counts);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_seg_f");
  } else if (S->nnz > 0) {
    int64_t threads = S->n_rows * 32;
    if (f32)
      k_keys<uint64_t><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(S->indptr, S->indices, S->values, S->n_rows, d,
                                                                        tile, L.n_tiles, ka, va64, sentinel_key);
    else
      k_keys<uint32_t><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(S->indptr, S->indices, S->values, S->n_rows, d,
                                                                        tile, L.n_tiles, ka, va, sentinel_key);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_keys");
    size_t tb = W.cub_bytes;
    e = f32 ? cub::DeviceRadixSort::SortPairs(cubtmp, tb, ka, kb, va64, vb64, (int)S->nnz, 0, end_bit_for(L.n_off - 1), st)
            : cub::DeviceRadixSort::SortPairs(cubtmp, tb, ka, kb, va, vb, (int)S->nnz, 0, end_bit_for(L.n_off - 1), st);
    if (e != cudaSuccess) return cuda_fail(e, "radix sort");
    k_seg_first<<<gnnz, 256, 0, st>>>(kb, S->nnz, sentinel_key, first);
    k_seg_count<<<gnnz, 256, 0, st>>>(kb, S->nnz, sentinel_key, first, counts);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_seg");
  }
  k_df<<<(unsigned)(((int64_t)d * 32 + 255) / 256), 256, 0, st>>>(counts, d, L.n_tiles, df);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_df");
  k_head_select<<<1, kTopThreads, 0, st>>>(df, d, min_df, head_max, head_slot, head_feat);
  k_units<<<(unsigned)((L.n_off + 255) / 256), 256, 0, st>>>(counts, units, L.n_off, L.n_tiles, head_slot);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_units");
  {
    size_t tb = W.cub_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(cubtmp, tb, units, off, (int)L.n_off, st)) != cudaSuccess) return cuda_fail(e, "scan off");
  }
  k_fill_pads<<<(unsigned)((L.unit_cap + 255) / 256), 256, 0, st>>>((uint4*)ids, L.unit_cap, (uint32_t)tile);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_fill_pads");
  if (S->nnz > 0) {
    if (fkey)
      k_scatter_f<<<gnnz, 256, 0, st>>>(kb, vb, S->nnz, d, wshift, (uint32_t)tile, L.n_tiles, off, first, units, ids, vals);
    else if (f32)
      k_scatter<<<gnnz, 256, 0, st>>>(kb, vb64, S->nnz, off, first, units, sentinel_key, ids, vals32);
    else
      k_scatter<<<gnnz, 256, 0, st>>>(kb, vb, S->nnz, off, first, units, sentinel_key, ids, vals);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_scatter");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (L.n_off - 1 + 7) / 8;
    const int64_t cap = (int64_t)sms * 16;
    const unsigned grid = (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
    if (f32)
      k_block_layout<<<grid, 256, 0, st>>>(off, units, L.n_off - 1, (uint32_t)tile, ids, vals32);
    else
      k_block_layout<<<grid, 256, 0, st>>>(off, units, L.n_off - 1, (uint32_t)tile, ids, vals);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_block_layout");
    if (head_max > 0) {
      int64_t threads = S->n_rows * 32;
      k_head_cols<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(S->indptr, S->indices, S->n_rows, d, head_slot,
                                                                   head_cols);
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_head_cols");
    }
  }
  const bool prune = opt && opt->prune;
  int64_t* fwd_ptr = nullptr;
  int32_t* fwd_idx = nullptr;
  uint8_t* fwd_val = nullptr;
  uint32_t* fmax = nullptr;
  if (prune) {  // forward rows for the exact completions of pruned queries (a6) / residual rows s' (f1)
    const knnjoin_csr* F = opt->forward ? opt->forward : S;
    if (F->n_rows > 0 && (!F->indptr || (F->nnz > 0 && (!F->indices || (S->dtype == KNNJOIN_INT8 && !F->values))))) {
      set_error("forward CSR pointers are NULL");
      return KNNJOIN_ERR_ARG;
    }
    fwd_ptr = (int64_t*)(sb + L.fwd_ptr_at);
    fwd_idx = (int32_t*)(sb + L.fwd_idx_at);
    if (F->n_rows > 0 &&
        (e = cudaMemcpyAsync(fwd_ptr, F->indptr, 8 * (size_t)(F->n_rows + 1), cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "copy forward indptr");
    if (F->n_rows == 0 && (e = cudaMemsetAsync(fwd_ptr, 0, 8, st)) != cudaSuccess) return cuda_fail(e, "memset indptr");
    if (F->nnz > 0 &&
        (e = cudaMemcpyAsync(fwd_idx, F->indices, 4 * (size_t)F->nnz, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "copy forward indices");
    if (S->dtype == KNNJOIN_INT8) {
      fwd_val = (uint8_t*)(sb + L.fwd_val_at);
      fmax = (uint32_t*)(sb + L.fmax_at);
      if (F->nnz > 0 &&
          (e = cudaMemcpyAsync(fwd_val, F->values, (size_t)F->nnz, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "copy forward values");
      if ((e = cudaMemsetAsync(fmax, 0, 4 * (size_t)d, st)) != cudaSuccess) return cuda_fail(e, "memset fmax");
      if (S->nnz > 0) {
        k_fmax<<<gnnz, 256, 0, st>>>(S->indices, (const int8_t*)S->values, S->nnz, d, fmax);
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_fmax");
      }
    }
  }
  knnjoin_index* h = new (std::nothrow) knnjoin_index();
  if (!h) { set_error("host allocation failed"); return KNNJOIN_ERR_ARG; }
  h->n_s = S->n_rows;
  h->s_id_base = s_id_base;
  h->d = d;
  h->tile = tile;
  h->n_tiles = L.n_tiles;
  h->n_off = L.n_off;
  h->unit_cap = L.unit_cap;
  h->s_dtype = S->dtype;
  h->head_min_df = min_df;
  h->head_max = head_max;
  h->off = off;
  h->df = df;
  h->head_slot = head_slot;
  h->head_feat = head_feat;
  h->head_cols = head_cols;
  h->ids = ids;
  h->vals = vals;
  h->vals32 = vals32;
  h->wmax = wmax;
  h->prune = prune ? 1 : 0;
  h->alpha = prune ? (opt->alpha > 0.0f ? opt->alpha : kDefaultPruneAlpha) : 0.0f;
  h->fwd_ptr = fwd_ptr;
  h->fwd_idx = fwd_idx;
  h->fwd_val = fwd_val;
  h->fmax = fmax;
  h->storage_bytes = L.total;
  h->fwd_bytes = prune ? L.total - L.fwd_ptr_at : 0;
  *out = h;
  return KNNJOIN_OK;
}

KJ_API knnjoin_status knnjoin_index_stats(const knnjoin_index* idx, knnjoin_index_info* out) {
  if (!idx || !out) { set_error("NULL argument"); return KNNJOIN_ERR_ARG; }
  out->n_s = idx->n_s;
  out->s_id_base = idx->s_id_base;
  out->d = idx->d;
  out->tile = idx->tile;
  out->n_tiles = idx->n_tiles;
  out->offsets = idx->n_off;
  out->unit_capacity = idx->unit_cap;
  out->storage_bytes = (int64_t)idx->storage_bytes;
  out->s_dtype = idx->s_dtype;
  out->head_min_df = idx->head_min_df == 0xFFFFFFFFu ? -1 : (int64_t)idx->head_min_df;
  out->head_max = idx->head_max;
  out->prune = idx->prune;
  out->alpha = idx->alpha;
  return KNNJOIN_OK;
}

KJ_API void knnjoin_free_index(knnjoin_index* idx) { delete idx; }
