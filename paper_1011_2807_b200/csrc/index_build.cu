// index_build.cu -- K1: the tiled inverted index of S, built on the device.
//
// This is Create_Inverted_List_IIB (Alg. 3 lines 5-8: "for every feature (d, w) of
// every s insert (s, w) into I_d") re-shaped for the GPU: the lists are partitioned into S-id tiles of
// `tile` ids (the analogue of Alg. 1's S blocks, sized so one tile's score array fits in shared memory)
// and laid out feature-major so that slice (f, t) = I_f ∩ tile t is contiguous:
//
//   off[f*(n_tiles+1) + t] .. off[f*(n_tiles+1) + t + 1]   16-byte posting units of slice (f, t)
//   ids[8*u .. 8*u+8)                                        8 local ids (s - t*tile) per unit; padding
//                                                            entries hold tile + (u mod 32), a dummy column
//   vals[8*u .. 8*u+8)                                       INT8 S weights (same positions)
//
// Steps (all stream-ordered, integer, deterministic, no contended atomics -- Zipf head features put every
// row of a tile on the same key, so a global-atomic histogram would serialise):
//   1. k_keys      key(s, f) = f*(n_tiles+1) + t(s) for every nonzero, value = (local id, weight)
//   2. CUB stable radix sort of (key, value) pairs -- CSR order is ascending s, so each key's postings come
//      out in ascending s (Alg. 3 inserts "in B_s scan order")
//   3. k_seg_first / k_seg_count: run-length of equal keys -> first[key], counts[key]; k_df: df[f] = |I_f|
//   4. k_units     units(key) = ceil(count/8) (16-byte alignment), or tile/128 for a bitmap slice;
//      CUB exclusive scan: off = scan(units)
//   5. k_scatter   posting of sorted rank rho inside slice goes to block rho/256, and inside a block of m
//      units to lane i = rho%m, slot j = rho/m (unit i holds sorted postings i, i+m, ..., i+7m): when a
//      warp's lane i loads unit i and issues atomic j, the 32 lanes hit 32 consecutive ids of a dense
//      slice -> 32 distinct shared-memory banks.
//      Dense slices (>= dense_min postings, BINARY S) are instead a tile-wide bitmap (bit = local id).
//   6. k_mark_dense sets bit 31 of a dense slice's start offset.
// The paper counts this as Eq. 4's first term, sum |s_i| postings.
#include <cub/cub.cuh>

#include "common.cuh"

namespace kj {

int32_t resolve_tile(const knnjoin_options* opt) {
  int32_t t = (opt && opt->tile) ? opt->tile : kDefaultTile;
  if (t <= 0 || t > kMaxTile || t % kTileQuantum != 0) return -1;
  return t;
}

bool index_layout(const knnjoin_csr* S, int32_t d, int32_t tile, IndexLayout* L) {
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
  L->ids_at = at;
  at = align_up(at + 16 * (size_t)L->unit_cap, 256);
  L->vals_at = at;
  if (S->dtype == KNNJOIN_INT8) at = align_up(at + 8 * (size_t)L->unit_cap, 256);
  L->total = at;
  return true;
}

// postings from which a slice is stored as a bitmap (0xFFFFFFFF = never); BINARY S only
uint32_t dense_threshold(const knnjoin_csr* S, int32_t tile, const knnjoin_options* opt) {
  if (S->dtype != KNNJOIN_BINARY) return 0xFFFFFFFFu;
  int32_t v = opt ? opt->dense_min : 0;
  if (v < 0) return 0xFFFFFFFFu;
  if (v == 0) v = tile / 4;
  if (v < tile / 16) v = tile / 16;
  return (uint32_t)v;
}

namespace {

struct BuildWs {
  size_t counts_at, units_at, first_at, ka_at, kb_at, va_at, vb_at, cub_at, cub_bytes, total;
};

int end_bit_for(int64_t max_key) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) <= max_key) ++b;
  return b;
}

bool build_ws_layout(const knnjoin_csr* S, const IndexLayout& L, BuildWs* W) {
  size_t nnz = (size_t)S->nnz, n_off = (size_t)L.n_off;
  size_t sort_bytes = 0, scan_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)nnz, 0,
                                                  end_bit_for(L.n_off - 1));
  if (e != cudaSuccess) return false;
  e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n_off);
  if (e != cudaSuccess) return false;
  size_t at = 0;
  W->counts_at = at; at = align_up(at + 4 * n_off, 256);
  W->units_at = at;  at = align_up(at + 4 * n_off, 256);
  W->first_at = at;  at = align_up(at + 4 * n_off, 256);
  W->ka_at = at;     at = align_up(at + 4 * nnz, 256);
  W->kb_at = at;     at = align_up(at + 4 * nnz, 256);
  W->va_at = at;     at = align_up(at + 4 * nnz, 256);
  W->vb_at = at;     at = align_up(at + 4 * nnz, 256);
  W->cub_at = at;
  W->cub_bytes = sort_bytes > scan_bytes ? sort_bytes : scan_bytes;
  at = align_up(at + W->cub_bytes, 256);
  W->total = at;
  return true;
}

bool check_build_args(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt, int32_t* tile) {
  if (!S) { set_error("S is NULL"); return false; }
  if (d <= 0) { set_error("d must be > 0 (got %d)", d); return false; }
  if (d >= (1 << 24)) { set_error("d must be < 2^24 (feature ids share a word with an 8-row mask)"); return false; }
  if (S->n_rows < 0 || S->nnz < 0) { set_error("negative S size"); return false; }
  if (S->dtype != KNNJOIN_BINARY && S->dtype != KNNJOIN_INT8) {
    set_error("S dtype %d unsupported: S must be BINARY or INT8 (DESIGN.md: fixed-point scores)", (int)S->dtype);
    return false;
  }
  if (S->nnz >= ((int64_t)1 << 31)) { set_error("nnz(S) must be < 2^31 per index (shard S)"); return false; }
  *tile = resolve_tile(opt);
  if (*tile < 0) { set_error("tile must be a multiple of %d in [%d, %d]", kTileQuantum, kTileQuantum, kMaxTile); return false; }
  if (opt && (opt->prune != 0)) { set_error("pruned mode is not available in this build (options.prune must be 0)"); return false; }
  if ((int64_t)d * ((S->n_rows + *tile - 1) / *tile + 1) + 1 >= ((int64_t)1 << 31)) {
    set_error("d * (n_tiles+1) too large for 32-bit slice keys; shard S or raise the tile width");
    return false;
  }
  return true;
}

// warp per S row
__global__ void k_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                       const int8_t* __restrict__ values, int64_t n_s, int32_t d, int32_t tile, int64_t n_tiles,
                       uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t sentinel_key) {
  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= n_s) return;
  int64_t t = row / tile;
  uint32_t local = (uint32_t)(row - t * tile);
  for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32) {
    int32_t f = indices[j];
    if (f >= 0 && f < d) {
      keys[j] = (uint32_t)((int64_t)f * (n_tiles + 1) + t);
      vals[j] = local | ((values ? (uint32_t)(uint8_t)values[j] : 0u) << 16);
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

// warp per feature: df[f] = sum over tiles of counts[f][t]
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

// padding entries point at one of 32 dummy score columns [tile, tile+32) (spread over banks by unit index),
// so the accumulation kernel issues its shared-memory atomics without a per-posting predicate
__global__ void k_fill_pads(uint4* __restrict__ ids, int64_t units, uint32_t tile) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= units) return;
  uint32_t pad = tile + (uint32_t)(u & 31);
  pad |= pad << 16;
  ids[u] = make_uint4(pad, pad, pad, pad);
}

__global__ void k_units(const uint32_t* __restrict__ counts, uint32_t* __restrict__ units, int64_t n,
                        uint32_t dense_min, uint32_t dense_units) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t c = counts[i];
    units[i] = c >= dense_min ? dense_units : (c + 7u) >> 3;
  }
}

// zero the bitmap of every dense slice (the pad fill wrote dummy ids there)
__global__ void k_zero_dense(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ off, int64_t n,
                             uint32_t dense_min, uint32_t dense_units, uint4* __restrict__ ids) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || counts[i] < dense_min) return;
  uint4* b = ids + off[i];
  for (uint32_t u = 0; u < dense_units; ++u) b[u] = make_uint4(0, 0, 0, 0);
}

__global__ void k_mark_dense(const uint32_t* __restrict__ counts, uint32_t* __restrict__ off, int64_t n,
                             uint32_t dense_min) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && counts[i] >= dense_min) off[i] |= kDenseFlag;
}

__global__ void k_scatter(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t nnz,
                          const uint32_t* __restrict__ off, const uint32_t* __restrict__ first,
                          const uint32_t* __restrict__ counts, uint32_t dense_min, uint32_t sentinel_key,
                          uint16_t* __restrict__ ids, uint8_t* __restrict__ wvals) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  uint32_t key = keys[i];
  if (key >= sentinel_key) return;
  uint32_t u0 = off[key];
  if (counts[key] >= dense_min) {  // bitmap slice: bit `local id`
    uint32_t local = vals[i] & 0xFFFFu;
    atomicOr((uint32_t*)ids + (size_t)u0 * 4 + (local >> 5), 1u << (local & 31));
    return;
  }
  uint32_t rank = (uint32_t)i - first[key];
  uint32_t U = off[key + 1] - u0;
  uint32_t beta = rank >> 8, iota = rank & 255u;
  uint32_t m = U - 32u * beta;
  if (m > 32u) m = 32u;
  uint32_t ii = iota % m, jj = iota / m;
  size_t pos = (size_t)u0 * 8 + (size_t)beta * 256 + ii * 8 + jj;
  uint32_t v = vals[i];
  ids[pos] = (uint16_t)(v & 0xFFFFu);
  if (wvals) wvals[pos] = (uint8_t)(v >> 16);
}

}  // namespace
}  // namespace kj

using namespace kj;

KJ_API size_t knnjoin_index_bytes(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt) {
  int32_t tile;
  if (!check_build_args(S, d, opt, &tile)) return 0;
  IndexLayout L;
  if (!index_layout(S, d, tile, &L)) { set_error("bad index layout arguments"); return 0; }
  return L.total;
}

KJ_API size_t knnjoin_build_workspace_bytes(const knnjoin_csr* S, int32_t d, const knnjoin_options* opt) {
  int32_t tile;
  if (!check_build_args(S, d, opt, &tile)) return 0;
  IndexLayout L;
  BuildWs W;
  if (!index_layout(S, d, tile, &L) || !build_ws_layout(S, L, &W)) { set_error("workspace sizing failed"); return 0; }
  return W.total;
}

KJ_API knnjoin_status knnjoin_build_index(const knnjoin_csr* S, int32_t d, int64_t s_id_base,
                                          const knnjoin_options* opt, void* storage, size_t storage_bytes,
                                          void* workspace, size_t workspace_bytes, void* stream,
                                          knnjoin_index** out) {
  if (!out) { set_error("out is NULL"); return KNNJOIN_ERR_ARG; }
  *out = nullptr;
  int32_t tile;
  if (!check_build_args(S, d, opt, &tile)) return (S && d <= 0) ? KNNJOIN_ERR_DIM : KNNJOIN_ERR_ARG;
  if (S->dtype != KNNJOIN_BINARY && S->dtype != KNNJOIN_INT8) return KNNJOIN_ERR_UNSUPPORTED;
  if (s_id_base < 0 || s_id_base + S->n_rows > (int64_t)0x7FFFFFFF) {
    set_error("global S ids must fit in int32 (s_id_base + n_rows < 2^31)");
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if (S->n_rows > 0 && (!S->indptr || (S->nnz > 0 && !S->indices))) { set_error("S pointers are NULL"); return KNNJOIN_ERR_ARG; }
  if (S->dtype == KNNJOIN_INT8 && S->nnz > 0 && !S->values) { set_error("INT8 S needs values"); return KNNJOIN_ERR_ARG; }
  IndexLayout L;
  BuildWs W;
  if (!index_layout(S, d, tile, &L) || !build_ws_layout(S, L, &W)) { set_error("layout failed"); return KNNJOIN_ERR_ARG; }
  if (!storage || storage_bytes < L.total) { set_error("index storage %zu < %zu bytes", storage_bytes, L.total); return KNNJOIN_ERR_WORKSPACE; }
  if (!workspace || workspace_bytes < W.total) { set_error("build workspace %zu < %zu bytes", workspace_bytes, W.total); return KNNJOIN_ERR_WORKSPACE; }
  if (((uintptr_t)storage & 255) || ((uintptr_t)workspace & 255)) { set_error("storage and workspace must be 256-byte aligned"); return KNNJOIN_ERR_ARG; }

  cudaStream_t st = (cudaStream_t)stream;
  char* sb = (char*)storage;
  char* wb = (char*)workspace;
  uint32_t* off = (uint32_t*)(sb + L.off_at);
  int32_t* df = (int32_t*)(sb + L.df_at);
  uint16_t* ids = (uint16_t*)(sb + L.ids_at);
  uint8_t* vals = S->dtype == KNNJOIN_INT8 ? (uint8_t*)(sb + L.vals_at) : nullptr;
  uint32_t* counts = (uint32_t*)(wb + W.counts_at);
  uint32_t* units = (uint32_t*)(wb + W.units_at);
  uint32_t* first = (uint32_t*)(wb + W.first_at);
  uint32_t* ka = (uint32_t*)(wb + W.ka_at);
  uint32_t* kb = (uint32_t*)(wb + W.kb_at);
  uint32_t* va = (uint32_t*)(wb + W.va_at);
  uint32_t* vb = (uint32_t*)(wb + W.vb_at);
  void* cubtmp = wb + W.cub_at;
  uint32_t sentinel_key = (uint32_t)(L.n_off - 1);
  const uint32_t dense_min = dense_threshold(S, tile, opt);
  const uint32_t dense_units = (uint32_t)tile / 128u;

  cudaError_t e;
  if ((e = cudaMemsetAsync(counts, 0, 4 * (size_t)L.n_off, st)) != cudaSuccess) return cuda_fail(e, "memset counts");
  if (vals && (e = cudaMemsetAsync(vals, 0, 8 * (size_t)L.unit_cap, st)) != cudaSuccess) return cuda_fail(e, "memset vals");
  const unsigned gnnz = (unsigned)((S->nnz + 255) / 256);
  if (S->nnz > 0) {
    int64_t threads = S->n_rows * 32;
    k_keys<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(S->indptr, S->indices, (const int8_t*)S->values,
                                                            S->n_rows, d, tile, L.n_tiles, ka, va, sentinel_key);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_keys");
    size_t tb = W.cub_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(cubtmp, tb, ka, kb, va, vb, (int)S->nnz, 0, end_bit_for(L.n_off - 1), st)) != cudaSuccess)
      return cuda_fail(e, "radix sort");
    k_seg_first<<<gnnz, 256, 0, st>>>(kb, S->nnz, sentinel_key, first);
    k_seg_count<<<gnnz, 256, 0, st>>>(kb, S->nnz, sentinel_key, first, counts);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_seg");
  }
  k_df<<<(unsigned)(((int64_t)d * 32 + 255) / 256), 256, 0, st>>>(counts, d, L.n_tiles, df);
  k_units<<<(unsigned)((L.n_off + 255) / 256), 256, 0, st>>>(counts, units, L.n_off, dense_min, dense_units);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_units");
  {
    size_t tb = W.cub_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(cubtmp, tb, units, off, (int)L.n_off, st)) != cudaSuccess) return cuda_fail(e, "scan off");
  }
  k_fill_pads<<<(unsigned)((L.unit_cap + 255) / 256), 256, 0, st>>>((uint4*)ids, L.unit_cap, (uint32_t)tile);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_fill_pads");
  if (S->nnz > 0) {
    if (dense_min != 0xFFFFFFFFu) {
      k_zero_dense<<<(unsigned)((L.n_off - 1 + 255) / 256), 256, 0, st>>>(counts, off, L.n_off - 1, dense_min,
                                                                        dense_units, (uint4*)ids);
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_zero_dense");
    }
    k_scatter<<<gnnz, 256, 0, st>>>(kb, vb, S->nnz, off, first, counts, dense_min, sentinel_key, ids, vals);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_scatter");
    if (dense_min != 0xFFFFFFFFu) {
      k_mark_dense<<<(unsigned)((L.n_off - 1 + 255) / 256), 256, 0, st>>>(counts, off, L.n_off - 1, dense_min);
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_mark_dense");
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
  h->dense_min = dense_min == 0xFFFFFFFFu ? 0x7FFFFFFF : (int32_t)dense_min;
  h->off = off;
  h->df = df;
  h->ids = ids;
  h->vals = vals;
  h->storage_bytes = L.total;
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
  out->dense_min = idx->dense_min;
  return KNNJOIN_OK;
}

KJ_API void knnjoin_free_index(knnjoin_index* idx) { delete idx; }
