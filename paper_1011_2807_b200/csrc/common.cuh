// common.cuh -- internal declarations shared by the translation units of libknnjoin.so.
// Nothing here is shared with oracle/ (the CPU oracle); see DESIGN.md "Boundary".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/knnjoin.h"

#define KJ_API extern "C" __attribute__((visibility("default")))

// NVTX range over a C-ABI entry point (SURVEY.md §5 tracing): header-only nvtx3, a no-op unless a tool (nsys, ncu
// --nvtx) is attached.  The ranges mark host-side enqueue; the kernels they launch carry the same names in traces.
#include <nvtx3/nvToolsExt.h>
struct KjNvtxRange {
  explicit KjNvtxRange(const char* name) { nvtxRangePushA(name); }
  ~KjNvtxRange() { nvtxRangePop(); }
};
#define KJ_NVTX(name) KjNvtxRange kj_nvtx_range_(name)

struct knnjoin_index;

namespace kj {

constexpr int kMaxK = 256;
constexpr int kDefaultTile = 8192;
// Posting ids are stored as BYTE offsets of their score column, 4 * (s - tile base) (padding: 4 * (tile + 0..31),
// dummy columns), so the accumulation kernel adds them to a row base without a shift: 4 * (tile + 32) < 2^16.
constexpr int kMaxTile = 14336;
constexpr int kTileQuantum = 2048;     // tile must split into 16 warps' column strips of 128-column steps
constexpr int kMaxHead = 32;                  // head features per index (one 32-bit word per S row)
constexpr float kDefaultHeadDensity = 0.125f;  // df >= |S|/8 makes a feature a head candidate
constexpr int kPadCols = 32;           // dummy score columns per row that absorb padding postings
constexpr uint64_t kKeyFloor = 0x00000000FFFFFFFFull;  // score 0 with every id: admits nothing
constexpr double kFixedOne = 1073741824.0;              // 2^30: per-row fixed-point scale numerator

// Checked builds (-DKJ_CHECKS, tools/checked_build.sh): device-side bounds checks on every index the kernels form
// into shared and global memory (the stand-in for compute-sanitizer, which this pool does not allow); a failed check
// prints its site and traps.  KNNJOIN_MAX_CTAS caps the persistent grids so results can be compared across very
// different schedules (race detection by determinism).  Release builds compile both out.
#ifdef KJ_CHECKS
#define KJ_CHECK(cond)                                                                          \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("KJ_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define KJ_CHECK(cond) \
  do {                 \
  } while (0)
#endif
int64_t checked_grid_cap(int64_t grid);  // grid, or min(grid, KNNJOIN_MAX_CTAS) in checked builds

void set_error(const char* fmt, ...);
knnjoin_status cuda_fail(cudaError_t e, const char* what);

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// host-side layout of the index storage (all offsets 256-byte aligned)
struct IndexLayout {
  int64_t n_tiles = 0, n_off = 0, unit_cap = 0;
  size_t off_at = 0, df_at = 0, head_slot_at = 0, head_feat_at = 0, head_cols_at = 0, ids_at = 0, vals_at = 0, wmax_at = 0,
         fwd_ptr_at = 0, fwd_idx_at = 0, fwd_val_at = 0, fmax_at = 0, total = 0;
};
// prune: also reserve S's forward rows and (INT8 S) the per-feature maximum weight (pruned queries, a6)
// F: the CSR whose rows are kept as forward rows (S itself, or options.forward)
bool index_layout(const knnjoin_csr* S, int32_t d, int32_t tile, bool prune, IndexLayout* L,
                  const knnjoin_csr* F = nullptr);
constexpr float kDefaultPruneAlpha = 0.25f;
int32_t resolve_tile(const knnjoin_options* opt);

// per-row score scale: sigma[r] = 2^30 / (sum_d r_d * smax) for FP32 R,
// 1 for integer R.  inv_sigma[r] = 1 / sigma[r] converts a fixed-point sum back to a score.
// err (optional): E_r = smax * sum_{d in r} |q_d - r_d sigma_r|, the bound on the absolute error of any pair's
// fixed-point score (certification in wide.cu)
void launch_row_scale(const knnjoin_csr* R, int32_t d, int32_t smax, double* sigma, double* inv_sigma, double* err,
                      cudaStream_t st);

// finalize / merge helpers implemented in merge.cu
int ks_for_k(int32_t k);
// K4: rank merge of P sorted key lists per row ([P][n][k], disjoint S ids) into the outputs
cudaError_t launch_merge_keys(const uint64_t* keys, int32_t P, int64_t n, int32_t k, const double* inv_sigma,
                              uint64_t* out_keys, int32_t* out_ids, float* out_scores, cudaStream_t st);
// float_keys: scores are fp32 bits (wide queries); row_list/row_count: position i -> output row row_list[i]
// n: slab stride in rows; limit: list positions merged (<= n)
cudaError_t launch_merge_keys_ex(const uint64_t* keys, int32_t P, int64_t n, int64_t limit, int32_t k,
                                 const double* inv_sigma, int float_keys, const int32_t* row_list,
                                 const int32_t* row_count, int keys_by_row, uint64_t* out_keys, int32_t* out_ids,
                                 float* out_scores, cudaStream_t st);
// 64-bit fixed-point queries (wide.cu)
size_t wide_part_bytes(int32_t k, int64_t n_tiles, int sms, int32_t* G_out);
cudaError_t launch_wide(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k, int64_t t0, int64_t t1,
                        const int32_t* row_list, const int32_t* row_count, const uint64_t* resume,
                        const uint64_t* theta_in, double* sigma64, double* inv64, uint32_t* item_counter,
                        uint64_t* part_keys, int32_t G, unsigned long long* counters, uint64_t* out_keys,
                        int32_t* out_ids, float* out_scores, int sms, cudaStream_t st);
// K4 for the split-mode lists of one candidate shape (gate as in the accumulate kernel)
cudaError_t launch_merge_keys_gated(const uint64_t* keys, int32_t P, int64_t n, int32_t k, const double* inv_sigma,
                                    const int32_t* gate, int gate_heads, uint64_t* out_keys, int32_t* out_ids,
                                    float* out_scores, cudaStream_t st);
cudaError_t launch_certify(const uint64_t* keys, const double* err, int64_t n, int32_t k, double tau, int32_t* list,
                           cudaStream_t st);
constexpr double kDefaultTolerance = 1e-5;  // BASELINE.json north_star: fp32 scores within 1e-5 relative

}  // namespace kj

struct knnjoin_index {
  int64_t n_s = 0, s_id_base = 0;
  int32_t d = 0, tile = 0;
  int64_t n_tiles = 0, n_off = 0, unit_cap = 0;
  knnjoin_dtype s_dtype = KNNJOIN_BINARY;
  uint32_t head_min_df = 0xFFFFFFFFu;  // df threshold of head features (0xFFFFFFFF: none)
  int32_t head_max = 0;                // cap on head features (0: none)
  const uint32_t* off = nullptr;       // [n_off] posting-unit (16 B) offsets, feature-major: f*(n_tiles+1)+t
  const int32_t* df = nullptr;         // [d] |I_d| (document frequency of each feature in S)
  const int32_t* head_slot = nullptr;  // [d] head slot of a feature, -1 if not a head feature
  const int32_t* head_feat = nullptr;  // [kMaxHead + 1] feature of each head slot (-1 unused); [kMaxHead] = n_head
  const uint32_t* head_cols = nullptr; // [n_tiles * tile] bit i: S row has head feature head_feat[i]
  const uint16_t* ids = nullptr;       // [unit_cap*8] local S ids (< tile); padding = tile + (u mod 32)
  const uint8_t* vals = nullptr;       // [unit_cap*8] INT8 S weights (nullptr for BINARY / FP32 S)
  const uint32_t* vals32 = nullptr;    // [unit_cap*8] FP32 S weight bits (FP32 S only; queried at 64 bits, wide.cu)
  const uint32_t* wmax = nullptr;      // [1] largest S weight: u32 (BINARY 1, INT8) or float bits (FP32)
  // pruned mode (options.prune = 1): forward rows of S (local row ids) and per-feature max weight
  int32_t prune = 0;
  float alpha = 0.0f;                  // default alpha of pruned queries
  const int64_t* fwd_ptr = nullptr;    // [n_s + 1]
  const int32_t* fwd_idx = nullptr;    // [nnz] features, ascending per row
  const uint8_t* fwd_val = nullptr;    // [nnz] INT8 S weights (nullptr for BINARY S)
  const uint32_t* fmax = nullptr;      // [d] largest weight of each feature (nullptr for BINARY S: 1)
  size_t storage_bytes = 0;
  size_t fwd_bytes = 0;                // part of storage_bytes holding the forward rows (not swept per tile)
};
