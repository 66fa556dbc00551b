// wide.cu -- 64-bit fixed-point ("wide") queries and the certification of 32-bit fixed-point results.
//
// The fast path (accumulate.cuh) accumulates FP32-R scores in 32-bit per-row fixed point, q_d = rint(r_d sigma_r)
// with sigma_r = 2^30 / (sum_d r_d * smax).  Its absolute error per pair is at most
//     E_r = smax * sum_{d in r} |q_d - r_d sigma_r|      (fixed-point units)
// (DESIGN.md §5), which is tiny against the k-th score on every BASELINE config but not for rows whose weights
// span many decades (a 1e5 peak next to unit weights, "intensity used directly"): there the
// k-th score may sit below the resolution the peak leaves.  So:
//   * k_row_scale (query.cu) also returns E_r;  k_certify checks every row's final list: with y_min = the
//     smallest positive fixed score in the list, the list meets the tolerance rule of reading c15 (every
//     position within tau of the exact order, every score within tau) when E_r (2 + tau) <= (tau - 2^-23) y_min
//     (the i-th largest of a set moves by at most E_r under a perturbation of at most E_r);
//   * rows that fail are recomputed here at 64-bit fixed point: sigma64_r = 2^62 / (sum_d r_d * wmax) with wmax
//     the largest S weight of the index; per posting the product r_d sigma64 w rounds once, so the error is
//     below n_r / 2 units of 2^-62 (sum_d r_d wmax) -- relative 1e-16 of the row's largest possible score;
//   * FP32 S (row a1) is always queried here (its weights are not integers).
// Scores of wide results are keyed by the fp32 value of y / sigma64 (positive floats order like their bits):
// key = (f32 bits << 32) | (0xFFFFFFFF - global id), so candidates within fp32 rounding (6e-8 relative, inside
// the 1e-5 rule) tie and go to the lower id; keys from different indexes (S shards) compare directly.
//
// Kernel k_accumulate_wide: persistent, 8-warp CTAs, one item = (listed row, S tile group).  Per tile: the row's
// features are staged 256 at a time (slice bounds, block scan into a flat unit stream), every lane takes a
// 16-byte unit of ids (+ weights) and adds its 8 products with 64-bit shared atomics; head features (BINARY S)
// are added in the scan from the row's per-slot q; the scan zeroes the array and offers keys to the warp's
// register top-k list (topk.cuh); at the end of an item the 8 lists are merged by rank.
#include "common.cuh"
#include "topk.cuh"

namespace kj {
namespace {

constexpr int kWideNW = 8;               // warps per CTA
constexpr int kWideThreads = kWideNW * 32;
constexpr int kWideChunk = kWideThreads; // features staged per chunk (one per thread)
constexpr double kFixedOne64 = 4611686018427387904.0;  // 2^62
// the first kWideCapRows listed rows are split into G tile groups (one row's tiles over several CTAs; lists
// merged by rank afterwards), later rows run whole: a fallback for a few rows still spreads over the GPU
constexpr int64_t kWideCapRows = 64;

struct WP {
  const uint32_t* off;
  const uint16_t* ids;
  const uint8_t* vals8;      // INT8 S weights or nullptr
  const uint32_t* vals32;    // FP32 S weight bits or nullptr
  const int32_t* head_slot;
  const int32_t* head_feat;
  const uint32_t* head_cols;
  int32_t d, T;
  int64_t NT, s_id_base, t0, t1;
  // R
  const int64_t* indptr;
  const int32_t* indices;
  const void* values;
  knnjoin_dtype r_dtype;
  const double* sigma;       // [n_r] sigma64
  const double* inv_sigma;   // [n_r] 1 / sigma64
  const int32_t* row_list;   // [count] rows to process, or nullptr (all rows)
  const int32_t* row_count;  // device count of row_list (nullptr: n_list)
  int64_t n_list;            // rows when row_list is nullptr; capacity otherwise
  int32_t k;
  int32_t G;                 // tile groups of each of the first cap_rows listed rows
  int64_t tiles_per_group;
  int64_t cap_rows;
  const uint64_t* resume;    // [n_r][k] float-keyed lists to continue (input row order) or nullptr
  const uint64_t* theta_in;  // [n_r] key floors or nullptr
  uint64_t* part_keys;       // G > 1: [G][cap_rows][k]
  uint32_t* item_counter;
  uint64_t* out_keys;
  int32_t* out_ids;
  float* out_scores;
  unsigned long long* counters;
};

__host__ __device__ inline size_t wide_smem_bytes(int T, int k) {
  const size_t acc = (size_t)(T + kPadCols) * 8, merge = (size_t)kWideNW * k * 8;
  return align_up(acc > merge ? acc : merge, 16) + (size_t)kWideChunk * 8 /* q */ + (size_t)kWideChunk * 4 /* u0 */ +
         (size_t)(kWideChunk + 1) * 4 /* P */ + (size_t)kMaxHead * 8 /* head q */ + 64 /* misc */ +
         (size_t)kWideNW * 4 /* scan partials */;
}

template <int KS>
__global__ void __launch_bounds__(kWideThreads, 2) k_accumulate_wide(WP p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = p.T, k = p.k;
  unsigned long long* acc = (unsigned long long*)smem;
  const size_t acc_bytes = align_up((size_t)(T + kPadCols) * 8 > (size_t)kWideNW * k * 8 ? (size_t)(T + kPadCols) * 8
                                                                                          : (size_t)kWideNW * k * 8, 16);
  double* s_q = (double*)(smem + acc_bytes);                 // FP32 S: r_d * sigma64 (real); else q64 bits
  uint32_t* s_u0 = (uint32_t*)(s_q + kWideChunk);
  uint32_t* s_P = s_u0 + kWideChunk;
  unsigned long long* s_qh = (unsigned long long*)(((uintptr_t)(s_P + kWideChunk + 1) + 7) & ~(uintptr_t)7);
  uint32_t* s_misc = (uint32_t*)(s_qh + kMaxHead);          // [0] item, [1] head mask, [2] total units
  uint32_t* s_scan = s_misc + 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool fp32s = p.vals32 != nullptr;
  const int n_head = p.head_feat[kMaxHead];
  const int64_t count = p.row_count ? (int64_t)*p.row_count : p.n_list;
  const int64_t n_grouped = p.G > 1 ? min(count, p.cap_rows) : 0;
  const int64_t n_items = n_grouped * p.G + (count - n_grouped);
  unsigned long long n_visits = 0;

  for (int i = tid; i < T + kPadCols; i += kWideThreads) acc[i] = 0ull;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_misc[0] = atomicAdd(p.item_counter, 1u);
    __syncthreads();
    const int64_t item = s_misc[0];
    if (item >= n_items) break;
    const bool grouped = item < n_grouped * p.G;
    const int64_t li = grouped ? item / p.G : n_grouped + (item - n_grouped * p.G);  // list position
    const int g = grouped ? (int)(item - li * p.G) : 0;                               // tile group
    const int64_t row = p.row_list ? (int64_t)p.row_list[li] : li;
    const int64_t tb = grouped ? p.t0 + (int64_t)g * p.tiles_per_group : p.t0;
    const int64_t te = grouped ? min(p.t1, tb + p.tiles_per_group) : p.t1;
    const int64_t rs = p.indptr[row], re = p.indptr[row + 1];
    const double sg = p.sigma[row];
    auto run_q = [&](int64_t j) -> double {  // r_d * sigma64 (real)
      const double r = p.r_dtype == KNNJOIN_FP32 ? (double)((const float*)p.values)[j]
                                                 : (p.r_dtype == KNNJOIN_INT8 ? (double)((const int8_t*)p.values)[j] : 1.0);
      return r * sg;
    };
    auto int_q = [](double x) -> unsigned long long {  // integer S: q64 = max(1, rint(r_d sigma64))
      const double q = rint(x);
      return q < 1.0 ? 1ull : (unsigned long long)q;
    };
    // head features of this row: per-slot q (integer S only: head features exist for BINARY S)
    if (n_head) {
      if (tid < kMaxHead) s_qh[tid] = 0;
      if (tid == 0) s_misc[1] = 0;
      __syncthreads();
      for (int64_t j = rs + tid; j < re; j += kWideThreads) {
        const int32_t f = p.indices[j];
        if (f < p.d) {
          const int sl = p.head_slot[f];
          if (sl >= 0) {
            s_qh[sl] = int_q(run_q(j));
            atomicOr(&s_misc[1], 1u << sl);
          }
        }
      }
      __syncthreads();
    }
    const uint32_t hmask = n_head ? s_misc[1] : 0u;

    uint64_t L[KS];
#pragma unroll
    for (int s = 0; s < KS; ++s) L[s] = 0;
    uint64_t theta = kKeyFloor;
    if (p.resume && g == 0 && warp == 0) {
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int pos = s * 32 + lane;
        if (pos < k) L[s] = __ldg((const unsigned long long*)p.resume + (size_t)row * k + pos);
      }
      theta = list_kth<KS>(L, k);
    }
    if (p.theta_in) {
      const uint64_t f = __ldg((const unsigned long long*)p.theta_in + row);
      if (f > 0 && f - 1 > theta) theta = f - 1;
    }

    for (int64_t t = tb; t < te; ++t) {
      // ------------------------------------------------------------------ accumulate (a4, 64-bit)
      for (int64_t c0 = rs; c0 < re; c0 += kWideChunk) {
        const int64_t j = c0 + tid;
        uint32_t u0 = 0, U = 0;
        double qv = 0.0;
        if (j < re) {
          const int32_t f = p.indices[j];
          if (f < p.d) {
            const uint32_t* o = p.off + (size_t)f * (size_t)(p.NT + 1) + (size_t)t;
            u0 = o[0];
            U = o[1] - u0;
            qv = run_q(j);
          }
        }
        // block exclusive scan of U
        uint32_t x = U;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) s_scan[warp] = x;
        __syncthreads();
        uint32_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kWideNW; ++w) {
          const uint32_t v = s_scan[w];
          if (w < warp) before += v;
          total += v;
        }
        const uint32_t P = before + x - U;
        s_u0[tid] = u0;
        s_P[tid] = P;
        if (fp32s) s_q[tid] = qv;
        else ((unsigned long long*)s_q)[tid] = U ? int_q(qv) : 0ull;
        if (tid == 0) s_P[kWideChunk] = total;
        __syncthreads();
        for (uint32_t pp = tid; pp < total; pp += kWideThreads) {
          int lo = 0, hi = kWideChunk - 1;  // largest e with P[e] <= pp (its range is non-empty)
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_P[mid] <= pp) lo = mid; else hi = mid - 1;
          }
          const uint32_t unit = s_u0[lo] + (pp - s_P[lo]);
          KJ_CHECK(pp >= s_P[lo] && pp < s_P[lo + 1]);
          const uint4 idw = __ldg((const uint4*)(p.ids + (size_t)unit * 8));
          const uint32_t wd[4] = {idw.x, idw.y, idw.z, idw.w};
          if (fp32s) {
            const double qd = s_q[lo];
            const uint4 wa = __ldg((const uint4*)(p.vals32 + (size_t)unit * 8));
            const uint4 wb = __ldg((const uint4*)(p.vals32 + (size_t)unit * 8 + 4));
            const uint32_t ww[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const uint32_t id = ((wd[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu) >> 2;  // ids are byte offsets
              KJ_CHECK(id < (uint32_t)(T + kPadCols));
              const double prod = qd * (double)__uint_as_float(ww[jj]);
              if (ww[jj]) atomicAdd(&acc[id], (unsigned long long)rint(prod));
            }
          } else {
            const unsigned long long q = ((const unsigned long long*)s_q)[lo];
            uint2 w8 = make_uint2(0x01010101u, 0x01010101u);
            if (p.vals8) w8 = __ldg((const uint2*)(p.vals8 + (size_t)unit * 8));
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const uint32_t id = ((wd[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu) >> 2;  // ids are byte offsets
              KJ_CHECK(id < (uint32_t)(T + kPadCols));
              const uint32_t w = ((jj < 4 ? w8.x : w8.y) >> (8 * (jj & 3))) & 0xFFu;
              atomicAdd(&acc[id], q * (unsigned long long)w);
            }
          }
          if (p.counters) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) n_visits += (((wd[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu) < 4u * (uint32_t)T) ? 1 : 0;
          }
        }
        __syncthreads();
      }
      // ------------------------------------------------------------------ scan + top-k (a5)
      {
        const int cols = T / kWideNW;
        const int cbase = warp * cols;
        for (int c = lane; c < cols; c += 32) {
          const int col = cbase + c;
          unsigned long long y = acc[col];
          acc[col] = 0ull;
          if (n_head) {
            uint32_t hw = __ldg(p.head_cols + (size_t)t * T + col) & hmask;
            if (p.counters) n_visits += __popc(hw);
            while (hw) {
              const int b = __ffs(hw) - 1;
              hw &= hw - 1;
              y += s_qh[b];
            }
          }
          uint64_t key = 0;
          if (y) {
            const float xs = (float)((double)y * p.inv_sigma[row]);
            uint32_t bits = __float_as_uint(xs);
            if (bits == 0) bits = 1;  // a positive score stays admissible
            key = make_key(bits, (uint32_t)(p.s_id_base + t * (int64_t)T + col));
          }
          list_offer_lanes<KS>(L, key, theta, k, lane);
        }
        __syncthreads();
      }
    }
    // ---------------------------------------------------------------------- merge the warps' lists (a7)
    {
      uint64_t* scratch = (uint64_t*)acc;  // [NW][k]; acc columns < T are all zero here
#pragma unroll
      for (int s = 0; s < KS; ++s)
        if (s * 32 + lane < k) scratch[(size_t)warp * k + s * 32 + lane] = L[s];
      __syncthreads();
      auto emit = [&](int pos, uint64_t key) {
        if (grouped) {
          p.part_keys[((size_t)g * p.cap_rows + li) * k + pos] = key;
          return;
        }
        const size_t o = (size_t)row * k + pos;
        if (key == 0) {
          if (p.out_keys) p.out_keys[o] = 0;
          if (p.out_ids) p.out_ids[o] = -1;
          if (p.out_scores) p.out_scores[o] = 0.0f;
        } else {
          if (p.out_keys) p.out_keys[o] = key;
          if (p.out_ids) p.out_ids[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)key);
          if (p.out_scores) p.out_scores[o] = __uint_as_float((uint32_t)(key >> 32));
        }
      };
      auto count_gt = [&](const uint64_t* lst, uint64_t x) {
        int lo = 0, hi = k;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (lst[mid] > x) lo = mid + 1; else hi = mid;
        }
        return lo;
      };
      for (int i = tid; i < kWideNW * k; i += kWideThreads) {
        const int w = i / k, pos = i % k;
        const uint64_t x = scratch[i];
        if (x == 0) continue;
        int rank = pos;
        for (int w2 = 0; w2 < kWideNW && rank < k; ++w2)
          if (w2 != w) rank += count_gt(scratch + (size_t)w2 * k, x);
        if (rank < k) emit(rank, x);
      }
      for (int pos = tid; pos < k; pos += kWideThreads) {
        int npos = 0;
        for (int w = 0; w < kWideNW && npos <= pos; ++w) npos += count_gt(scratch + (size_t)w * k, 0);
        if (pos >= npos) emit(pos, 0);
      }
      __syncthreads();
      for (int i = tid; i < kWideNW * k; i += kWideThreads) scratch[i] = 0;
    }
  }
  if (p.counters) {
#pragma unroll
    for (int o = 16; o; o >>= 1) n_visits += __shfl_xor_sync(0xffffffffu, n_visits, o);
    if (lane == 0) atomicAdd(&p.counters[0], n_visits);
  }
}

// per-row 64-bit scale: sigma64 = 2^62 / (sum_{d in r, d < D} r_d * wmax); warp per row
__global__ void k_row_scale64(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                              const void* __restrict__ values, knnjoin_dtype rdt, int64_t n, int32_t d,
                              const uint32_t* __restrict__ wmax, knnjoin_dtype sdt, double* __restrict__ sigma,
                              double* __restrict__ inv_sigma) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int64_t j = indptr[row] + lane; j < indptr[row + 1]; j += 32)
    if (indices[j] < d)
      s += rdt == KNNJOIN_FP32 ? (double)((const float*)values)[j]
                               : (rdt == KNNJOIN_INT8 ? (double)((const int8_t*)values)[j] : 1.0);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const uint32_t wb = *wmax;
    const double wm = sdt == KNNJOIN_FP32 ? (double)__uint_as_float(wb) : (double)(wb ? wb : 1u);
    double sg = 1.0;
    if (s > 0.0 && wm > 0.0) sg = kFixedOne64 / (s * wm);
    sigma[row] = sg;
    inv_sigma[row] = 1.0 / sg;
  }
}

// certification of 32-bit fixed-point lists (see the header comment); warp per row.  keys: [n][k] fixed keys in
// input row order; err: E_r per row (fixed units); appends failing rows to list[1..] (count in list[0])
__global__ void k_certify(const uint64_t* __restrict__ keys, const double* __restrict__ err, int64_t n, int32_t k,
                          double tau, int32_t* __restrict__ list) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  uint32_t ymin = 0xFFFFFFFFu;  // smallest positive score of the list
  for (int i = lane; i < k; i += 32) {
    const uint32_t y = (uint32_t)(__ldg((const unsigned long long*)keys + (size_t)row * k + i) >> 32);
    if (y) ymin = min(ymin, y);
  }
  ymin = __reduce_min_sync(0xffffffffu, ymin);
  if (lane == 0 && ymin != 0xFFFFFFFFu) {
    const double e = err[row];
    if (!(e * (2.0 + tau) <= (tau - 0x1p-23) * (double)ymin)) list[1 + atomicAdd(list, 1)] = (int32_t)row;
  }
}

}  // namespace

int wide_ctas(int sms) { return sms * 2; }

size_t wide_part_bytes(int32_t k, int64_t n_tiles, int sms, int32_t* G_out) {
  // G groups for each of the first kWideCapRows rows: two waves of CTAs when only those rows are listed
  int64_t G = (2 * wide_ctas(sms) + kWideCapRows - 1) / kWideCapRows;
  if (G > n_tiles) G = n_tiles > 0 ? n_tiles : 1;
  if (G < 1) G = 1;
  *G_out = (int32_t)G;
  return G > 1 ? (size_t)G * kWideCapRows * (size_t)k * 8 : 0;
}

cudaError_t launch_wide(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k, int64_t t0, int64_t t1,
                        const int32_t* row_list, const int32_t* row_count, const uint64_t* resume,
                        const uint64_t* theta_in, double* sigma64, double* inv64, uint32_t* item_counter,
                        uint64_t* part_keys, int32_t G, unsigned long long* counters, uint64_t* out_keys,
                        int32_t* out_ids, float* out_scores, int sms, cudaStream_t st) {
  cudaError_t e;
  if (R->n_rows <= 0) return cudaSuccess;
  k_row_scale64<<<(unsigned)((R->n_rows * 32 + 255) / 256), 256, 0, st>>>(R->indptr, R->indices, R->values, R->dtype,
                                                                          R->n_rows, idx->d, idx->wmax, idx->s_dtype,
                                                                          sigma64, inv64);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(item_counter, 0, 4, st)) != cudaSuccess) return e;
  WP p;
  p.off = idx->off;
  p.ids = idx->ids;
  p.vals8 = idx->s_dtype == KNNJOIN_INT8 ? idx->vals : nullptr;
  p.vals32 = idx->s_dtype == KNNJOIN_FP32 ? idx->vals32 : nullptr;
  p.head_slot = idx->head_slot;
  p.head_feat = idx->head_feat;
  p.head_cols = idx->head_cols;
  p.d = idx->d;
  p.T = idx->tile;
  p.NT = idx->n_tiles;
  p.s_id_base = idx->s_id_base;
  p.t0 = t0;
  p.t1 = t1;
  p.indptr = R->indptr;
  p.indices = R->indices;
  p.values = R->values;
  p.r_dtype = R->dtype;
  p.sigma = sigma64;
  p.inv_sigma = inv64;
  p.row_list = row_list;
  p.row_count = row_count;
  p.n_list = R->n_rows;
  p.k = k;
  const int64_t span = t1 - t0;
  if (G > span) G = span > 1 ? (int32_t)span : 1;
  p.G = G;
  p.tiles_per_group = span > 0 ? (span + G - 1) / G : 1;
  p.cap_rows = kWideCapRows;
  p.resume = resume;
  p.theta_in = theta_in;
  p.part_keys = part_keys;
  p.item_counter = item_counter;
  p.out_keys = out_keys;
  p.out_ids = out_ids;
  p.out_scores = out_scores;
  p.counters = counters;
  const size_t sm = wide_smem_bytes(idx->tile, k);
  int64_t grid = checked_grid_cap(wide_ctas(sms));
  const int64_t max_items = R->n_rows + (G > 1 ? kWideCapRows * (G - 1) : 0);
  if (grid > max_items) grid = max_items;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e2 != cudaSuccess) return e2;
    kern<<<(unsigned)grid, kWideThreads, sm, st>>>(p);
    return cudaGetLastError();
  };
  const int KS = ks_for_k(k);
  e = KS == 1 ? go(k_accumulate_wide<1>) : (KS == 4 ? go(k_accumulate_wide<4>) : go(k_accumulate_wide<8>));
  if (e != cudaSuccess) return e;
  if (G > 1) {
    // the part lists have a stride of kWideCapRows rows; positions >= min(count, kWideCapRows) are not grouped
    const int64_t limit = row_list ? kWideCapRows : (R->n_rows < kWideCapRows ? R->n_rows : kWideCapRows);
    return launch_merge_keys_ex(part_keys, G, kWideCapRows, limit, k, nullptr, 1, row_list, row_count, 0, out_keys,
                                out_ids, out_scores, st);
  }
  return cudaSuccess;
}

cudaError_t launch_certify(const uint64_t* keys, const double* err, int64_t n, int32_t k, double tau, int32_t* list,
                           cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(list, 0, 4, st);
  if (e != cudaSuccess || n <= 0) return e;
  k_certify<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(keys, err, n, k, tau, list);
  return cudaGetLastError();
}

}  // namespace kj

using namespace kj;

KJ_API knnjoin_status knnjoin_certify(const uint64_t* keys, const knnjoin_csr* R, int32_t d, knnjoin_dtype s_dtype,
                                      int32_t k, float tolerance, int32_t* out_list, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  KJ_NVTX("knnjoin_certify");
  if (!R || k < 1 || k > kMaxK || !out_list) { set_error("bad certify arguments"); return KNNJOIN_ERR_ARG; }
  if (d <= 0) { set_error("d must be > 0"); return KNNJOIN_ERR_DIM; }
  if (s_dtype != KNNJOIN_BINARY && s_dtype != KNNJOIN_INT8) {
    set_error("certify applies to 32-bit fixed-point keys (BINARY / INT8 S)");
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  if (!(tolerance >= 0.0f && tolerance < 1.0f)) { set_error("tolerance must be in [0, 1)"); return KNNJOIN_ERR_ARG; }
  const size_t need = align_up(8 * (size_t)R->n_rows, 256) + 256;
  if (!workspace || workspace_bytes < need) { set_error("certify workspace %zu < %zu", workspace_bytes, need); return KNNJOIN_ERR_WORKSPACE; }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (R->n_rows == 0) {
    if ((e = cudaMemsetAsync(out_list, 0, 4, st)) != cudaSuccess) return cuda_fail(e, "certify");
    return KNNJOIN_OK;
  }
  if (!keys) { set_error("keys is NULL"); return KNNJOIN_ERR_ARG; }
  double* err = (double*)workspace;
  launch_row_scale(R, d, s_dtype == KNNJOIN_INT8 ? 127 : 1, nullptr, nullptr, err, st);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "row error");
  if (R->dtype != KNNJOIN_FP32) {  // integer scores are exact: nothing to certify
    if ((e = cudaMemsetAsync(out_list, 0, 4, st)) != cudaSuccess) return cuda_fail(e, "certify");
    return KNNJOIN_OK;
  }
  if ((e = launch_certify(keys, err, R->n_rows, k, tolerance > 0.0f ? (double)tolerance : 1e-5, out_list, st)) !=
      cudaSuccess)
    return cuda_fail(e, "k_certify");
  return KNNJOIN_OK;
}

KJ_API size_t knnjoin_certify_workspace_bytes(const knnjoin_csr* R) {
  if (!R || R->n_rows < 0) { set_error("bad R"); return 0; }
  return align_up(8 * (size_t)R->n_rows, 256) + 256;
}
