// query.cu -- K2 (query prep) and K3 (score accumulation fused with per-tile top-k) of the KNN join.
//
// What is computed: for every r in R, Find_Matches_IIB (Alg. 3 lines 9-17):
//   A[s] += r[d] * s[d] for every posting (s, s[d]) of I_d, for every feature (d, r[d]) of r  (a4)
//   then every s with A[s] > pruneScore(r) enters r's candidate set                          (a5)
// with S split into tiles (the S blocks of Alg. 1) and pruneScore carried across tiles.
//
// GPU mapping:
//  * k_row_scale  (a3) per-row fixed-point scale sigma_r = 2^30 / (sum_d r_d * smax) for FP32 R, 1 otherwise.
//  * k_build_runs (a3) one warp per batch of B rows: B-way merge of the rows' ascending feature lists
//    into "runs" (feature f, mask of batch rows that contain f, q_b = r_b[f] quantised).  A run's
//    posting slice is loaded once and applied to every row in its mask (cross-row reuse).
//  * k_accumulate_topk (a4 + a5 + a7), persistent, one CTA (16 warps) per SM:
//      for each batch (B rows) taken from a global counter:
//        for each S tile t (ascending, so ids arrive in ascending order):
//          stage: every thread reads the (f, t) slice bounds of one run; a block scan compacts
//                 non-empty runs and gives each its position P in the tile's flattened unit stream.
//          accumulate: each warp owns a contiguous range of 32-unit windows of that stream; lane l
//                 takes unit p0+l, finds its run by a 5-step shuffle search, loads 16 B (8 local ids,
//                 + 8 INT8 weights) with ld.global.nc, and issues atomicAdd(acc[b][id], q_b*w) for each
//                 row b of the run.  Integer atomics make the sum order-independent (bit-reproducible).
//          scan:  warp w owns columns [w*T/16, (w+1)*T/16) of every row: 128-bit reads, zero-fill, and
//                 candidates with key > theta go into the warp's register top-k list; theta_row (shared,
//                 atomicMax of every warp's k-th key) tightens every warp's filter.
//        merge the 16 per-warp lists of each row, finalize (ids, scores, keys).
#include "common.cuh"
#include "topk.cuh"

namespace kj {
namespace {

struct QP {
  // index
  const uint32_t* off;
  const uint16_t* ids;
  const uint8_t* vals;
  int32_t d, T;
  int64_t NT;
  int64_t s_id_base;
  // R / batches
  int64_t n_r;
  int32_t k;
  int64_t n_batches;
  const int64_t* r_indptr;
  const uint32_t* runs_f;
  const int32_t* runs_q;
  const uint32_t* batch_nruns;
  const double* inv_sigma;
  uint32_t* batch_counter;
  unsigned long long* counters;
  // out
  uint64_t* out_keys;
  int32_t* out_ids;
  float* out_scores;
};

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// ------------------------------------------------------------------------------------------- a3 prep
__global__ void k_row_scale_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                   const float* __restrict__ values, int64_t n, int32_t d, int32_t smax,
                                   double* __restrict__ sigma, double* __restrict__ inv_sigma) {
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
  if (lane == 0) {
    double sg = 1.0;
    if (values && s > 0.0) sg = kFixedOne / (s * (double)smax);
    if (sigma) sigma[row] = sg;
    if (inv_sigma) inv_sigma[row] = 1.0 / sg;
  }
}

// one warp per batch of B rows
__global__ void k_build_runs(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                             const void* __restrict__ values, knnjoin_dtype rdt, int64_t n_r, int32_t d, int B,
                             int64_t n_batches, const double* __restrict__ sigma, uint32_t* __restrict__ runs_f,
                             int32_t* __restrict__ runs_q, uint32_t* __restrict__ batch_nruns) {
  int64_t batch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (batch >= n_batches) return;
  int64_t row = batch * B + lane;
  bool mine = lane < B && row < n_r;
  int64_t ptr = 0, end = 0;
  double sg = 1.0;
  if (mine) {
    ptr = indptr[row];
    end = indptr[row + 1];
    sg = sigma[row];
  }
  int64_t base = indptr[batch * B];
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
        if (rdt == KNNJOIN_FP32) {
          double v = (double)((const float*)values)[ptr] * sg;
          q = (int32_t)rint(v);
          if (q < 1) q = 1;
        } else if (rdt == KNNJOIN_INT8) {
          q = (int32_t)((const int8_t*)values)[ptr];
        } else {
          q = 1;
        }
        ++ptr;
      }
      runs_q[run * B + lane] = q;
    }
    if (lane == 0) runs_f[run] = (uint32_t)fmin | (mask << 24);
    ++nruns;
  }
  if (lane == 0) batch_nruns[batch] = nruns;
}

// -------------------------------------------------------------------------- block-wide scan helper
__device__ __forceinline__ uint64_t block_exclusive_scan_u64(uint64_t v, uint64_t* s_warp, uint64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < kWarps ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kWarps) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  uint64_t before = warp ? s_warp[warp - 1] : 0;
  *total = s_warp[kWarps - 1];
  return before + x - v;
}

// ------------------------------------------------------------------------------ a4 + a5 + a7 kernel
// Score rows have stride T + kPadCols: columns [T, T+32) absorb padding postings (never scanned).
__host__ __device__ inline int acc_stride(int T) { return T + kPadCols; }

// the score array doubles as the scratch of the end-of-batch list merge ([kWarps][B][k] keys)
__host__ __device__ inline size_t acc_region_bytes(int B, int T, int k) {
  size_t a = (size_t)B * acc_stride(T) * 4, m = (size_t)kWarps * B * k * 8;
  return align_up(a > m ? a : m, 16);
}

template <int B>
struct Smem {
  static size_t bytes(int T, int k) {
    size_t at = acc_region_bytes(B, T, k);          // acc / merge scratch
    at += (size_t)kCap * 4;                        // ustart
    at += (size_t)(kCap + 1) * 4;                  // P
    at += (size_t)kCap * 4;                        // fm
    at += (size_t)kCap * B * 4;                    // q
    at = align_up(at, 16);
    at += kWarps * 8;                              // scan partials
    at += 8 * 8;                                   // theta_row (B <= 8)
    at += 16;                                      // misc
    return at;
  }
};

__device__ __forceinline__ void red_add_shared(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

constexpr int kWinChunk = 4;  // 32-unit windows a warp takes per grab of the dynamic window counter

template <int B, int KS, bool SINT8>
__global__ void __launch_bounds__(kThreads, 1) k_accumulate_topk(QP p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = p.T;
  const int TS = acc_stride(T);
  uint32_t* acc = (uint32_t*)smem;
  const uint32_t acc_s = (uint32_t)__cvta_generic_to_shared(acc);
  uint32_t* s_ustart = (uint32_t*)(smem + acc_region_bytes(B, T, p.k));
  uint32_t* s_P = s_ustart + kCap;
  uint32_t* s_fm = s_P + kCap + 1;
  int32_t* s_q = (int32_t*)(s_fm + kCap);
  size_t at = align_up(acc_region_bytes(B, T, p.k) + (size_t)kCap * 4 + (size_t)(kCap + 1) * 4 + (size_t)kCap * 4 +
                           (size_t)kCap * B * 4, 16);
  uint64_t* s_warp = (uint64_t*)(smem + at);
  uint64_t* s_theta = s_warp + kWarps;
  int* s_misc = (int*)(s_theta + 8);  // [0] batch, [1] n_items, [2] TOT, [3] window counter

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = p.k;
  constexpr bool wint8 = SINT8;
  unsigned long long n_visits = 0, n_inserts = 0;

  for (int i = tid; i < (int)(acc_region_bytes(B, T, k) / 16); i += kThreads) ((uint4*)acc)[i] = make_uint4(0, 0, 0, 0);

  for (;;) {
    __syncthreads();
    if (tid == 0) s_misc[0] = (int)atomicAdd(p.batch_counter, 1u);
    __syncthreads();
    const int64_t batch = s_misc[0];
    if (batch >= p.n_batches) break;
    const int64_t row0 = batch * B;
    const int nb = (int)min((int64_t)B, p.n_r - row0);
    const int64_t run_base = p.r_indptr[row0];
    const int nruns = (int)p.batch_nruns[batch];
    if (tid < 8) s_theta[tid] = kKeyFloor;

    uint64_t L[B][KS];
    uint64_t own[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      own[b] = kKeyFloor;
#pragma unroll
      for (int s = 0; s < KS; ++s) L[b][s] = 0;
    }
    __syncthreads();

    const int64_t ntiles = nruns > 0 ? p.NT : 0;
    for (int64_t t = 0; t < ntiles; ++t) {
      for (int c0 = 0; c0 < nruns; c0 += kCap) {
        // ---------------------------------------------------------------- stage chunk of runs
        {
          const int i = c0 + tid;
          uint32_t fm = 0, u0 = 0, U = 0;
          size_t run = (size_t)(run_base + i);
          if (i < nruns) {
            fm = p.runs_f[run];
            const uint32_t* o = p.off + (size_t)(fm & 0xFFFFFFu) * (size_t)(p.NT + 1) + (size_t)t;
            u0 = o[0];
            U = o[1] - u0;
          }
          const uint64_t packed = ((uint64_t)(U > 0) << 32) | U;
          uint64_t total;
          const uint64_t ex = block_exclusive_scan_u64(packed, s_warp, &total);
          if (U > 0) {
            const uint32_t c = (uint32_t)(ex >> 32);
            s_ustart[c] = u0;
            s_P[c] = (uint32_t)ex;
            s_fm[c] = fm;
#pragma unroll
            for (int b = 0; b < B; ++b) s_q[c * B + b] = p.runs_q[run * B + b];
          }
          if (tid == 0) {
            s_misc[1] = (int)(total >> 32);
            s_misc[2] = (int)(uint32_t)total;
            s_misc[3] = 0;
            s_P[(uint32_t)(total >> 32)] = (uint32_t)total;
          }
          __syncthreads();
        }
        // ---------------------------------------------------------------- accumulate (a4)
        {
          const int n_items = s_misc[1];
          const uint32_t TOT = (uint32_t)s_misc[2];
          const uint32_t nwin = (TOT + 31) >> 5;
          for (;;) {
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd((unsigned*)&s_misc[3], (unsigned)kWinChunk);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c >= nwin) break;
            const uint32_t p_begin = c * 32, p_end = min(TOT, (c + kWinChunk) * 32);
            int lo = 0, hi = n_items - 1;  // largest e with P[e] <= p_begin
            while (lo < hi) {
              int mid = (lo + hi + 1) >> 1;
              if (s_P[mid] <= p_begin) lo = mid; else hi = mid - 1;
            }
            int e_cur = lo;
            auto lookup = [&](uint32_t p0, int& e_out, uint32_t& unit, bool& valid) {
              const uint32_t nxt = s_P[e_cur + 1];
              int e = e_cur;
              if (p0 + 32 > nxt) {
                const int j = min(e_cur + 1 + lane, n_items);
                const uint32_t o = s_P[j];
                const uint32_t pp = p0 + lane;
                int cc = 0;
#pragma unroll
                for (int st = 16; st; st >>= 1) {
                  uint32_t v = __shfl_sync(0xffffffffu, o, cc + st - 1);
                  if (v <= pp) cc += st;
                }
                e = e_cur + cc;
              }
              const uint32_t pp = p0 + lane;
              valid = pp < p_end;
              if (!valid) e = e_cur;
              e_out = e;
              unit = s_ustart[e] + (pp - s_P[e]);
              const int e31 = __shfl_sync(0xffffffffu, e, 31);
              e_cur = e31 + (s_P[e31 + 1] <= p0 + 32 ? 1 : 0);
              if (e_cur > n_items - 1) e_cur = n_items - 1;
            };
            int eA;
            uint32_t uA;
            bool vA;
            lookup(p_begin, eA, uA, vA);
            uint4 idA = make_uint4(0, 0, 0, 0);
            uint2 wA = make_uint2(0, 0);
            if (vA) {
              idA = ldg_nc_v4(p.ids + (size_t)uA * 8);
              if (wint8) wA = ldg_nc_v2(p.vals + (size_t)uA * 8);
            }
            for (uint32_t p0 = p_begin; p0 < p_end; p0 += 32) {
              int eB = 0;
              uint32_t uB = 0;
              bool vB = false;
              uint4 idB = make_uint4(0, 0, 0, 0);
              uint2 wB = make_uint2(0, 0);
              if (p0 + 32 < p_end) {
                lookup(p0 + 32, eB, uB, vB);
                if (vB) {
                  idB = ldg_nc_v4(p.ids + (size_t)uB * 8);
                  if (wint8) wB = ldg_nc_v2(p.vals + (size_t)uB * 8);
                }
              }
              if (vA) {
                const uint32_t mask = s_fm[eA] >> 24;
                const uint32_t wd[4] = {idA.x, idA.y, idA.z, idA.w};
                uint32_t off4[8], w8[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  off4[j] = ((wd[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu) * 4u;
                  w8[j] = wint8 ? (((j < 4 ? wA.x : wA.y) >> (8 * (j & 3))) & 0xFFu) : 1u;
                }
#pragma unroll
                for (int b = 0; b < B; ++b) {
                  if (mask & (1u << b)) {
                    const uint32_t q = (uint32_t)s_q[eA * B + b];
                    const uint32_t rb = acc_s + (uint32_t)(b * TS * 4);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                      red_add_shared(rb + off4[j], wint8 ? q * w8[j] : q);
                    }
                  }
                }
                if (p.counters) {
                  int nid = 0;
#pragma unroll
                  for (int j = 0; j < 8; ++j) nid += off4[j] < (uint32_t)T * 4u;
                  n_visits += (unsigned long long)nid * __popc(mask);
                }
              }
              eA = eB; uA = uB; vA = vB; idA = idB; wA = wB;
            }
          }
          __syncthreads();
        }
      }
      // -------------------------------------------------------------------- scan + top-k (a5)
      {
        const int cols = T / kWarps;
        const int cbase = warp * cols;
        const uint32_t gbase = (uint32_t)(p.s_id_base + t * (int64_t)T);
#pragma unroll
        for (int b = 0; b < B; ++b) {
          if (b < nb) {
            uint64_t th = own[b];
            {
              const uint64_t sh = *(volatile uint64_t*)&s_theta[b];
              if (sh > th) th = sh;
            }
            uint32_t* row = acc + (size_t)b * TS;
            for (int c = 0; c < cols; c += 128) {
              const int col = cbase + c + lane * 4;
              uint4 v = *(uint4*)(row + col);
              *(uint4*)(row + col) = make_uint4(0, 0, 0, 0);
              const uint32_t thh = (uint32_t)(th >> 32), thl = (uint32_t)th;
              const uint32_t g0 = gbase + (uint32_t)col;
              const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
              bool any = false;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                any |= vv[j] > thh || (vv[j] == thh && (0xFFFFFFFFu - (g0 + j)) > thl);
              if (__any_sync(0xffffffffu, any)) {
                {
                  const uint64_t sh = *(volatile uint64_t*)&s_theta[b];
                  if (sh > th) th = sh;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint64_t key = vv[j] ? make_key(vv[j], g0 + j) : 0;
                  int n = list_offer_lanes<KS>(L[b], key, th, k, lane);
                  n_inserts += (lane == 0) ? n : 0;
                }
                const uint64_t nk = list_kth<KS>(L[b], k);
                if (nk > own[b]) {
                  own[b] = nk;
                  if (lane == 0) atomicMax((unsigned long long*)&s_theta[b], (unsigned long long)nk);
                }
              }
            }
          }
        }
        __syncthreads();
      }
    }
    // ---------------------------------------------------------------------- merge lists + finalize (a7)
    {
      uint64_t* scratch = (uint64_t*)acc;  // [kWarps][B][k]; acc columns < T are all zero here
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int s = 0; s < KS; ++s)
          if (s * 32 + lane < k) scratch[((size_t)warp * B + b) * k + s * 32 + lane] = L[b][s];
      __syncthreads();
      if (warp < nb) {
        uint64_t M[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s) M[s] = 0;
        uint64_t th = kKeyFloor;
        for (int w = 0; w < kWarps; ++w) {
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            const int pos = s * 32 + lane;
            uint64_t c = pos < k ? scratch[((size_t)w * B + warp) * k + pos] : 0;
            list_offer_lanes<KS>(M, c, th, k, lane);
          }
        }
        const int64_t r = row0 + warp;
        list_finalize<KS>(M, k, r, p.inv_sigma[r], p.out_keys, p.out_ids, p.out_scores, lane);
      }
      __syncthreads();
      for (int i = tid; i < kWarps * B * k; i += kThreads) scratch[i] = 0;
    }
  }
  if (p.counters) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n_visits += __shfl_xor_sync(0xffffffffu, n_visits, o);
      n_inserts += __shfl_xor_sync(0xffffffffu, n_inserts, o);
    }
    if (lane == 0) {
      atomicAdd(&p.counters[0], n_visits);
      atomicAdd(&p.counters[1], n_inserts);
    }
  }
}

// ------------------------------------------------------------------------------------ host dispatch
struct QueryWs {
  size_t sigma_at, inv_at, runs_f_at, runs_q_at, nruns_at, counter_at, total;
};

const int kBChoices[] = {8, 6, 4, 2, 1};

int pick_batch_rows(int T, int k, int requested) {
  int KS = ks_for_k(k);
  auto fits = [&](int B) -> bool {
    size_t bytes = 0;
    switch (B) {
      case 1: bytes = Smem<1>::bytes(T, k); break;
      case 2: bytes = Smem<2>::bytes(T, k); break;
      case 4: bytes = Smem<4>::bytes(T, k); break;
      case 6: bytes = Smem<6>::bytes(T, k); break;
      case 8: bytes = Smem<8>::bytes(T, k); break;
      default: return false;
    }
    if (B * KS > 24) return false;
    return bytes <= 227 * 1024;
  };
  if (requested) return fits(requested) ? requested : -1;
  for (int B : kBChoices)
    if (fits(B)) return B;
  return -1;
}

bool query_ws_layout(int64_t n_r, int64_t nnz_r, int B, QueryWs* W) {
  int64_t n_batches = (n_r + B - 1) / B;
  size_t at = 0;
  W->sigma_at = at;   at = align_up(at + 8 * (size_t)n_r, 256);
  W->inv_at = at;     at = align_up(at + 8 * (size_t)n_r, 256);
  W->runs_f_at = at;  at = align_up(at + 4 * (size_t)nnz_r, 256);
  W->runs_q_at = at;  at = align_up(at + 4 * (size_t)nnz_r * B, 256);
  W->nruns_at = at;   at = align_up(at + 4 * (size_t)n_batches, 256);
  W->counter_at = at; at = align_up(at + 16, 256);
  W->total = at;
  return true;
}

template <int B, int KS, bool SINT8>
cudaError_t launch_main3(const QP& p, int grid, cudaStream_t st) {
  size_t sm = Smem<B>::bytes(p.T, p.k);
  cudaError_t e = cudaFuncSetAttribute(k_accumulate_topk<B, KS, SINT8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_accumulate_topk<B, KS, SINT8><<<grid, kThreads, sm, st>>>(p);
  return cudaGetLastError();
}

template <int B, int KS>
cudaError_t launch_main(const QP& p, int grid, cudaStream_t st) {
  return p.vals ? launch_main3<B, KS, true>(p, grid, st) : launch_main3<B, KS, false>(p, grid, st);
}

template <int B>
cudaError_t launch_ks(const QP& p, int grid, cudaStream_t st) {
  switch (ks_for_k(p.k)) {
    case 1: return launch_main<B, 1>(p, grid, st);
    case 4: if constexpr (B * 4 <= 24) return launch_main<B, 4>(p, grid, st); else return cudaErrorInvalidValue;
    case 8: if constexpr (B * 8 <= 24) return launch_main<B, 8>(p, grid, st); else return cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

bool check_query_args(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k) {
  if (!idx || !R) { set_error("index or R is NULL"); return false; }
  if (k < 1 || k > kMaxK) { set_error("k must be in [1, %d] (got %d)", kMaxK, k); return false; }
  if (R->n_rows < 0 || R->nnz < 0) { set_error("negative R size"); return false; }
  if (R->dtype != KNNJOIN_BINARY && R->dtype != KNNJOIN_INT8 && R->dtype != KNNJOIN_FP32) { set_error("bad R dtype"); return false; }
  return true;
}

}  // namespace

void launch_row_scale(const knnjoin_csr* R, int32_t d, int32_t smax, double* sigma, double* inv_sigma,
                      cudaStream_t st) {
  if (R->n_rows <= 0) return;
  int64_t threads = R->n_rows * 32;
  k_row_scale_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      R->indptr, R->indices, R->dtype == KNNJOIN_FP32 ? (const float*)R->values : nullptr, R->n_rows, d, smax, sigma,
      inv_sigma);
}

}  // namespace kj

using namespace kj;

KJ_API size_t knnjoin_query_workspace_bytes(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k,
                                            const knnjoin_query_options* qopt) {
  if (!check_query_args(idx, R, k)) return 0;
  int B = pick_batch_rows(idx->tile, k, qopt ? qopt->batch_rows : 0);
  if (B < 0) { set_error("no batch size fits shared memory for tile %d, k %d", idx->tile, k); return 0; }
  QueryWs W;
  query_ws_layout(R->n_rows, R->nnz, B, &W);
  return W.total;
}

KJ_API knnjoin_status knnjoin_query(const knnjoin_index* idx, const knnjoin_csr* R, int32_t k,
                                    const knnjoin_query_options* qopt, uint64_t* out_keys, int32_t* out_ids,
                                    float* out_scores, void* workspace, size_t workspace_bytes, void* stream) {
  if (!check_query_args(idx, R, k)) return KNNJOIN_ERR_ARG;
  if (R->n_rows == 0) return KNNJOIN_OK;  // empty R: nothing to write
  if (!out_keys && (!out_ids || !out_scores)) { set_error("need out_keys or both out_ids and out_scores"); return KNNJOIN_ERR_ARG; }
  const bool integer = R->dtype != KNNJOIN_FP32;
  if (integer && (double)idx->d * 127.0 * 127.0 >= 4294967296.0) {
    set_error("integer scores may overflow 32 bits for d = %d", idx->d);
    return KNNJOIN_ERR_UNSUPPORTED;
  }
  int B = pick_batch_rows(idx->tile, k, qopt ? qopt->batch_rows : 0);
  if (B < 0) { set_error("batch_rows %d unsupported for tile %d, k %d", qopt ? qopt->batch_rows : 0, idx->tile, k); return KNNJOIN_ERR_UNSUPPORTED; }
  QueryWs W;
  query_ws_layout(R->n_rows, R->nnz, B, &W);
  if (!workspace || workspace_bytes < W.total) { set_error("query workspace %zu < %zu bytes", workspace_bytes, W.total); return KNNJOIN_ERR_WORKSPACE; }
  if ((uintptr_t)workspace & 255) { set_error("workspace must be 256-byte aligned"); return KNNJOIN_ERR_ARG; }
  if (R->n_rows == 0) return KNNJOIN_OK;
  if (!R->indptr || (R->nnz > 0 && !R->indices) || (R->dtype != KNNJOIN_BINARY && R->nnz > 0 && !R->values)) {
    set_error("R pointers are NULL");
    return KNNJOIN_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* wb = (char*)workspace;
  double* sigma = (double*)(wb + W.sigma_at);
  double* inv_sigma = (double*)(wb + W.inv_at);
  uint32_t* runs_f = (uint32_t*)(wb + W.runs_f_at);
  int32_t* runs_q = (int32_t*)(wb + W.runs_q_at);
  uint32_t* nruns = (uint32_t*)(wb + W.nruns_at);
  uint32_t* counter = (uint32_t*)(wb + W.counter_at);
  const int32_t smax = idx->s_dtype == KNNJOIN_INT8 ? 127 : 1;
  const int64_t n_batches = (R->n_rows + B - 1) / B;
  cudaError_t e;
  if ((e = cudaMemsetAsync(counter, 0, 16, st)) != cudaSuccess) return cuda_fail(e, "memset counter");
  launch_row_scale(R, idx->d, smax, sigma, inv_sigma, st);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_row_scale");
  {
    int64_t threads = n_batches * 32;
    k_build_runs<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(R->indptr, R->indices, R->values, R->dtype,
                                                                   R->n_rows, idx->d, B, n_batches, sigma, runs_f,
                                                                   runs_q, nruns);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_build_runs");
  }
  QP p;
  p.off = idx->off;
  p.ids = idx->ids;
  p.vals = idx->vals;
  p.d = idx->d;
  p.T = idx->tile;
  p.NT = idx->n_tiles;
  p.s_id_base = idx->s_id_base;
  p.n_r = R->n_rows;
  p.k = k;
  p.n_batches = n_batches;
  p.r_indptr = R->indptr;
  p.runs_f = runs_f;
  p.runs_q = runs_q;
  p.batch_nruns = nruns;
  p.inv_sigma = inv_sigma;
  p.batch_counter = counter;
  p.counters = (unsigned long long*)(qopt ? qopt->counters : nullptr);
  p.out_keys = out_keys;
  p.out_ids = out_ids;
  p.out_scores = out_scores;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = (int)(n_batches < sms ? n_batches : sms);
  if (qopt && qopt->ev_begin) cudaEventRecord((cudaEvent_t)qopt->ev_begin, st);
  switch (B) {
    case 1: e = launch_ks<1>(p, grid, st); break;
    case 2: e = launch_ks<2>(p, grid, st); break;
    case 4: e = launch_ks<4>(p, grid, st); break;
    case 6: e = launch_ks<6>(p, grid, st); break;
    case 8: e = launch_ks<8>(p, grid, st); break;
    default: e = cudaErrorInvalidValue;
  }
  if (qopt && qopt->ev_end) cudaEventRecord((cudaEvent_t)qopt->ev_end, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_accumulate_topk");
  return KNNJOIN_OK;
}
