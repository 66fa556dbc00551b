// accumulate.cuh -- K3: score accumulation (a4) fused with the per-tile top-k (a5) and the output (a7).
// Included by query.cu (host dispatch, shared-memory layout) and by accumulate_ks{1,4,8}.cu, which each
// instantiate the kernel for one top-k list width KS (slots per lane) so the instances compile in parallel.
#pragma once
#include "common.cuh"
#include "topk.cuh"

namespace kj {

struct QP {
  // index
  const uint32_t* off;
  const uint16_t* ids;
  int64_t unit_cap;          // 16-byte units of ids in the index (bounds checks of checked builds)
  const uint8_t* vals;
  const int32_t* head_slot;  // [d] head slot or -1
  const int32_t* head_feat;  // [kMaxHead + 1]; [kMaxHead] = number of head features
  const uint32_t* head_cols; // [n_tiles * T] head-feature bits per S row
  const int32_t* gate;       // nullptr, or the index's head count (device): the launch runs only when
  int32_t gate_heads;        //   (count > 0) == gate_heads (knnjoin_query launches both candidate shapes)
  int32_t d, T;
  int64_t NT;
  int64_t s_id_base;
  int32_t head_smem;         // shared memory holds head tables (0 only when the index has no head features)
  // R / batches
  int64_t n_r;
  int32_t k;
  int64_t n_batches;
  const int64_t* r_indptr;
  const int32_t* perm;      // [n_r] original row of each work-sorted position (nullptr: input order)
  const int64_t* rbase;     // [n_r] first run slot of each sorted position's row (nullptr: r_indptr)
  const uint32_t* runs_f;
  const int32_t* runs_q;
  const uint32_t* batch_nruns;
  const double* inv_sigma;
  uint32_t* batch_counter;
  int64_t t0, t1;           // S tiles [t0, t1) of the index this query covers
  const uint64_t* theta_in; // [n_r] per-row key floor (input row order): keys below it are not kept, or nullptr
  const uint64_t* resume;   // [n_r][k] keys of an earlier query over other tiles to continue from, or nullptr
  int64_t tiles_per_pass;   // S tiles per pass: all batches sweep pass 0, then pass 1, ... (L2 locality)
  int64_t n_passes;
  uint64_t* state_keys;     // [n_r][k] top-k keys carried between passes (n_passes > 1)
  uint32_t* pass_done;      // [n_batches] number of passes finished per batch
  int32_t split;            // 1: passes are independent tile groups (small R), each writing part_keys
  uint64_t* part_keys;      // [n_passes][n_r][k] per-group lists (split), merged by knnjoin's rank merge
  unsigned long long* counters;
  unsigned long long* phase;  // [8] cycles per phase (profiling), or nullptr
  // threshold pruning (a6; PRUNE instances only)
  float alpha;               // non-essential budget = min(alpha * theta, theta - 1)
  const uint2* prune_suf;    // [runs] per run: {sum of c over the runs at or after it in c-descending order, c}
  const int64_t* fwd_ptr;    // [n_s + 1] forward rows of S (local row ids)
  const int32_t* fwd_idx;    // [nnz(S)]
  const uint8_t* fwd_val;    // [nnz(S)] INT8 S weights, or nullptr (BINARY)
  const uint32_t* fmax;      // [d] largest S weight per feature, or nullptr (BINARY: 1)
  int32_t prune_words;       // (d + 31) / 32: shared bitmap of the row's non-essential features
  int32_t residual;          // f1 (IIIB-literal): every run is "non-essential" for the completion (its bit is
                             // set) but its slice is loaded; every touched s is completed with dot(r, s')
  // out
  uint64_t* out_keys;
  int32_t* out_ids;
  float* out_scores;
};

// Posting loads skip L1 (no reuse inside an SM) but must stay in L2 at normal priority: the slab of S tiles of
// the current pass is re-read by every batch.  (A bare L1::no_allocate load is issued as L2 evict-first on
// sm_100a -- ncu showed 80 % of C5's index sectors missing L2 -- so the L2 policy is given explicitly.)
__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}

// Streaming data read once per work item (a one-row item's runs): L2 evict-first, so that it does not push the
// pass slab of the index out of L2.  (The top-k state carried between passes keeps the default policy: evict-
// first on it measured 2-3 % slower on C2 / C4, whose items wait for it at entry.)
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t ldg_stream_u32(const void* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

namespace {

// -------------------------------------------------------------------------- block-wide scan helper
template <int NW>
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
  // every thread adds up the warp totals itself (one barrier instead of a second pass by warp 0 and another barrier)
  uint64_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint64_t y = s_warp[w];
    before += w < warp ? y : 0;
    tot += y;
  }
  *total = tot;
  return before + x - v;
}

// ------------------------------------------------------------------------------ a4 + a5 + a7 kernel
// Score rows have stride T + kPadCols: columns [T, T+32) absorb padding postings (never scanned).
__host__ __device__ inline int acc_stride(int T) { return T + kPadCols; }

// the score array doubles as the scratch of the end-of-batch list merge ([NW][B][k] keys)
__host__ __device__ inline size_t acc_region_bytes(int B, int T, int k, int NW) {
  size_t a = (size_t)B * acc_stride(T) * 4, m = (size_t)NW * B * k * 8;
  return align_up(a > m ? a : m, 16);
}

// shared-memory layout of k_accumulate_topk<B, ., ., NW>; the kernel derives its pointers from the same sums.
// Staging of one chunk of runs: q[cap][B], ustart[cap], fm[cap], P[cap + 1]; cap = runs per chunk (320 for
// 8-warp CTAs so that three CTAs with B = 2 fit on one SM, 512 for 16-warp CTAs).
__host__ __device__ constexpr int kcap(int NW) { return NW == 4 ? 256 : (NW == 8 ? 320 : 512); }
__host__ __device__ inline size_t staging_at(int B, int T, int k, int NW) { return acc_region_bytes(B, T, k, NW); }
// Head tables: lut[kMaxHead/4 groups][B][16] u32 (entry m of group g, row b = sum of q over the set bits of
// m among head slots 4g..4g+3), cum[B][kMaxHead+1] u32 (cum[b][p] = sum of the p largest head q of row b:
// an upper bound of the head part of any score whose S row shares p head features with r_b) and
// head_mask[B] u32 (head slots present in row b).  The per-slot q values they are built from
// (q_head[kMaxHead][B]) alias the staging area, which is free during batch setup.
// One-row head-free CTAs (B = 1, no head features: the per-warp path of k_accumulate_topk) use the staging area
// for per-warp run tables instead: warp w holds the runs [nruns*w/NW, nruns*(w+1)/NW) of the row, kRowRPL per lane
// in registers, and per tile a table of its non-empty slices -- start P in the warp's flattened unit stream
// ([kRowCapW + 1] u32) and {first unit - P, q} ([kRowCapW] uint2).
constexpr int kRowRPL = 6;
constexpr int kRowCapW = 32 * kRowRPL;
constexpr int kRowDepth = 2;    // windows whose posting loads are in flight while one is processed
__host__ __device__ inline size_t row_table_P_bytes() { return align_up((size_t)(kRowCapW + 1) * 4, 16); }
__host__ __device__ inline size_t row_table_warp_bytes() {
  return row_table_P_bytes() + (size_t)kRowCapW * 8;
}
__host__ __device__ inline size_t staging_bytes(int B, int NW, bool heads) {
  // (B <= 2: one 16-byte record {first unit - start, feature | row mask, q0, q1} per staged run, then the starts)
  const size_t chunk = (size_t)kcap(NW) * (B > 2 ? B : 2) * 4 + (size_t)kcap(NW) * 8 + (size_t)(kcap(NW) + 1) * 4;
  const size_t rows = (B == 1 && !heads) ? (size_t)NW * row_table_warp_bytes() : 0;
  return chunk > rows ? chunk : rows;
}
__host__ __device__ inline size_t head_at(int B, int T, int k, int NW, bool heads) {
  return align_up(staging_at(B, T, k, NW) + staging_bytes(B, NW, heads), 16);
}
// (heads = false: the index has no head features; the head tables and completion queues are left out so that
// six one-row CTAs fit on an SM)
__host__ __device__ inline size_t head_bytes(int B, bool heads) {
  return heads ? (size_t)(kMaxHead / 4) * B * 16 * 4 + (size_t)B * (kMaxHead + 1) * 4 + (size_t)B * 4 : 0;
}
__host__ __device__ inline size_t tail_at(int B, int T, int k, int NW, bool heads) {
  return align_up(head_at(B, T, k, NW, heads) + head_bytes(B, heads), 16);
}
__host__ __device__ inline size_t smem_bytes(int B, int T, int k, int NW, bool heads) {
  return tail_at(B, T, k, NW, heads) + (size_t)NW * 8 /* scan partials */ + (size_t)B * 8 /* theta */ +
         32 /* misc */ + (heads ? (size_t)NW * 32 * 4 : 0) /* completion queues */;
}

// read 4 scores and zero them in one instruction (ATOMS.EXCH.128: 110 B/clk/SM of scores against 64 for LDS.128 +
// STS.128, tools/microbench_scan2.cu; used by the head-free scan -- the head scan keeps LDS + STS, where the
// exchange measured 1.5-3 % slower)
__device__ __forceinline__ uint4 xchg_v4_zero(uint32_t addr) {
  uint4 r;
  asm volatile("{ .reg .b128 d, z; mov.b128 z, {%4,%4,%4,%4}; atom.shared.exch.b128 d, [%5], z; mov.b128 {%0,%1,%2,%3}, d; }"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(0u), "r"(addr) : "memory");
  return r;
}


__device__ __forceinline__ void red_add_shared(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));  // ordered by __syncthreads, not by clobbers
}


// HEADS = false: instance for indexes without head features (the head tables, bounds and completions are
// compiled out, which leaves the one-row short-slice path more registers).
// PRUNE = true (B = 1, HEADS = false only): threshold pruning, SURVEY.md §8(a) a6 -- the r-side form of IIIB's
// threshold refinement (Alg. 4).  Per tile, with theta = the score of the
// row's running k-th key, the runs whose c-descending suffix sum (prune_suf) is <= budget =
// min(alpha * theta, theta - 1) are non-essential (N): their slices are not loaded.  In the scan an s with
// partial score x > 0 is completed exactly (its forward row merged against N) when x + U_N >= theta, where
// U_N = sum of c over N's non-empty slices of the tile; any other s has score <= x + U_N < theta (or, with
// x = 0, <= U_N <= budget < theta) and cannot enter.
template <int B, int KS, bool SINT8, int NW, bool HEADS, bool PRUNE = false>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? ((B == 1 && !HEADS && !PRUNE) ? (KS >= 4 ? 4 : 5) : 6) : (NW == 8 ? (KS >= 8 ? 2 : 3) : 1))
    k_accumulate_topk(QP p) {
  static_assert(!PRUNE || (B == 1 && !HEADS), "pruned instances are one-row and head-free");
  constexpr bool ROWP = B == 1 && !HEADS && !PRUNE;  // one-row head-free instance: per-warp accumulate
  if (p.gate && ((*p.gate > 0) != (p.gate_heads != 0))) return;  // the other candidate shape runs
  constexpr int NT_ = NW * 32;        // threads per CTA
  constexpr int kCap = kcap(NW);      // runs staged per chunk
  constexpr int IPT = (kCap + NT_ - 1) / NT_;  // staged runs per thread (the last may be partial)
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = p.T;
  const int TS = acc_stride(T);
  uint32_t* acc = (uint32_t*)smem;
  const uint32_t acc_s = (uint32_t)__cvta_generic_to_shared(acc);
  constexpr int QS = B;
  int32_t* s_q = (int32_t*)(smem + staging_at(B, T, p.k, NW));
  uint32_t* s_ustart = (uint32_t*)(s_q + kCap * QS);
  uint32_t* s_fm = s_ustart + kCap;
  uint32_t* s_P = s_fm + kCap;
  uint4* s_ent = (uint4*)s_q;                // B <= 2: staged run records {first unit - start, fm, q0, q1}
  uint32_t* s_P2 = (uint32_t*)(s_ent + kCap);  //   and their starts (+ the total at [n])
  uint32_t* s_lut = (uint32_t*)(smem + head_at(B, T, p.k, NW, p.head_smem != 0));  // [kMaxHead/4][B][16]
  uint32_t* s_cum = s_lut + (kMaxHead / 4) * B * 16;                 // [B][kMaxHead + 1]
  uint32_t* s_hmask = s_cum + B * (kMaxHead + 1);                    // [B]
  int32_t* s_qh = s_q;                                                // [kMaxHead][B], aliases staging
  static_assert(kMaxHead * B <= kcap(NW) * B, "q_head must fit in the staging area");
  uint64_t* s_warp = (uint64_t*)(smem + tail_at(B, T, p.k, NW, p.head_smem));
  // [B] (u64 slots, low words used): max over the warps of the SCORE of their k-th key per row.  (score << 32) is a
  // lower bound of that key, so it is a valid admission floor; a 32-bit shared max is one native ATOMS.MAX where the
  // 64-bit key max was a CAS loop (ATOMS.CAST.SPIN.64)
  uint64_t* s_theta = s_warp + NW;
  uint32_t* s_tscore = (uint32_t*)s_theta;
  int* s_misc = (int*)(s_theta + B);         // [0] batch, [1] n sparse items, [2] TOT, [4] U_N (a6/f1)

  // lane from an opaque move: the compiler may not re-materialise it (an S2R + LOP3 per window, whose S2R latency
  // showed as short-scoreboard stalls in the posting loop)
  int lane_reg;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane_reg));
  const int tid = threadIdx.x, lane = lane_reg, warp = tid >> 5;
  uint32_t* s_queue = (uint32_t*)(s_misc + 8) + warp * 32;  // this warp's head-completion queue (heads only)
  // a6: bit f set <=> feature f of the batch row is non-essential in the current tile (placed after everything
  // else; the budget only grows within an item, so the bits of earlier tiles stay valid)
  uint32_t* s_nbits = (uint32_t*)(smem + align_up(smem_bytes(B, T, p.k, NW, p.head_smem), 16));
  const int k = p.k;
  constexpr bool wint8 = SINT8;
  const bool timing = p.phase != nullptr && tid == 0;
  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long t_mark = timing ? clock64() : 0;
  auto phase_mark = [&](int i) {
    if (timing) {
      const long long now = clock64();
      ph[i] += (unsigned long long)(now - t_mark);
      t_mark = now;
    }
  };
  unsigned long long n_visits = 0, n_inserts = 0, n_complete = 0, n_skipped = 0;
  const uint64_t l2pol = l2_policy_normal();
  const uint64_t l2first = l2_policy_first();
  const int n_head = (HEADS && p.head_smem) ? p.head_feat[kMaxHead] : 0;  // host: head_smem when n_head > 0
  const int n_groups = HEADS ? (n_head + 3) >> 2 : 0;

  for (int i = tid; i < (int)(acc_region_bytes(B, T, k, NW) / 16); i += NT_) ((uint4*)acc)[i] = make_uint4(0, 0, 0, 0);

  // Work items are (pass, batch) in pass-major order: every CTA sweeps the tiles of one pass (a slab of the
  // index sized to stay L2-resident) over all batches before any moves to the next pass.  A batch's top-k
  // keys are carried between its passes in global memory (state_keys); item (pass g, batch b) waits until
  // item (g - 1, b) -- fetched earlier, so already running or done -- has published them.
  const int64_t n_items = p.n_batches * p.n_passes;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_misc[0] = (int)atomicAdd(p.batch_counter, 1u);
    __syncthreads();
    const int64_t item = s_misc[0];
    if (item >= n_items) break;
    const int64_t pass = item / p.n_batches;
    const int64_t batch = item - pass * p.n_batches;
    const int64_t t_begin = p.t0 + pass * p.tiles_per_pass;
    const int64_t t_end = min(p.t1, t_begin + p.tiles_per_pass);
    const bool last_pass = pass == p.n_passes - 1;
    const int64_t row0 = batch * B;
    const int nb = (int)min((int64_t)B, p.n_r - row0);
    const int64_t run_base = p.rbase ? p.rbase[row0] : p.r_indptr[row0];
    const int nruns = (int)p.batch_nruns[batch];
    if (pass > 0 && !p.split) {
      if (tid == 0) {
        while (*(volatile uint32_t*)&p.pass_done[batch] < (uint32_t)pass) __nanosleep(200);
        __threadfence();
      }
      __syncthreads();
    }

    uint64_t L[B][KS];
    uint64_t own[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      own[b] = kKeyFloor;
#pragma unroll
      for (int s = 0; s < KS; ++s) L[b][s] = 0;
      if (pass > 0 && !p.split && warp == 0 && b < nb) {  // warp 0 resumes from the batch's merged list
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const int pos = s * 32 + lane;
          if (pos < k) L[b][s] = __ldcg((const unsigned long long*)p.state_keys + (size_t)(row0 + b) * k + pos);
        }
        own[b] = list_kth<KS>(L[b], k);
      } else if (pass == 0 && p.resume && warp == 0 && b < nb) {  // continue an earlier query's lists
        const int64_t r = p.perm ? (int64_t)p.perm[row0 + b] : row0 + b;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const int pos = s * 32 + lane;
          if (pos < k) L[b][s] = __ldg((const unsigned long long*)p.resume + (size_t)r * k + pos);
        }
        own[b] = list_kth<KS>(L[b], k);
      }
      if (p.theta_in && b < nb) {  // floor from other S shards (f2): keep keys >= floor only
        const int64_t r = p.perm ? (int64_t)p.perm[row0 + b] : row0 + b;
        const uint64_t f = __ldg((const unsigned long long*)p.theta_in + r);
        if (f > 0 && f - 1 > own[b]) own[b] = f - 1;
      }
    }
    if (warp == 0 && lane == 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) s_tscore[b] = (uint32_t)(own[b] >> 32);
    }
    if constexpr (PRUNE)
      for (int i = tid; i < p.prune_words; i += NT_) s_nbits[i] = 0;
    // ------------------------------------------------------------------ head tables of this batch
    if (n_groups) {
      for (int i = tid; i < kMaxHead * B; i += NT_) s_qh[i] = 0;
      if (tid < B) s_hmask[tid] = 0;
      __syncthreads();
      for (int i = tid; i < nruns; i += NT_) {
        const size_t run = (size_t)(run_base + i);
        const uint32_t fm = p.runs_f[run];
        const int sl = p.head_slot[fm & 0xFFFFFFu];
        if (sl >= 0) {
#pragma unroll
          for (int b = 0; b < B; ++b) s_qh[sl * B + b] = p.runs_q[run * B + b];
#pragma unroll
          for (int b = 0; b < B; ++b)
            if (fm & (1u << (24 + b))) atomicOr(&s_hmask[b], 1u << sl);
        }
      }
      __syncthreads();
      for (int i = tid; i < n_groups * B * 16; i += NT_) {
        const int g = i / (B * 16), b = (i / 16) % B, m = i & 15;
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (m & (1 << j)) v += (uint32_t)s_qh[(4 * g + j) * B + b];
        s_lut[i] = v;
      }
      if (warp < B) {  // cum[b]: prefix sums of row b's head q sorted descending (warp bitonic sort)
        uint32_t x = (uint32_t)s_qh[lane * B + warp];
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
          for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x, jj);
            const bool up = (lane & kk) == 0;           // descending overall
            const bool lower = (lane & jj) == 0;
            x = (lower == up) ? max(x, y) : min(x, y);
          }
        }
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        s_cum[warp * (kMaxHead + 1) + lane + 1] = incl;
        if (lane == 0) s_cum[warp * (kMaxHead + 1)] = 0;
      }
    }
    __syncthreads();
    phase_mark(5);

    const int64_t t_stop = nruns > 0 ? t_end : t_begin;
    // batches whose runs fit one staging chunk: the runs' features are loaded once per item instead of once
    // per tile (one dependent L2 round trip less in every stage)
    const bool one_chunk = nruns <= kCap;
    uint32_t fm_c[IPT];
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
      const int li = tid + it * NT_;
      fm_c[it] = (!ROWP && one_chunk && li < kCap && li < nruns) ? __ldg(p.runs_f + run_base + li) : 0u;
    }
    // One-row path (ROWP): warp w takes the runs [wr0, wr1) of the row for every tile -- no block-wide staging.
    // The first kRowCapW of them stay in registers for the whole item (kRowRPL per lane), and the end of each of
    // their slices in tile t+1 is loaded while tile t accumulates (a slice of tile t+1 starts where that of tile t
    // ends: units are feature-major); further runs (rows longer than NW * kRowCapW) are loaded per tile.
    const int wr0 = ROWP ? (int)(((int64_t)nruns * warp) / NW) : 0;
    const int wr1 = ROWP ? (int)(((int64_t)nruns * (warp + 1)) / NW) : 0;
    uint32_t r_o[kRowRPL];                // feature f of each held run (0xFFFFFFFF: none)
    uint32_t r_q[kRowRPL];                // its q
    uint32_t r_s[kRowRPL], r_e[kRowRPL];  // slice of the current tile: units [r_s, r_e) (r_e: loaded ahead)
    if constexpr (ROWP) {
#pragma unroll
      for (int g = 0; g < kRowRPL; ++g) {
        const int i = wr0 + 32 * g + lane;
        const bool v = i < wr1 && t_begin < t_stop;
        r_o[g] = v ? (ldg_stream_u32(p.runs_f + run_base + i, l2first) & 0xFFFFFFu) : 0xFFFFFFFFu;
        r_q[g] = v ? ldg_stream_u32(p.runs_q + run_base + i, l2first) : 0u;
        r_s[g] = v ? __ldg(p.off + (size_t)r_o[g] * (size_t)(p.NT + 1) + t_begin) : 0u;
        r_e[g] = v ? __ldg(p.off + (size_t)r_o[g] * (size_t)(p.NT + 1) + t_begin + 1) : 0u;
      }
    }
    for (int64_t t = t_begin; t < t_stop; ++t) {
      // a6: the non-essential budget of this tile, from the row's k-th key so far (every thread reads the same
      // value: s_theta is only written during scans, which are fenced by __syncthreads)
      uint32_t budget = 0;
      if constexpr (PRUNE) {
        const uint32_t th_s = *(volatile uint32_t*)&s_tscore[0];
        if (th_s > 0) {
          const double a = (double)p.alpha * (double)th_s;
          budget = a >= (double)(th_s - 1) ? th_s - 1 : (uint32_t)a;
        }
      }
      if constexpr (ROWP) {
        // ------------------------------------------------- one-row accumulate (a4): per-warp tables, no barrier
        unsigned char* wbase = smem + staging_at(B, T, k, NW) + (size_t)warp * row_table_warp_bytes();
        uint32_t* w_P = (uint32_t*)wbase;                                  // [n_ent + 1] starts
        uint2* w_bq = (uint2*)(wbase + row_table_P_bytes());               // [n_ent] {first unit - start, q}
        const uint32_t lt_mask = (1u << lane) - 1u;
        const int n_sc = (wr1 - wr0 + kRowCapW - 1) / kRowCapW;
        for (int sc = 0; sc < n_sc; ++sc) {
          const int cb = wr0 + sc * kRowCapW;  // first run of this super-chunk
          uint2 cu[kRowRPL];
          uint32_t cq[kRowRPL];
          if (sc == 0) {
#pragma unroll
            for (int g = 0; g < kRowRPL; ++g) {
              cu[g] = make_uint2(r_s[g], r_e[g]);
              cq[g] = r_q[g];
              if (r_o[g] != 0xFFFFFFFFu) {
                r_s[g] = r_e[g];
                if (t + 1 < t_stop) r_e[g] = __ldg(p.off + (size_t)r_o[g] * (size_t)(p.NT + 1) + t + 2);
              }
            }
          } else {  // rows with more than NW * kRowCapW runs: the further super-chunks are loaded per tile
#pragma unroll
            for (int g = 0; g < kRowRPL; ++g) {
              const int i = cb + 32 * g + lane;
              cu[g] = make_uint2(0u, 0u);
              cq[g] = i < wr1 ? __ldg(p.runs_q + run_base + i) : 0u;
              if (i < wr1) {
                const uint32_t* o = p.off + (size_t)(__ldg(p.runs_f + run_base + i) & 0xFFFFFFu) * (size_t)(p.NT + 1) + t;
                cu[g] = make_uint2(__ldg(o), __ldg(o + 1));
              }
            }
          }
          // table of the non-empty slices in run order: start P in the warp's unit stream, {first unit - P, q}
          uint32_t tot = 0, n_ent = 0;
#pragma unroll
          for (int g = 0; g < kRowRPL; ++g) {
            if (cb + 32 * g < wr1) {  // warp-uniform
              const uint32_t L = cu[g].y - cu[g].x;
              uint32_t incl = L;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
              }
              const uint32_t ne = __ballot_sync(0xffffffffu, L > 0);
              if (L > 0) {
                const uint32_t c = n_ent + __popc(ne & lt_mask);
                const uint32_t P = tot + incl - L;
                KJ_CHECK(c < (uint32_t)kRowCapW && (int64_t)cu[g].y <= p.unit_cap);
                w_P[c] = P;
                w_bq[c] = make_uint2(cu[g].x - P, cq[g]);
              }
              tot += __shfl_sync(0xffffffffu, incl, 31);
              n_ent += __popc(ne);
            }
          }
          if (lane == 0) w_P[n_ent] = tot;
          __syncwarp();
          phase_mark(0);
          const uint32_t wend = (tot + 31) >> 5;
          if (wend) {
            // software pipeline over the windows of 32 units (lane l takes unit 32m + l): R (the entries starting
            // inside window m, one OR-reduction of the next 32 starts past e_cur, the entry covering its first
            // unit) -> C (posting loads) -> process.  Every stage consumes shared-memory results loaded one step
            // earlier, so no step waits on a load issued in the same step; kRowDepth windows' posting loads are in
            // flight while one is processed.
            struct St {
              uint4 id;
              uint2 w;
              uint32_t q;
              bool v;
            };
            const int n_items = (int)n_ent;
            int e_cur = 0;  // entry covering the first unit of the next window stage R handles
            auto ldP = [&]() { return w_P[min(e_cur + 1 + lane, n_items)]; };
            // stage R for window m: pS = starts after e_cur (loaded one step earlier); returns {first unit - start,
            // q} of lane l's entry (a shared load consumed one step later) and advances e_cur, reloading pS
            auto stR = [&](uint32_t m, uint32_t& pS) -> uint2 {
              if (m >= wend) return make_uint2(0u, 0u);
              const uint32_t o = pS - m * 32;  // >= 1: e_cur covers unit 32m, so the next start lies past it
              const uint32_t M = __reduce_or_sync(0xffffffffu, o < 32 ? (1u << o) : 0u);
              const int e = e_cur + __popc(M & (lt_mask | (1u << lane)));
              const int e_next = e_cur + __popc(M) + (__ballot_sync(0xffffffffu, o == 32) ? 1 : 0);
              e_cur = min(e_next, n_items - 1);
              // lanes past the warp's last unit (tail of the last window) may count the end of the stream as a
              // start (e == n_items); their entry is clamped and stage C skips them
              KJ_CHECK(e >= 0 && (e < n_items || m * 32 + (uint32_t)lane >= tot));
              const uint2 bq = w_bq[min(e, n_items - 1)];
              pS = ldP();
              return bq;
            };
            auto stC = [&](uint32_t m, uint2 bq, St& S) {
              const uint32_t pp = m * 32 + lane;
              S.v = m < wend && pp < tot;
              if (S.v) {
                const uint32_t unit = bq.x + pp;
                KJ_CHECK((int64_t)unit < p.unit_cap);
                S.q = bq.y;
                if (wint8) S.w = ldg_nc_v2(p.vals + (size_t)unit * 8, l2pol);
                S.id = ldg_nc_v4(p.ids + (size_t)unit * 8, l2pol);
              }
            };
            auto process = [&](const St& S) {
              if (!S.v) return;
              const uint32_t wd[4] = {S.id.x, S.id.y, S.id.z, S.id.w};
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t o4 = (j & 1) ? (wd[j >> 1] >> 16) : (wd[j >> 1] & 0xFFFFu);  // byte offsets
                KJ_CHECK(o4 < 4u * (uint32_t)TS && (o4 & 3u) == 0);
                const uint32_t w8 = wint8 ? __byte_perm(j < 4 ? S.w.x : S.w.y, 0u, 0x4440u | (uint32_t)(j & 3)) : 1u;
                red_add_shared(acc_s + o4, wint8 ? S.q * w8 : S.q);
              }
              if (p.counters) {
                int nid = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) nid += ((j & 1) ? (wd[j >> 1] >> 16) : (wd[j >> 1] & 0xFFFFu)) < (uint32_t)T * 4u;
                n_visits += (unsigned long long)nid;
              }
            };
            constexpr int LD = kRowDepth;  // windows whose loads are in flight
            St D[LD + 1];
#pragma unroll
            for (int j = 0; j <= LD; ++j) {
              D[j].id = make_uint4(0, 0, 0, 0);
              D[j].w = make_uint2(0, 0);
              D[j].q = 0;
              D[j].v = false;
            }
            // each slot is refilled right after it is processed, so the loads of LD + 1 windows are in flight
            // while one is processed and a window's loads are issued LD + 1 steps before their use
            uint32_t pS = ldP();
#pragma unroll
            for (int j = 0; j <= LD; ++j) stC(j, stR(j, pS), D[j]);
            uint2 bqC = stR(LD + 1, pS);
            for (uint32_t w = 0; w < wend; w += LD + 1) {
#pragma unroll
              for (int j = 0; j <= LD; ++j) {
                process(D[j]);
                stC(w + j + LD + 1, bqC, D[j]);
                bqC = stR(w + j + LD + 2, pS);
              }
            }
          }
          __syncwarp();  // table reads done before the next super-chunk rewrites it
        }
        __syncthreads();
        phase_mark(1);
      } else
      for (int c0 = 0; c0 < nruns; c0 += kCap) {
        // ---------------------------------------------------------------- stage chunk of runs
        // non-empty slices are compacted with their position P in the flattened unit stream (head
        // features have empty slices: their postings live in head_cols)
        {
          uint32_t fm[IPT], u0[IPT], U[IPT];
          uint64_t pk[IPT], mine = 0;
          uint32_t un_mine = 0;  // a6: c of this thread's skipped non-empty slices
#pragma unroll
          for (int it = 0; it < IPT; ++it) {
            const int li = tid + it * NT_;  // run li of this chunk
            const int i = c0 + li;
            fm[it] = 0; u0[it] = 0; U[it] = 0;
            if (li < kCap && i < nruns) {
              fm[it] = one_chunk ? fm_c[it] : p.runs_f[(size_t)(run_base + i)];
              const uint32_t* o = p.off + (size_t)(fm[it] & 0xFFFFFFu) * (size_t)(p.NT + 1) + (size_t)t;
              u0[it] = o[0];
              U[it] = o[1] - u0[it];
              if constexpr (PRUNE) {
                const uint2 sc = p.residual ? make_uint2(0xFFFFFFFFu, 0u) : __ldg(p.prune_suf + run_base + i);
                if (p.residual) {  // f1: r's feature set for dot(r, s'), slices all loaded
                  const uint32_t f = fm[it] & 0xFFFFFFu;
                  atomicOr(&s_nbits[f >> 5], 1u << (f & 31u));
                } else if (sc.x <= budget) {  // non-essential: slice not loaded
                  const uint32_t f = fm[it] & 0xFFFFFFu;
                  atomicOr(&s_nbits[f >> 5], 1u << (f & 31u));
                  if (U[it] > 0) {
                    un_mine += sc.y;
                    n_skipped += U[it];
                  }
                  U[it] = 0;
                }
              }
            }
            pk[it] = ((uint64_t)(U[it] > 0) << 32) | U[it];
            mine += pk[it];
          }
          // U_N of this tile (read after the accumulate; f1 completes every touched s whatever U_N)
          if (PRUNE && c0 == 0 && tid == 0) s_misc[4] = 0;
          uint64_t total;
          uint64_t ex = block_exclusive_scan_u64<NW>(mine, s_warp, &total);
          if (PRUNE && un_mine) atomicAdd((unsigned*)&s_misc[4], un_mine);
#pragma unroll
          for (int it = 0; it < IPT; ++it) {
            if (U[it] > 0) {
              const uint32_t c = (uint32_t)(ex >> 32);
              KJ_CHECK(c < (uint32_t)kCap && (int64_t)u0[it] + U[it] <= p.unit_cap);
              const size_t run = (size_t)(run_base + c0 + tid + it * NT_);
              if constexpr (B <= 2) {
                const uint32_t P = (uint32_t)ex;
                s_ent[c] = make_uint4(u0[it] - P, fm[it], (uint32_t)p.runs_q[run * B],
                                      B == 2 ? (uint32_t)p.runs_q[run * B + 1] : 0u);
                s_P2[c] = P;
              } else {
                s_ustart[c] = u0[it];
                s_P[c] = (uint32_t)ex;
                s_fm[c] = fm[it];
#pragma unroll
                for (int b = 0; b < B; ++b) s_q[c * QS + b] = p.runs_q[run * B + b];
              }
            }
            ex += pk[it];
          }
          if (tid == 0) {
            const uint32_t ns = (uint32_t)(total >> 32);
            s_misc[1] = (int)ns;
            s_misc[2] = (int)(uint32_t)total;
            if constexpr (B <= 2) s_P2[ns] = (uint32_t)total;
            else s_P[ns] = (uint32_t)total;
          }
          __syncthreads();
          phase_mark(0);
        }
        // ---------------------------------------------------------------- accumulate (a4)
        {
          const int n_items = s_misc[1];
          const uint32_t TOT = (uint32_t)s_misc[2];
          const uint32_t nwin = (TOT + 31) >> 5;
          // Warp w takes the contiguous windows [nwin*w/NW, nwin*(w+1)/NW): balanced to one window, one binary
          // search per warp, one continuous load pipeline.  (With several rows a window costs one atomic per
          // posting per row of its run; grabbing 8-window chunks from a shared counter, or splitting by that
          // cost, both measured slower on C2/C4: 4.10 / 4.24 ms against 3.86 ms for this split.)
          {
            const uint32_t w0 = (uint32_t)(((uint64_t)nwin * warp) / NW);
            const uint32_t w1 = (uint32_t)(((uint64_t)nwin * (warp + 1)) / NW);
            if (w0 < w1) {
            const uint32_t p_begin = w0 * 32, p_end = min(TOT, w1 * 32);
            const uint32_t* sP = B <= 2 ? s_P2 : s_P;
            int lo = 0, hi = n_items - 1;  // largest e with P[e] <= p_begin
            while (lo < hi) {
              int mid = (lo + hi + 1) >> 1;
              if (sP[mid] <= p_begin) lo = mid; else hi = mid - 1;
            }
            if constexpr (B <= 2) {
              // software pipeline (as in the one-row path): R (entry of each lane: one OR-reduction of the next 32
              // starts past e_cur; the record load) -> C (posting loads) -> process, each stage consuming shared
              // loads issued one step earlier
              int e_cur = lo;
              struct St2 {
                uint4 id;
                uint2 w;
                uint32_t fm, q0, q1;
                bool v;
              };
              const uint32_t le_mask = (2u << lane) - 1u;
              auto ldP = [&]() { return s_P2[min(e_cur + 1 + lane, n_items)]; };
              auto stR = [&](uint32_t p0, uint32_t& pS) -> uint4 {
                if (p0 >= p_end) return make_uint4(0u, 0u, 0u, 0u);
                const uint32_t o = pS - p0;  // >= 1
                const uint32_t M = __reduce_or_sync(0xffffffffu, o < 32 ? (1u << o) : 0u);
                const int e = e_cur + __popc(M & le_mask);
                const int e_next = e_cur + __popc(M) + (__ballot_sync(0xffffffffu, o == 32) ? 1 : 0);
                e_cur = min(e_next, n_items - 1);
                KJ_CHECK(e >= 0 && (e < n_items || p0 + lane >= p_end));
                const uint4 ent = s_ent[min(e, n_items - 1)];
                pS = ldP();
                return ent;
              };
              auto stC = [&](uint32_t p0, const uint4& ent, St2& S) {
                const uint32_t pp = p0 + lane;
                S.v = p0 < p_end && pp < p_end;
                if (S.v) {
                  const uint32_t unit = ent.x + pp;
                  KJ_CHECK((int64_t)unit < p.unit_cap);
                  S.fm = ent.y >> 24;
                  S.q0 = ent.z;
                  S.q1 = ent.w;
                  S.id = ldg_nc_v4(p.ids + (size_t)unit * 8, l2pol);
                  if (wint8) S.w = ldg_nc_v2(p.vals + (size_t)unit * 8, l2pol);
                }
              };
              auto process2 = [&](const St2& S) {
                if (!S.v) return;
                const uint32_t wd[4] = {S.id.x, S.id.y, S.id.z, S.id.w};
                uint32_t off4[8], w8[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  off4[j] = (j & 1) ? (wd[j >> 1] >> 16) : (wd[j >> 1] & 0xFFFFu);
                  KJ_CHECK(off4[j] < 4u * (uint32_t)TS && (off4[j] & 3u) == 0);
                  w8[j] = wint8 ? __byte_perm(j < 4 ? S.w.x : S.w.y, 0u, 0x4440u | (uint32_t)(j & 3)) : 1u;
                }
#pragma unroll
                for (int b = 0; b < B; ++b) {
                  if (S.fm & (1u << b)) {
                    const uint32_t q = b == 0 ? S.q0 : S.q1;
                    const uint32_t rb = acc_s + (uint32_t)(b * TS * 4);
#pragma unroll
                    for (int j = 0; j < 8; ++j) red_add_shared(rb + off4[j], wint8 ? q * w8[j] : q);
                  }
                }
                if (p.counters) {
                  int nid = 0;
#pragma unroll
                  for (int j = 0; j < 8; ++j) nid += off4[j] < (uint32_t)T * 4u;
                  n_visits += (unsigned long long)nid * __popc(S.fm & ((1u << B) - 1u));
                }
              };
              constexpr int LD = B == 1 ? 2 : 1;  // windows whose posting loads are in flight
              St2 D[LD + 1];
#pragma unroll
              for (int j = 0; j <= LD; ++j) {
                D[j].id = make_uint4(0, 0, 0, 0);
                D[j].w = make_uint2(0, 0);
                D[j].fm = D[j].q0 = D[j].q1 = 0;
                D[j].v = false;
              }
              uint32_t pS = ldP();
#pragma unroll
              for (int j = 0; j < LD; ++j) stC(p_begin + 32 * j, stR(p_begin + 32 * j, pS), D[j]);
              uint4 entC = stR(p_begin + 32 * LD, pS);
              for (uint32_t p0 = p_begin; p0 < p_end; p0 += 32 * (LD + 1)) {
#pragma unroll
                for (int j = 0; j <= LD; ++j) {
                  stC(p0 + 32 * (j + LD), entC, D[(j + LD) % (LD + 1)]);
                  entC = stR(p0 + 32 * (j + LD + 1), pS);
                  process2(D[j]);
                }
              }
            } else {
            int e_cur = lo;
            struct Stage {
              uint4 id;
              uint2 w;
              int e;
              bool v;
            };
            // lane l takes unit p0 + l.  e_cur is the item covering p0; the items starting inside the window
            // are found with one OR-reduction of their start offsets (starts are strictly increasing).
            // Windows must be fetched in ascending order (e_cur advances).
            auto fetch = [&](Stage& S, uint32_t p0) {
              S.v = false;
              S.e = e_cur;
              if (p0 >= p_end) return;
              const uint32_t nxt = s_P[e_cur + 1];
              int e = e_cur, e_next;
              if (p0 + 32 > nxt) {
                const int j = min(e_cur + 1 + lane, n_items);
                const uint32_t o = s_P[j] - p0;  // >= 1
                const uint32_t M = __reduce_or_sync(0xffffffffu, o < 32 ? (1u << o) : 0u);
                e = e_cur + __popc(M & (0xFFFFFFFFu >> (31 - lane)));
                e_next = e_cur + __popc(M) + (__ballot_sync(0xffffffffu, o == 32) ? 1 : 0);
              } else {
                e_next = e_cur + (nxt == p0 + 32 ? 1 : 0);
              }
              const uint32_t pp = p0 + lane;
              S.v = pp < p_end;
              if (!S.v) e = e_cur;
              S.e = e;
              e_cur = min(e_next, n_items - 1);
              if (S.v) {
                const uint32_t unit = s_ustart[e] + (pp - s_P[e]);
                KJ_CHECK(e >= 0 && e < n_items && pp >= s_P[e] && pp < s_P[e + 1] && (int64_t)unit < p.unit_cap);
                S.id = ldg_nc_v4(p.ids + (size_t)unit * 8, l2pol);
                if (wint8) S.w = ldg_nc_v2(p.vals + (size_t)unit * 8, l2pol);
              }
            };
            auto process = [&](const Stage& S) {
              if (!S.v) return;
              const uint32_t mask = s_fm[S.e] >> 24;
              const uint32_t wd[4] = {S.id.x, S.id.y, S.id.z, S.id.w};
              uint32_t off4[8], w8[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                off4[j] = (j & 1) ? (wd[j >> 1] >> 16) : (wd[j >> 1] & 0xFFFFu);  // stored as byte offsets
                KJ_CHECK(off4[j] < 4u * (uint32_t)TS && (off4[j] & 3u) == 0);
                // byte j & 3 zero-extended in one PRMT (selector nibbles 4 = a zero byte of the second operand)
                w8[j] = wint8 ? __byte_perm(j < 4 ? S.w.x : S.w.y, 0u, 0x4440u | (uint32_t)(j & 3)) : 1u;
              }
#pragma unroll
              for (int b = 0; b < B; ++b) {
                if (mask & (1u << b)) {
                  const uint32_t q = (uint32_t)s_q[S.e * QS + b];
                  const uint32_t rb = acc_s + (uint32_t)(b * TS * 4);
#pragma unroll
                  for (int j = 0; j < 8; ++j) red_add_shared(rb + off4[j], wint8 ? q * w8[j] : q);
                }
              }
              if (p.counters) {
                int nid = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) nid += off4[j] < (uint32_t)T * 4u;
                n_visits += (unsigned long long)nid * __popc(mask);
              }
            };
            Stage A, Bs, C;
            A.id = Bs.id = C.id = make_uint4(0, 0, 0, 0);
            A.w = Bs.w = C.w = make_uint2(0, 0);
            fetch(A, p_begin);
            if constexpr (B == 1) {  // two windows in flight (registers are plentiful at one row)
              fetch(Bs, p_begin + 32);
              for (uint32_t p0 = p_begin; p0 < p_end; p0 += 96) {
                fetch(C, p0 + 64);
                process(A);
                fetch(A, p0 + 96);
                process(Bs);
                fetch(Bs, p0 + 128);
                process(C);
              }
            } else {  // one window in flight
              for (uint32_t p0 = p_begin; p0 < p_end; p0 += 32) {
                fetch(Bs, p0 + 32);
                process(A);
                A = Bs;
              }
            }
            }  // B > 2
            }
          }
          __syncthreads();
          phase_mark(1);
        }
      }
      // -------------------------------------------------------------------- scan + top-k (a5)
      // warp w owns columns [w*T/NW, (w+1)*T/NW); per 128-column step every lane reads the 4 accumulated
      // scores (id-list features) of each row and offers keys above theta to the warp's register top-k list
      // of that row, then zero-fills.  With head features the accumulated score is only part of the score:
      // it is completed exactly, from the lookup tables, only where the upper bound
      //     acc + cum[b][popc(head bits of s & head mask of r_b)]   (the largest head weights of r_b)
      // reaches theta (the threshold refinement of IIIB) -- a pair whose bound is below
      // theta cannot enter the top-k, so skipping its completion changes nothing.
      {
        const int cols = T / NW;
        const int cbase = warp * cols;
        const uint32_t gbase = (uint32_t)(p.s_id_base + t * (int64_t)T);
        const uint32_t* hcols = p.head_cols + (size_t)t * T + cbase + lane * 4;
        uint4 hq = make_uint4(0, 0, 0, 0);
        if (n_groups) hq = __ldg((const uint4*)hcols);
        // theta of row b = max over the warps' k-th keys (k keys at least that large exist in one list, so a
        // candidate key below it cannot be in the row's final top-k; reading c1 total order)
        auto row_theta = [&](int b) {
          const uint64_t sh = (uint64_t)(*(volatile uint32_t*)&s_tscore[b]) << 32;
          return sh > own[b] ? sh : own[b];
        };
        // cheap superset test: key > theta needs score >= t32 (theta's score, +1 when theta's id part admits
        // no id); the exact 64-bit key comparison happens in list_offer_lanes
        auto t32_of = [](uint64_t th) {
          return (uint32_t)(th >> 32) + ((uint32_t)th == 0xFFFFFFFFu ? 1u : 0u);
        };
        auto publish = [&](int b) {
          const uint64_t nk = list_kth<KS>(L[b], k);
          if (nk > own[b]) {
            own[b] = nk;
            if (lane == 0) atomicMax(&s_tscore[b], (uint32_t)(nk >> 32));
          }
        };
        uint64_t th[B];
#pragma unroll
        for (int b = 0; b < B; ++b) th[b] = row_theta(b);
        if (n_groups == 0) {
          // no head features: the accumulated score is the score.  Per 128-column step a lane reads 4 scores
          // of each row (32-bit shared addresses), zero-fills, and only a warp with a score >= theta's score
          // leaves the fast loop to offer its keys.
          uint32_t t32[B];
#pragma unroll
          for (int b = 0; b < B; ++b) t32[b] = t32_of(th[b]);
          const uint32_t a0 = acc_s + (uint32_t)(cbase + lane * 4) * 4u;
          // a6: U_N of this tile (0 when nothing was skipped: the plain filter)
          const uint32_t un = PRUNE ? (uint32_t)s_misc[4] : 0u;  // <= budget < theta: x + un cannot wrap
          const bool all_touched = PRUNE && p.residual;           // f1: complete every s with x != 0
          // a6 exact completion of s = local column col: add r's non-essential features that s has, merging s's
          // forward row against the row's runs (both ascending by feature)
          auto complete = [&](uint32_t col) -> uint32_t {
            uint32_t add = 0;
            if constexpr (PRUNE) {
              const int64_t srow = t * (int64_t)T + col;
              const int64_t e0 = __ldg(p.fwd_ptr + srow), e1 = __ldg(p.fwd_ptr + srow + 1);
              int lo = 0;
              // s's features are tested against the shared bitmap of N; a hit (rare: |s & N| is small) finds
              // its q by a binary search of the row's runs (ascending features) from the previous hit on
              for (int64_t e = e0; e < e1; e += 4) {
                uint32_t fs[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) fs[j] = e + j < e1 ? (uint32_t)__ldg(p.fwd_idx + e + j) : 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint32_t f = fs[j];
                  if (f == 0xFFFFFFFFu || f >= (uint32_t)p.d || !((s_nbits[f >> 5] >> (f & 31u)) & 1u)) continue;
                  int hi = nruns;  // lower bound of f in runs [lo, nruns): f is a feature of r, so it is found
                  while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if ((__ldg(p.runs_f + run_base + mid) & 0xFFFFFFu) < f) lo = mid + 1; else hi = mid;
                  }
                  add += (uint32_t)__ldg(p.runs_q + run_base + lo) * (p.fwd_val ? (uint32_t)__ldg(p.fwd_val + e + j) : 1u);
                  ++lo;
                }
              }
              ++n_complete;
            }
            return add;
          };
#pragma unroll 2
          for (int c = 0; c < cols; c += 128) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
              if (b < nb) {
                const uint32_t a = a0 + (uint32_t)(b * TS + c) * 4u;
                const uint4 x = xchg_v4_zero(a);
                const uint32_t mx = max(max(x.x, x.y), max(x.z, x.w));
                if (__any_sync(0xffffffffu, PRUNE ? (mx != 0u && (all_touched || mx + un >= t32[b])) : mx >= t32[b])) {
                  th[b] = row_theta(b);
                  const uint32_t g0 = gbase + (uint32_t)(cbase + c + lane * 4);
                  uint32_t xv[4] = {x.x, x.y, x.z, x.w};
                  if constexpr (PRUNE) {
                    if (un || all_touched) {
                      const uint32_t tc = t32_of(th[b]);
#pragma unroll
                      for (int j = 0; j < 4; ++j)
                        if (xv[j] != 0u && (all_touched || xv[j] + un >= tc))
                          xv[j] += complete((uint32_t)(cbase + c + lane * 4 + j));
                    }
                  }
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const uint64_t key = xv[j] ? make_key(xv[j], g0 + j) : 0;
                    const int n = list_offer_lanes<KS>(L[b], key, th[b], k, lane);  // warp-collective
                    n_inserts += (lane == 0) ? n : 0;
                  }
                  publish(b);
                  t32[b] = t32_of(th[b]);
                }
              }
            }
          }
        }
        // deferred exact completion of queued (row, column) pairs: lane l completes entry l -- the head part
        // from the lookup tables, added to the partial score left in the score array, which it then zeroes
        int qn = 0;  // queued pairs (warp-uniform)
        auto flush = [&]() {
          if (qn == 0) return;
          uint64_t key = 0;
          int pb = -1;
          if (lane < qn) {
            const uint32_t ent = s_queue[lane];
            pb = (int)(ent >> 16);
            const int cl = (int)(ent & 0xFFFFu);  // column within the tile
            KJ_CHECK(pb >= 0 && pb < B && cl < T);
            const uint32_t w = __ldg(p.head_cols + (size_t)t * T + cl);
            uint32_t* ap = acc + (size_t)pb * TS + cl;
            uint32_t sc = *ap;
            *ap = 0;
            const uint32_t* lutb = s_lut + pb * 16;
            for (int g = 0; g < n_groups; ++g) sc += lutb[g * B * 16 + ((w >> (4 * g)) & 15u)];
            uint64_t thb = th[0];
#pragma unroll
            for (int b = 1; b < B; ++b)
              if (pb == b) thb = th[b];
            key = make_key(sc, gbase + (uint32_t)cl);
            if (!(sc && key > thb)) key = 0;  // the exact score does not beat this row's theta
          }
          __syncwarp();
          if (__ballot_sync(0xffffffffu, key != 0)) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
              if (__ballot_sync(0xffffffffu, key != 0 && pb == b)) {
                const int n = list_offer_lanes<KS>(L[b], pb == b ? key : 0, th[b], k, lane);
                n_inserts += (lane == 0) ? n : 0;
                if (n) publish(b);
              }
            }
          }
          qn = 0;
        };
        uint32_t hmr[B];  // head slots present in each row (constant over the item)
#pragma unroll
        for (int b = 0; b < B; ++b) hmr[b] = n_groups ? s_hmask[b] : 0u;
        if (n_groups)
        for (int c = 0; c < cols; c += 128) {
          const int col = cbase + c + lane * 4;
          const uint32_t g0 = gbase + (uint32_t)col;
          uint32_t v[B][4];
#pragma unroll
          for (int b = 0; b < B; ++b) {
            if (b < nb) {
              const uint4 x = *(const uint4*)(acc + (size_t)b * TS + col);
              v[b][0] = x.x; v[b][1] = x.y; v[b][2] = x.z; v[b][3] = x.w;
            } else {
              v[b][0] = v[b][1] = v[b][2] = v[b][3] = 0;
            }
          }
          bool plain = n_groups == 0;
          uint32_t keep = 0;  // bit 4b+j: pair left in the score array for the deferred completion
          if (n_groups) {
            const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
            if (c + 128 < cols) hq = __ldg((const uint4*)(hcols + c + 128));  // next step's head words
            uint32_t pend = 0;  // bit 4b+j: pair (row b, column col+j) may reach theta
            uint32_t tsb[B];    // the rows' shared floors, one 64-bit load for two rows
            if constexpr (B == 2) {
              const unsigned long long t2 = *(volatile unsigned long long*)s_tscore;
              tsb[0] = (uint32_t)t2;
              tsb[1] = (uint32_t)(t2 >> 32);
            } else {
#pragma unroll
              for (int b = 0; b < B; ++b) tsb[b] = *(volatile uint32_t*)&s_tscore[b];
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
              if (b < nb) {
                const uint64_t sh = (uint64_t)tsb[b] << 32;
                th[b] = sh > own[b] ? sh : own[b];
                const uint32_t t32 = t32_of(th[b]);
                const uint32_t hm = hmr[b];
                const uint32_t* cum = s_cum + b * (kMaxHead + 1);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint32_t nh = __popc(hw[j] & hm);
                  const bool need = v[b][j] + cum[nh] >= t32;
                  if (need) pend |= 1u << (4 * b + j);
                  if (p.counters) {
                    n_visits += nh;
                    n_complete += need;
                    n_skipped += need ? 0u : nh;
                  }
                }
              }
            }
            // usually no pair of the step can reach theta: one vote, and the count (REDUX) only when some can
            const int npend = __any_sync(0xffffffffu, pend != 0u) ? __reduce_add_sync(0xffffffffu, __popc(pend)) : 0;
            if (npend > 32) {
              // many pairs may reach theta (the first tiles of a batch, theta still low): complete every pair
              // from the tables and take the plain filter below
#pragma unroll 1
              for (int g = 0; g < n_groups; ++g) {
                const uint32_t* lutg = s_lut + g * B * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint32_t m = (hw[j] >> (4 * g)) & 15u;
#pragma unroll
                  for (int b = 0; b < B; ++b) v[b][j] += lutg[b * 16 + m];
                }
              }
              plain = true;
            } else if (npend) {
              // exact completion is deferred: the pending pairs are appended to the warp's queue (their partial
              // scores stay in the score array) and completed 32 at a time, one per lane
              if (qn + npend > 32) flush();
              int excl = __popc(pend);
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, excl, o);
                if (lane >= o) excl += y;
              }
              excl -= __popc(pend);
              uint32_t pp = pend;
              for (int e = qn + excl; pp; ++e) {
                const int i = __ffs(pp) - 1;
                pp &= pp - 1;
                s_queue[e] = ((uint32_t)(i >> 2) << 16) | (uint32_t)(col + (i & 3));
              }
              qn += npend;
              __syncwarp();
              keep = pend;
            }
          }
          if (plain) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
              if (b < nb) {
                const uint32_t t32 = t32_of(th[b]);
                const bool any = (v[b][0] >= t32) | (v[b][1] >= t32) | (v[b][2] >= t32) | (v[b][3] >= t32);
                if (__any_sync(0xffffffffu, any) && t32 != 0u) {
                  th[b] = row_theta(b);
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const uint64_t key = v[b][j] ? make_key(v[b][j], g0 + j) : 0;
                    int n = list_offer_lanes<KS>(L[b], key, th[b], k, lane);
                    n_inserts += (lane == 0) ? n : 0;
                  }
                  publish(b);
                }
              }
            }
          }
          if (keep == 0u) {  // the usual case: zero-fill the lane's 4 columns of every row
#pragma unroll
            for (int b = 0; b < B; ++b)
              if (b < nb) *(uint4*)(acc + (size_t)b * TS + col) = make_uint4(0u, 0u, 0u, 0u);
          } else {
#pragma unroll
            for (int b = 0; b < B; ++b)
              if (b < nb) {  // zero-fill, except queued pairs (their completion reads and then zeroes them)
                const uint32_t kb = keep >> (4 * b);
                *(uint4*)(acc + (size_t)b * TS + col) =
                    make_uint4(kb & 1u ? v[b][0] : 0u, kb & 2u ? v[b][1] : 0u, kb & 4u ? v[b][2] : 0u,
                               kb & 8u ? v[b][3] : 0u);
              }
          }
        }
        flush();
        __syncthreads();
        phase_mark(3);
      }
    }
    // ---------------------------------------------------------------------- merge lists + finalize (a7)
    {
      uint64_t* scratch = (uint64_t*)acc;  // [NW][B][k]; acc columns < T are all zero here
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int s = 0; s < KS; ++s)
          if (s * 32 + lane < k) scratch[((size_t)warp * B + b) * k + s * 32 + lane] = L[b][s];
      __syncthreads();
      // The NW lists of a row are sorted and hold distinct keys (distinct columns), so the merged position
      // of a key is its position in its own list plus the number of larger keys in the other lists (binary
      // searches): every thread places keys independently.  Positions past the row's positive keys are
      // padding (reading c2).
      auto emit = [&](int b, int pos, uint64_t key) {
        if (p.split) {  // independent tile groups: this group's list, merged by rank after the kernel
          const int64_t r = p.perm ? (int64_t)p.perm[row0 + b] : row0 + b;
          p.part_keys[((size_t)pass * p.n_r + r) * k + pos] = key;
          return;
        }
        if (!last_pass) {  // state is kept per sorted position
          __stcg((unsigned long long*)p.state_keys + (size_t)(row0 + b) * k + pos, (unsigned long long)key);
          return;
        }
        const int64_t r = p.perm ? (int64_t)p.perm[row0 + b] : row0 + b;
        const size_t o = (size_t)r * k + pos;
        const uint32_t score = (uint32_t)(key >> 32);
        if (score == 0) {
          if (p.out_keys) p.out_keys[o] = 0;
          if (p.out_ids) p.out_ids[o] = -1;
          if (p.out_scores) p.out_scores[o] = 0.0f;
        } else {
          if (p.out_keys) p.out_keys[o] = key;
          if (p.out_ids) p.out_ids[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)key);
          if (p.out_scores) p.out_scores[o] = (float)((double)score * p.inv_sigma[r]);
        }
      };
      auto count_gt = [&](const uint64_t* lst, uint64_t x) {  // keys > x in a descending list of k
        int lo = 0, hi = k;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (lst[mid] > x) lo = mid + 1; else hi = mid;
        }
        return lo;
      };
      for (int i = tid; i < NW * B * k; i += NT_) {
        const int w = i / (B * k), b = (i / k) % B, pos = i % k;
        if (b >= nb) continue;
        const uint64_t x = scratch[i];
        if (x == 0) continue;
        int rank = pos;
        for (int w2 = 0; w2 < NW && rank < k; ++w2)
          if (w2 != w) rank += count_gt(scratch + ((size_t)w2 * B + b) * k, x);
        if (rank < k) emit(b, rank, x);
      }
      for (int i = tid; i < B * k; i += NT_) {
        const int b = i / k, pos = i % k;
        if (b >= nb) continue;
        int npos = 0;
        for (int w = 0; w < NW && npos <= pos; ++w) npos += count_gt(scratch + ((size_t)w * B + b) * k, 0);
        if (pos >= npos) emit(b, pos, 0);
      }
      __syncthreads();
      if (!last_pass && !p.split && tid == 0) {
        __threadfence();
        atomicExch(&p.pass_done[batch], (uint32_t)(pass + 1));
      }
      for (int i = tid; i < NW * B * k; i += NT_) scratch[i] = 0;
      phase_mark(4);
    }
  }
  if (timing) {
#pragma unroll
    for (int i = 0; i < 6; ++i) atomicAdd(&p.phase[i], ph[i]);
  }
  if (p.counters) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n_visits += __shfl_xor_sync(0xffffffffu, n_visits, o);
      n_inserts += __shfl_xor_sync(0xffffffffu, n_inserts, o);
      n_complete += __shfl_xor_sync(0xffffffffu, n_complete, o);
      n_skipped += __shfl_xor_sync(0xffffffffu, n_skipped, o);
    }
    if (lane == 0) {
      atomicAdd(&p.counters[0], n_visits);
      atomicAdd(&p.counters[1], n_inserts);
      atomicAdd(&p.counters[2], n_skipped);
      atomicAdd(&p.counters[3], n_complete);
    }
  }
}

}  // namespace

struct Shape {
  int B, NW;
};

// launches k_accumulate_topk<B, KS, ...> for the shape; defined (explicitly instantiated) in accumulate_ks<KS>.cu
template <int KS>
cudaError_t launch_accumulate(const Shape& sh, const QP& p, int sms, cudaStream_t st);

#ifdef KJ_ACCUMULATE_INSTANCES
namespace {
template <int B, int KS, bool SINT8, int NW, bool HEADS, bool PRUNE = false>
cudaError_t launch_main4(const QP& p, int sms, cudaStream_t st) {
  const size_t sm = align_up(smem_bytes(B, p.T, p.k, NW, p.head_smem != 0), 16) + (PRUNE ? 4 * (size_t)p.prune_words : 0);
  auto kern = k_accumulate_topk<B, KS, SINT8, NW, HEADS, PRUNE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, sm)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > p.n_batches * p.n_passes) grid = p.n_batches * p.n_passes;
  grid = checked_grid_cap(grid);
  kern<<<(unsigned)grid, NW * 32, sm, st>>>(p);
  return cudaGetLastError();
}

template <int B, int KS, int NW>
cudaError_t launch_main(const QP& p, int sms, cudaStream_t st) {
  if constexpr (B * KS <= 24 && B <= NW) {
    if constexpr (B == 1 && NW == 4) {  // the auto shape of indexes without head features
      if (p.prune_suf || p.residual)  // pruned queries (a6), residual completion (f1)
        return p.vals ? launch_main4<B, KS, true, NW, false, true>(p, sms, st)
                      : launch_main4<B, KS, false, NW, false, true>(p, sms, st);
      if (!p.head_smem)
        return p.vals ? launch_main4<B, KS, true, NW, false>(p, sms, st) : launch_main4<B, KS, false, NW, false>(p, sms, st);
    }
    return p.vals ? launch_main4<B, KS, true, NW, true>(p, sms, st) : launch_main4<B, KS, false, NW, true>(p, sms, st);
  } else {
    return cudaErrorInvalidValue;
  }
}
}  // namespace

template <int KS>
cudaError_t launch_accumulate(const Shape& sh, const QP& p, int sms, cudaStream_t st) {
  if (sh.NW == 4) {
    switch (sh.B) {
      case 1: return launch_main<1, KS, 4>(p, sms, st);
      case 2: return launch_main<2, KS, 4>(p, sms, st);
    }
  } else if (sh.NW == 8) {
    switch (sh.B) {
      case 1: return launch_main<1, KS, 8>(p, sms, st);
      case 2: return launch_main<2, KS, 8>(p, sms, st);
      case 3: return launch_main<3, KS, 8>(p, sms, st);
      case 4: return launch_main<4, KS, 8>(p, sms, st);
    }
  } else {
    switch (sh.B) {
      case 1: return launch_main<1, KS, 16>(p, sms, st);
      case 2: return launch_main<2, KS, 16>(p, sms, st);
      case 4: return launch_main<4, KS, 16>(p, sms, st);
      case 6: return launch_main<6, KS, 16>(p, sms, st);
      case 8: return launch_main<8, KS, 16>(p, sms, st);
    }
  }
  return cudaErrorInvalidValue;
}
#endif

}  // namespace kj
