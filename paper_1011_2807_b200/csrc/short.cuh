// short.cuh -- K3 for indexes WITHOUT head features, one R row per work item (the auto shape of C1, C3, C5: uniform or
// banded features, short posting slices).  Same computation as k_accumulate_topk<1, KS, SINT8, 4, false> (a4 + a5 +
// a7 of SURVEY.md §8), organised as a warp-specialised bulk-copy pipeline:
//
//   warp 0 (producer)   for each item (pass, row) and S tile: reads the row's slice bounds from the offset table
//                       (32 runs per step), packs the tile's slices into pipeline stages (<= kCU 16-byte units,
//                       <= kCR pieces per stage; a slice longer than a stage's room is split into pieces) and moves
//                       each piece into shared memory with cp.async.bulk (TMA 1-D copies: the ids, and for INT8 S
//                       the weights), completion tracked by the stage's "full" mbarrier (expect_tx per copy);
//   warps 1..7 (consumers)  wait for a stage, scatter its postings into the row's score array with shared-memory
//                       atomics (lane = unit: a per-unit piece index gives the run's q without any search), release
//                       the stage ("empty" mbarrier); at the end of a tile they scan the score array with the
//                       running top-k filter (a5) and, at the end of the item, merge their lists by rank (a7).
//
// The slices of C3 / C5 are 4-8 units: the old kernel fetched them with dependent 16-byte loads (a lookup of the
// unit's run, then an L2 round trip per window), so its warps spent a third of their time on long-scoreboard
// stalls.  Here the copies of a whole stage are in flight at once, issued by one warp ahead of the consumers,
// and the consumers read posting data from shared memory.
#pragma once
#include "accumulate.cuh"

namespace kj {
namespace shortk {

constexpr int kNW = 8;                // warps per CTA
constexpr int kNC = kNW - 1;          // consumer warps
constexpr int kThreads = kNW * 32;
constexpr int kNST = 3;               // pipeline stages
constexpr int kCU = 512;              // 16-byte id units per stage
constexpr int kCR = 128;              // pieces (slice parts) per stage
constexpr uint32_t kFirst = 1, kTileEnd = 2, kItemEnd = 4, kStop = 8;

// stage layout (byte offsets)
__host__ __device__ constexpr size_t st_ids() { return 0; }
__host__ __device__ constexpr size_t st_vals() { return 16 * (size_t)kCU; }
// piece starts: bit u of pbits <=> a piece starts at unit u; pbase[w] = piece starts in words < w
__host__ __device__ constexpr size_t st_pbits(bool i8) { return st_vals() + (i8 ? 8 * (size_t)(kCU + 2 * kCR) : 0); }
__host__ __device__ constexpr size_t st_pbase(bool i8) { return st_pbits(i8) + 4 * (size_t)(kCU / 32); }
__host__ __device__ constexpr size_t st_q(bool i8) { return st_pbase(i8) + 4 * (size_t)(kCU / 32); }
__host__ __device__ constexpr size_t st_P(bool i8) { return st_q(i8) + 4 * (size_t)kCR; }
__host__ __device__ constexpr size_t st_dv(bool i8) { return st_P(i8) + 2 * (size_t)kCR; }
__host__ __device__ constexpr size_t st_meta(bool i8) { return st_dv(i8) + 2 * (size_t)kCR; }
__host__ __device__ constexpr size_t stage_bytes(bool i8) { return (st_meta(i8) + 32 + 127) / 128 * 128; }

__host__ __device__ inline size_t acc_bytes(int T, int k) {
  const size_t a = (size_t)(T + kPadCols) * 4, m = (size_t)kNC * k * 8;
  return align_up(a > m ? a : m, 128);
}
constexpr int kRunCap = 1024;  // runs of the item cached in shared memory (features, q, slice bounds of two tiles)
// [acc][stages][full mbarriers][empty mbarriers][theta u64][misc][run f][run q][slice bounds 2 x run x 2]
__host__ __device__ inline size_t smem_total(int T, int k, bool i8) {
  return acc_bytes(T, k) + kNST * stage_bytes(i8) + 2 * kNST * 8 + 8 + 56 + (size_t)kRunCap * (4 + 4 + 16);
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(sa(bar))
               : "memory");
}
__device__ __forceinline__ void consumers_sync() {  // the kNC consumer warps only (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(kNC * 32) : "memory");
}

template <int KS, bool SINT8>
__global__ void __launch_bounds__(kThreads, 2) k_accumulate_short(QP p) {
  if (p.gate && ((*p.gate > 0) != (p.gate_heads != 0))) return;  // the other candidate shape runs
  extern __shared__ __align__(128) unsigned char smem[];
  const int T = p.T, k = p.k;
  uint32_t* acc = (uint32_t*)smem;
  const uint32_t acc_s = sa(acc);
  unsigned char* stages = smem + acc_bytes(T, k);
  constexpr size_t SB = stage_bytes(SINT8);
  uint64_t* full = (uint64_t*)(stages + kNST * SB);
  uint64_t* empty = full + kNST;
  uint64_t* s_theta = empty + kNST;
  uint32_t* s_misc = (uint32_t*)(s_theta + 1);
  uint32_t* s_rf = s_misc + 14;                   // [kRunCap] features of the item's runs (producer)
  int32_t* s_rq = (int32_t*)(s_rf + kRunCap);     // [kRunCap] q of the runs
  uint32_t* s_off = (uint32_t*)(s_rq + kRunCap);  // [2][kRunCap][2] slice bounds of the current / next tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_items = p.n_batches * p.n_passes;

  for (int i = tid; i < (int)(acc_bytes(T, k) / 16); i += kThreads) ((uint4*)acc)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < kNST; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], kNC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ======================================================================== producer
    uint32_t n = 0;                  // stages produced
    int fill_u = 0, fill_s = 0, fill_v = 0;
    bool open = false;
    unsigned char* st = stages;
    const uint64_t pol = l2_policy_normal();
    (void)pol;
    auto open_stage = [&]() {
      const int s = (int)(n % kNST);
      if (n >= (uint32_t)kNST) mbar_wait(&empty[s], ((n / kNST) - 1) & 1);
      st = stages + s * SB;
      if (lane < kCU / 32) ((uint32_t*)(st + st_pbits(SINT8)))[lane] = 0;
      __syncwarp();
      fill_u = fill_s = fill_v = 0;
      open = true;
    };
    auto commit = [&](uint32_t flags, uint32_t item, uint32_t tile) {
      if (!open) open_stage();
      __syncwarp();  // the piece-start bits of every lane are in place
      if (lane < kCU / 32) {  // pbase: exclusive prefix of the words' piece-start counts
        uint32_t c = __popc(((const uint32_t*)(st + st_pbits(SINT8)))[lane]), x = c;
#pragma unroll
        for (int o = 1; o < kCU / 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFu, x, o);
          if (lane >= o) x += y;
        }
        ((uint32_t*)(st + st_pbase(SINT8)))[lane] = x - c;
      }
      if (lane == 0) {
        uint32_t* meta = (uint32_t*)(st + st_meta(SINT8));
        meta[0] = (uint32_t)fill_u;
        meta[1] = (uint32_t)fill_s;
        meta[2] = flags;
        meta[3] = item;
        meta[4] = tile;
      }
      __syncwarp();
      mbar_arrive(&full[n % kNST]);  // 32 arrivals: each lane releases its own header / piece-index writes
      ++n;
      open = false;
    };
    for (;;) {
      uint32_t item32 = 0;
      if (lane == 0) item32 = atomicAdd(p.batch_counter, 1u);
      item32 = __shfl_sync(0xffffffffu, item32, 0);
      const int64_t item = item32;
      if (item >= n_items) {
        commit(kStop, 0, 0);
        break;
      }
      const int64_t pass = item / p.n_batches;
      const int64_t batch = item - pass * p.n_batches;
      const int64_t t_begin = p.t0 + pass * p.tiles_per_pass;
      const int64_t t_end = min(p.t1, t_begin + p.tiles_per_pass);
      const int64_t run_base = p.rbase ? p.rbase[batch] : p.r_indptr[batch];
      const int nruns = (int)p.batch_nruns[batch];
      uint32_t first = kFirst;
      // the item's runs are cached in shared memory and the slice bounds of tile t+1 are fetched with cp.async
      // while tile t is packed (rows with more than kRunCap runs read both from global memory)
      const bool cached = nruns <= kRunCap;
      auto prefetch_bounds = [&](int64_t tt, int slot) {
        for (int i = lane; i < nruns; i += 32) {
          const uint32_t* o = p.off + (size_t)s_rf[i] * (size_t)(p.NT + 1) + (size_t)tt;
          const uint32_t dst = sa(s_off + ((size_t)slot * kRunCap + i) * 2);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(o) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4), "l"(o + 1) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      if (cached && nruns > 0) {
        for (int i = lane; i < nruns; i += 32) {
          s_rf[i] = __ldg(p.runs_f + run_base + i) & 0xFFFFFFu;
          s_rq[i] = __ldg(p.runs_q + run_base + i);
        }
        __syncwarp();
        if (t_begin < t_end) prefetch_bounds(t_begin, 0);
      }
      for (int64_t t = t_begin; nruns > 0 && t < t_end; ++t) {
        bool tile_any = false;
        const int slot = (int)((t - t_begin) & 1);
        if (cached) {
          if (t + 1 < t_end) {
            prefetch_bounds(t + 1, slot ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
        }
        for (int g0 = 0; g0 < nruns; g0 += 32) {
          const int i = g0 + lane;
          uint32_t u0 = 0, rem = 0;
          int32_t q = 0;
          if (i < nruns) {
            if (cached) {
              const uint2 b = *(const uint2*)(s_off + ((size_t)slot * kRunCap + i) * 2);
              q = s_rq[i];
              u0 = b.x;
              rem = b.y - b.x;
            } else {
              const uint32_t f = __ldg(p.runs_f + run_base + i) & 0xFFFFFFu;
              q = __ldg(p.runs_q + run_base + i);
              const uint32_t* o = p.off + (size_t)f * (size_t)(p.NT + 1) + (size_t)t;
              u0 = __ldg(o);
              rem = __ldg(o + 1) - u0;
            }
          }
          while (__any_sync(0xffffffffu, rem > 0)) {
            tile_any = true;
            if (!open) open_stage();
            const bool has = rem > 0;
            const uint32_t lt = (1u << lane) - 1u;
            const int rank = __popc(__ballot_sync(0xffffffffu, has) & lt);
            uint32_t x = has ? rem : 0u;  // exclusive prefix of the pending units
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
              if (lane >= o) x += y;
            }
            x -= has ? rem : 0u;
            const uint32_t cap_u = (uint32_t)(kCU - fill_u), cap_s = (uint32_t)(kCR - fill_s);
            uint32_t take = 0;
            if (has && (uint32_t)rank < cap_s && x < cap_u) take = min(rem, cap_u - x);
            // weights (INT8 S): the copy is widened to 16-byte ends, [v0, v1) in 8-byte units
            const uint32_t v0 = u0 & ~1u, v1 = (u0 + take + 1u) & ~1u, vun = take ? v1 - v0 : 0u;
            uint32_t xv = vun;  // exclusive prefix of the weight units
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, xv, o);
              if (lane >= o) xv += y;
            }
            xv -= vun;
            if (take) {
              uint64_t* bar = &full[n % kNST];
              const int e = fill_s + rank;
              const uint32_t P = (uint32_t)fill_u + x;
              const uint32_t dv = (uint32_t)fill_v + xv;
              ((int32_t*)(st + st_q(SINT8)))[e] = q;
              ((uint16_t*)(st + st_P(SINT8)))[e] = (uint16_t)P;
              ((uint16_t*)(st + st_dv(SINT8)))[e] = (uint16_t)(dv + (u0 - v0));
              atomicOr((uint32_t*)(st + st_pbits(SINT8)) + (P >> 5), 1u << (P & 31u));
              mbar_expect_tx(bar, 16u * take);
              bulk_g2s(sa(st + st_ids() + 16 * (size_t)P), p.ids + (size_t)u0 * 8, 16u * take, bar);
              if constexpr (SINT8) {
                mbar_expect_tx(bar, 8u * vun);
                bulk_g2s(sa(st + st_vals() + 8 * (size_t)dv), p.vals + (size_t)v0 * 8, 8u * vun, bar);
              }
            }
            fill_s += __popc(__ballot_sync(0xffffffffu, take > 0));
            fill_u += (int)__reduce_add_sync(0xffffffffu, take);
            fill_v += (int)__reduce_add_sync(0xffffffffu, vun);
            u0 += take;
            rem -= take;
            if (__any_sync(0xffffffffu, rem > 0)) {  // the stage is full: hand it over, continue in the next
              commit(first, (uint32_t)item, (uint32_t)t);
              first = 0;
            }
          }
        }
        if (tile_any) {
          commit(first | kTileEnd, (uint32_t)item, (uint32_t)t);
          first = 0;
        }
      }
      commit(first | kItemEnd, (uint32_t)item, 0);
    }
    return;
  }

  // ========================================================================== consumers (warps 1..7)
  const int c = warp - 1;
  const int ctid = tid - 32;
  uint64_t L[KS];
  uint64_t own = kKeyFloor, th = kKeyFloor;
  unsigned long long n_visits = 0, n_inserts = 0;
  int64_t item = -1, pass = 0, batch = 0;
  bool last_pass = true;
  auto row_theta = [&]() {
    const uint64_t sh = *(volatile uint64_t*)s_theta;
    return sh > own ? sh : own;
  };
  auto t32_of = [](uint64_t x) { return (uint32_t)(x >> 32) + ((uint32_t)x == 0xFFFFFFFFu ? 1u : 0u); };
  auto publish = [&]() {
    const uint64_t nk = list_kth<KS>(L, k);
    if (nk > own) {
      own = nk;
      if (lane == 0) atomicMax((unsigned long long*)s_theta, (unsigned long long)nk);
    }
  };
  uint32_t n = 0;
  for (;;) {
    const int s = (int)(n % kNST);
    mbar_wait(&full[s], (n / kNST) & 1);
    const unsigned char* st = stages + s * SB;
    const uint32_t* meta = (const uint32_t*)(st + st_meta(SINT8));
    const uint32_t n_units = meta[0], flags = meta[2], tile = meta[4];  // read before the stage is released
    if (flags & kStop) break;
    if (flags & kFirst) {
      // ------------------------------------------------------------------ item start: the row's running list
      item = meta[3];
      pass = item / p.n_batches;
      batch = item - pass * p.n_batches;
      last_pass = pass == p.n_passes - 1;
      if (pass > 0 && !p.split) {
        if (ctid == 0) {
          while (*(volatile uint32_t*)&p.pass_done[batch] < (uint32_t)pass) __nanosleep(200);
          __threadfence();
        }
        consumers_sync();
      }
      own = kKeyFloor;
#pragma unroll
      for (int ss = 0; ss < KS; ++ss) L[ss] = 0;
      if (pass > 0 && !p.split && c == 0) {
#pragma unroll
        for (int ss = 0; ss < KS; ++ss) {
          const int pos = ss * 32 + lane;
          if (pos < k) L[ss] = __ldcg((const unsigned long long*)p.state_keys + (size_t)batch * k + pos);
        }
        own = list_kth<KS>(L, k);
      } else if (pass == 0 && p.resume && c == 0) {
        const int64_t r = p.perm ? (int64_t)p.perm[batch] : batch;
#pragma unroll
        for (int ss = 0; ss < KS; ++ss) {
          const int pos = ss * 32 + lane;
          if (pos < k) L[ss] = __ldg((const unsigned long long*)p.resume + (size_t)r * k + pos);
        }
        own = list_kth<KS>(L, k);
      }
      if (p.theta_in) {
        const int64_t r = p.perm ? (int64_t)p.perm[batch] : batch;
        const uint64_t f = __ldg((const unsigned long long*)p.theta_in + r);
        if (f > 0 && f - 1 > own) own = f - 1;
      }
      if (c == 0 && lane == 0) *s_theta = own;
      consumers_sync();
      th = row_theta();
    }
    // -------------------------------------------------------------------- accumulate the stage (a4)
    {
      const uint32_t* pbits = (const uint32_t*)(st + st_pbits(SINT8));
      const uint32_t* pbase = (const uint32_t*)(st + st_pbase(SINT8));
      const int32_t* sq = (const int32_t*)(st + st_q(SINT8));
      const uint16_t* sP = (const uint16_t*)(st + st_P(SINT8));
      const uint16_t* sdv = (const uint16_t*)(st + st_dv(SINT8));
      for (uint32_t w = (uint32_t)c * 32; w < n_units; w += kNC * 32) {
        const uint32_t pp = w + lane;
        if (pp < n_units) {
          const int e = (int)(pbase[pp >> 5] + __popc(pbits[pp >> 5] & (0xFFFFFFFFu >> (31u - (pp & 31u))))) - 1;
          const uint32_t q = (uint32_t)sq[e];
          const uint4 id = *(const uint4*)(st + st_ids() + 16 * (size_t)pp);
          const uint32_t wd[4] = {id.x, id.y, id.z, id.w};
          uint2 wv = make_uint2(0, 0);
          if constexpr (SINT8) wv = *(const uint2*)(st + st_vals() + 8 * (size_t)(sdv[e] + (pp - sP[e])));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t off = (j & 1) ? (wd[j >> 1] >> 16) : (wd[j >> 1] & 0xFFFFu);
            uint32_t v = q;
            if constexpr (SINT8) v = q * __byte_perm(j < 4 ? wv.x : wv.y, 0u, 0x4440u | (uint32_t)(j & 3));
            red_add_shared(acc_s + off, v);
            if (p.counters) n_visits += off < 4u * (uint32_t)T ? 1 : 0;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++n;
    }
    if (flags & kTileEnd) {
      // ------------------------------------------------------------------ scan + top-k of the tile (a5)
      consumers_sync();  // every atomic of the tile has landed
      const int64_t t = tile;
      const uint32_t gbase = (uint32_t)(p.s_id_base + t * (int64_t)T);
      th = row_theta();
      uint32_t t32 = t32_of(th);
      for (int cs = c * 128; cs < T; cs += kNC * 128) {
        const int col = cs + lane * 4;
        const uint32_t a = acc_s + (uint32_t)col * 4u;
        const uint4 x = lds_v4(a);
        sts_v4_zero(a);
        const uint32_t mx = max(max(x.x, x.y), max(x.z, x.w));
        if (__any_sync(0xffffffffu, mx >= t32)) {
          th = row_theta();
          const uint32_t xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t key = xv[j] ? make_key(xv[j], gbase + (uint32_t)(col + j)) : 0;
            const int ni = list_offer_lanes<KS>(L, key, th, k, lane);  // warp-collective
            n_inserts += (lane == 0) ? ni : 0;
          }
          publish();
          t32 = t32_of(th);
        }
      }
      consumers_sync();  // the score array is zero again before the next tile's atomics
    }
    if (flags & kItemEnd) {
      // ------------------------------------------------------------------ merge the consumers' lists (a7)
      uint64_t* scratch = (uint64_t*)acc;  // [kNC][k]; acc columns < T are all zero here
#pragma unroll
      for (int ss = 0; ss < KS; ++ss)
        if (ss * 32 + lane < k) scratch[(size_t)c * k + ss * 32 + lane] = L[ss];
      consumers_sync();
      auto emit = [&](int pos, uint64_t key) {
        if (p.split) {
          const int64_t r = p.perm ? (int64_t)p.perm[batch] : batch;
          p.part_keys[((size_t)pass * p.n_r + r) * k + pos] = key;
          return;
        }
        if (!last_pass) {
          __stcg((unsigned long long*)p.state_keys + (size_t)batch * k + pos, (unsigned long long)key);
          return;
        }
        const int64_t r = p.perm ? (int64_t)p.perm[batch] : batch;
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
      auto count_gt = [&](const uint64_t* lst, uint64_t x) {
        int lo = 0, hi = k;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (lst[mid] > x) lo = mid + 1; else hi = mid;
        }
        return lo;
      };
      for (int i = ctid; i < kNC * k; i += kNC * 32) {
        const int w = i / k, pos = i % k;
        const uint64_t x = scratch[i];
        if (x == 0) continue;
        int rank = pos;
        for (int w2 = 0; w2 < kNC && rank < k; ++w2)
          if (w2 != w) rank += count_gt(scratch + (size_t)w2 * k, x);
        if (rank < k) emit(rank, x);
      }
      for (int pos = ctid; pos < k; pos += kNC * 32) {
        int npos = 0;
        for (int w = 0; w < kNC && npos <= pos; ++w) npos += count_gt(scratch + (size_t)w * k, 0);
        if (pos >= npos) emit(pos, 0);
      }
      consumers_sync();
      if (!last_pass && !p.split && ctid == 0) {
        __threadfence();
        atomicExch(&p.pass_done[batch], (uint32_t)(pass + 1));
      }
      for (int i = ctid; i < kNC * k; i += kNC * 32) scratch[i] = 0;
      consumers_sync();
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

}  // namespace shortk

// host launch (accumulate_short.cu)
template <int KS>
cudaError_t launch_short(const QP& p, int sms, cudaStream_t st);

}  // namespace kj
