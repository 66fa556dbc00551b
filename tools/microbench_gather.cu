// Microbenchmark: the posting-window gather of the accumulate kernel in isolation.  A warp reads "windows" of 32
// 16-byte units; the window is made of 32/m contiguous segments of m units (m lanes each) at random unit-aligned
// places of a buffer (L2-resident 40 MB, or 2 GB from HBM).  Each warp keeps ILP windows in flight (independent
// 128-bit loads per lane), CTAs of 128 threads, W warps per SM.  Reports bytes/s chip-wide and bytes/clk/SM: the
// ceiling of the one-row path's load stream for a given slice length m and pipeline depth.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbgather tools/microbench_gather.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_v4(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint4 ldg_v8x(const void* p, uint64_t pol) {  // 256-bit load, folded to 128 bits
  uint32_t r[8];
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p), "l"(pol));
  return make_uint4(r[0] ^ r[4], r[1] ^ r[5], r[2] ^ r[6], r[3] ^ r[7]);
}

// VEC = 16 or 32 bytes per lane (units of VEC bytes)
template <int ILP, int VEC>
__global__ void __launch_bounds__(128) k_gather(const uint4* __restrict__ src, uint32_t n_units, int m_log2, int rounds,
                                                uint32_t* out) {
  const int lane = threadIdx.x & 31;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  uint32_t x = 0x9E3779B9u * (blockIdx.x * 4 + (threadIdx.x >> 5) + 1);
  const int seg = lane >> m_log2, inseg = lane & ((1 << m_log2) - 1);
  uint32_t acc = 0;
  for (int r = 0; r < rounds; ++r) {
    uint4 v[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      // segment start: a hash of (warp state, round, i, seg), the same for the m lanes of a segment
      uint32_t h = (x + (uint32_t)(r * ILP + i) * 0x85EBCA6Bu) ^ (uint32_t)seg * 0xC2B2AE35u;
      h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
      const uint32_t u = ((h % (n_units >> m_log2)) << m_log2) + inseg;
      v[i] = VEC == 16 ? ldg_v4(src + u, pol) : ldg_v8x(src + 2 * (size_t)u, pol);
    }
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  const size_t big = (size_t)2 << 30;
  uint4* buf;
  uint32_t* out;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 1, big));
  CK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  // "l2": effective L2 capacity for random 32-byte reads -- throughput against the working-set size
  if (argc > 1) {
    for (size_t mb : {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 192}) {
      const size_t span = mb << 20;
      const uint32_t n_units = (uint32_t)(span / 16);
      const int grid = sms * 5;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_gather<4, 16><<<grid, 128>>>(buf, n_units, 1, 1024, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bps = (double)grid * 128 * 4096 * 16 / (ms * 1e-3);
      printf("{\"l2_span_mb\": %zu, \"GBps\": %.1f, \"B_per_clk_per_sm\": %.2f}\n", mb, bps / 1e9, bps / sms / (clk * 1e3));
    }
    return 0;
  }
  for (int vec : {16, 32})
  for (size_t span : {(size_t)40 << 20, big}) {
    const uint32_t n_units = (uint32_t)(span / vec);
    for (int m_log2 : {0, 1, 2, 3, 5}) {
      for (int ctas : {5, 12}) {
        for (int ilp : {1, 4}) {
          const int grid = sms * ctas;
          const int rounds = 4096 / ilp;
          auto run = [&]() {
            if (vec == 16) {
              if (ilp == 1) k_gather<1, 16><<<grid, 128>>>(buf, n_units, m_log2, rounds, out);
              else k_gather<4, 16><<<grid, 128>>>(buf, n_units, m_log2, rounds, out);
            } else {
              if (ilp == 1) k_gather<1, 32><<<grid, 128>>>(buf, n_units, m_log2, rounds, out);
              else k_gather<4, 32><<<grid, 128>>>(buf, n_units, m_log2, rounds, out);
            }
          };
          run();
          CK(cudaDeviceSynchronize());
          cudaEventRecord(e0);
          run();
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = (double)grid * 128 * 4096 * vec;
          const double bps = bytes / (ms * 1e-3);
          printf("{\"vec\": %d, \"span_mb\": %zu, \"seg_units\": %d, \"warps_per_sm\": %d, \"ilp\": %d, \"ms\": %.3f, \"GBps\": %.1f, "
                 "\"B_per_clk_per_sm\": %.2f}\n",
                 vec, span >> 20, 1 << m_log2, ctas * 4, ilp, ms, bps / 1e9, bps / sms / (clk * 1e3));
        }
      }
    }
  }
  return 0;
}
