// Microbenchmark: does a bulk (TMA) copy INTO shared memory take shared-memory bandwidth from LDS / STS?
// Kernel: every warp streams LDS.128 (conflict-free) over buffer X; optionally warp 0 lane 0 keeps refilling buffer
// Y (32 KB, the one-row score array) from a zeroed global buffer with cp.async.bulk (mbarrier-completed).  Reports
// the LDS rate (bytes/clk/SM) with and without the concurrent bulk copies, and the bulk bytes/clk/SM.  If the LDS
// rate does not drop, zero-filling the score array by bulk copy would free the STS half of the scan.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbtma tools/microbench_tma_zero.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kY = 32768;  // bytes per bulk copy
constexpr int kX = 16384;  // LDS buffer

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool TMA, bool STS>
__global__ void __launch_bounds__(256) k_bench(const uint8_t* __restrict__ zeros, int iters, unsigned long long* out,
                                               unsigned long long* copies) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  uint8_t* X = sm;
  uint8_t* Y = sm + kX;
  const int tid = threadIdx.x;
  for (int i = tid; i < kX / 16; i += 256) ((uint4*)X)[i] = make_uint4(i, i, i, i);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t acc = 0;
  unsigned long long ncopy = 0;
  uint32_t phase = 0;
  bool inflight = false;
  const uint32_t base = sa(X) + (tid & 31) * 16 + (tid >> 5) * 512;
  for (int it = 0; it < iters; ++it) {
    if (TMA && tid == 0) {
      bool done = !inflight;
      if (inflight) {
        uint32_t ok;
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(&bar)), "r"(phase) : "memory");
        if (ok) { done = true; phase ^= 1; ++ncopy; }
      }
      if (done) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(kY) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(Y)), "l"(zeros), "r"(kY), "r"(sa(&bar)) : "memory");
        inflight = true;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t a = base + ((j * 4096) & (kX - 1));
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
      if (STS) asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(acc & 0));
    }
  }
  if (TMA && tid == 0 && inflight) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&bar)), "r"(phase) : "memory");
    ++ncopy;
  }
  if (acc == 0x12345u) out[0] = acc;
  if (tid == 0) atomicAdd(copies, ncopy);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  uint8_t* zeros;
  unsigned long long *out, *copies;
  CK(cudaMalloc(&zeros, kY));
  CK(cudaMemset(zeros, 0, kY));
  CK(cudaMalloc(&out, 8));
  CK(cudaMalloc(&copies, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = kX + kY;
  const int iters = 20000;
  for (int ctas : {1, 2, 4}) {
    for (int mode = 0; mode < 4; ++mode) {
      const bool tma = mode & 1, sts = mode & 2;
      auto kern = tma ? (sts ? k_bench<true, true> : k_bench<true, false>) : (sts ? k_bench<false, true> : k_bench<false, false>);
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaMemset(copies, 0, 8));
      kern<<<sms * ctas, 256, smem>>>(zeros, iters, out, copies);
      CK(cudaDeviceSynchronize());
      CK(cudaMemset(copies, 0, 8));
      cudaEventRecord(e0);
      kern<<<sms * ctas, 256, smem>>>(zeros, iters, out, copies);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long nc = 0;
      CK(cudaMemcpy(&nc, copies, 8, cudaMemcpyDeviceToHost));
      const double clks = ms * 1e-3 * clk * 1e3;
      const double lds_bytes = (double)sms * ctas * 256 * iters * 8 * 16 * (sts ? 2 : 1);
      printf("{\"ctas_per_sm\": %d, \"tma\": %d, \"sts\": %d, \"ms\": %.3f, \"lds_sts_B_per_clk_per_sm\": %.1f, "
             "\"bulk_B_per_clk_per_sm\": %.1f}\n",
             ctas, (int)tma, (int)sts, ms, lds_bytes / sms / clks, (double)nc * kY / sms / clks);
    }
  }
  return 0;
}
