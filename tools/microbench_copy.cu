// Microbenchmark: moving many SMALL L2-resident slices (the posting slices of the short-slice configs, C3 / C5:
// 64-256 B each) into shared memory.  Compares, at the same bytes per round:
//   bulk   -- cp.async.bulk (UBLKCP) global -> shared, one copy per slice issued by every thread, mbarrier
//             complete_tx, two rounds in flight (double-buffered)
//   ldgsts -- cp.async.cg 16-byte copies (LDGSTS), S/16 per slice per thread, commit groups, two rounds in flight
//   ldg    -- plain 128-bit loads into registers (what k_accumulate_topk does today)
// Sources are random 16-byte-aligned slices of a 32 MB buffer (L2-resident).  Prints slices/s and GB/s chip-wide.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbcopy tools/microbench_copy.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NT = 128;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_addr(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

template <int MODE, int S>
__global__ void __launch_bounds__(NT) k_copy(const uint8_t* __restrict__ src, size_t span, int rounds, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[2];
  const int tid = threadIdx.x;
  uint32_t x = 0x9E3779B9u * (blockIdx.x * NT + tid + 1);
  uint32_t acc = 0;
  if (MODE == 0) {
    if (tid == 0) { mbar_init(&bars[0], NT); mbar_init(&bars[1], NT); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
  }
  for (int r = 0; r < rounds; ++r) {
    const int buf = r & 1;
    uint8_t* dst = sm + (size_t)buf * NT * S + (size_t)tid * S;
    x = x * 1664525u + 1013904223u;
    const size_t off = ((size_t)x * 16) % (span - S);
    const uint8_t* s = src + (off & ~(size_t)15);
    if (MODE == 0) {
      mbar_arrive_tx(&bars[buf], S);
      bulk_g2s(dst, s, S, &bars[buf]);
      if (r > 0) {
        mbar_wait(&bars[buf ^ 1], ((r - 1) >> 1) & 1);
        acc += sm[(size_t)(buf ^ 1) * NT * S + (size_t)tid * S];
      }
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < S / 16; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + 16 * i)), "l"(s + 16 * i) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (r > 0) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        acc += sm[(size_t)(buf ^ 1) * NT * S + (size_t)tid * S];
      }
    } else {
#pragma unroll
      for (int i = 0; i < S / 16; ++i) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + 16 * i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    __syncwarp();
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE, int S>
int run(const uint8_t* src, size_t span, int sms, uint32_t* out, const char* name, int ctas_per_sm) {
  const size_t smem = 2 * (size_t)NT * S;
  CK(cudaFuncSetAttribute(k_copy<MODE, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = sms * ctas_per_sm, rounds = 2000;
  k_copy<MODE, S><<<grid, NT, smem>>>(src, span, 10, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_copy<MODE, S><<<grid, NT, smem>>>(src, span, rounds, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double slices = (double)grid * NT * rounds;
  printf("{\"bench\": \"%s\", \"slice_bytes\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"slices_per_s\": %.4e, "
         "\"GBps\": %.1f, \"slices_per_sm_per_clk_at_1.965GHz\": %.3f}\n",
         name, S, ctas_per_sm, ms, slices / (ms * 1e-3), slices * S / (ms * 1e-3) / 1e9,
         slices / (ms * 1e-3) / sms / 1.965e9);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t span = (size_t)32 << 20;
  uint8_t* src;
  CK(cudaMalloc(&src, span));
  CK(cudaMemset(src, 3, span));
  uint32_t* out;
  CK(cudaMalloc(&out, 4));
  for (int c : {2, 6}) {
    run<0, 64>(src, span, sms, out, "bulk", c);
    run<0, 128>(src, span, sms, out, "bulk", c);
    run<0, 256>(src, span, sms, out, "bulk", c);
    run<1, 64>(src, span, sms, out, "ldgsts", c);
    run<1, 128>(src, span, sms, out, "ldgsts", c);
    run<1, 256>(src, span, sms, out, "ldgsts", c);
    run<2, 64>(src, span, sms, out, "ldg", c);
    run<2, 128>(src, span, sms, out, "ldg", c);
    run<2, 256>(src, span, sms, out, "ldg", c);
  }
  return 0;
}
