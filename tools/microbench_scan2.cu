// Scan-side shared-memory microbenchmarks (round 2, session 3): can the score array's read + zero-fill and the
// per-pair head-bound lookup leave the LSU data pipe less busy than K3's LDS.128 + STS.128 and LDS.32 lookups?
//   scan_ldsts   : LDS.128 then STS.128 of zero (K3's scan today)
//   scan_xchg128 : ATOMS.EXCH.128 with zero (read and zero in one instruction)
//   scan_xchg32  : ATOMS.EXCH.32 x 4
//   lut_lds      : 8 data-dependent LDS.32 lookups into a 33-entry table per lane (the cum[] bound)
//   lut_shfl     : the same 8 lookups as SHFL.IDX from a register-held table (lane i holds entry i)
//   scan+lut_*   : the scan with 8 lookups per 128 columns beside it (does SHFL share the LSU data pipe?)
// Rates are per SM per clock (one CTA of 16 warps per SM, 148 CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbscan tools/microbench_scan2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NCOL = 2 * 8192;  // two score rows of one tile

// LUT: 0 none, 1 eight LDS.32 cum lookups per 128 columns (K3's B = 2 scan), 2 the same as SHFL.IDX
template <int MODE, int LUT = 0>
__global__ void __launch_bounds__(512, 1) k_scan(int iters, unsigned long long* cyc, int* out) {
  extern __shared__ __align__(16) uint32_t acc[];
  __shared__ uint32_t cum[33];
  for (int i = threadIdx.x; i < NCOL; i += blockDim.x) acc[i] = i & 7;
  if (threadIdx.x < 33) cum[threadIdx.x] = threadIdx.x * 1000u;
  __syncthreads();
  const uint32_t creg = (threadIdx.x & 31) * 1000u;
  uint32_t h = 0x9E3779B9u * (threadIdx.x + 1);
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(acc);
  uint32_t cnt = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = threadIdx.x * 4; c < NCOL; c += blockDim.x * 4) {
      const uint32_t a = base + c * 4;
      uint32_t x0, x1, x2, x3;
      if (MODE == 0) {
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(a) : "memory");
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0u) : "memory");
      } else if (MODE == 1) {
        asm volatile("{ .reg .b128 d, z; mov.b128 z, {%4,%4,%4,%4}; atom.shared.exch.b128 d, [%5], z; mov.b128 {%0,%1,%2,%3}, d; }"
                     : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(0u), "r"(a) : "memory");
      } else {
        asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(x0) : "r"(a), "r"(0u) : "memory");
        asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(x1) : "r"(a + 4), "r"(0u) : "memory");
        asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(x2) : "r"(a + 8), "r"(0u) : "memory");
        asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(x3) : "r"(a + 12), "r"(0u) : "memory");
      }
      cnt += max(max(x0, x1), max(x2, x3));
      if (LUT) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t nh = __popc((h >> j) & 0x0F0F0F0Fu);
          cnt += LUT == 1 ? cum[nh] : __shfl_sync(0xffffffffu, creg, nh);
        }
        h = h * 1664525u + cnt;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  if (cnt == 0x7fffffffu) out[0] = cnt;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_lut(int iters, unsigned long long* cyc, int* out) {
  __shared__ uint32_t cum[33];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 33) cum[threadIdx.x] = threadIdx.x * 1000u;
  __syncthreads();
  const uint32_t creg = lane * 1000u;
  uint32_t h = 0x9E3779B9u * (threadIdx.x + 1), acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      h = h * 1664525u + 1013904223u;
      const uint32_t nh = __popc(h & 0x0F0F0F0Fu);  // 0..16
      acc += MODE == 0 ? cum[nh] : __shfl_sync(0xffffffffu, creg, nh);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  if (acc == 0x7fffffffu) out[0] = acc;
}

int main() {
  unsigned long long* cyc;
  int* out;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&out, 4));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms, threads = 512;  // one CTA per SM
  const size_t smem = NCOL * 4;
  auto run_scan = [&](auto kern, const char* name, int iters) -> int {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, threads, smem>>>(2, cyc, out);
    CK(cudaMemset(cyc, 0, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, threads, smem>>>(iters, cyc, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    const double cyc_per_cta = (double)c / grid;
    const double bytes_per_cta = (double)iters * NCOL * 4;
    // one CTA per SM at a time (launch_bounds 512 x 1; 64 KB smem): per-SM bytes per clock = bytes / cycles
    printf("%-14s %8.3f ms  %6.1f B/clk/SM (read+zero of score bytes)  %.3f clk per 128 cols per warp\n", name, ms,
           bytes_per_cta / cyc_per_cta, cyc_per_cta / ((double)iters * NCOL / 128 / 16));
    return 0;
  };
  auto run_lut = [&](auto kern, const char* name, int iters) -> int {
    kern<<<grid, threads>>>(2, cyc, out);
    CK(cudaMemset(cyc, 0, 8));
    kern<<<grid, threads>>>(iters, cyc, out);
    CK(cudaDeviceSynchronize());
    unsigned long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    const double cyc_per_cta = (double)c / grid;
    const double lookups = (double)iters * 8 * 16;  // warp lookups per CTA
    printf("%-14s %6.3f warp lookups / clk / SM\n", name, lookups / cyc_per_cta);
    return 0;
  };
  if (run_scan(k_scan<0>, "scan_ldsts", 2000)) return 1;
  if (run_scan(k_scan<1>, "scan_xchg128", 2000)) return 1;
  if (run_scan(k_scan<2>, "scan_xchg32", 2000)) return 1;
  if (run_scan(k_scan<0, 1>, "scan+lut_lds", 2000)) return 1;
  if (run_scan(k_scan<0, 2>, "scan+lut_shfl", 2000)) return 1;
  if (run_scan(k_scan<1, 1>, "xchg128+lds", 2000)) return 1;
  if (run_lut(k_lut<0>, "lut_lds", 20000)) return 1;
  if (run_lut(k_lut<1>, "lut_shfl", 20000)) return 1;
  return 0;
}
