// Microbenchmarks for the peaks MEASURED_PEAKS.json lacks (SURVEY.md §8(d) "Peaks MP lacks"):
// shared-memory atomics / RMW / scan throughput and L2-resident + HBM streaming read bandwidth.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int T = 8192;
constexpr int B = 6;
// mode 0: atomicAdd conflict-free; 1: ld/add/st RMW conflict-free; 2: atomicAdd random (within a row)
// 3: red (atomicAdd result unused) conflict-free via inline PTX red.shared
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_smem(int iters, unsigned seed, int* out) {
  extern __shared__ int acc[];
  for (int i = threadIdx.x; i < B * T; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 97u);
  int row = warp % B;
  int* base = acc + row * T;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int id;
      if (MODE == 2) { x = x * 1664525u + 1013904223u; id = (x >> 8) & (T - 1); }
      else id = ((it * 8 + j) * 32 + lane + warp * 256) & (T - 1);
      if (MODE == 0) atomicAdd(base + id, j + 1);
      else if (MODE == 1) { if (warp < B) base[id] += j + 1; else { base = acc + (warp % B) * T; base[id ^ 4096] += j + 1; } }
      else if (MODE == 2) atomicAdd(base + id, j + 1);
      else { asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(base + id)), "r"(j + 1)); }
    }
  }
  __syncthreads();
  int s = 0;
  for (int i = threadIdx.x; i < B * T; i += blockDim.x) s += acc[i];
  if (s == 0x7fffffff) out[0] = s;
}

// scan: LDS.128 + compare + STS.128 zero
__global__ void __launch_bounds__(512, 1) k_scan(int iters, int* out) {
  extern __shared__ int4 acc4[];
  int n4 = B * T / 4;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) acc4[i] = make_int4(i, 1, 2, 3);
  __syncthreads();
  int cnt = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
      int4 v = acc4[i];
      cnt += (v.x > 1000000) + (v.y > 1000000) + (v.z > 1000000) + (v.w > 1000000);
      acc4[i] = make_int4(it, 0, 0, 0);
    }
  }
  if (cnt == 12345) out[0] = cnt;
}

__global__ void k_read(const int4* __restrict__ p, size_t n4, int reps, int* out) {
  int4 acc = make_int4(0, 0, 0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      int4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) out[0] = 1;
}

int main() {
  int dev = 0, sms = 0, l2 = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"clock_khz_attr\": %d}\n", sms, l2, clk);
  int* out; CK(cudaMalloc(&out, 4));
  size_t smem = (size_t)B * T * 4;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run_smem = [&](auto kern, const char* name, int iters, double ops_per_iter_thread) -> int {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int w = 0; w < 2; ++w) kern<<<sms, 512, smem>>>(iters, 1u, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kern<<<sms, 512, smem>>>(iters, 1u, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 512 * iters * ops_per_iter_thread;
    printf("{\"bench\": \"%s\", \"ms\": %.4f, \"lane_ops_per_s\": %.4e, \"per_sm_per_ns\": %.3f}\n", name, ms, ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / 1e9);
    return 0;
  };
  run_smem(k_smem<0>, "smem_atomicAdd_conflict_free", 4000, 8);
  run_smem(k_smem<1>, "smem_rmw_conflict_free", 4000, 8);
  run_smem(k_smem<2>, "smem_atomicAdd_random", 4000, 8);
  run_smem(k_smem<3>, "smem_red_conflict_free", 4000, 8);
  {
    CK(cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int iters = 2000;
    for (int w = 0; w < 2; ++w) k_scan<<<sms, 512, smem>>>(iters, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_scan<<<sms, 512, smem>>>(iters, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)sms * B * T * iters;
    printf("{\"bench\": \"smem_scan_zero\", \"ms\": %.4f, \"pairs_per_s\": %.4e, \"per_sm_per_ns\": %.3f}\n", ms, pairs / (ms * 1e-3), pairs / (ms * 1e-3) / sms / 1e9);
  }
  for (size_t bytes : {(size_t)8 << 20, (size_t)64 << 20, (size_t)4 << 30}) {
    int4* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 1, bytes));
    int reps = bytes < ((size_t)1 << 30) ? 200 : 5;
    for (int threads : {256, 512, 1024}) {
      int grid = sms * (2048 / threads);
      k_read<<<grid, threads>>>(p, bytes / 16, 1, out);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); k_read<<<grid, threads>>>(p, bytes / 16, reps, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"bench\": \"read_%zuMB_t%d\", \"ms\": %.4f, \"GBps\": %.1f}\n", bytes >> 20, threads, ms, (double)bytes * reps / (ms * 1e-3) / 1e9);
    }
    cudaFree(p);
  }
  return 0;
}
