// accumulate_short.cu -- instances and launcher of the warp-specialised bulk-copy K3 (short.cuh) for indexes without
// head features, one R row per item.
#include "short.cuh"

namespace kj {

template <int KS>
cudaError_t launch_short(const QP& p, int sms, cudaStream_t st) {
  auto go = [&](auto kern, bool i8) -> cudaError_t {
    const size_t sm = shortk::smem_total(p.T, p.k, i8);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, shortk::kThreads, sm)) != cudaSuccess)
      return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > p.n_batches * p.n_passes) grid = p.n_batches * p.n_passes;
    kern<<<(unsigned)grid, shortk::kThreads, sm, st>>>(p);
    return cudaGetLastError();
  };
  return p.vals ? go(shortk::k_accumulate_short<KS, true>, true) : go(shortk::k_accumulate_short<KS, false>, false);
}

template cudaError_t launch_short<1>(const QP& p, int sms, cudaStream_t st);
template cudaError_t launch_short<4>(const QP& p, int sms, cudaStream_t st);
template cudaError_t launch_short<8>(const QP& p, int sms, cudaStream_t st);

}  // namespace kj
