// accumulate_ks1.cu -- instances of k_accumulate_topk with KS = 1 top-k slots per lane (k <= 32).
#define KJ_ACCUMULATE_INSTANCES
#include "accumulate.cuh"

namespace kj {
template cudaError_t launch_accumulate<1>(const Shape& sh, const QP& p, int sms, cudaStream_t st);
}  // namespace kj
