// accumulate_ks8.cu -- instances of k_accumulate_topk with KS = 8 top-k slots per lane (k <= 256).
#define KJ_ACCUMULATE_INSTANCES
#include "accumulate.cuh"

namespace kj {
template cudaError_t launch_accumulate<8>(const Shape& sh, const QP& p, int sms, cudaStream_t st);
}  // namespace kj
