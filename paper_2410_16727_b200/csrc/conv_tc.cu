// bf16 tcgen05 U-Net (mode 1) -- placeholder until the tcgen05 kernels land.
#include "common.cuh"
#include "sampler.cuh"

namespace ps {
size_t tc_workspace_bytes(int B, int T) { return (size_t)B * T * 64; }
int unet_eval_tc(const Layout&, const char*, float*, int, int, int, const float*, const float*, float*, float*,
                 const TcStep*, cudaStream_t) {
    return PS_ERR_SHAPE;
}
}  // namespace ps
