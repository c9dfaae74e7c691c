// Shared declarations of the sampler (sampler.cu) and the tcgen05 U-Net (conv_tc.cu).
#pragma once
#include <cuda_bf16.h>

#include <functional>

#include "unet_arch.h"

namespace ps {

struct PackMap;

struct Layout {
    int mode = 0;             // 0: fp32 SIMT, 1: bf16 tcgen05
    size_t n_params = 0;
    size_t w_elems = 0;       // packed weight elements (float or bf16)
    size_t w_bytes = 0;       // aligned weight region size
    size_t side_elems = 0;    // fp32 side table (biases, GN, FiLM, time MLP, out 1x1)
    PBlock blk[U_NBLK];
    PConv down[2], up[2], fin, out;
    size_t outw_f32 = 0;
    size_t t1w = 0, t1b = 0, t2w = 0, t2b = 0;
    size_t film_wt = 0, film_wc = 0, film_b = 0;
    size_t total_bytes = 0;

    const float* side(const char* packed) const { return reinterpret_cast<const float*>(packed + w_bytes); }
};

Layout make_layout(int mode, PackMap* M);

struct StepCoef {
    int k;            // 1-based step index
    int last;         // final step: emit trajectories
    int ddpm;         // 1: posterior + noise, 0: deterministic DDIM
    float sq1m, rsq;  // x0 reconstruction
    float c0, c1, sig;
    float sqn, sq1mn;  // DDIM: next index coefficients
};

struct TcStep {
    StepCoef sc;
    int p0;
    unsigned key;
    const float* q_start;
    float* traj;
    float lo, hi;
};

size_t tc_workspace_bytes(int B, int T);
int unet_eval_tc(const Layout& L, const char* packed, float* x, int B, int T, int S, const float* film_a,
                 const float* film_b_row, float* ws, float* eps, const TcStep* step, cudaStream_t st);

}  // namespace ps
