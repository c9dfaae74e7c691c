// Shared declarations of the sampler (sampler.cu) and the tcgen05 U-Net (conv_tc.cu).
#pragma once
#include <cuda_bf16.h>

#include <cuda.h>

#include <functional>
#include <vector>

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
    int xb_ready = 0;   // the bf16 state view already holds x (written by the previous step's FINAL epilogue)
};

// One conv layer of the tcgen05 U-Net.  src[0..2]: activation views (bf16 [B][Tv][ld]); the
// main conv's segments read src[seg.src], the residual 1x1 reads src[seg.src + res_shift].
struct TcLayer {
    const PConv* c;
    const PConv* res;
    int epi;
    const __nv_bfloat16* src[3];
    int ld[3];
    int res_shift;
    int Tv;
    __nv_bfloat16* out;
    const __nv_bfloat16* res_src;
    int xb_src = -1;   // source index that is the 8-channel bf16 state view
};

// activation slots of the tcgen05 workspace (tc_workspace_bytes)
struct UnetSlots {
    __nv_bfloat16 *a0, *cur, *nxt, *h, *skip1, *skip2;
    float* film;
};
UnetSlots unet_slots(void* ws, int B, int T);
void unet_layer_list(const Layout& L, int T, const UnetSlots& u, bool split_res256, std::vector<TcLayer>& out);
int tc_xb(const float* x, size_t rows, __nv_bfloat16* xb, cudaStream_t st);

// tensor maps (conv_tc.cu)
bool get_encoder();
bool make_ts_map(CUtensorMap* tm, const void* base, int B, int Tv, int C, int nb);
bool make_xb_map(CUtensorMap* tm, const void* base, int B, int Tv, int nb);
bool make_w_map(CUtensorMap* tm, const void* base, int N, int Kp, int box_rows = 0);

// persistent small-batch sampler (unet_small.cu); unet_persist_launch returns US_NOT_RESIDENT
// (nothing launched) when its cooperative grid cannot be resident, e.g. while other work holds
// SMs: callers then run the layered kernels instead
constexpr int US_NOT_RESIDENT = 100;
bool unet_persist_eligible(int B, int T);
int unet_persist_prepare(const Layout& L, const char* packed, void* ws, int B, int T, const StepCoef* sc_h,
                         int n_steps);
int unet_persist_mark_used(void* ws, cudaStream_t st);
int unet_persist_launch(const Layout& L, const char* packed, void* ws, float* x, int B, int T, int S, int p0,
                        unsigned key, const float* film_a, const float* film_b, int n_steps, const float* q_start,
                        float* traj, float lo, float hi, float* eps_out, cudaStream_t st);

size_t tc_workspace_bytes(int B, int T);
int unet_eval_tc(const Layout& L, const char* packed, float* x, int B, int T, int S, const float* film_a,
                 const float* film_b_row, float* ws, float* eps, const TcStep* step, cudaStream_t st);

}  // namespace ps
