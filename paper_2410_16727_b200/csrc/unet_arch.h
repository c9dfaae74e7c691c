// Host-side description of the BASELINE 1-D temporal U-Net (spec.py: UNetArch) and of
// the packed per-layer device layout.  Every convolution is expressed as a stride-1
// implicit GEMM over a *view* of its input:
//
//   out[b, t, n] = bias[n] + sum_seg sum_{c<nc} in_seg[b, t + dt, c0 + c] * W[k_seg + c, n]
//
// with zero padding outside [0, Tv).  Stride-2 downsampling reads the input as
// [B, T/2, 2C] (time pairs), transposed-conv upsampling writes [B, T, 2C] pairs; see
// DESIGN.md "Convolutions as segment GEMMs".
#pragma once
#include <cstddef>
#include <string>
#include <vector>

namespace ps {

constexpr int U_DOF = 7;
constexpr int U_COND = 270;
constexpr int U_TEMB = 128;
constexpr int U_THID = 512;
constexpr int U_FILM_IN = U_TEMB + U_COND;
constexpr int U_GROUPS = 8;
constexpr int U_NBLK = 12;
constexpr int U_FILM_COLS = 2 * (64 * 4 + 128 * 4 + 256 * 4);  // 3584
constexpr int U_MAXSEG = 12;

struct PSeg {
    int src;   // 0 = primary input, 1 = secondary (skip) input
    int dt;    // time offset
    int c0;    // first channel in the source view
    int nc;    // channels
    int k0;    // first packed K row
};

enum Epi { EPI_PLAIN = 0, EPI_GN_FILM = 1, EPI_GN_RES = 2, EPI_FINAL = 3, EPI_RELU2D = 4 };

struct PConv {
    int K = 0, N = 0;
    int n_seg = 0;
    PSeg seg[U_MAXSEG];
    size_t w_off = 0;      // packed weight offset (elements of the weight dtype)
    size_t b_off = 0;      // fp32 offsets into the fp32 side table
    long long g_off = -1, be_off = -1;
    int film_col = -1;     // FiLM scale column in the 3584-wide table (shift = +N)
};

struct PBlock {
    std::string name;
    int c_in, c_out, level;
    PConv c0, c1, res;     // res.K == 0 => identity residual
};

struct ParamEntry {
    std::string name;
    std::vector<int> shape;
    size_t off;            // element offset in the PSCK-order fp32 blob
    size_t numel() const {
        size_t n = 1;
        for (int s : shape) n *= (size_t)s;
        return n;
    }
};

// Table identical (names, shapes, order) to spec.UNetArch().param_shapes().
std::vector<ParamEntry> unet_param_table();
const ParamEntry* find_param(const std::vector<ParamEntry>& t, const std::string& name);

}  // namespace ps
