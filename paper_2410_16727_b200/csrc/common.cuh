// Shared device helpers for the sm_100a kernels of the seeding hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ps_b200.h"

#define PS_FULL 0xffffffffu

#include <cstdio>
#include <cstdlib>

// Error returns log file:line when PS_DEBUG is set in the environment.
inline int ps_fail(int code, const char* file, int line) {
    static const bool dbg = std::getenv("PS_DEBUG") != nullptr;
    if (dbg) std::fprintf(stderr, "[ps_b200] status %d at %s:%d\n", code, file, line);
    return code;
}
#define PS_FAIL(code) ps_fail((code), __FILE__, __LINE__)

#include <atomic>
// Every kernel launch site goes through PS_CHECK_LAUNCH, which counts it
// (ps_launch_count() in the C-ABI; bench.py reports launches per step).
inline std::atomic<long long>& ps_launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}

#define PS_CHECK_LAUNCH()                                                   \
    do {                                                                    \
        ps_launch_counter().fetch_add(1, std::memory_order_relaxed);        \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) {                                            \
            if (std::getenv("PS_DEBUG"))                                    \
                std::fprintf(stderr, "[ps_b200] %s\n", cudaGetErrorString(e_)); \
            return PS_FAIL(PS_ERR_CUDA);                                    \
        }                                                                   \
    } while (0)

namespace ps {

// ---------------------------------------------------------------------------
// Canonical fp32 math.  Files that include
// these are compiled with --fmad=false: every fused multiply-add is an explicit
// fmaf(), so results are bit-identical to oracle/c/bl_oracle.c.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void c_sincos(float x, float& s, float& c) {
    float j = rintf(x * 0.636619772367581343f);
    int q = (int)j;
    float r = fmaf(-j, 1.5703125f, x);
    r = fmaf(-j, 4.83751296997e-04f, r);
    r = fmaf(-j, 7.54978995489e-08f, r);
    float r2 = r * r;
    float sp = fmaf(fmaf(fmaf(-1.9515295891e-4f, r2, 8.3321608736e-3f), r2, -1.6666654611e-1f) * r2, r, r);
    float cp = fmaf(fmaf(fmaf(fmaf(2.443315711809948e-5f, r2, -1.388731625493765e-3f), r2,
                              4.166664568298827e-2f), r2, -0.5f), r2, 1.0f);
    switch (q & 3) {
        case 0: s = sp; c = cp; break;
        case 1: s = cp; c = -sp; break;
        case 2: s = -sp; c = -cp; break;
        default: s = -cp; c = sp; break;
    }
}

struct f3 {
    float x, y, z;
};

__device__ __forceinline__ f3 c_cross(const f3& a, const f3& b) {
    return f3{fmaf(a.y, b.z, -(a.z * b.y)), fmaf(a.z, b.x, -(a.x * b.z)), fmaf(a.x, b.y, -(a.y * b.x))};
}

struct Grid {
    const float* __restrict__ v;
    int nx, ny, nz;
    float ox, oy, oz, inv_h;
};

// Trilinear value + in-cell analytic gradient + clamp flag; generalises
// planseed/_kernels.py:_bilinear (:23-57) to 3-D.  Manual fp32 weights, never
// texture filtering (8-bit fractional weights would break parity).
__device__ __forceinline__ float c_trilinear(const Grid& g, const f3& p, f3& grad, bool& clamped) {
    float ux = (p.x - g.ox) * g.inv_h;
    float uy = (p.y - g.oy) * g.inv_h;
    float uz = (p.z - g.oz) * g.inv_h;
    clamped = (ux < 0.f) | (ux > (float)(g.nx - 1)) | (uy < 0.f) | (uy > (float)(g.ny - 1)) |
              (uz < 0.f) | (uz > (float)(g.nz - 1));
    float fi = fminf(fmaxf(floorf(ux), 0.f), (float)(g.nx - 2));
    float fj = fminf(fmaxf(floorf(uy), 0.f), (float)(g.ny - 2));
    float fk = fminf(fmaxf(floorf(uz), 0.f), (float)(g.nz - 2));
    float tx = fminf(fmaxf(ux - fi, 0.f), 1.f);
    float ty = fminf(fmaxf(uy - fj, 0.f), 1.f);
    float tz = fminf(fmaxf(uz - fk, 0.f), 1.f);
    const size_t sy = (size_t)g.nz, sx = (size_t)g.ny * (size_t)g.nz;
    const float* v = g.v + ((size_t)(int)fi * sx + (size_t)(int)fj * sy + (size_t)(int)fk);
    float v000 = __ldg(v), v001 = __ldg(v + 1), v010 = __ldg(v + sy), v011 = __ldg(v + sy + 1);
    float v100 = __ldg(v + sx), v101 = __ldg(v + sx + 1), v110 = __ldg(v + sx + sy),
          v111 = __ldg(v + sx + sy + 1);
    float z00 = v001 - v000, z01 = v011 - v010, z10 = v101 - v100, z11 = v111 - v110;
    float c00 = fmaf(tz, z00, v000), c01 = fmaf(tz, z01, v010);
    float c10 = fmaf(tz, z10, v100), c11 = fmaf(tz, z11, v110);
    float e0 = c01 - c00, e1 = c11 - c10;
    float c0 = fmaf(ty, e0, c00), c1 = fmaf(ty, e1, c10);
    float dxv = c1 - c0;
    float d = fmaf(tx, dxv, c0);
    float dyv = fmaf(tx, e1 - e0, e0);
    float zy0 = fmaf(ty, z01 - z00, z00), zy1 = fmaf(ty, z11 - z10, z10);
    float dzv = fmaf(tx, zy1 - zy0, zy0);
    grad = f3{dxv * g.inv_h, dyv * g.inv_h, dzv * g.inv_h};
    return d;
}

__device__ __forceinline__ float warp_sum_butterfly(float v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(PS_FULL, v, off);
    return v;
}

}  // namespace ps
