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
    int brick;   // 0: C order (z fastest); 1: 4x4x4 bricks (see esdf_brick_index); 2: quad bricks
};

// 4x4x4-brick layout of an (nx, ny, nz) grid with all extents multiples of 4: brick
// (i/4, j/4, k/4) in C order, 64 contiguous floats per brick, node (i&3, j&3, k&3) at
// 16 (i&3) + 4 (j&3) + (k&3).  A trilinear cell's 8 corners then share one or two 128-B
// lines most of the time (C order: four lines 256 B / 64 KB apart), so a problem's ESDF
// working set takes a fraction of the L2 lines.
__host__ __device__ __forceinline__ size_t esdf_brick_index(int i, int j, int k, int ny, int nz) {
    return (((size_t)(i >> 2) * (size_t)(ny >> 2) + (size_t)(j >> 2)) * (size_t)(nz >> 2) + (size_t)(k >> 2)) * 64 +
           (size_t)((i & 3) * 16 + (j & 3) * 4 + (k & 3));
}

// Quad-brick layout (layout 2): node (i, j, k) holds the float4 (v(i,j,k), v(i,j,k+1), v(i,j+1,k),
// v(i,j+1,k+1)) (neighbours clamped at the upper faces, never read as cell corners), entries in the
// 4^3-brick order of esdf_brick_index.  A trilinear cell's 8 corners are the entries of (i, j, k)
// and (i+1, j, k): two 16-B loads instead of eight scalar gathers (L1TEX wavefronts / 4), at 4x
// the storage -- the layout for an ESDF shared by a large batch (BASELINE config 2: 33.6 MB,
// L2-resident).

// Trilinear value + in-cell analytic gradient + clamp flag; generalises
// planseed/_kernels.py:_bilinear (:23-57) to 3-D.  Manual fp32 weights, never
// texture filtering (8-bit fractional weights would break parity).
// Split in two stages so a caller can have several lookups' gathers in flight: tri_gather
// (cell, fractions, the 8 corner loads) and tri_eval (the interpolation arithmetic).
struct TriCell {
    float v000, v001, v010, v011, v100, v101, v110, v111;
    float tx, ty, tz;
    bool clamped;
};

__device__ __forceinline__ void tri_gather(const Grid& g, const f3& p, TriCell& c) {
    float ux = (p.x - g.ox) * g.inv_h;
    float uy = (p.y - g.oy) * g.inv_h;
    float uz = (p.z - g.oz) * g.inv_h;
    c.clamped = (ux < 0.f) | (ux > (float)(g.nx - 1)) | (uy < 0.f) | (uy > (float)(g.ny - 1)) |
                (uz < 0.f) | (uz > (float)(g.nz - 1));
    float fi = fminf(fmaxf(floorf(ux), 0.f), (float)(g.nx - 2));
    float fj = fminf(fmaxf(floorf(uy), 0.f), (float)(g.ny - 2));
    float fk = fminf(fmaxf(floorf(uz), 0.f), (float)(g.nz - 2));
    c.tx = fminf(fmaxf(ux - fi, 0.f), 1.f);
    c.ty = fminf(fmaxf(uy - fj, 0.f), 1.f);
    c.tz = fminf(fmaxf(uz - fk, 0.f), 1.f);
    const float* v;
    size_t sx, sy, sz;
    if (g.brick == 2) {   // quad bricks: two 16-B loads hold the cell's 8 corners
        const int ii = (int)fi, jj = (int)fj, kk = (int)fk;
        const float4* q4 = reinterpret_cast<const float4*>(g.v) + esdf_brick_index(ii, jj, kk, g.ny, g.nz);
        const size_t s4 = (ii & 3) == 3 ? (size_t)(g.ny >> 2) * (size_t)(g.nz >> 2) * 64 - 48 : 16;
        const float4 a = __ldg(q4), b = __ldg(q4 + s4);
        c.v000 = a.x; c.v001 = a.y; c.v010 = a.z; c.v011 = a.w;
        c.v100 = b.x; c.v101 = b.y; c.v110 = b.z; c.v111 = b.w;
        return;
    }
    if (g.brick) {   // neighbour steps stay inside a brick unless the cell sits on its edge
        const int ii = (int)fi, jj = (int)fj, kk = (int)fk;
        v = g.v + esdf_brick_index(ii, jj, kk, g.ny, g.nz);
        sz = (kk & 3) == 3 ? 61 : 1;
        sy = (jj & 3) == 3 ? (size_t)(g.nz >> 2) * 64 - 12 : 4;
        sx = (ii & 3) == 3 ? (size_t)(g.ny >> 2) * (size_t)(g.nz >> 2) * 64 - 48 : 16;
    } else {
        sz = 1;
        sy = (size_t)g.nz;
        sx = (size_t)g.ny * (size_t)g.nz;
        v = g.v + ((size_t)(int)fi * sx + (size_t)(int)fj * sy + (size_t)(int)fk);
    }
    c.v000 = __ldg(v); c.v001 = __ldg(v + sz); c.v010 = __ldg(v + sy); c.v011 = __ldg(v + sy + sz);
    c.v100 = __ldg(v + sx); c.v101 = __ldg(v + sx + sz); c.v110 = __ldg(v + sx + sy); c.v111 = __ldg(v + sx + sy + sz);
}

__device__ __forceinline__ float tri_eval(const Grid& g, const TriCell& c, f3& grad) {
    const float tx = c.tx, ty = c.ty, tz = c.tz;
    float z00 = c.v001 - c.v000, z01 = c.v011 - c.v010, z10 = c.v101 - c.v100, z11 = c.v111 - c.v110;
    float c00 = fmaf(tz, z00, c.v000), c01 = fmaf(tz, z01, c.v010);
    float c10 = fmaf(tz, z10, c.v100), c11 = fmaf(tz, z11, c.v110);
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

__device__ __forceinline__ float c_trilinear(const Grid& g, const f3& p, f3& grad, bool& clamped) {
    TriCell c;
    tri_gather(g, p, c);
    clamped = c.clamped;
    return tri_eval(g, c, grad);
}

__device__ __forceinline__ float warp_sum_butterfly(float v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(PS_FULL, v, off);
    return v;
}

}  // namespace ps
