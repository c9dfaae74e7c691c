// bf16 tcgen05 U-Net (mode 1): implicit-GEMM temporal convolutions on the 5th-gen
// tensor cores with fused epilogues.
//
// One CTA computes a 128-row tile (rows = (sample, time) pairs, whole samples) for ALL
// output channels N (64..256), so GroupNorm statistics are complete inside the tile.
//   warp 0     TMA producer: per K chunk a [128 x 64] bf16 activation box (3-D map over
//              the [B, Tv, C] view, time offset dt -> out-of-range rows zero-filled by
//              TMA = the conv's zero padding) and an [N x 64] weight box, SW128.
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer (M=128, N, K=16),
//              accumulator(s) in TMEM; optional second accumulator for the residual 1x1.
//   warps 2-5  epilogue: tcgen05.ld -> +bias -> GroupNorm(8) -> Mish -> FiLM / residual
//              -> bf16 store; FINAL fuses the 64->7 projection, the DDPM/DDIM update of
//              the fp32 state and the Philox noise injection.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "sampler.cuh"
#include "tc_ptx.cuh"

namespace ps {

// ---------------------------------------------------------------------------
// kernel arguments
// ---------------------------------------------------------------------------
constexpr int TC_MAX_CHUNKS = 64;

struct TcChunk {
    int16_t c;      // channel offset in the source view
    int16_t kcol;   // K column in the weight matrix
    int8_t src;     // activation source map 0..2
    int8_t dt;      // time offset
    int8_t res;     // 1: residual GEMM
    int8_t first;   // 1: first chunk of its accumulator
    int8_t dx;      // 2-D geometry: x-pair offset
    int8_t par;     // 2-D geometry: row parity
};

struct TcArgs {
    CUtensorMap tmA[3];
    CUtensorMap tmW;
    CUtensorMap tmR;
    TcChunk chunk[TC_MAX_CHUNKS];
    int n_chunks, stages;
    int rows, Tv, S;
    const float* bias;
    const float* gamma;
    const float* beta;
    const float* rbias;
    const __nv_bfloat16* res_src;   // identity residual (same [rows, N] layout)
    const float* film;              // [P][3584] step FiLM, this block's scale at film + col
    int film_col;
    __nv_bfloat16* out;             // [rows, N]
    // FINAL
    const float* wout;              // [7][64]
    const float* bout;
    float* x;                       // fp32 state [rows][7]
    StepCoef sc;
    int p0;
    unsigned key;
    const float* q_start;
    float* traj;
    float lo, hi;
    float* eps_out;                 // optional: write eps (forward-only calls)
    // 2-D geometry (encoder): tile = ry output rows x wx output columns of one image
    int geom;                       // 0: [B][Tv] samples, 1: 2-D image tiles
    int Ho, Wo, Hp, wx, ry, tiles_x, tiles_y;
    int dbg;                        // PS_TC_DBG: 1 = skip epilogue math, 2 = skip MMAs
};

// columns of one accumulator buffer (main [+ residual])
template <int N, bool RES>
__host__ __device__ constexpr int acc_cols() { return RES ? 2 * N : N; }
// double-buffer the accumulators when two fit in the 512 TMEM columns
template <int N, bool RES>
__host__ __device__ constexpr int n_accbuf() { return 2 * acc_cols<N, RES>() <= 512 ? 2 : 1; }
template <int N, bool RES>
__host__ __device__ constexpr int tmem_alloc_cols() {
    return acc_cols<N, RES>() * n_accbuf<N, RES>() <= 32    ? 32
           : acc_cols<N, RES>() * n_accbuf<N, RES>() <= 64  ? 64
           : acc_cols<N, RES>() * n_accbuf<N, RES>() <= 128 ? 128
           : acc_cols<N, RES>() * n_accbuf<N, RES>() <= 256 ? 256
                                                            : 512;
}

constexpr int TC_EPI_WG = 2;                         // epilogue warpgroups
constexpr int TC_FILM_P = 2;                         // FiLM rows (problems) staged per tile
constexpr int TC_THREADS = 64 + 128 * TC_EPI_WG;     // producer warp, MMA warp, epilogue

// Persistent: CTA c handles tiles c, c + gridDim.x, ...  The producer streams every
// tile's K chunks through the smem ring; the MMA warp fills accumulator buffer j % NBUF
// for local tile j; epilogue warpgroup j % 2 drains it and releases the buffer, so the
// epilogue of one tile overlaps the MMAs (and loads) of the next.
template <int N, int EPI, bool RES>
__global__ void __launch_bounds__(TC_THREADS, 1) conv_tc_kernel(const __grid_constant__ TcArgs a) {
    constexpr int A_BYTES = 128 * 128;
    constexpr int B_BYTES = N * 128;
    constexpr int STAGE = A_BYTES + B_BYTES;
    constexpr int ACC = acc_cols<N, RES>();
    constexpr int NBUF = n_accbuf<N, RES>();
    constexpr int NCOLS = tmem_alloc_cols<N, RES>();
    constexpr int CG = N / 8;  // channels per group
    // single accumulator buffer: both epilogue warpgroups drain every tile, each taking
    // half of the GroupNorm groups (NSPLIT = 2); otherwise warpgroups alternate tiles.
    constexpr int NSPLIT = NBUF == 1 ? 2 : 1;
    constexpr int NC = N / NSPLIT;   // columns per warpgroup
    constexpr int NG = 8 / NSPLIT;   // groups per warpgroup
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int stages = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * STAGE);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;   // [2]
    uint64_t* tempty = tfull + 2;       // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    float* sv = reinterpret_cast<float*>(tmem_holder + 4);
    float* s_bias = sv;
    float* s_gamma = sv + N;
    float* s_beta = sv + 2 * N;
    float* s_rbias = sv + 3 * N;
    float* s_red = sv + 4 * N;          // [2 WG][4 quadrants][16]
    float* s_wout = s_red + 128;        // [7][64]
    float* s_film = s_wout + 7 * 64;    // [2 WG][TC_FILM_P][2N]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles = a.geom ? a.rows : (a.rows + 127) / 128;   // geom 1: rows = #tiles
    const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128 * NSPLIT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.tmA[0]) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.tmW) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "r"(NCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp >= 2) {
        for (int i = threadIdx.x - 64; i < N; i += 128 * TC_EPI_WG) {
            s_bias[i] = a.bias[i];
            if (EPI != EPI_PLAIN && EPI != EPI_RELU2D) {
                s_gamma[i] = a.gamma[i];
                s_beta[i] = a.beta[i];
            }
            if (RES) s_rbias[i] = a.rbias[i];
        }
        if (EPI == EPI_FINAL)
            for (int i = threadIdx.x - 64; i < U_DOF * 64; i += 128 * TC_EPI_WG) s_wout[i] = a.wout[i];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int j = 0; j < my_tiles; ++j) {
                const int tile = blockIdx.x + j * gridDim.x;
                const int b0 = a.geom ? 0 : tile * 128 / a.Tv;
                int img = 0, y0 = 0, x0 = 0;
                if (a.geom) {
                    const int per_img = a.tiles_x * a.tiles_y;
                    img = tile / per_img;
                    const int tt = tile % per_img;
                    y0 = (tt / a.tiles_x) * a.ry;
                    x0 = (tt % a.tiles_x) * a.wx;
                }
                for (int i = 0; i < a.n_chunks; ++i, ++it) {
                    const int s = it % stages;
                    const uint32_t ph = (uint32_t)(it / stages) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    mbar_expect_tx(&full[s], STAGE);
                    const TcChunk ch = a.chunk[i];
                    uint8_t* sa = smem + (size_t)s * STAGE;
                    if (a.geom)
                        tma_load_5d(sa, &a.tmA[ch.src], &full[s], ch.c, x0 + ch.dx, ch.par, y0 + ch.dt, img);
                    else
                        tma_load_3d(sa, &a.tmA[ch.src], &full[s], ch.c, ch.dt, b0);
                    tma_load_2d(sa + A_BYTES, ch.res ? &a.tmR : &a.tmW, &full[s], ch.kcol, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(128, N);
            int it = 0;
            for (int j = 0; j < my_tiles; ++j) {
                const int buf = j % NBUF;
                const uint32_t use = (uint32_t)(j / NBUF);
                mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t acc0 = tmem_base + (uint32_t)(buf * ACC);
                for (int i = 0; i < a.n_chunks; ++i, ++it) {
                    const int s = it % stages;
                    const uint32_t ph = (uint32_t)(it / stages) & 1u;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const TcChunk ch = a.chunk[i];
                    const uint8_t* sa = smem + (size_t)s * STAGE;
                    const uint64_t da = umma_desc_sw128(sa);
                    const uint64_t db = umma_desc_sw128(sa + A_BYTES);
                    const uint32_t d_tmem = acc0 + (ch.res ? (uint32_t)N : 0u);
                    if (!(a.dbg & 2)) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_bf16(d_tmem, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc,
                                      (ch.first && kk == 0) ? 0u : 1u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else {
        // ============================ epilogue ============================
        const int wg = (warp - 2) >> 2;   // warpgroup
        const int q = warp & 3;           // TMEM lane quadrant of this warp
        const int r = q * 32 + lane;
        const int Tv = a.Tv;
        const int seg = Tv < 32 ? Tv : 32;
        const float inv_n = 1.0f / (float)(Tv * CG);
        float* red = s_red + wg * 64;
        const int cbase = NSPLIT == 2 ? wg * NC : 0;   // first column of this warpgroup
        const int j0 = NSPLIT == 2 ? 0 : wg;
        const int jstep = NSPLIT == 2 ? 1 : TC_EPI_WG;
        for (int j = j0; j < my_tiles; j += jstep) {
            const int tile = blockIdx.x + j * gridDim.x;
            const int buf = j % NBUF;
            const uint32_t use = (uint32_t)(j / NBUF);
            const int grow = tile * 128 + r;
            const bool valid = grow < a.rows;
            const uint32_t t_lane = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * ACC + cbase);
            mbar_wait(&tfull[buf], use & 1u);
            tc_fence_after();

            if (a.dbg & 1) {
                // debug: drain without epilogue work
            } else if constexpr (EPI == EPI_RELU2D) {
                const int per_img = a.tiles_x * a.tiles_y;
                const int img = tile / per_img, tt = tile % per_img;
                const int y = (tt / a.tiles_x) * a.ry + r / a.wx, x = (tt % a.tiles_x) * a.wx + r % a.wx;
                const bool ok = y < a.Ho && x < a.Wo;
                __nv_bfloat16* o = a.out + (((size_t)img * a.Hp + y) * a.Wo + x) * N;
#pragma unroll 1
                for (int cc = 0; cc < NC; cc += 32) {
                    float v[32];
                    tmem_ld32(t_lane + cc, v);
                    if (ok) {
                        const int c0 = cbase + cc;
#pragma unroll
                        for (int jj = 0; jj < 32; jj += 8) {
                            __align__(16) __nv_bfloat162 pk[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                pk[u] = __floats2bfloat162_rn(fmaxf(v[jj + 2 * u] + s_bias[c0 + jj + 2 * u], 0.f),
                                                              fmaxf(v[jj + 2 * u + 1] + s_bias[c0 + jj + 2 * u + 1], 0.f));
                            *reinterpret_cast<uint4*>(o + c0 + jj) = *reinterpret_cast<uint4*>(pk);
                        }
                    }
                }
            } else if constexpr (EPI == EPI_PLAIN) {
#pragma unroll 1
                for (int cc = 0; cc < NC; cc += 32) {
                    float v[32];
                    tmem_ld32(t_lane + cc, v);
                    if (valid) {
                        const int c0 = cbase + cc;
                        __nv_bfloat16* o = a.out + (size_t)grow * N + c0;
#pragma unroll
                        for (int jj = 0; jj < 32; jj += 8) {
                            __align__(16) __nv_bfloat162 pk[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                pk[u] = __floats2bfloat162_rn(v[jj + 2 * u] + s_bias[c0 + jj + 2 * u],
                                                              v[jj + 2 * u + 1] + s_bias[c0 + jj + 2 * u + 1]);
                            *reinterpret_cast<uint4*>(o + jj) = *reinterpret_cast<uint4*>(pk);
                        }
                    }
                }
            } else {
                // ---- GroupNorm statistics (local groups of this warpgroup), one pass
                float s1[NG], s2[NG], mean[NG], rstd[NG];
#pragma unroll
                for (int g = 0; g < NG; ++g) s1[g] = s2[g] = 0.f;
#pragma unroll
                for (int cc = 0; cc < NC; cc += 32) {
                    float v[32];
                    tmem_ld32(t_lane + cc, v);
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        const float xv = v[jj] + s_bias[cbase + cc + jj];
                        s1[(cc + jj) / CG] += xv;
                        s2[(cc + jj) / CG] = fmaf(xv, xv, s2[(cc + jj) / CG]);
                    }
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    if (off < seg)
#pragma unroll
                        for (int g = 0; g < NG; ++g) {
                            s1[g] += __shfl_xor_sync(PS_FULL, s1[g], off);
                            s2[g] += __shfl_xor_sync(PS_FULL, s2[g], off);
                        }
                if (Tv > 32) {  // a sample spans two warps (quadrants q, q^1)
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
                    if (lane == 0)
#pragma unroll
                        for (int g = 0; g < NG; ++g) {
                            red[q * 16 + g] = s1[g];
                            red[q * 16 + 8 + g] = s2[g];
                        }
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        s1[g] = red[q * 16 + g] + red[(q ^ 1) * 16 + g];
                        s2[g] = red[q * 16 + 8 + g] + red[(q ^ 1) * 16 + 8 + g];
                    }
                }
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    mean[g] = s1[g] * inv_n;
                    rstd[g] = rsqrtf(fmaxf(fmaf(s2[g], inv_n, -mean[g] * mean[g]), 0.f) + 1e-5f);
                }

                const int b = grow / Tv;
                const int p = b / a.S;
                if constexpr (EPI == EPI_FINAL) {
                    static_assert(N == 64 && NSPLIT == 1, "final layer has 64 channels");
                    float y[64];
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        float v[32];
                        tmem_ld32(t_lane + c0, v);
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            const int c = c0 + jj;
                            const float t = (v[jj] + s_bias[c] - mean[c / CG]) * rstd[c / CG];
                            y[c] = mish_fast(fmaf(t, s_gamma[c], s_beta[c]));
                        }
                    }
                    if (valid) {
                        float eps[U_DOF];
#pragma unroll
                        for (int d = 0; d < U_DOF; ++d) {
                            float acc = a.bout[d];
#pragma unroll
                            for (int c = 0; c < 64; ++c) acc = fmaf(y[c], s_wout[d * 64 + c], acc);
                            eps[d] = acc;
                        }
                        const int t = grow % Tv;
                        float* xr = a.x + (size_t)grow * U_DOF;
                        if (a.eps_out) {
#pragma unroll
                            for (int d = 0; d < U_DOF; ++d) a.eps_out[(size_t)grow * U_DOF + d] = eps[d];
                        } else {
                            const StepCoef sc = a.sc;
#pragma unroll
                            for (int d = 0; d < U_DOF; ++d) {
                                const float xv = xr[d];
                                float x0 = (xv - sc.sq1m * eps[d]) * sc.rsq;
                                x0 = fminf(fmaxf(x0, -0.1f), 1.1f);
                                if (sc.last) {
                                    a.traj[(size_t)grow * U_DOF + d] =
                                        (t == 0) ? a.q_start[(size_t)p * U_DOF + d] : a.lo + x0 * (a.hi - a.lo);
                                } else if (sc.ddpm) {
                                    const float z = normal_tc((uint32_t)sc.k, (uint32_t)(a.p0 + p),
                                                              (uint32_t)(b % a.S), (uint32_t)(t * U_DOF + d), a.key);
                                    xr[d] = sc.c0 * x0 + sc.c1 * xv + sc.sig * z;
                                } else {
                                    xr[d] = sc.sqn * x0 + sc.sq1mn * eps[d];
                                }
                            }
                        }
                    }
                } else {
                    // FiLM (scale, shift) for the <= TC_FILM_P problems of this tile, staged in smem
                    const float* film_row = nullptr;
                    if constexpr (EPI == EPI_GN_FILM) {
                        const int last_row = min(tile * 128 + 127, a.rows - 1);
                        const int p_lo = (tile * 128 / Tv) / a.S, p_hi = (last_row / Tv) / a.S;
                        float* sf = s_film + wg * (TC_FILM_P * 2 * N);
                        if (p_hi - p_lo < TC_FILM_P) {
                            asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
                            const int n = (p_hi - p_lo + 1) * 2 * N;
                            for (int i = r; i < n; i += 128) {
                                const int pp = p_lo + i / (2 * N), c = i % (2 * N);
                                sf[i] = __ldg(a.film + (size_t)pp * 3584 + a.film_col + c);
                            }
                            asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
                            film_row = sf + (p - p_lo) * 2 * N;
                        } else {
                            film_row = a.film + (size_t)p * 3584 + a.film_col;
                        }
                    }
                    if (valid) {
#pragma unroll 1
                        for (int cc = 0; cc < NC; cc += 16) {
                            const int c0 = cbase + cc;
                            float v[32];
                            // 16 columns per step keeps the register footprint below the cap
                            uint32_t rr[16];
                            asm volatile(
                                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                                : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]),
                                  "=r"(rr[6]), "=r"(rr[7]), "=r"(rr[8]), "=r"(rr[9]), "=r"(rr[10]), "=r"(rr[11]),
                                  "=r"(rr[12]), "=r"(rr[13]), "=r"(rr[14]), "=r"(rr[15])
                                : "r"(t_lane + cc));
                            if constexpr (RES) {
                                uint32_t rq[16];
                                asm volatile(
                                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                                    : "=r"(rq[0]), "=r"(rq[1]), "=r"(rq[2]), "=r"(rq[3]), "=r"(rq[4]), "=r"(rq[5]),
                                      "=r"(rq[6]), "=r"(rq[7]), "=r"(rq[8]), "=r"(rq[9]), "=r"(rq[10]), "=r"(rq[11]),
                                      "=r"(rq[12]), "=r"(rq[13]), "=r"(rq[14]), "=r"(rq[15])
                                    : "r"(t_lane + N + cc));
                                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj) v[16 + jj] = __uint_as_float(rq[jj]);
                            } else {
                                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                            }
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(rr[jj]);
                            const int gi = cc / CG;
                            const float mu = sel(mean, gi), rs = sel(rstd, gi);
                            const float mu2 = CG < 16 ? sel(mean, gi + 1) : mu;
                            const float rs2 = CG < 16 ? sel(rstd, gi + 1) : rs;
                            float y[16];
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) {
                                const int c = c0 + jj;
                                const bool hi = CG < 16 && jj >= CG;
                                const float t = (v[jj] + s_bias[c] - (hi ? mu2 : mu)) * (hi ? rs2 : rs);
                                y[jj] = mish_fast(fmaf(t, s_gamma[c], s_beta[c]));
                            }
                            if constexpr (EPI == EPI_GN_FILM) {
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj)
                                    y[jj] = fmaf(y[jj], 1.f + film_row[c0 + jj], film_row[N + c0 + jj]);
                            } else if constexpr (RES) {
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj) y[jj] += v[16 + jj] + s_rbias[c0 + jj];
                            } else {
                                const uint4* rsrc = reinterpret_cast<const uint4*>(a.res_src + (size_t)grow * N + c0);
#pragma unroll
                                for (int jj = 0; jj < 16; jj += 8) {
                                    uint4 u = __ldg(rsrc + jj / 8);
                                    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                                    for (int k2 = 0; k2 < 4; ++k2) {
                                        const float2 f = __bfloat1622float2(h2[k2]);
                                        y[jj + 2 * k2] += f.x;
                                        y[jj + 2 * k2 + 1] += f.y;
                                    }
                                }
                            }
                            __nv_bfloat16* o = a.out + (size_t)grow * N + c0;
#pragma unroll
                            for (int jj = 0; jj < 16; jj += 8) {
                                __align__(16) __nv_bfloat162 pk[4];
#pragma unroll
                                for (int u = 0; u < 4; ++u) pk[u] = __floats2bfloat162_rn(y[jj + 2 * u], y[jj + 2 * u + 1]);
                                *reinterpret_cast<uint4*>(o + jj) = *reinterpret_cast<uint4*>(pk);
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[buf]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NCOLS));
    }
}

__global__ void gather_bf16_kernel(const float* __restrict__ blob, const long long* __restrict__ src, size_t n,
                                   __nv_bfloat16* __restrict__ dst) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __float2bfloat16_rn(src[i] >= 0 ? blob[src[i]] : 0.f);
}
__global__ void gather_f32_kernel(const float* __restrict__ blob, const long long* __restrict__ src, size_t n,
                                  float* __restrict__ dst) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i] >= 0 ? blob[src[i]] : 0.f;
}

// bf16 view of the fp32 state for the first layer: xb[row] = (x[row][0..6], 0), 16 B per
// row; the first layer's taps are row shifts of this view inside the MMA descriptors.
__global__ void xb_kernel(const float* __restrict__ x, size_t rows, __nv_bfloat16* __restrict__ xb) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int u = 0; u < U_DOF; ++u) v[u] = __float2bfloat16_rn(__ldg(x + i * U_DOF + u));
    v[7] = __float2bfloat16_rn(0.f);
    reinterpret_cast<uint4*>(xb)[i] = *reinterpret_cast<uint4*>(v);
}

// ---------------------------------------------------------------------------
// host side: tensor maps and launches
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encoder() {
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    return g_encode != nullptr;
}

// weights [N][Kp] bf16, box {64, N}
bool make_w_map(CUtensorMap* tm, const void* base, int N, int Kp, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)Kp * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(box_rows ? box_rows : N)};
    cuuint32_t es[2] = {1, 1};
    return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static size_t kpad(int K) { return (size_t)((K + 63) / 64) * 64; }

template <int N, int EPI, bool RES>
static int launch_tc(TcArgs& a, int n_tiles, cudaStream_t st) {
    constexpr int STAGE = 128 * 128 + N * 128;
    const int stages = N == 256 ? 4 : (N == 128 ? 6 : 8);
    a.stages = stages;
    const size_t smem = 1024 + (size_t)stages * STAGE + (2 * stages + 4) * 8 + 16 +
                        (4 * N + 128 + 7 * 64 + TC_EPI_WG * TC_FILM_P * 2 * N) * 4;
    auto kern = conv_tc_kernel<N, EPI, RES>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return PS_FAIL(PS_ERR_CUDA);
        attr_set = true;
    }
    static const int dbg = std::getenv("PS_TC_DBG") ? std::atoi(std::getenv("PS_TC_DBG")) : 0;
    a.dbg = dbg;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = n_tiles < n_sm ? n_tiles : n_sm;
    kern<<<grid, TC_THREADS, smem, st>>>(a);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

// ===========================================================================
// U-Net layers: (time, sample)-ordered tiles with one activation load per channel
// chunk.  Tile rows are r = t * nb + s (nb = 128 / Tv samples), so a conv tap dt is
// a uniform shift of dt * nb rows: each 64-channel activation chunk is loaded ONCE
// per tile as a [(Tv + 4) x nb] box whose two halo rows on each side are TMA
// zero-fill (the conv's zero padding), and the 1..5 taps that read it issue their
// MMAs from shifted smem descriptors (SW128 base-offset field set for row shifts that
// are not multiples of 8).  Weights stream through a separate ring, one [N x 64] box
// per (tap, chunk).
// ===========================================================================
constexpr int UT_MAXG = 24;   // activation chunk groups per tile
constexpr int UT_MAXTAP = 64;

struct UtGroup {
    int16_t c;      // channel offset in the source view
    int8_t src;     // activation map
    int8_t ntap;    // taps reading this chunk
    int16_t tap0;   // index of its first tap
    int8_t xb;      // 1: the 8-channel bf16 state view (no swizzle, 16-B rows)
};
struct UtTap {
    int16_t kcol;   // weight K column
    int8_t dt;      // time shift
    int8_t res;     // residual accumulator
    int8_t first;   // first MMA into its accumulator
};

constexpr int UT_EPI_WG = 4;                       // U-Net epilogue warpgroups
#ifndef PS_GN_PIPE
#define PS_GN_PIPE 0   // 1: GroupNorm statistics pipelined one tile ahead (4 TMEM buffers); measured 0.7% slower
#endif
constexpr int UT_THREADS = 64 + 128 * UT_EPI_WG;
// GroupNorm partials in shared memory: [2 tile parity][WG][4 quadrants][32 samples][2 * NG];
// FINAL (one warpgroup per tile, all 8 groups): [WG][4 quadrants][32 samples][16]
template <int EPI, int NG>
__host__ __device__ constexpr int ut_red_floats() {
    return EPI == EPI_FINAL ? UT_EPI_WG * 4 * 32 * 16 : 2 * UT_EPI_WG * 4 * 32 * 2 * NG;
}

struct UtArgs {
    CUtensorMap tmA[3];
    CUtensorMap tmW;
    CUtensorMap tmR;
    CUtensorMap tmO;   // output view [B][Tv][N], (time, sample)-ordered boxes {16, nb, 128/nb}
    CUtensorMap tmRes; // identity residual view, same geometry as tmO
    UtGroup grp[UT_MAXG];
    UtTap tap[UT_MAXTAP];
    int n_grp, n_tap;
    int sa_stages, sb_stages;
    int resident;   // 1: every tap's weight box stays in B stage <tap> for the whole kernel
    int B, Tv, nb, S;
    unsigned long long s_magic;   // ceil(2^40 / S): x / S = (x * s_magic) >> 40 for x < 2^40 / S
    const float* bias;
    const float* gamma;
    const float* beta;
    const float* rbias;
    const __nv_bfloat16* res_src;
    const float* film;        // per-problem FiLM part [P][3584]
    const float* film_b;      // this step's per-step part [3584], added when the tile's rows are staged
    int film_col;
    __nv_bfloat16* out;
    __nv_bfloat16* xb_next;   // FINAL: bf16 view of the updated state for the next step's first layer
    const float* wout;
    const float* bout;
    float* x;
    StepCoef sc;
    int p0;
    unsigned key;
    const float* q_start;
    float* traj;
    float lo, hi;
    float* eps_out;
    int dbg;
};

// sample -> problem index without an integer division (exact for x < 2^40 / S)
__device__ __forceinline__ int div_s(const UtArgs& a, int x) {
    return (int)(((unsigned long long)(unsigned)x * a.s_magic) >> 40);
}

// SW128 K-major descriptor for a matrix starting `row` rows into a 1024-B aligned slot
// (measured on B200: the MMA applies the SW128 XOR pattern from absolute smem address
// bits, so a row-shifted start needs no base-offset field; setting it breaks results)
__device__ __forceinline__ uint64_t umma_desc_sw128_rows(const void* slot, int row) {
    const uint32_t a = smem_u32(slot) + (uint32_t)row * 128u;
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// no-swizzle K-major descriptor over 16-B rows in (time, sample) order: core matrices are
// 8 consecutive rows (SBO = 128 B to the next 8 rows); LBO = nb * 16 B steps K by one time shift
__device__ __forceinline__ uint64_t xb_desc(const void* base, int nb) {
    const uint32_t a = smem_u32(base);
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);
    d |= (uint64_t)(((uint32_t)nb * 16u) >> 4) << 16;   // LBO: K direction
    d |= (uint64_t)(128 >> 4) << 32;                     // SBO: M direction
    d |= (uint64_t)1 << 46;
    return d;                                            // layout type 0: SWIZZLE_NONE
}

// MB = M-blocks (128 rows) per tile: every weight stage feeds MB x 4 MMAs.
// PAIR: CTA pairs (cluster of 2, cta_group::2): the two CTAs hold adjacent 128-row tiles
// and HALF of every weight box each; the leader issues M=256 MMAs over both CTAs' smem
// (half the weight bytes per SM, in shared memory traffic and in L2 reads).
// SPLIT: N-split for latency-bound small batches: a work item is (tile, channel slice of N
// = NF / SPLIT channels, whole GroupNorm groups); the template N is the slice width.
template <int N, int EPI, bool RES, int MB, bool PAIR, int SPLIT>
__global__ void __launch_bounds__(UT_THREADS, 1) unet_tc_kernel(const __grid_constant__ UtArgs a) {
    constexpr int NF = N * SPLIT;   // the layer's output channels
    constexpr int B_BYTES = PAIR ? N * 64 : N * 128;   // this CTA's share of a weight stage
    constexpr int ACC1 = acc_cols<N, RES>();          // columns of one M-block
    constexpr int ACC = MB * ACC1;                     // columns of one tile
    constexpr bool FIN = EPI == EPI_FINAL;
    // TMEM accumulator buffers: up to 4, so the commit -> epilogue -> release round trip of a
    // tile hides behind the MMAs of the following tiles even when a tile's K loop is short.
    // FINAL: 7 x 64 columns + the warpgroups' 4 x 16 projection columns = all 512, so the MMAs
    // run up to three tiles ahead of the four warpgroup-owned tiles in flight
    constexpr int NBUF = FIN ? 7 : 4 * ACC <= 512 ? 4 : 2 * ACC <= 512 ? 2 : 1;
    // FINAL: the 64->7 projection runs on the tensor core from a bf16 tile in smem into
    // 16 TMEM columns per epilogue warpgroup after the accumulators
    constexpr int PROJ_COL = NBUF * ACC;
    constexpr int NUSED = NBUF * ACC + (FIN ? 16 * UT_EPI_WG : 0);
    constexpr int NCOLS = NUSED <= 32 ? 32 : NUSED <= 64 ? 64 : NUSED <= 128 ? 128 : NUSED <= 256 ? 256 : 512;
    constexpr int CG = NF / 8;   // channels per GroupNorm group (of the full layer)
    // both warpgroups drain every tile, each half of the channels / GroupNorm groups
    constexpr int NSPLIT = UT_EPI_WG;
    constexpr int NC = N / NSPLIT;
    constexpr int NG = 8 / (SPLIT * NSPLIT);
    extern __shared__ __align__(1024) uint8_t smem_dyn[];
    // SW128 tiles need 1024-B alignment; offset within the shared array (keeps LDS/STS)
    uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
    const int Tv = a.Tv, nb = a.nb;
    const int A_BYTES = (Tv + 4) * nb * 128;
    const int SA = a.sa_stages, SB = a.sb_stages;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)SA * A_BYTES;
    // FINAL only: per epilogue warpgroup a projection A tile [128 x 64] bf16 SW128 and the
    // tile's noise [128 x 7]; W_out^T [16 x 64] bf16 SW128
    uint8_t* sP = sB + (size_t)SB * B_BYTES;
    uint8_t* sWo = sP + (FIN ? UT_EPI_WG * 16384 : 0);
    float* sZ = reinterpret_cast<float*>(sWo + (FIN ? 2048 : 0));
    // output staging (non-FINAL): per warpgroup two [128 rows x 16 ch] bf16 buffers that
    // TMA-store 16-channel column slabs of the tile (coalesced writes off the LSU path)
    uint8_t* sOut = reinterpret_cast<uint8_t*>(sZ) + (FIN ? UT_EPI_WG * 128 * U_DOF * 4 : 0);
    uint64_t* a_full = reinterpret_cast<uint64_t*>(sOut + (FIN ? 0 : UT_EPI_WG * 2 * 4096));
    uint64_t* a_empty = a_full + SA;
    uint64_t* b_full = a_empty + SA;
    uint64_t* b_empty = b_full + SB;
    uint64_t* tfull = b_empty + SB;
    uint64_t* tempty = tfull + 8;
    uint64_t* pbar = tempty + 8;                 // FINAL: projection MMA done, per warpgroup
    uint64_t* rbar = pbar + 4;                   // identity residual slabs: [epilogue warp][2]
    uint64_t* gnbar = rbar + 8 * UT_EPI_WG;      // GroupNorm partials posted: [epilogue warpgroup][2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gnbar + 2 * UT_EPI_WG);
    float* s_bias = reinterpret_cast<float*>(tmem_holder + 4);
    float* s_gamma = s_bias + NF;
    float* s_beta = s_gamma + NF;
    float* s_rbias = s_beta + NF;
    float* s_wout = s_rbias + NF;                // [7][64]
    float* s_red = s_wout + 7 * 64;              // [2 tile parity][WG][4 quadrants][32 samples][2*NG]
    float* s_film = s_red + ut_red_floats<EPI, NG>();  // [3 tiles][WG][TC_FILM_P][2*NC]
    UtGroup* s_grp = reinterpret_cast<UtGroup*>(s_film + 3 * UT_EPI_WG * TC_FILM_P * 2 * NC);
    UtTap* s_tap = reinterpret_cast<UtTap*>(s_grp + UT_MAXG);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles = (a.B + nb - 1) / nb;
    // tile sequence: single CTAs stride over tiles; pairs stride over tile pairs, rank r of
    // the pair takes tile 2 * pair + r (a phantom tile past the end when n_tiles is odd:
    // its loads are zero-filled and its stores clipped)
    const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
    const bool leader = crank == 0;
    // work items: (tile or tile pair) x channel slice
    const int n_units = (PAIR ? (n_tiles + 1) / 2 : n_tiles) * SPLIT;
    const int unit0 = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    const int ustride = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
    const int my_tiles = unit0 < n_units ? (n_units - 1 - unit0) / ustride + 1 : 0;
    auto tile_of = [&](int j) {
        const int u = (unit0 + j * ustride) / SPLIT;
        return PAIR ? 2 * u + (int)crank : u;
    };
    auto slice_of = [&](int j) { return (unit0 + j * ustride) % SPLIT; };

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < SA; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < SB; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            // one arrival per epilogue warp (both CTAs); FINAL: the 4 warps of the tile's warpgroup
            mbar_init(&tempty[b], FIN ? 4 : (PAIR ? 2 : 1) * 4 * NSPLIT);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&pbar[i], 1);
        for (int i = 0; i < 8 * UT_EPI_WG; ++i) mbar_init(&rbar[i], 1);
        for (int i = 0; i < 2 * UT_EPI_WG; ++i) mbar_init(&gnbar[i], 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.tmA[0]) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.tmW) : "memory");
    }
    if (warp == 1) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                         "r"(NCOLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                         "r"(NCOLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    if (warp >= 2) {
        for (int i = threadIdx.x - 64; i < NF; i += 128 * UT_EPI_WG) {
            s_bias[i] = a.bias[i];
            if (EPI != EPI_PLAIN) {
                s_gamma[i] = a.gamma[i];
                s_beta[i] = a.beta[i];
            }
            if (RES) s_rbias[i] = a.rbias[i];
        }
        if constexpr (FIN) {
            // W_out^T as the projection's B operand: row n = joint (7 used of 16), K = 64 channels,
            // 16-B chunk j of row n at chunk position j ^ (n & 7) (SW128, absolute-address swizzle)
            for (int i = threadIdx.x - 64; i < 16 * 8; i += 128 * UT_EPI_WG) {
                const int n = i >> 3, jc = i & 7;
                __align__(16) __nv_bfloat16 w8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) w8[u] = __float2bfloat16_rn(n < U_DOF ? a.wout[n * 64 + jc * 8 + u] : 0.f);
                *reinterpret_cast<uint4*>(sWo + n * 128 + ((jc ^ (n & 7)) << 4)) = *reinterpret_cast<uint4*>(w8);
            }
            if (threadIdx.x - 64 < U_DOF) s_wout[threadIdx.x - 64] = a.bout[threadIdx.x - 64];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        for (int i = threadIdx.x - 64; i < a.n_grp; i += 128 * UT_EPI_WG) s_grp[i] = a.grp[i];
        for (int i = threadIdx.x - 64; i < a.n_tap; i += 128 * UT_EPI_WG) s_tap[i] = a.tap[i];
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync_all();   // both CTAs' barriers initialised before any remote signal
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // weight box of tap t into B stage `stage` (this CTA's half for pairs); the leader's
    // b_full counts both halves
    auto load_w = [&](int stage, int t, int slice) {
        const UtTap tp = s_tap[t];
        const CUtensorMap* tm = tp.res ? &a.tmR : &a.tmW;
        if constexpr (PAIR) {
            if (leader) mbar_expect_tx(&b_full[stage], (uint32_t)(2 * B_BYTES));
            tma_load_2d_cg2(sB + (size_t)stage * B_BYTES, tm, leader_addr(&b_full[stage]), tp.kcol,
                            slice * N + (int)crank * (N / 2));
        } else {
            mbar_expect_tx(&b_full[stage], (uint32_t)B_BYTES);
            tma_load_2d(sB + (size_t)stage * B_BYTES, tm, &b_full[stage], tp.kcol, slice * N);
        }
    };
    // programmatic dependent launch: the prologue above overlapped the previous layer's
    // tail.  The producer first sends the first tile's weight boxes (no kernel writes
    // weights), then every thread waits for the previous grid before touching activations,
    // and the next layer's CTAs may launch (they become resident as this kernel's CTAs exit)
    int pre = 0;   // weight boxes issued before the dependency wait (stages 0..pre-1)
    if (warp == 0 && lane == 0 && my_tiles > 0 && !(a.dbg & (16 | 64))) {
        pre = a.resident ? a.n_tap : (a.n_tap < SB ? a.n_tap : SB);
        for (int t = 0; t < pre; ++t) load_w(t, t, slice_of(0));
    }
    pdl_wait();
    pdl_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            int sa = 0, sb = 0;
            uint32_t pa = 0, pb = 0;   // phase bits of the A / B rings
            const int n_grp = a.n_grp;
            const bool resident = a.resident != 0;
            if (resident && my_tiles > 0)
                for (int t = pre; t < a.n_tap; ++t) load_w(t, t, 0);   // weights loaded once, reused by every tile
            int issued = 0;   // streamed weight boxes counted from the start of the kernel
            for (int j = 0; j < my_tiles; ++j) {
                const int b0 = tile_of(j) * nb;
                for (int g = 0; g < n_grp; ++g) {
                    const UtGroup gr = s_grp[g];
                    mbar_wait(&a_empty[sa], pa ^ 1u);
                    if (a.dbg & 8) {
                        mbar_arrive(&a_full[sa]);
                    } else if constexpr (PAIR) {   // (pairs never use the 8-channel state view)
                        if (leader) mbar_expect_tx(&a_full[sa], (uint32_t)(2 * A_BYTES));
                        tma_load_3d_cg2(sA + (size_t)sa * A_BYTES, &a.tmA[gr.src], leader_addr(&a_full[sa]), gr.c, b0, -2);
                    } else {
                        mbar_expect_tx(&a_full[sa], (uint32_t)(gr.xb ? (Tv + 5) * nb * 16 : A_BYTES));
                        tma_load_3d(sA + (size_t)sa * A_BYTES, &a.tmA[gr.src], &a_full[sa], gr.c, b0, -2);
                    }
                    if (++sa == SA) { sa = 0; pa ^= 1u; }
                    if (resident) continue;
                    for (int k = 0; k < gr.ntap; ++k, ++issued) {
                        if (issued < pre) {   // sent before the dependency wait
                            if (++sb == SB) { sb = 0; pb ^= 1u; }
                            continue;
                        }
                        mbar_wait(&b_empty[sb], pb ^ 1u);
                        if (a.dbg & 16) {
                            mbar_arrive(&b_full[sb]);
                        } else {
                            load_w(sb, gr.tap0 + k, slice_of(j));
                        }
                        if (++sb == SB) { sb = 0; pb ^= 1u; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {   // the whole warp runs the issue loop; elect.sync picks the issuing lane
            constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, N);
            int sa = 0, sb = 0;
            uint32_t pa = 0, pb = 0;
            const int n_grp = a.n_grp;
            const bool do_mma = !(a.dbg & 2);
            const bool resident = a.resident != 0;
            const uint64_t dA0 = umma_desc_sw128(sA), dB0 = umma_desc_sw128(sB);
            const uint64_t a_step = (uint64_t)(A_BYTES >> 4), b_step = (uint64_t)(B_BYTES >> 4);
            const uint64_t row_step = (uint64_t)((nb * 128) >> 4);
            int buf = 0;
            uint32_t tph = 0;
            auto mma_ = [&](uint32_t d, uint64_t da_, uint64_t db_, uint32_t id, uint32_t acc) {
                if constexpr (PAIR) umma_bf16_w2(d, da_, db_, id, acc);
                else umma_bf16_w(d, da_, db_, id, acc);
            };
            auto commit_ = [&](uint64_t* bar) {
                if constexpr (PAIR) umma_commit_w2(bar);
                else umma_commit_w(bar);
            };
            for (int j = 0; j < my_tiles; ++j) {
                mbar_wait(&tempty[buf], tph ^ 1u);
                tc_fence_after();
                const uint32_t acc0 = tmem_base + (uint32_t)(buf * ACC);
                for (int g = 0; g < n_grp; ++g) {
                    const UtGroup gr = s_grp[g];
                    mbar_wait(&a_full[sa], pa);
                    const uint64_t dA = dA0 + (uint64_t)sa * a_step;
                    for (int k = 0; k < gr.ntap; ++k) {
                        const UtTap tp = s_tap[gr.tap0 + k];
                        const int bs = resident ? gr.tap0 + k : sb;   // resident: stage = tap
                        mbar_wait(&b_full[bs], resident ? 0u : pb);
                        tc_fence_after();
                        const uint64_t da = dA + (uint64_t)(2 + tp.dt) * row_step;
                        const uint64_t db = dB0 + (uint64_t)bs * b_step;
                        const uint32_t d_tmem = acc0 + (tp.res ? (uint32_t)N : 0u);
                        if (gr.xb) {
                            // state view: no-swizzle K-major, 16-B rows; a K=16 MMA reads two
                            // 8-channel core-matrix columns LBO = one time step apart, so the
                            // 5 taps are 3 MMAs (shifts -2/-1, 0/1, 2/3) and the 1x1 residual one
                            const uint64_t dX = xb_desc(sA + (size_t)sa * A_BYTES, nb);
                            const int nk = tp.res ? 1 : 3;
                            if (do_mma)
#pragma unroll
                                for (int mb = 0; mb < MB; ++mb)
                                    for (int kk = 0; kk < nk; ++kk) {
                                        const int sh = tp.res ? 0 : 2 * kk - 2;
                                        mma_(d_tmem + (uint32_t)(mb * ACC1),
                                                  dX + (uint64_t)((((2 + sh) * nb + mb * 128) * 16) >> 4),
                                                  db + (uint64_t)(kk * 2), idesc, (tp.first && kk == 0) ? 0u : 1u);
                                    }
                        } else if (do_mma) {
#pragma unroll
                            for (int mb = 0; mb < MB; ++mb)
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    mma_(d_tmem + (uint32_t)(mb * ACC1), da + (uint64_t)(mb * 128 * 128 / 16 + kk * 2),
                                              db + (uint64_t)(kk * 2), idesc, (tp.first && kk == 0) ? 0u : 1u);
                        }
                        if (!resident) {
                            commit_(&b_empty[sb]);
                            if (++sb == SB) { sb = 0; pb ^= 1u; }
                        }
                    }
                    commit_(&a_empty[sa]);
                    if (++sa == SA) { sa = 0; pa ^= 1u; }
                }
                commit_(&tfull[buf]);
                if (++buf == NBUF) { buf = 0; tph ^= 1u; }
            }
        }
        __syncwarp();
    } else if constexpr (FIN) {
        // ======================= final-layer epilogue =======================
        // Warpgroup w drains the CTA's tiles j = w, w + 4, ... alone: all 64 channels of its
        // 128 rows (TMEM buffer w), Mish(GN(acc + bias)) as a bf16 SW128 tile in its own smem
        // buffer, the 64->7 projection as one M128 x N16 tcgen05 MMA into its own 16 TMEM
        // columns (its own barrier), then x0 clip + DDPM posterior / DDIM / denormalise for its
        // rows.  No barrier spans warpgroups, so four tiles' epilogues overlap.  The statistics
        // keep the summation order of the channel-split epilogue (per 8-channel group: packed
        // pair sums, then the time shuffles, then the 4 quadrants in order).
        static_assert(N == 64 && MB == 1 && UT_EPI_WG == 4 && CG == 8 && NCOLS == 512, "final layer shape");
        const int wg = (warp - 2) >> 2;
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const int t = r / nb, sl = r % nb;
        const float inv_n = 1.0f / (float)(Tv * CG);
        float* red = s_red + wg * (4 * 32 * 16);
        uint8_t* sPw = sP + wg * 16384;
        float* sZw = sZ + wg * (128 * U_DOF);
        const uint32_t t_lane = tmem_base + ((uint32_t)(q * 32) << 16);
        const uint32_t pcol = (uint32_t)(PROJ_COL + 16 * wg);
        const StepCoef sc = a.sc;
        const bool noisy = !a.eps_out && !sc.last && sc.ddpm;
        const int per = Tv * U_DOF / 4;   // Philox blocks per sample
        int it = 0;
        for (int j = wg; j < my_tiles; j += 4, ++it) {
            const int tile = tile_of(j);
            const int b = tile * nb + sl;
            const bool valid = b < a.B;
            const int buf = j % NBUF;
            const uint32_t t_lane0 = t_lane + (uint32_t)(buf * ACC);
            mbar_wait(&tfull[buf], (uint32_t)(j / NBUF) & 1u);
            tc_fence_after();
            if (a.dbg & 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
                continue;
            }
            float s1[8], s2[8];
#pragma unroll
            for (int cc = 0; cc < 64; cc += 16) {
                uint32_t rr[16];
                tmem_ld16(t_lane0 + cc, rr);
                tmem_wait_ld();
                float2 a1[2], a2[2];
#pragma unroll
                for (int g = 0; g < 2; ++g) a1[g] = a2[g] = f2(0.f, 0.f);
#pragma unroll
                for (int jj = 0; jj < 16; jj += 2) {
                    const int g = jj / 8;
                    const float2 bb = *reinterpret_cast<const float2*>(s_bias + cc + jj);
                    const float2 xv = fadd2(f2(__uint_as_float(rr[jj]), __uint_as_float(rr[jj + 1])), bb);
                    a1[g] = fadd2(a1[g], xv);
                    a2[g] = ffma2(xv, xv, a2[g]);
                }
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    s1[cc / 8 + g] = 0.f + (a1[g].x + a1[g].y);
                    s2[cc / 8 + g] = 0.f + (a2[g].x + a2[g].y);
                }
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1)
                if (off >= nb)
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        s1[g] += __shfl_xor_sync(PS_FULL, s1[g], off);
                        s2[g] += __shfl_xor_sync(PS_FULL, s2[g], off);
                    }
            if (lane < nb) {
                float4* rp = reinterpret_cast<float4*>(red + (q * 32 + sl) * 16);
                rp[0] = make_float4(s1[0], s1[1], s1[2], s1[3]);
                rp[1] = make_float4(s1[4], s1[5], s1[6], s1[7]);
                rp[2] = make_float4(s2[0], s2[1], s2[2], s2[3]);
                rp[3] = make_float4(s2[4], s2[5], s2[6], s2[7]);
            }
            asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
            float mean[8], rstd[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                float a1 = 0.f, a2 = 0.f;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    a1 += red[(qq * 32 + sl) * 16 + g];
                    a2 += red[(qq * 32 + sl) * 16 + 8 + g];
                }
                mean[g] = a1 * inv_n;
                rstd[g] = rsqrtf(fmaxf(fmaf(a2, inv_n, -mean[g] * mean[g]), 0.f) + 1e-5f);
            }
            // y = Mish(GN(acc + bias)) -> bf16 projection tile (row r: 128 B, SW128)
#pragma unroll
            for (int cc = 0; cc < 64; cc += 16) {
                uint32_t rr[16];
                tmem_ld16(t_lane0 + cc, rr);
                tmem_wait_ld();
                __align__(16) __nv_bfloat162 pk[8];
#pragma unroll
                for (int jj = 0; jj < 16; jj += 2) {
                    const int c = cc + jj, g = c / 8;
                    const float2 bb = *reinterpret_cast<const float2*>(s_bias + c);
                    const float2 ga = *reinterpret_cast<const float2*>(s_gamma + c);
                    const float2 be = *reinterpret_cast<const float2*>(s_beta + c);
                    const float2 xv = fadd2(f2(__uint_as_float(rr[jj]), __uint_as_float(rr[jj + 1])), bb);
                    const float nm = -mean[g] * rstd[g];
                    const float2 tt = ffma2(xv, f2(rstd[g], rstd[g]), f2(nm, nm));
                    const float2 yv = mish2(ffma2(tt, ga, be));
                    pk[jj / 2] = __floats2bfloat162_rn(yv.x, yv.y);
                }
                const int jc = cc >> 3;
                *reinterpret_cast<uint4*>(sPw + r * 128 + (((jc) ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(&pk[0]);
                *reinterpret_cast<uint4*>(sPw + r * 128 + (((jc + 1) ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(&pk[4]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);   // accumulator drained: its next tile's MMAs may start
            // the rows' state, loaded ahead of the projection (only the DDPM / DDIM update reads it)
            const int grow = b * Tv + t;
            float xs[U_DOF];
#pragma unroll
            for (int d = 0; d < U_DOF; ++d) xs[d] = 0.f;
            if (valid && !a.eps_out)
#pragma unroll
                for (int d = 0; d < U_DOF; ++d) xs[d] = a.x[(size_t)grow * U_DOF + d];
            if (noisy) {
                // the tile's Philox blocks (nb samples x Tv*7/4)
                for (int i = r; i < nb * per; i += 128) {
                    const int s2_ = i / per, blk = i - s2_ * per;
                    const int b2 = tile * nb + s2_;
                    float n4[4] = {0.f, 0.f, 0.f, 0.f};
                    if (b2 < a.B) {
                        const int p2 = div_s(a, b2);
                        normal4_tc((uint32_t)sc.k, (uint32_t)(a.p0 + p2), (uint32_t)(b2 - p2 * a.S), (uint32_t)blk, a.key, n4);
                    }
                    *reinterpret_cast<float4*>(sZw + s2_ * Tv * U_DOF + blk * 4) = make_float4(n4[0], n4[1], n4[2], n4[3]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
            if (threadIdx.x == 64 + 128 * wg) {
                tc_fence_after();
                constexpr uint32_t idp = idesc_bf16(128, 16);
                const uint64_t dP = umma_desc_sw128(sPw), dW = umma_desc_sw128(sWo);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    umma_bf16(tmem_base + pcol, dP + (uint64_t)(kk * 2), dW + (uint64_t)(kk * 2), idp, kk > 0 ? 1u : 0u);
                umma_commit(&pbar[wg]);
            }
            __syncwarp();
            mbar_wait(&pbar[wg], (uint32_t)it & 1u);
            tc_fence_after();
            uint32_t pr[16];
            tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + pcol, pr);
            tmem_wait_ld();
            float eps[U_DOF];
#pragma unroll
            for (int d = 0; d < U_DOF; ++d) eps[d] = __uint_as_float(pr[d]) + s_wout[d];
            if (valid) {
                const int p = div_s(a, b);
                float* xr = a.x + (size_t)grow * U_DOF;
                if (a.eps_out) {
#pragma unroll
                    for (int d = 0; d < U_DOF; ++d) a.eps_out[(size_t)grow * U_DOF + d] = eps[d];
                } else {
                    const float* zr = sZw + sl * Tv * U_DOF + t * U_DOF;
                    __align__(16) __nv_bfloat16 xv8[8];
                    xv8[7] = __float2bfloat16_rn(0.f);
#pragma unroll
                    for (int d = 0; d < U_DOF; ++d) {
                        const float xv = xs[d];
                        float x0 = (xv - sc.sq1m * eps[d]) * sc.rsq;
                        x0 = fminf(fmaxf(x0, -0.1f), 1.1f);
                        if (sc.last) {
                            a.traj[(size_t)grow * U_DOF + d] =
                                (t == 0) ? a.q_start[(size_t)p * U_DOF + d] : a.lo + x0 * (a.hi - a.lo);
                        } else {
                            const float xn = sc.ddpm ? sc.c0 * x0 + sc.c1 * xv + sc.sig * zr[d]
                                                     : sc.sqn * x0 + sc.sq1mn * eps[d];
                            xr[d] = xn;
                            xv8[d] = __float2bfloat16_rn(xn);
                        }
                    }
                    if (!sc.last && a.xb_next)
                        *reinterpret_cast<uint4*>(a.xb_next + (size_t)grow * 8) = *reinterpret_cast<const uint4*>(xv8);
                }
            }
        }
    } else {
        // ============================ epilogue ============================
        const int wg = (warp - 2) >> 2;
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const int sl = r % nb;  // tile row = (time, sample); M-block mb adds 128/nb time steps
        const int tstep = 128 / nb;
        const float inv_n = 1.0f / (float)(Tv * CG);
        float* red = s_red + wg * (4 * 32 * 2 * NG);
        const int cbase = NSPLIT > 1 ? wg * NC : 0;   // first column of this warpgroup
        const int ew = warp - 2;                       // epilogue warp 0..4*WG-1
        const float* s_bias_all = s_bias;
        const float* s_gamma_all = s_gamma;
        const float* s_beta_all = s_beta;
        const float* s_rbias_all = s_rbias;
        const int t_w = (q * 32) / nb;                 // first time row of this warp's 32 rows
        uint32_t ob = 0;   // staging buffer counter of this warp
        int cur_tile = 0, cur_noff = 0;
        // 16 channels of this thread's row -> the warp's staging buffer (1 KB) -> TMA store of
        // the warp's [32 rows x 16 ch] box; lane 0 first waits until the store from the other
        // buffer has been read out, so the next slab can be written right after __syncwarp
        auto stage_store = [&](const __nv_bfloat162* pk, int c0, int mb) {
            uint8_t* so = sOut + (size_t)(ew * 2 + (ob & 1u)) * 1024;
            *reinterpret_cast<uint4*>(so + lane * 32) = reinterpret_cast<const uint4*>(pk)[0];
            *reinterpret_cast<uint4*>(so + lane * 32 + 16) = reinterpret_cast<const uint4*>(pk)[1];
            fence_proxy_async_smem();
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
            if (lane == 0) {
                tma_store_3d(&a.tmO, so, c0 + cur_noff, cur_tile * nb, mb * tstep + t_w);
                bulk_commit();
            }
            ++ob;
        };
        // identity residual (GN_RES without a projection): the warp's residual box is TMA-loaded
        // into its staging buffer one slab ahead; each lane adds its row and writes the output
        // back in place, and the same buffer is TMA-stored
        constexpr bool IDRES = EPI == EPI_GN_RES && !RES;
        const int n_slab = MB * (NC / 16);
        auto res_load = [&](uint32_t o, int tile_, int slab, int noff_) {
            constexpr int SPM = NC >= 16 ? NC / 16 : 1;   // 16-channel slabs per M-block
            const int mb_ = slab / SPM, c_ = noff_ + cbase + (slab % SPM) * 16;
            uint64_t* bar = &rbar[ew * 2 + (o & 1u)];
            mbar_expect_tx(bar, 1024u);
            tma_load_3d(sOut + (size_t)(ew * 2 + (o & 1u)) * 1024, &a.tmRes, bar, c_, tile_ * nb,
                        mb_ * tstep + t_w);
        };
        auto stage_store_res = [&](float* y, int c0, int mb, int j_, int slab) {
            const uint32_t bi = ob & 1u;
            uint8_t* so = sOut + (size_t)(ew * 2 + bi) * 1024;
            mbar_wait(&rbar[ew * 2 + bi], (ob >> 1) & 1u);
            const uint4 q0 = *reinterpret_cast<const uint4*>(so + lane * 32);
            const uint4 q1 = *reinterpret_cast<const uint4*>(so + lane * 32 + 16);
            const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&q0);
            const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&q1);
            __align__(16) __nv_bfloat162 pk[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f0 = __bfloat1622float2(h0[u]), f1 = __bfloat1622float2(h1[u]);
                pk[u] = __floats2bfloat162_rn(y[2 * u] + f0.x, y[2 * u + 1] + f0.y);
                pk[4 + u] = __floats2bfloat162_rn(y[8 + 2 * u] + f1.x, y[8 + 2 * u + 1] + f1.y);
            }
            *reinterpret_cast<uint4*>(so + lane * 32) = reinterpret_cast<const uint4*>(pk)[0];
            *reinterpret_cast<uint4*>(so + lane * 32 + 16) = reinterpret_cast<const uint4*>(pk)[1];
            fence_proxy_async_smem();
            if (lane == 0) {
                bulk_wait_read0();   // the other buffer's store has been read out: prefetch into it
                if (slab + 1 < n_slab) res_load(ob + 1, cur_tile, slab + 1, cur_noff);
                else if (j_ + 1 < my_tiles) res_load(ob + 1, tile_of(j_ + 1), 0, slice_of(j_ + 1) * N);
            }
            __syncwarp();
            if (lane == 0) {
                tma_store_3d(&a.tmO, so, c0 + cur_noff, cur_tile * nb, mb * tstep + t_w);
                bulk_commit();
            }
            ++ob;
        };
        if (IDRES && lane == 0 && my_tiles > 0) res_load(0, tile_of(0), 0, slice_of(0) * N);
        // every warpgroup drains every tile (its N / 4 channels)
        if constexpr (EPI == EPI_PLAIN) {
            for (int j = 0; j < my_tiles; ++j) {
                cur_tile = tile_of(j);
                cur_noff = slice_of(j) * N;
                const float* s_bias = s_bias_all + cur_noff;
                const int buf = j % NBUF;
                const uint32_t t_lane0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * ACC + cbase);
                mbar_wait(&tfull[buf], (uint32_t)(j / NBUF) & 1u);
                tc_fence_after();
                if (!(a.dbg & 1)) {
#pragma unroll 1
                    for (int mb = 0; mb < MB; ++mb) {
                        const uint32_t t_lane = t_lane0 + (uint32_t)(mb * ACC1);
                        constexpr int PC = NC < 32 ? NC : 32;
#pragma unroll 1
                        for (int cc = 0; cc < NC; cc += PC) {
                            float v[PC];
                            if constexpr (PC == 32) {
                                tmem_ld32(t_lane + cc, v);
                            } else {
                                uint32_t rr[16];
                                tmem_ld16(t_lane + cc, rr);
                                tmem_wait_ld();
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(rr[jj]);
                            }
                            const int c0 = cbase + cc;
#pragma unroll
                            for (int h = 0; h < PC; h += 16) {
                                __align__(16) __nv_bfloat162 pk[8];
#pragma unroll
                                for (int u = 0; u < 8; ++u)
                                    pk[u] = __floats2bfloat162_rn(v[h + 2 * u] + s_bias[c0 + h + 2 * u],
                                                                  v[h + 2 * u + 1] + s_bias[c0 + h + 2 * u + 1]);
                                stage_store(pk, c0 + h, mb);
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR && !leader) mbar_arrive_remote(leader_addr(&tempty[buf]));
                    else mbar_arrive(&tempty[buf]);
                }
            }
        } else {
            // GroupNorm layers, software-pipelined by one tile (PIPE): the statistics of tile j + 1 (wait
            // for its accumulator, sums per (sample, group), time shuffles, the warp's partials and
            // the tile's FiLM rows to smem, an arrival on the warpgroup's barrier) run before the
            // normalise pass of tile j, so nobody waits on the slowest warp of a tile: by the time a
            // warp needs tile j's partials, a whole normalise pass has passed since they were
            // posted.  Partials are double-buffered (a warp writes tile j + 2's only after every warp
            // arrived for j + 1, i.e. read tile j's); staged FiLM rows, read in the normalise pass
            // after that arrival, are triple-buffered.  Same arithmetic and summation order as the
            // unpipelined epilogue.  (PS_TC_DBG bit 1 is ignored here.)
            uint64_t* gnb = gnbar + wg * 2;
            // pipelining holds two accumulator buffers in the epilogue: only with 4 buffers (with 2 the
            // MMAs of the next tile could not start before the normalise pass of this one ends)
            constexpr bool PIPE = PS_GN_PIPE && NBUF >= 4;
            // KEEP (unpipelined 16-channel slices): the biased accumulator values stay in registers
            // between the statistics and the normalise pass (one TMEM read per tile)
            constexpr bool KEEP = !PIPE && NC == 16;
            float kv[KEEP ? MB : 1][16];
            auto film_rows = [&](int tile_, int& plo, int& phi) {
                plo = div_s(a, tile_ * nb);
                phi = div_s(a, min(tile_ * nb + nb - 1, a.B - 1));
            };
            auto stats = [&](int jn) {
                const int tile_n = tile_of(jn);
                const int noff_n = slice_of(jn) * N;
                const int buf_n = jn % NBUF;
                const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf_n * ACC + cbase);
                const float* sb_n = s_bias_all + noff_n;
                // FiLM rows of the tile's problems: loaded (L2) before waiting for the accumulator
                float fpre[2] = {0.f, 0.f};
                int f_plo = 0, f_n = 0;
                if constexpr (EPI == EPI_GN_FILM) {
                    static_assert(TC_FILM_P * 2 * NC <= 256, "two FiLM values per thread");
                    int p_hi;
                    film_rows(tile_n, f_plo, p_hi);
                    if (p_hi - f_plo < TC_FILM_P) {
                        f_n = (p_hi - f_plo + 1) * 2 * NC;
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int i = r + 128 * u;
                            if (i < f_n) {
                                const int pp = i / (2 * NC), w = i % (2 * NC);
                                const int c = cbase + (w < NC ? w : w - NC);
                                const int col = a.film_col + noff_n + (w < NC ? c : NF + c);
                                fpre[u] = __ldg(a.film + (size_t)(f_plo + pp) * 3584 + col) + __ldg(a.film_b + col);
                            }
                        }
                    }
                }
                mbar_wait(&tfull[buf_n], (uint32_t)(jn / NBUF) & 1u);
                tc_fence_after();
                float s1[NG], s2[NG];
#pragma unroll
                for (int g = 0; g < NG; ++g) s1[g] = s2[g] = 0.f;
                constexpr int SC = NC < 32 ? NC : 32;   // stats chunk width
                // 16-channel slices: every M-block's accumulator row is loaded before one wait
                uint32_t rr_all[NC == 16 ? MB : 1][16];
                if constexpr (NC == 16) {
#pragma unroll
                    for (int mb = 0; mb < MB; ++mb) tmem_ld16(tl + (uint32_t)(mb * ACC1), rr_all[mb]);
                    tmem_wait_ld();
                }
#pragma unroll
                for (int mb = 0; mb < MB; ++mb)
#pragma unroll
                    for (int cc = 0; cc < NC; cc += SC) {
                        float v[SC];
                        if constexpr (SC == 32) {
                            tmem_ld32(tl + (uint32_t)(mb * ACC1) + cc, v);
                        } else if constexpr (NC == 16) {
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(rr_all[NC == 16 ? mb : 0][jj]);
                        } else {
                            uint32_t rr[16];
                            tmem_ld16(tl + (uint32_t)(mb * ACC1) + cc, rr);
                            tmem_wait_ld();
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(rr[jj]);
                        }
                        // packed: channel pairs (2c, 2c+1) share a group (CG >= 8)
                        float2 a1[NG], a2[NG];
#pragma unroll
                        for (int g = 0; g < NG; ++g) a1[g] = a2[g] = f2(0.f, 0.f);
#pragma unroll
                        for (int jj = 0; jj < SC; jj += 2) {
                            const int g = (cc + jj) / CG;
                            const float2 bb = *reinterpret_cast<const float2*>(sb_n + cbase + cc + jj);
                            const float2 xv = fadd2(f2(v[jj], v[jj + 1]), bb);
                            if constexpr (KEEP) {
                                kv[KEEP ? mb : 0][(cc + jj) & 15] = xv.x;
                                kv[KEEP ? mb : 0][(cc + jj + 1) & 15] = xv.y;
                            }
                            a1[g] = fadd2(a1[g], xv);
                            a2[g] = ffma2(xv, xv, a2[g]);
                        }
#pragma unroll
                        for (int g = 0; g < NG; ++g) {
                            s1[g] += a1[g].x + a1[g].y;
                            s2[g] += a2[g].x + a2[g].y;
                        }
                    }
                // rows of one sample share `sl` across all 4 warps (and both M-blocks); the summation
                // order depends on the tile shape, which run_layer chooses from the trajectory count
                // alone, so every batch on the same side of that threshold gives the same bits
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    if (off >= nb)
#pragma unroll
                        for (int g = 0; g < NG; ++g) {
                            s1[g] += __shfl_xor_sync(PS_FULL, s1[g], off);
                            s2[g] += __shfl_xor_sync(PS_FULL, s2[g], off);
                        }
                float* redj = red + (jn & 1) * (UT_EPI_WG * 4 * 32 * 2 * NG);
                if (lane < nb)
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        redj[(q * 32 + sl) * 2 * NG + g] = s1[g];
                        redj[(q * 32 + sl) * 2 * NG + NG + g] = s2[g];
                    }
                if constexpr (EPI == EPI_GN_FILM) {
                    float* sf = s_film + ((jn % 3) * UT_EPI_WG + wg) * (TC_FILM_P * 2 * NC);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int i = r + 128 * u;
                        if (i < f_n) {
                            const int pp = i / (2 * NC), w = i % (2 * NC);
                            sf[pp * 2 * NC + w] = w < NC ? 1.f + fpre[u] : fpre[u];
                        }
                    }
                }
                mbar_arrive(&gnb[jn & 1]);
            };
            if (PIPE && my_tiles > 0) stats(0);
            for (int j = 0; j < my_tiles; ++j) {
                if (!PIPE) stats(j);
                const int tile = tile_of(j);
                cur_tile = tile;
                cur_noff = slice_of(j) * N;
                // this item's channel slice of the per-channel vectors
                const float* s_bias = s_bias_all + cur_noff;
                const float* s_gamma = s_gamma_all + cur_noff;
                const float* s_beta = s_beta_all + cur_noff;
                const float* s_rbias = s_rbias_all + cur_noff;
                const int buf = j % NBUF;
                const int b = tile * nb + sl;
                const bool valid = b < a.B;
                const uint32_t t_lane0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * ACC + cbase);
                mbar_wait(&gnb[j & 1], (uint32_t)(j >> 1) & 1u);
                float mean[NG], rstd[NG];
                const float* redj = red + (j & 1) * (UT_EPI_WG * 4 * 32 * 2 * NG);
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    float a1 = 0.f, a2 = 0.f;
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        a1 += redj[(qq * 32 + sl) * 2 * NG + g];
                        a2 += redj[(qq * 32 + sl) * 2 * NG + NG + g];
                    }
                    mean[g] = a1 * inv_n;
                    rstd[g] = rsqrtf(fmaxf(fmaf(a2, inv_n, -mean[g] * mean[g]), 0.f) + 1e-5f);
                }
                if (PIPE && j + 1 < my_tiles) stats(j + 1);
                const int p = div_s(a, b);
                // per-tile FiLM rows staged as (1 + scale, shift) for this warpgroup's columns
                const float* fs1 = nullptr;
                const float* fsh = nullptr;
                if constexpr (EPI == EPI_GN_FILM) {
                    int p_lo, p_hi;
                    film_rows(tile, p_lo, p_hi);
                    if (p_hi - p_lo < TC_FILM_P) {
                        fs1 = s_film + ((j % 3) * UT_EPI_WG + wg) * (TC_FILM_P * 2 * NC) + (p - p_lo) * 2 * NC;
                        fsh = fs1 + NC;
                    }
                }
                float nmr[NG];
#pragma unroll
                for (int g = 0; g < NG; ++g) nmr[g] = -mean[g] * rstd[g];
                // no early-out on `valid`: tcgen05.ld is .sync.aligned and lanes of one warp
                // belong to different samples, so only global accesses are predicated
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    const uint32_t t_lane = t_lane0 + (uint32_t)(mb * ACC1);
#pragma unroll
                    for (int cc = 0; cc < NC; cc += 16) {
                        const int c0 = cbase + cc;
                        uint32_t rr[16], rq[16];
                        if constexpr (!KEEP) tmem_ld16(t_lane + cc, rr);
                        if constexpr (RES) tmem_ld16(t_lane + N + cc, rq);
                        if constexpr (!KEEP || RES) tmem_wait_ld();
                        const int gi = cc / CG;
                        const float rs = sel(rstd, gi), nm = sel(nmr, gi);
                        const float rs2 = CG < 16 ? sel(rstd, gi + 1) : rs;
                        const float nm2 = CG < 16 ? sel(nmr, gi + 1) : nm;
                        float y[16];
#pragma unroll
                        for (int jj = 0; jj < 16; jj += 4) {
                            const float4 bi = *reinterpret_cast<const float4*>(s_bias + c0 + jj);
                            const float4 ga = *reinterpret_cast<const float4*>(s_gamma + c0 + jj);
                            const float4 be = *reinterpret_cast<const float4*>(s_beta + c0 + jj);
                            // packed pairs: (jj, jj+1) and (jj+2, jj+3) lie in one group each
                            const bool hi = CG < 16 && jj >= CG;
                            const float2 rsv = hi ? f2(rs2, rs2) : f2(rs, rs), nmv = hi ? f2(nm2, nm2) : f2(nm, nm);
                            float2 x0, x1;
                            if constexpr (KEEP) {
                                x0 = f2(kv[KEEP ? mb : 0][jj], kv[KEEP ? mb : 0][jj + 1]);
                                x1 = f2(kv[KEEP ? mb : 0][jj + 2], kv[KEEP ? mb : 0][jj + 3]);
                            } else {
                                x0 = fadd2(f2(__uint_as_float(rr[jj]), __uint_as_float(rr[jj + 1])), f2(bi.x, bi.y));
                                x1 = fadd2(f2(__uint_as_float(rr[jj + 2]), __uint_as_float(rr[jj + 3])), f2(bi.z, bi.w));
                            }
                            const float2 z0 = ffma2(ffma2(x0, rsv, nmv), f2(ga.x, ga.y), f2(be.x, be.y));
                            const float2 z1 = ffma2(ffma2(x1, rsv, nmv), f2(ga.z, ga.w), f2(be.z, be.w));
                            const float2 y0 = mish2(z0), y1 = mish2(z1);
                            y[jj] = y0.x; y[jj + 1] = y0.y; y[jj + 2] = y1.x; y[jj + 3] = y1.y;
                        }
                        if constexpr (EPI == EPI_GN_FILM) {
                            if (fs1 && valid) {
#pragma unroll
                                for (int jj = 0; jj < 16; jj += 4) {
                                    const float4 m1 = *reinterpret_cast<const float4*>(fs1 + cc + jj);
                                    const float4 sh = *reinterpret_cast<const float4*>(fsh + cc + jj);
                                    const float2 u0 = ffma2(f2(y[jj], y[jj + 1]), f2(m1.x, m1.y), f2(sh.x, sh.y));
                                    const float2 u1 = ffma2(f2(y[jj + 2], y[jj + 3]), f2(m1.z, m1.w), f2(sh.z, sh.w));
                                    y[jj] = u0.x; y[jj + 1] = u0.y; y[jj + 2] = u1.x; y[jj + 3] = u1.y;
                                }
                            } else if (valid) {
                                const float* fr = a.film + (size_t)p * 3584 + a.film_col + cur_noff;
                                const float* fq = a.film_b + a.film_col + cur_noff;
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj)
                                    y[jj] = fmaf(y[jj], 1.f + (__ldg(fr + c0 + jj) + __ldg(fq + c0 + jj)),
                                                 __ldg(fr + NF + c0 + jj) + __ldg(fq + NF + c0 + jj));
                            }
                        } else if constexpr (RES) {
                            // packed, with 16-B loads of the projection bias (4 LDS wavefronts per 16
                            // channels instead of 16)
#pragma unroll
                            for (int jj = 0; jj < 16; jj += 4) {
                                const float4 rb = *reinterpret_cast<const float4*>(s_rbias + c0 + jj);
                                const float2 u0 = fadd2(f2(y[jj], y[jj + 1]),
                                                        fadd2(f2(__uint_as_float(rq[jj]), __uint_as_float(rq[jj + 1])), f2(rb.x, rb.y)));
                                const float2 u1 = fadd2(f2(y[jj + 2], y[jj + 3]),
                                                        fadd2(f2(__uint_as_float(rq[jj + 2]), __uint_as_float(rq[jj + 3])), f2(rb.z, rb.w)));
                                y[jj] = u0.x; y[jj + 1] = u0.y; y[jj + 2] = u1.x; y[jj + 3] = u1.y;
                            }
                        } else {
                            stage_store_res(y, c0, mb, j, mb * (NC / 16) + cc / 16);
                            continue;
                        }
                        __align__(16) __nv_bfloat162 pk[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) pk[u] = __floats2bfloat162_rn(y[2 * u], y[2 * u + 1]);
                        stage_store(pk, c0, mb);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR && !leader) mbar_arrive_remote(leader_addr(&tempty[buf]));
                    else mbar_arrive(&tempty[buf]);
                }
            }
        }
        if (!FIN && lane == 0) bulk_wait0();   // output stores complete before the grid ends
    }
    __syncthreads();
    if constexpr (PAIR) {
        cluster_sync_all();   // the pair's MMAs, remote arrivals and TMA completions are done
        if (warp == 1) {
            tc_fence_after();
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NCOLS));
        }
    } else if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NCOLS));
    }
}

// activation view [B][Tv][C] bf16 read in (time, sample) order: dims (C, B, Tv), box {64, nb, Tv+4}
bool make_ts_map(CUtensorMap* tm, const void* base, int B, int Tv, int C, int nb) {
    cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)B, (cuuint64_t)Tv};
    cuuint64_t strides[2] = {(cuuint64_t)Tv * C * 2, (cuuint64_t)C * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)nb, (cuuint32_t)(Tv + 4)};
    cuuint32_t es[3] = {1, 1, 1};
    return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// output [B][Tv][N] bf16 written in (time, sample)-ordered 16-channel slabs: box {16, nb, 32/nb}
static bool make_out_map(CUtensorMap* tm, void* base, int B, int Tv, int N, int nb) {
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)B, (cuuint64_t)Tv};
    cuuint64_t strides[2] = {(cuuint64_t)Tv * N * 2, (cuuint64_t)N * 2};
    cuuint32_t box[3] = {16, (cuuint32_t)nb, (cuuint32_t)(32 / nb)};   // one epilogue warp's 32 rows
    cuuint32_t es[3] = {1, 1, 1};
    return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bf16 state view [B][Tv][8] in (time, sample) order, no swizzle: box {8, nb, Tv+5}
// (time shifts -2..+3: the MMA pairing taps 2/3 also reads the zero-weight shift +3, whose
// rows must be zero-filled by TMA, not stale shared memory -- NaN * 0 = NaN)
bool make_xb_map(CUtensorMap* tm, const void* base, int B, int Tv, int nb) {
    cuuint64_t dims[3] = {8, (cuuint64_t)B, (cuuint64_t)Tv};
    cuuint64_t strides[2] = {(cuuint64_t)Tv * 16, 16};
    cuuint32_t box[3] = {8, (cuuint32_t)nb, (cuuint32_t)(Tv + 5)};
    cuuint32_t es[3] = {1, 1, 1};
    return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N, int EPI, bool RES, int MB, bool PAIR, int SPLIT>
static int launch_ut(UtArgs& a, cudaStream_t st) {
    const int A_BYTES = (a.Tv + 4) * a.nb * 128;
    constexpr int B_BYTES = PAIR ? N * 64 : N * 128;
    // the kernel's shared layout (unet_tc_kernel): per-channel vectors, w_out, GN partials,
    // staged FiLM, tap tables
    constexpr int NSPLIT_ = UT_EPI_WG;
    constexpr int NG_ = 8 / (SPLIT * NSPLIT_), NC_ = N / NSPLIT_;
    const size_t vec = (size_t)(4 * N * SPLIT + 7 * 64 + ut_red_floats<EPI, NG_>() + 3 * UT_EPI_WG * TC_FILM_P * 2 * NC_) * 4 +
                       UT_MAXG * sizeof(UtGroup) + UT_MAXTAP * sizeof(UtTap) + 64;
    const size_t fin = EPI == EPI_FINAL ? UT_EPI_WG * (16384 + 128 * U_DOF * 4) + 2048 : (size_t)UT_EPI_WG * 2 * 4096;
    const size_t budget = 225 * 1024 - vec - 2048 - fin;
    a.sa_stages = 3 * (size_t)A_BYTES <= 110 * 1024 ? 3 : 2;
    const int sb_fit = (int)((budget - (size_t)a.sa_stages * A_BYTES) / B_BYTES);
    // small layers keep all their weights resident (one box per tap), the rest stream them
    a.resident = (SPLIT == 1 && a.n_tap <= std::min(sb_fit, 12)) ? 1 : 0;   // one slice per kernel only
    static const bool no_res = std::getenv("PS_NO_RESIDENT") != nullptr;
    if (no_res) a.resident = 0;
    if (a.resident) {   // spend the smem the weight ring no longer needs on activation stages
        a.sb_stages = a.n_tap;
        a.sa_stages = (int)std::max<size_t>(a.sa_stages, std::min<size_t>(4, (budget - (size_t)a.n_tap * B_BYTES) / A_BYTES));
    } else {            // streamed weights: two activation stages, as deep a weight ring as fits, then a third A stage
        a.sa_stages = 2;
        a.sb_stages = (int)std::min<size_t>(8, (budget - 2 * (size_t)A_BYTES) / B_BYTES);
        if (a.sb_stages >= 4 && budget >= 3 * (size_t)A_BYTES + (size_t)a.sb_stages * B_BYTES) a.sa_stages = 3;
    }
    if (a.sb_stages < 2 && !a.resident) return PS_FAIL(PS_ERR_SHAPE);
    const size_t smem = 1024 + (size_t)a.sa_stages * A_BYTES + (size_t)a.sb_stages * B_BYTES + fin +
                        (2 * (a.sa_stages + a.sb_stages) + 20 + 10 * UT_EPI_WG) * 8 + 16 + vec;
    auto kern = unet_tc_kernel<N, EPI, RES, MB, PAIR, SPLIT>;
    static int set_bytes = 0;
    if ((int)smem > set_bytes) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return PS_FAIL(PS_ERR_CUDA);
        set_bytes = (int)smem;
    }
    static const int dbg = std::getenv("PS_TC_DBG") ? std::atoi(std::getenv("PS_TC_DBG")) : 0;
    a.dbg = dbg;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int n_tiles = (a.B + a.nb - 1) / a.nb;
    const int n_units = (PAIR ? (n_tiles + 1) / 2 : n_tiles) * SPLIT;
    const int units = n_units < (PAIR ? n_sm / 2 : n_sm) ? n_units : (PAIR ? n_sm / 2 : n_sm);
    const int grid = PAIR ? 2 * units : units;
    static const bool trace = std::getenv("PS_DEBUG") && std::atoi(std::getenv("PS_DEBUG")) >= 2;
    if (trace) std::fprintf(stderr, "[ps_b200] unet_tc N=%d EPI=%d RES=%d MB=%d B=%d Tv=%d nb=%d grid=%d groups=%d taps=%d\n",
                            N, EPI, (int)RES, MB, a.B, a.Tv, a.nb, grid, a.n_grp, a.n_tap);
    {
        const int e_ = PAIR ? launch_pdl_pair(kern, dim3(grid), dim3(UT_THREADS), smem, st, a)
                            : launch_pdl(kern, dim3(grid), dim3(UT_THREADS), smem, st, a);
        if (e_) return e_;
    }
    if (trace && cudaStreamSynchronize(st) != cudaSuccess) return PS_FAIL(PS_ERR_CUDA);
    return PS_OK;
}


static int run_layer(const Layout& L, const char* packed, const TcLayer& ly, int B, int S, const float* film,
                     const float* film_b, float* x, __nv_bfloat16* xb_next, const TcStep* step, float* eps_out,
                     cudaStream_t st) {
    UtArgs a;
    memset(&a, 0, sizeof(a));
    const PConv& c = *ly.c;
    const int N = c.N;
    const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(packed);
    // two M-blocks per tile where the TMEM budget still allows double buffering
    // two M-blocks per tile where the TMEM budget allows double buffering, unless the batch is
    // too small to give every SM a tile (small batches are latency-bound: more, smaller tiles)
    static int n_sm_rl = 0;
    if (!n_sm_rl) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm_rl, cudaDevAttrMultiProcessorCount, dev);
    }
    // Two M-blocks per tile (each weight stage feeds 8 MMAs) unless the batch is too small to give
    // every SM a two-block tile at the full horizon.  The choice depends on the trajectory count
    // only (not on the layer's level), so any two batches on the same side of the threshold
    // (B * 32 rows vs 256 x #SM) tile every layer alike and give the same bits per trajectory.
    const bool small = (long long)B * 32 < 256LL * n_sm_rl;
    const int MBv = (!small && ly.epi != EPI_FINAL && (N == 64 || (N == 128 && !ly.res))) ? 2 : 1;
    const int nb = MBv * 128 / ly.Tv;
    for (int s = 0; s < 3; ++s)
        // maps span >= nb samples (the workspace is padded to TC_MIN_B): a TMA box larger than
        // the tensor extent never completes its transaction
        if (ly.src[s] && !(s == ly.xb_src ? make_xb_map(&a.tmA[s], ly.src[s], std::max(B, nb), ly.Tv, nb)
                                          : make_ts_map(&a.tmA[s], ly.src[s], std::max(B, nb), ly.Tv, ly.ld[s], nb)))
            return PS_FAIL(PS_ERR_CUDA);
    // CTA pairs for the weight-heavy layers (K >= 1024; PS_NO_PAIR=1 disables): each CTA loads half of
    // every weight box and the leader issues M = 256 MMAs over both CTAs
    static const bool no_pair = std::getenv("PS_NO_PAIR") != nullptr;
    const int k_total = c.K + (ly.res ? ly.res->K : 0);
    // (never for the 8-channel state view: its 16-B-row boxes have no CTA-pair load path)
    static const int pair_k = std::getenv("PS_PAIR_K") ? std::atoi(std::getenv("PS_PAIR_K")) : 1024;   // A/B knob
    const bool pair = !no_pair && k_total >= pair_k && ly.epi != EPI_FINAL && ly.xb_src < 0;   // weight-heavy layers
    // small batches: N-split the N >= 128 layers into two channel slices (whole GroupNorm
    // groups), doubling the CTAs per tile and halving each CTA's weight stream and MMA chain
    static const bool no_split = std::getenv("PS_NO_SPLIT") != nullptr;
    const bool tiny = 2LL * ((long long)B * ly.Tv + 127) / 128 <= n_sm_rl;   // both slices still fit on the SMs
    const int split = (!no_split && tiny && N >= 128 && ly.epi != EPI_FINAL) ? 2 : 1;
    const int wrows = N / split / (pair ? 2 : 1);
    if (!make_w_map(&a.tmW, W + c.w_off, N, (int)kpad(c.K), wrows)) return PS_FAIL(PS_ERR_CUDA);
    if (ly.epi != EPI_FINAL && !make_out_map(&a.tmO, ly.out, std::max(B, nb), ly.Tv, N, nb))
        return PS_FAIL(PS_ERR_CUDA);
    if (ly.res_src && !make_out_map(&a.tmRes, const_cast<__nv_bfloat16*>(ly.res_src), std::max(B, nb), ly.Tv, N, nb))
        return PS_FAIL(PS_ERR_CUDA);
    if (ly.res && !make_w_map(&a.tmR, W + ly.res->w_off, N, (int)kpad(ly.res->K), wrows))
        return PS_FAIL(PS_ERR_CUDA);
    // group taps by the activation chunk they read: (src, channel offset)
    struct Tmp { int src, c; std::vector<UtTap> taps; };
    std::vector<Tmp> groups;
    bool first_main = true, first_res = true;
    auto add = [&](const PConv& cc, int res, int shift) {
        for (int i = 0; i < cc.n_seg; ++i) {
            const PSeg& sg = cc.seg[i];
            for (int j = 0; j < sg.nc; j += 64) {
                const int src = sg.src + shift, ch = sg.c0 + j;
                Tmp* gp = nullptr;
                for (auto& g : groups)
                    if (g.src == src && g.c == ch) gp = &g;
                if (!gp) {
                    groups.push_back(Tmp{src, ch, {}});
                    gp = &groups.back();
                }
                UtTap tp;
                tp.kcol = (int16_t)(sg.k0 + j);
                tp.dt = (int8_t)sg.dt;
                tp.res = (int8_t)res;
                tp.first = 0;
                gp->taps.push_back(tp);
            }
        }
    };
    add(c, 0, 0);
    if (ly.res) add(*ly.res, 1, ly.res_shift);
    if ((int)groups.size() > UT_MAXG) return PS_FAIL(PS_ERR_SHAPE);
    int nt = 0;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        UtGroup& g = a.grp[gi];
        g.c = (int16_t)groups[gi].c;
        g.src = (int8_t)groups[gi].src;
        g.ntap = (int8_t)groups[gi].taps.size();
        g.tap0 = (int16_t)nt;
        g.xb = (int8_t)(groups[gi].src == ly.xb_src ? 1 : 0);
        for (auto tp : groups[gi].taps) {
            if (nt >= UT_MAXTAP) return PS_FAIL(PS_ERR_SHAPE);
            bool& f = tp.res ? first_res : first_main;
            tp.first = f ? 1 : 0;
            f = false;
            a.tap[nt++] = tp;
        }
    }
    a.n_grp = (int)groups.size();
    a.n_tap = nt;
    a.B = B;
    a.Tv = ly.Tv;
    a.nb = nb;
    a.S = S;
    a.s_magic = ((1ull << 40) + (unsigned long long)S - 1) / (unsigned long long)S;
    const float* side = L.side(packed);
    a.bias = side + c.b_off;
    if (c.g_off >= 0) {
        a.gamma = side + c.g_off;
        a.beta = side + c.be_off;
    }
    if (ly.res) a.rbias = side + ly.res->b_off;
    a.res_src = ly.res_src;
    a.film = film;
    a.film_b = film_b;
    a.film_col = c.film_col;
    a.out = ly.out;
    if (ly.epi == EPI_FINAL) {
        a.wout = side + L.outw_f32;
        a.bout = side + L.out.b_off;
        a.x = x;
        a.xb_next = xb_next;
        a.eps_out = eps_out;
        if (step) {
            a.sc = step->sc;
            a.p0 = step->p0;
            a.key = step->key;
            a.q_start = step->q_start;
            a.traj = step->traj;
            a.lo = step->lo;
            a.hi = step->hi;
        }
        return launch_ut<64, EPI_FINAL, false, 1, false, 1>(a, st);
    }
#define PS_LAUNCH4(NN, MBR, MBN, PR, SP)                                                               \
    {                                                                                                  \
        if (ly.epi == EPI_PLAIN) return launch_ut<NN / SP, EPI_PLAIN, false, MBN, PR, SP>(a, st);       \
        if (ly.epi == EPI_GN_FILM) return launch_ut<NN / SP, EPI_GN_FILM, false, MBN, PR, SP>(a, st);   \
        if (ly.res) return launch_ut<NN / SP, EPI_GN_RES, true, MBR, PR, SP>(a, st);                    \
        return launch_ut<NN / SP, EPI_GN_RES, false, MBN, PR, SP>(a, st);                               \
    }
#define PS_DISPATCH(NN, MBR, MBN)                                                                      \
    if (N == NN) {                                                                                     \
        if (MBv == 1) {                                                                                \
            if (split == 2) {                                                                          \
                if (pair) PS_LAUNCH4(NN, 1, 1, true, 2)                                                \
                PS_LAUNCH4(NN, 1, 1, false, 2)                                                         \
            }                                                                                          \
            if (pair) PS_LAUNCH4(NN, 1, 1, true, 1)                                                    \
            PS_LAUNCH4(NN, 1, 1, false, 1)                                                             \
        }                                                                                              \
        if (pair) PS_LAUNCH4(NN, MBR, MBN, true, 1)                                                    \
        PS_LAUNCH4(NN, MBR, MBN, false, 1)                                                             \
    }
    PS_DISPATCH(64, 2, 2)
    PS_DISPATCH(128, 1, 2)
    PS_DISPATCH(256, 1, 1)
#undef PS_DISPATCH
#undef PS_LAUNCH4
    return PS_FAIL(PS_ERR_SHAPE);
}

constexpr int TC_MIN_B = 64;   // activation slots are padded to at least this many samples

size_t tc_workspace_bytes(int B, int T) {
    const size_t Bp = (size_t)std::max(B, TC_MIN_B);
    const size_t slot = Bp * T * 128 * 2;
    return Bp * T * 64 * 2 + 5 * slot + (size_t)B * 3584 * 4 + 4096;
}

#define PS_TRY_TC(x)        \
    do {                    \
        int s_ = (x);       \
        if (s_) return s_;  \
    } while (0)

UnetSlots unet_slots(void* ws, int B, int T) {
    const size_t Bp = (size_t)std::max(B, TC_MIN_B);
    const size_t slot = Bp * T * 128;
    UnetSlots u;
    u.a0 = reinterpret_cast<__nv_bfloat16*>(ws);
    u.cur = u.a0 + Bp * T * 64;
    u.nxt = u.cur + slot;
    u.h = u.nxt + slot;
    u.skip1 = u.h + slot;
    u.skip2 = u.skip1 + slot;
    u.film = reinterpret_cast<float*>(u.skip2 + slot);
    return u;
}

// The forward's 29 (30 with split_res256) layers in execution order.  split_res256: the
// 256-wide residual projection of d2r0 runs as its own 1x1 conv into a free slot (the
// layered kernels would otherwise need 512 TMEM columns for c1); the persistent small-batch
// kernel keeps it fused.
void unet_layer_list(const Layout& L, int T, const UnetSlots& u, bool split_res256, std::vector<TcLayer>& out) {
    out.clear();
    auto block = [&](int bi, const __nv_bfloat16* in0, int ld0, const __nv_bfloat16* in1, int ld1,
                     __nv_bfloat16* dst, __nv_bfloat16* res_tmp = nullptr) {
        const PBlock& bk = L.blk[bi];
        const int Tv = T >> bk.level;
        TcLayer l0{};
        l0.c = &bk.c0;
        l0.epi = EPI_GN_FILM;
        l0.src[0] = in0; l0.ld[0] = ld0;
        l0.src[1] = in1; l0.ld[1] = ld1;
        l0.Tv = Tv;
        l0.out = u.h;
        if (bi == 0) l0.xb_src = 0;
        out.push_back(l0);
        TcLayer l1{};
        l1.c = &bk.c1;
        l1.epi = EPI_GN_RES;
        l1.src[0] = u.h; l1.ld[0] = bk.c_out;
        l1.Tv = Tv;
        l1.out = dst;
        if (bk.res.K && bk.c_out == 256 && !in1 && res_tmp && split_res256) {
            TcLayer lr{};
            lr.c = &bk.res;
            lr.epi = EPI_PLAIN;
            lr.src[0] = in0; lr.ld[0] = ld0;
            lr.Tv = Tv;
            lr.out = res_tmp;
            out.push_back(lr);
            l1.res_src = res_tmp;
        } else if (bk.res.K) {
            l1.res = &bk.res;
            l1.res_shift = 1;
            l1.src[1] = in0; l1.ld[1] = ld0;
            l1.src[2] = in1; l1.ld[2] = ld1;
            if (bi == 0) l1.xb_src = 1;
        } else {
            l1.res_src = in0;
        }
        out.push_back(l1);
    };
    auto plain = [&](const PConv& c, const __nv_bfloat16* in, int ld, int Tv, __nv_bfloat16* dst) {
        TcLayer l{};
        l.c = &c;
        l.epi = EPI_PLAIN;
        l.src[0] = in; l.ld[0] = ld;
        l.Tv = Tv;
        l.out = dst;
        out.push_back(l);
    };
    block(0, u.a0, 64, nullptr, 0, u.cur);
    block(1, u.cur, 64, nullptr, 0, u.nxt);
    plain(L.down[0], u.nxt, 128, T / 2, u.cur);            // pair view [B, T/2, 128]
    block(2, u.cur, 64, nullptr, 0, u.nxt);
    block(3, u.nxt, 128, nullptr, 0, u.skip1);
    plain(L.down[1], u.skip1, 256, T / 4, u.cur);          // pair view [B, T/4, 256]
    block(4, u.cur, 128, nullptr, 0, u.nxt, u.skip2);   // skip2 is free until block 5 writes it
    block(5, u.nxt, 256, nullptr, 0, u.skip2);
    block(6, u.skip2, 256, nullptr, 0, u.cur);
    block(7, u.cur, 256, nullptr, 0, u.nxt);
    block(8, u.nxt, 256, u.skip2, 256, u.cur);
    block(9, u.cur, 128, nullptr, 0, u.nxt);
    plain(L.up[0], u.nxt, 128, T / 4, u.cur);              // writes pair view [B, T/4, 256]
    block(10, u.cur, 128, u.skip1, 128, u.nxt);
    block(11, u.nxt, 64, nullptr, 0, u.cur);
    plain(L.up[1], u.cur, 64, T / 2, u.nxt);               // writes pair view [B, T/2, 128]
    TcLayer lf{};
    lf.c = &L.fin;
    lf.epi = EPI_FINAL;
    lf.src[0] = u.nxt; lf.ld[0] = 64;
    lf.Tv = T;
    out.push_back(lf);
}

int tc_xb(const float* x, size_t rows, __nv_bfloat16* xb, cudaStream_t st) {
    xb_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(x, rows, xb);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

int unet_eval_tc(const Layout& L, const char* packed, float* x, int B, int T, int S, const float* film_a,
                 const float* film_b_row, float* ws, float* eps, const TcStep* step, cudaStream_t st) {
    if (!get_encoder()) return PS_FAIL(PS_ERR_CUDA);
    if (L.mode != 1) return PS_FAIL(PS_ERR_SHAPE);
    const UnetSlots u = unet_slots(ws, B, T);
    // the FiLM layers add this step's per-step part to the per-problem rows as they stage them; the
    // state's bf16 view comes from the previous step's FINAL epilogue when the caller says so
    static const bool no_fuse = std::getenv("PS_NO_XB_FUSE") != nullptr;   // A/B knob
    if (!step || !step->xb_ready || no_fuse) PS_TRY_TC(tc_xb(x, (size_t)B * T, u.a0, st));
    std::vector<TcLayer> layers;
    unet_layer_list(L, T, u, true, layers);
    for (const TcLayer& ly : layers) {
        const bool fin = ly.epi == EPI_FINAL;
        PS_TRY_TC(run_layer(L, packed, ly, B, S, film_a, film_b_row, x, fin && step && !no_fuse ? u.a0 : nullptr,
                            fin ? step : nullptr, fin && !step ? eps : nullptr, st));
    }
    return PS_OK;
}

// ===========================================================================
// Observation encoder on tcgen05: conv3x3 stride 2 pad 1 + ReLU as a segment GEMM
// over the 5-D pair view [img][H/2][2][W/2][2C] of an NHWC bf16 activation.
//   out[y][x] = sum_dy ( in[2y+dy-1][2x-1] W[.,.,dy,0] + in[2y+dy-1][2x..2x+1] W[.,.,dy,1..2] )
// row 2y+dy-1 -> (pair y-1, parity 1) | (y, 0) | (y, 1); column pair x-1 (odd pixel)
// and x (both pixels).  TMA zero-fills the top/left padding.
// ===========================================================================
constexpr int ENC_MAXL = 5;
static const int ENC_CH[ENC_MAXL] = {32, 64, 128, 256, 256};

struct EncLayerGeo {
    int C, N;            // in / out channels
    int Hin, Win, Hin_p; // input (Hin_p even, padded)
    int Ho, Wo, Ho_p;    // output (Ho_p even for the next layer's pair view)
    int wx, ry, tiles_x, tiles_y;
    int n_chunks;
    size_t w_off;        // bf16 offset in the packed encoder buffer
    size_t b_off;        // fp32 bias offset in the side table (elements)
};

static void enc_geometry(int H, int W, int n_layers, EncLayerGeo* g) {
    int h = H, w = W, c = 1;
    size_t woff = 0, boff = 0;
    for (int l = 0; l < n_layers; ++l) {
        EncLayerGeo& e = g[l];
        e.C = c;
        e.N = ENC_CH[l];
        e.Hin = h;
        e.Win = w;
        e.Hin_p = h + (h & 1);
        e.Ho = (h - 1) / 2 + 1;
        e.Wo = (w - 1) / 2 + 1;
        e.Ho_p = e.Ho + (e.Ho & 1);
        // tile shape: wx x ry = 128 minimising padding waste
        int best_wx = 8;
        double best = 1e30;
        for (int wx = 4; wx <= 128; wx *= 2) {
            const int ry = 128 / wx;
            const double cover = (double)((e.Wo + wx - 1) / wx * wx) * ((e.Ho + ry - 1) / ry * ry);
            if (cover < best - 1e-9) {
                best = cover;
                best_wx = wx;
            }
        }
        e.wx = best_wx;
        e.ry = 128 / best_wx;
        e.tiles_x = (e.Wo + e.wx - 1) / e.wx;
        e.tiles_y = (e.Ho + e.ry - 1) / e.ry;
        const int segA = c == 32 ? 1 : c / 64, segB = 2 * c / 64;
        e.n_chunks = l == 0 ? 0 : 3 * (segA + segB);
        e.w_off = woff;
        if (l > 0) woff += (size_t)e.N * e.n_chunks * 64;
        e.b_off = boff;
        boff += e.N;
        h = e.Ho;
        w = e.Wo;
        c = e.N;
    }
}

extern "C" long long ps_encoder_packed_bytes(int H, int W, int n_layers) {
    if (n_layers < 2 || n_layers > ENC_MAXL) return -1;
    EncLayerGeo g[ENC_MAXL];
    enc_geometry(H, W, n_layers, g);
    const EncLayerGeo& last = g[n_layers - 1];
    const size_t wb = (last.w_off + (size_t)last.N * last.n_chunks * 64) * 2;
    size_t side = 0;
    for (int l = 0; l < n_layers; ++l) side += g[l].N;
    side += 32 * 9;  // layer-1 weights (fp32)
    return (long long)(((wb + 255) / 256) * 256 + side * 4);
}

// blob: encoder params in table order (fp32, device).  Layer 1 stays fp32 (SIMT);
// layers 2.. are packed bf16 [N][chunks*64] in chunk order.
extern "C" int ps_encoder_pack(const float* blob, int H, int W, int n_layers, void* packed, void* stream) {
    if (n_layers < 2 || n_layers > ENC_MAXL) return PS_FAIL(PS_ERR_SHAPE);
    EncLayerGeo g[ENC_MAXL];
    enc_geometry(H, W, n_layers, g);
    // blob offsets
    size_t boff[ENC_MAXL], woff_blob[ENC_MAXL], o = 0;
    for (int l = 0; l < n_layers; ++l) {
        woff_blob[l] = o;
        o += (size_t)g[l].N * g[l].C * 9;
        boff[l] = o;
        o += g[l].N;
    }
    std::vector<long long> wsrc, ssrc;
    for (int l = 1; l < n_layers; ++l) {
        const EncLayerGeo& e = g[l];
        const int C = e.C;
        // chunk list (same order as the launcher): dy -> segA chunks -> segB chunks
        for (int n = 0; n < e.N; ++n) {
            for (int dy = 0; dy < 3; ++dy) {
                const int segA = C == 32 ? 1 : C / 64;
                for (int ci = 0; ci < segA; ++ci)
                    for (int k = 0; k < 64; ++k) {
                        // pair x-1: channel index within the pair = (C==32 ? k : C + 64ci + k); odd pixel
                        const int pc = C == 32 ? k : C + 64 * ci + k;
                        if (pc < C) {
                            wsrc.push_back(-1);
                            continue;
                        }
                        const int c = pc - C;
                        wsrc.push_back((long long)(woff_blob[l] + (((size_t)n * C + c) * 3 + dy) * 3 + 0));
                    }
                for (int ci = 0; ci < 2 * C / 64; ++ci)
                    for (int k = 0; k < 64; ++k) {
                        const int pc = 64 * ci + k;  // pair x: even pixel c (dx=1), odd pixel c (dx=2)
                        const int dx = pc < C ? 1 : 2, c = pc < C ? pc : pc - C;
                        wsrc.push_back((long long)(woff_blob[l] + (((size_t)n * C + c) * 3 + dy) * 3 + dx));
                    }
            }
        }
    }
    for (int l = 0; l < n_layers; ++l)
        for (int n = 0; n < g[l].N; ++n) ssrc.push_back((long long)(boff[l] + n));
    for (int i = 0; i < 32 * 9; ++i) ssrc.push_back((long long)(woff_blob[0] + i));
    const EncLayerGeo& last = g[n_layers - 1];
    const size_t wb = ((last.w_off + (size_t)last.N * last.n_chunks * 64) * 2 + 255) / 256 * 256;
    if (wsrc.size() * 2 > wb) return PS_FAIL(PS_ERR_SHAPE);
    cudaStream_t st = (cudaStream_t)stream;
    long long* d_idx = nullptr;
    const size_t nmax = std::max(wsrc.size(), ssrc.size());
    if (cudaMallocAsync(&d_idx, nmax * sizeof(long long), st) != cudaSuccess) return PS_FAIL(PS_ERR_CUDA);
    cudaMemcpyAsync(d_idx, wsrc.data(), wsrc.size() * sizeof(long long), cudaMemcpyHostToDevice, st);
    gather_bf16_kernel<<<(unsigned)((wsrc.size() + 255) / 256), 256, 0, st>>>(
        blob, d_idx, wsrc.size(), reinterpret_cast<__nv_bfloat16*>(packed));
    PS_CHECK_LAUNCH();
    if (cudaStreamSynchronize(st) != cudaSuccess) return PS_FAIL(PS_ERR_CUDA);
    cudaMemcpyAsync(d_idx, ssrc.data(), ssrc.size() * sizeof(long long), cudaMemcpyHostToDevice, st);
    gather_f32_kernel<<<(unsigned)((ssrc.size() + 255) / 256), 256, 0, st>>>(
        blob, d_idx, ssrc.size(), reinterpret_cast<float*>(reinterpret_cast<char*>(packed) + wb));
    PS_CHECK_LAUNCH();
    if (cudaStreamSynchronize(st) != cudaSuccess) return PS_FAIL(PS_ERR_CUDA);
    cudaFreeAsync(d_idx, st);
    return PS_OK;
}

// layer 1 (1 -> 32 channels) in fp32 SIMT: one output pixel x 32 channels per thread,
// input depth scaled by 1/2 (spec.DEPTH_SCALE), NHWC bf16 output with even-padded rows.
// Two horizontally adjacent output pixels per thread: the weights sit in shared memory as
// [tap][32 channels], so one 16-B broadcast load feeds 8 FMAs (4 channels x 2 pixels) instead of
// one load per FMA; the FMA order per output is unchanged (bias, then taps dy-major).
__global__ void enc_l1_kernel(const float* __restrict__ img, int n_img, int H, int W, const float* __restrict__ w,
                              const float* __restrict__ bias, int Ho, int Wo, int Ho_p,
                              __nv_bfloat16* __restrict__ out) {
    __shared__ __align__(16) float sw[9 * 32];
    __shared__ __align__(16) float sb[32];
    for (int i = threadIdx.x; i < 32 * 9; i += blockDim.x) sw[(i % 9) * 32 + i / 9] = w[i];   // w: [o][tap]
    for (int i = threadIdx.x; i < 32; i += blockDim.x) sb[i] = bias[i];
    __syncthreads();
    const int Wp = (Wo + 1) / 2;   // pixel pairs per row
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t n = (size_t)n_img * Ho_p * Wp;
    if (idx >= n) return;
    const int xp = (int)(idx % Wp), y = (int)((idx / Wp) % Ho_p), m = (int)(idx / ((size_t)Wp * Ho_p));
    const int x0 = 2 * xp;
    const bool has1 = x0 + 1 < Wo;
    float a0[32], a1[32];
#pragma unroll
    for (int o = 0; o < 32; o += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(sb + o);
        a0[o] = a1[o] = b4.x; a0[o + 1] = a1[o + 1] = b4.y; a0[o + 2] = a1[o + 2] = b4.z; a0[o + 3] = a1[o + 3] = b4.w;
    }
    if (y < Ho) {
        const float* ib = img + (size_t)m * H * W;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
            const int yy = 2 * y + dy - 1;
            const bool rowok = yy >= 0 && yy < H;
            // input columns 2 x0 - 1 .. 2 x0 + 3 cover both pixels' 3 taps
            float v[5];
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                const int xx = 2 * x0 - 1 + c;
                v[c] = (rowok && xx >= 0 && xx < W) ? ib[(size_t)yy * W + xx] * 0.5f : 0.f;
            }
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                const float* wt = sw + (dy * 3 + dx) * 32;
                const float p0 = v[dx], p1 = v[dx + 2];
#pragma unroll
                for (int o = 0; o < 32; o += 4) {
                    const float4 w4 = *reinterpret_cast<const float4*>(wt + o);
                    a0[o] = fmaf(p0, w4.x, a0[o]); a0[o + 1] = fmaf(p0, w4.y, a0[o + 1]);
                    a0[o + 2] = fmaf(p0, w4.z, a0[o + 2]); a0[o + 3] = fmaf(p0, w4.w, a0[o + 3]);
                    a1[o] = fmaf(p1, w4.x, a1[o]); a1[o + 1] = fmaf(p1, w4.y, a1[o + 1]);
                    a1[o + 2] = fmaf(p1, w4.z, a1[o + 2]); a1[o + 3] = fmaf(p1, w4.w, a1[o + 3]);
                }
            }
        }
    }
    const size_t pix = ((size_t)m * Ho_p + y) * Wo + x0;
    __align__(16) __nv_bfloat162 pk[16];
#pragma unroll
    for (int o = 0; o < 16; ++o)
        pk[o] = y < Ho ? __floats2bfloat162_rn(fmaxf(a0[2 * o], 0.f), fmaxf(a0[2 * o + 1], 0.f))
                       : __floats2bfloat162_rn(0.f, 0.f);
    uint4* dst = reinterpret_cast<uint4*>(out + pix * 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = reinterpret_cast<uint4*>(pk)[i];
    if (has1) {
#pragma unroll
        for (int o = 0; o < 16; ++o)
            pk[o] = y < Ho ? __floats2bfloat162_rn(fmaxf(a1[2 * o], 0.f), fmaxf(a1[2 * o + 1], 0.f))
                           : __floats2bfloat162_rn(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[4 + i] = reinterpret_cast<uint4*>(pk)[i];
    }
}

// global average pool of the last layer (NHWC bf16) averaged over each problem's images,
// then the condition vector [emb ; (q-lo)/(hi-lo) ; goal xyz/0.6 ; quat]
__global__ void enc_gap_cond_kernel(const __nv_bfloat16* __restrict__ feat, int n_img, int Ho, int Ho_p, int Wo,
                                    const float* __restrict__ q, const float* __restrict__ goal, float lo, float hi,
                                    float* __restrict__ cond) {
    const int p = blockIdx.x, c = threadIdx.x;  // 256 threads
    float acc = 0.f;
    for (int m = 0; m < n_img; ++m) {
        const __nv_bfloat16* f = feat + (size_t)(p * n_img + m) * Ho_p * Wo * 256 + c;
        float s = 0.f;
        for (int i = 0; i < Ho * Wo; ++i) s += __bfloat162float(f[(size_t)i * 256]);
        acc += s / (float)(Ho * Wo);
    }
    cond[(size_t)p * U_COND + c] = acc / (float)n_img;
    if (c < U_DOF) cond[(size_t)p * U_COND + 256 + c] = (q[p * U_DOF + c] - lo) / (hi - lo);
    if (c < 3) cond[(size_t)p * U_COND + 256 + U_DOF + c] = goal[p * 7 + c] / 0.6f;
    if (c < 4) cond[(size_t)p * U_COND + 256 + U_DOF + 3 + c] = goal[p * 7 + 3 + c];
}

// 5-D pair view of an NHWC bf16 tensor [img][Hp][W][C]: dims (2C, W/2, 2, Hp/2, img)
static bool make_pair_map(CUtensorMap* tm, const void* base, int n_img, int Hp, int W, int C, int wx, int ry) {
    cuuint64_t dims[5] = {(cuuint64_t)2 * C, (cuuint64_t)W / 2, 2, (cuuint64_t)Hp / 2, (cuuint64_t)n_img};
    cuuint64_t strides[4] = {(cuuint64_t)2 * C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)2 * W * C * 2,
                             (cuuint64_t)Hp * W * C * 2};
    cuuint32_t box[5] = {64, (cuuint32_t)wx, 1, (cuuint32_t)ry, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

extern "C" long long ps_encode_tc_workspace_bytes(int n_images, int H, int W, int n_layers) {
    if (n_layers < 2 || n_layers > ENC_MAXL) return -1;
    EncLayerGeo g[ENC_MAXL];
    enc_geometry(H, W, n_layers, g);
    size_t mx = 0;
    for (int l = 0; l < n_layers; ++l) mx = std::max(mx, (size_t)n_images * g[l].Ho_p * g[l].Wo * g[l].N);
    return (long long)(2 * ((mx * 2 + 255) / 256 * 256));
}

extern "C" int ps_encode_tc(const float* images, int P, int n_img, int H, int W, const void* packed, int n_layers,
                            const float* q_start, const float* goal, float lo, float hi, void* ws, float* cond,
                            void* stream) {
    if (P <= 0 || n_img <= 0 || n_layers < 2 || n_layers > ENC_MAXL || (W & 3)) return PS_FAIL(PS_ERR_SHAPE);
    if (!get_encoder()) return PS_FAIL(PS_ERR_CUDA);
    cudaStream_t st = (cudaStream_t)stream;
    EncLayerGeo g[ENC_MAXL];
    enc_geometry(H, W, n_layers, g);
    for (int l = 1; l < n_layers; ++l)
        if (g[l].Win & 1) return PS_FAIL(PS_ERR_SHAPE);
    const int NI = P * n_img;
    const size_t half = (size_t)(ps_encode_tc_workspace_bytes(NI, H, W, n_layers) / 2);
    __nv_bfloat16* buf[2] = {reinterpret_cast<__nv_bfloat16*>(ws),
                             reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(ws) + half)};
    const EncLayerGeo& last = g[n_layers - 1];
    const size_t wb = ((last.w_off + (size_t)last.N * last.n_chunks * 64) * 2 + 255) / 256 * 256;
    const float* side = reinterpret_cast<const float*>(reinterpret_cast<const char*>(packed) + wb);
    size_t bias_tot = 0;
    for (int l = 0; l < n_layers; ++l) bias_tot += g[l].N;
    const float* w1 = side + bias_tot;
    {
        const EncLayerGeo& e = g[0];
        const size_t n = (size_t)NI * e.Ho_p * ((e.Wo + 1) / 2);
        enc_l1_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(images, NI, H, W, w1, side + e.b_off, e.Ho,
                                                                    e.Wo, e.Ho_p, buf[0]);
        PS_CHECK_LAUNCH();
    }
    const __nv_bfloat16* W16 = reinterpret_cast<const __nv_bfloat16*>(packed);
    for (int l = 1; l < n_layers; ++l) {
        const EncLayerGeo& e = g[l];
        __nv_bfloat16* in = buf[(l - 1) & 1];
        __nv_bfloat16* out = buf[l & 1];
        if (e.Ho_p != e.Ho)  // zero the padding row the next layer's pair view reads
            cudaMemsetAsync(out, 0, (size_t)NI * e.Ho_p * e.Wo * e.N * 2, st);
        TcArgs a;
        memset(&a, 0, sizeof(a));
        if (!make_pair_map(&a.tmA[0], in, NI, e.Hin_p, e.Win, e.C, e.wx, e.ry)) return PS_FAIL(PS_ERR_CUDA);
        if (!make_w_map(&a.tmW, W16 + e.w_off, e.N, e.n_chunks * 64)) return PS_FAIL(PS_ERR_CUDA);
        int n = 0;
        const int C = e.C;
        for (int dy = 0; dy < 3; ++dy) {
            const int par = dy == 1 ? 0 : 1, dt = dy == 0 ? -1 : 0;
            const int segA = C == 32 ? 1 : C / 64;
            for (int ci = 0; ci < segA; ++ci) {
                TcChunk ch{};
                ch.c = (int16_t)(C == 32 ? 0 : C + 64 * ci);
                ch.kcol = (int16_t)(64 * n);
                ch.dt = (int8_t)dt;
                ch.par = (int8_t)par;
                ch.dx = -1;
                ch.first = n == 0;
                a.chunk[n++] = ch;
            }
            for (int ci = 0; ci < 2 * C / 64; ++ci) {
                TcChunk ch{};
                ch.c = (int16_t)(64 * ci);
                ch.kcol = (int16_t)(64 * n);
                ch.dt = (int8_t)dt;
                ch.par = (int8_t)par;
                ch.dx = 0;
                ch.first = n == 0;
                a.chunk[n++] = ch;
            }
        }
        if (n != e.n_chunks || n > TC_MAX_CHUNKS) return PS_FAIL(PS_ERR_SHAPE);
        a.n_chunks = n;
        a.geom = 1;
        a.rows = NI * e.tiles_x * e.tiles_y;   // number of tiles
        a.Tv = 1;
        a.S = 1;
        a.Ho = e.Ho;
        a.Wo = e.Wo;
        a.Hp = e.Ho_p;
        a.wx = e.wx;
        a.ry = e.ry;
        a.tiles_x = e.tiles_x;
        a.tiles_y = e.tiles_y;
        a.bias = side + e.b_off;
        a.out = out;
        int s;
        if (e.N == 64)
            s = launch_tc<64, EPI_RELU2D, false>(a, a.rows, st);
        else if (e.N == 128)
            s = launch_tc<128, EPI_RELU2D, false>(a, a.rows, st);
        else
            s = launch_tc<256, EPI_RELU2D, false>(a, a.rows, st);
        if (s) return s;
    }
    enc_gap_cond_kernel<<<P, 256, 0, st>>>(buf[(n_layers - 1) & 1], n_img, last.Ho, last.Ho_p, last.Wo, q_start, goal,
                                           lo, hi, cond);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
}  // namespace ps
