// PTX wrappers shared by the tcgen05 kernels (conv_tc.cu: encoder, unet_tc.cu: U-Net).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace ps {

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in the barrier unit until the
// phase completes (or ~the hint elapses) instead of spinning through issue slots that the
// epilogue warps need
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity), "r"(0x100000u)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
// programmatic dependent launch (griddepcontrol): no-ops for a normal launch
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// launch with cudaLaunchAttributeProgrammaticStreamSerialization: the kernel may start
// while the previous kernel on the stream drains; it must call pdl_wait() before touching
// memory the previous kernels produce or consume
template <typename Kern, typename Arg>
static inline int launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const Arg& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("PS_NO_PDL") != nullptr;
    cfg.numAttrs = no_pdl ? 0 : 1;
    ps_launch_counter().fetch_add(1, std::memory_order_relaxed);
    if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return PS_FAIL(PS_ERR_CUDA);
    return PS_OK;
}

// TMA store (shared -> global), bulk-group completion
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"((uint64_t)tm),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled UMMA shared-memory descriptor (rows of 128 B, 8-row atoms)
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* p) {
    const uint32_t a = smem_u32(p);
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)0 << 16;                       // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;             // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                       // version (sm100)
    d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
    return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, K-major both, M=128, N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// warp-uniform variants: the whole warp runs the issue loop (descriptor math stays in
// uniform registers) and one elected lane issues
__device__ __forceinline__ void umma_bf16_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}
// ---- CTA pairs (cta_group::2): rank, leader-mapped addresses, cluster barrier, 2-SM MMA
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same variable in the pair's leader (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's smem whose completion is counted on the leader's mbarrier
__device__ __forceinline__ void tma_load_3d_cg2(void* dst, const CUtensorMap* tm, uint32_t bar_cl, int c0, int c1,
                                                int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
        "%5}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)tm), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* tm, uint32_t bar_cl, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)tm), "r"(bar_cl), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_w2(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// completion of the pair's MMAs arrives on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void umma_commit_w2(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
            smem_u32(bar)),
        "h"((unsigned short)3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cl) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
template <typename Kern, typename Arg>
static inline int launch_pdl_pair(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const Arg& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("PS_NO_PDL") != nullptr;
    cfg.numAttrs = no_pdl ? 1 : 2;
    ps_launch_counter().fetch_add(1, std::memory_order_relaxed);
    if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return PS_FAIL(PS_ERR_CUDA);
    return PS_OK;
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// mish(x) = x tanh(softplus(x)) = x * n(n+2) / (n(n+2) + 2), n = e^x
__device__ __forceinline__ float mish_fast(float x) {
    const float n = __expf(fminf(x, 15.f));
    const float m = n * (n + 2.f);
    const float y = x * __fdividef(m, m + 2.f);
    return x > 15.f ? x : y;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// mish(x) = x - 2x / (n^2 + 2n + 2), n = e^min(x, 15)   (8 instructions; for x > 15 the
// correction underflows below fp32 resolution, so no branch/select is needed)
// packed fp32 (sm_100 FFMA2 / FADD2 / FMUL2): two lanes of math per instruction
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// mish8 on a pair (see mish8): the SFU ops stay scalar, the rest is packed
__device__ __forceinline__ float2 mish2(float2 z) {
    const float2 zl = fmul2(z, f2(1.4426950408889634f, 1.4426950408889634f));
    float2 n;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(n.x) : "f"(zl.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(n.y) : "f"(zl.y));
    const float2 m = ffma2(n, f2(-0.5f, -0.5f), f2(-1.f, -1.f));
    const float2 d = ffma2(n, m, f2(-1.f, -1.f));
    float2 r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(d.y));
    return ffma2(z, r, z);
}

__device__ __forceinline__ float mish8(float x) {
    // mish(x) = x - 2x / (n (n + 2) + 2), n = e^x, as x + x * r with r = 1 / (-d/2) = -2/d:
    // -d/2 = n * (-(n + 2)/2) - 1.  6 ops (2 on the SFU).  No clamp needed: n = inf gives
    // -d/2 = -inf, r = -0 and mish = x; n = 0 gives r = -1 and mish = 0.
    const float n = ex2_approx(x * 1.4426950408889634f);
    const float m = fmaf(n, -0.5f, -1.f);
    return fmaf(x, rcp_approx(fmaf(n, m, -1.f)), x);
}


__device__ __forceinline__ uint4 philox_tc(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ float normal_tc(uint32_t step, uint32_t prob, uint32_t seed, uint32_t e, uint32_t key) {
    const uint4 r = philox_tc(make_uint4(e >> 2, step, prob, seed), key, 0x5EED5EEDu);
    const uint32_t comp = e & 3u;
    const uint32_t a = comp < 2 ? r.x : r.z, b = comp < 2 ? r.y : r.w;
    const float u1 = ((float)(a >> 8) + 1.0f) * (1.0f / 16777216.0f);
    const float u2 = (float)(b >> 8) * (1.0f / 16777216.0f);
    const float rad = sqrtf(-2.0f * logf(u1));
    const float ang = 6.28318530717958648f * u2;
    return (comp & 1u) ? rad * sinf(ang) : rad * cosf(ang);
}

// Box-Muller pair of two raw Philox words (spec.py "Counter-based noise"), the fused-epilogue form.
// The radius uses the full-precision logf: near u1 = 1 the true -2 ln u1 is ~1.2e-7, below the
// absolute error of the SFU lg2.approx, whose sign could then flip (sqrtf of a negative -> NaN)
// or inflate the radius by ~4e-4.  logf is within 1 ulp, so the radius is within ~1e-6 of the exact
// transform for every one of the 2^24 values of a >> 8; the fmaxf guards u1 = 1 exactly.  The angle
// is taken centred, 2 pi (u2 - 1/2) in [-pi, pi) (u2 - 1/2 is exact), where the SFU sincos holds its
// documented 2^-21.4 absolute error; cos / sin of the centred angle are the negated uncentred ones.
// tests/test_noise_gpu.py checks both words exhaustively against the float64 transform.
__device__ __forceinline__ void box_muller_tc(uint32_t a, uint32_t b, float& z0, float& z1) {
    const float u1 = ((float)(a >> 8) + 1.0f) * (1.0f / 16777216.0f);
    const float u2 = (float)(b >> 8) * (1.0f / 16777216.0f);
    const float rad = sqrtf(fmaxf(-2.0f * logf(u1), 0.0f));
    float sn, cs;
    __sincosf(6.28318530717958648f * (u2 - 0.5f), &sn, &cs);
    z0 = -rad * cs;
    z1 = -rad * sn;
}

// the 4 normals of Philox block `blk` (elements 4*blk .. 4*blk+3); used by the fused DDPM epilogues
__device__ __forceinline__ void normal4_tc(uint32_t step, uint32_t prob, uint32_t seed, uint32_t blk, uint32_t key,
                                           float (&n)[4]) {
    const uint4 r = philox_tc(make_uint4(blk, step, prob, seed), key, 0x5EED5EEDu);
    box_muller_tc(r.x, r.y, n[0], n[1]);
    box_muller_tc(r.z, r.w, n[2], n[3]);
}

template <int NV>
__device__ __forceinline__ float sel(const float (&a)[NV], int i) {
    float r = a[0];
#pragma unroll
    for (int k = 1; k < NV; ++k) r = (i == k) ? a[k] : r;
    return r;
}


__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace ps
