// Test hooks for the fused-epilogue noise transform (tc_ptx.cuh: box_muller_tc / normal4_tc).
// The DDPM epilogues of the layered and persistent U-Net kernels draw their posterior noise with
// normal4_tc; these entry points run exactly that device function so tests/test_noise_gpu.py can
// check it exhaustively (every value of the radius and angle words) and at scale (>= 1e8 draws).
#include "tc_ptx.cuh"

namespace {

__global__ void box_muller_probe_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int n,
                                        float* __restrict__ z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float z0, z1;
    ps::box_muller_tc(a[i], b[i], z0, z1);
    z[2 * i] = z0;
    z[2 * i + 1] = z1;
}

__global__ void normal4_probe_kernel(float* __restrict__ out, int n_blocks, uint32_t step, uint32_t prob,
                                     uint32_t seed, uint32_t key) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_blocks) return;
    float n4[4];
    ps::normal4_tc(step, prob, seed, (uint32_t)i, key, n4);
    reinterpret_cast<float4*>(out)[i] = make_float4(n4[0], n4[1], n4[2], n4[3]);
}

// every (problem, seed, block) of one step: counts non-finite draws, accumulates max |z|, sum z and
// sum z^2 (for a moment check) -- grid-stride over n_prob x n_seed x n_blk Philox blocks
__global__ void noise_scan_kernel(uint32_t step, uint32_t n_prob, uint32_t n_seed, uint32_t n_blk, uint32_t key,
                                  unsigned long long* __restrict__ nonfinite, unsigned* __restrict__ maxabs_bits,
                                  double* __restrict__ moments) {
    const unsigned long long total = (unsigned long long)n_prob * n_seed * n_blk;
    unsigned long long bad = 0;
    float mx = 0.f;
    double s1 = 0.0, s2 = 0.0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t blk = (uint32_t)(i % n_blk);
        const unsigned long long r = i / n_blk;
        const uint32_t seed = (uint32_t)(r % n_seed), prob = (uint32_t)(r / n_seed);
        float n4[4];
        ps::normal4_tc(step, prob, seed, blk, key, n4);
        float ls1 = 0.f, ls2 = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!isfinite(n4[j])) {
                ++bad;
            } else {
                mx = fmaxf(mx, fabsf(n4[j]));
                ls1 += n4[j];
                ls2 += n4[j] * n4[j];
            }
        }
        s1 += ls1;
        s2 += ls2;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad += __shfl_xor_sync(PS_FULL, bad, o);
        mx = fmaxf(mx, __shfl_xor_sync(PS_FULL, mx, o));
        s1 += __shfl_xor_sync(PS_FULL, s1, o);
        s2 += __shfl_xor_sync(PS_FULL, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(nonfinite, bad);
        atomicMax(maxabs_bits, __float_as_uint(mx));   // non-negative floats order like their bits
        atomicAdd(&moments[0], s1);
        atomicAdd(&moments[1], s2);
    }
}

}  // namespace

extern "C" int ps_box_muller_probe(const unsigned* a, const unsigned* b, int n, float* z, void* stream) {
    if (n < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (n == 0) return PS_OK;
    box_muller_probe_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(a, b, n, z);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_normal4_probe(float* out, int n_blocks, int step, int prob, int seed, unsigned key,
                                void* stream) {
    if (n_blocks < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (n_blocks == 0) return PS_OK;
    normal4_probe_kernel<<<(n_blocks + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        out, n_blocks, (uint32_t)step, (uint32_t)prob, (uint32_t)seed, key);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_noise_scan(int step, int n_prob, int n_seed, int n_blk, unsigned key,
                             unsigned long long* nonfinite, unsigned* maxabs_bits, double* moments, void* stream) {
    if (n_prob <= 0 || n_seed <= 0 || n_blk <= 0) return PS_FAIL(PS_ERR_SHAPE);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    noise_scan_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>((uint32_t)step, (uint32_t)n_prob, (uint32_t)n_seed,
                                                                (uint32_t)n_blk, key, nonfinite, maxabs_bits,
                                                                moments);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
