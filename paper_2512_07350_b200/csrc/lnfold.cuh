// lnfold.cuh — the LayerNorm-fold producer arithmetic of the GEMM epilogue (gemm_tcgen05.cu,
// knob dit_lnfold), written with explicit round-to-nearest intrinsics (no contraction).
#pragma once

#include <cuda_bf16.h>

namespace lpb200 {

// LayerNorm partials of one part (a GEMM tile's columns), fed
// 32-value chunks in column order.  Shifted sums: K = the part's first value, then four
// independent (Σd, Σd²) accumulators over d = v - K (chain length 8 per chunk instead of a 32-deep
// serial Welford/Chan merge, which cost the residual GEMM epilogues ~4% of the step, r3k).  The
// shift keeps Σd² - (Σd)²/n well conditioned (K is within a few standard deviations of the mean).
struct LnAcc {
    float k = 0.f;
    float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
};
__device__ __forceinline__ void ln_acc_chunk(const float (&v)[32], int chunk, LnAcc& a) {
    if (chunk == 0) a.k = v[0];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const float d = __fsub_rn(v[j], a.k);
        a.s1[j & 3] = __fadd_rn(a.s1[j & 3], d);
        a.s2[j & 3] = __fmaf_rn(d, d, a.s2[j & 3]);
    }
}
// (mean, M2) of the part's n values, the form the consumer merges across parts
__device__ __forceinline__ float2 ln_acc_final(const LnAcc& a, float n) {
    const float S1 = __fadd_rn(__fadd_rn(a.s1[0], a.s1[1]), __fadd_rn(a.s1[2], a.s1[3]));
    const float S2 = __fadd_rn(__fadd_rn(a.s2[0], a.s2[1]), __fadd_rn(a.s2[2], a.s2[3]));
    const float m = __fdiv_rn(S1, n);
    return make_float2(__fadd_rn(a.k, m), fmaxf(__fmaf_rn(-S1, m, S2), 0.f));
}

// xq = bf16(x * g) (plus1: x * (1 + g)) for 8 consecutive values, packed
__device__ __forceinline__ uint4 ln_xq8(const float* v, const float* g, int plus1) {
    uint32_t w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const float g0 = plus1 ? __fadd_rn(1.f, g[2 * u]) : g[2 * u];
        const float g1 = plus1 ? __fadd_rn(1.f, g[2 * u + 1]) : g[2 * u + 1];
        __nv_bfloat162 p = __floats2bfloat162_rn(__fmul_rn(v[2 * u], g0), __fmul_rn(v[2 * u + 1], g1));
        w[u] = *reinterpret_cast<uint32_t*>(&p);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace lpb200
