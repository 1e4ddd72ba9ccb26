// lnfold.cuh — the LayerNorm-fold producer arithmetic shared by the GEMM epilogue
// (gemm_tcgen05.cu) and the stage-boundary pass (dit_kernels.cu), written with explicit
// round-to-nearest intrinsics so both compile to the same operations: a pipeline stage that
// recomputes the partials from x gets the bits the GEMM epilogue would have written.
#pragma once

#include <cuda_bf16.h>

namespace lpb200 {

// Merge the LayerNorm partials of one 32-value chunk (the chunk-th of its tile, counted from
// 0) into the tile's running (mean, M2) (Chan et al.; equal chunk sizes).
__device__ __forceinline__ void ln_chunk_merge(const float (&v)[32], int chunk, float& mean, float& m2) {
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) m = __fadd_rn(m, v[j]);
    m = __fmul_rn(m, 1.f / 32.f);
    float c2 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const float dlt = __fsub_rn(v[j], m);
        c2 = __fmaf_rn(dlt, dlt, c2);
    }
    const float dlt = __fsub_rn(m, mean), inv = __frcp_rn(static_cast<float>(chunk + 1));
    mean = __fmaf_rn(dlt, inv, mean);
    m2 = __fadd_rn(m2, __fmaf_rn(__fmul_rn(dlt, dlt), __fmul_rn(32.f * static_cast<float>(chunk), inv), c2));
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
