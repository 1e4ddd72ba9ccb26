// dit_ops.hpp — host-side launchers of the DiT kernels (tcgen05 GEMM and
// attention, fused norm/modulation/RoPE/CFG kernels).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace lpb200 {

enum GemmMode { EPI_BF16 = 0, EPI_BF16_GELU = 1, EPI_F32_RESID = 2, EPI_F32 = 3 };

struct GemmEpilogue {
    const float* bias;  // [N] or null
    void* out;          // bf16 / f32 [M, ldo]
    int64_t ldo;        // output row stride (elements)
    const float* gate;  // [N] or null (F32_RESID only)
    // LayerNorm folded into the next GEMM (dit.cpp, knob dit_lnfold), producer side (F32 /
    // F32_RESID): besides x the epilogue writes xq = bf16(x * g) (g_plus1: x * (1 + g); row
    // stride ldq) — the next LayerNorm's per-channel multiplier applied — and, per row and
    // N tile, the tile's LayerNorm partials (mean, M2 = sum (x - mean)^2) of x at
    // stats_out[row * (N / BN) + n_tile].  Null xq: off.
    __nv_bfloat16* xq;
    int64_t ldq;
    const float* g;
    int g_plus1;
    float2* stats_out;
    // consumer side (BF16 / BF16_GELU with A = xq): out = rstd * (acc - mean * cs[col]) + bias[col]
    // with (mean, rstd = 1/sqrt(var + eps)) merged from the row's `parts` partials of
    // cols_per_part columns each (stats_in[row * parts ...]).  Null stats_in: off.
    const float* cs;
    const float2* stats_in;
    int parts;
    float cols_per_part;
    float eps;
    // BF16 epilogue: per row and N tile, the sum of squares of the bf16 values written
    // (rms_out[row * (N / BN) + n_tile]) — the cross-attention q RMSNorm folded into attention
    // (dit.cpp, knob dit_xq_rms).  Null: off.
    float* rms_out;
};
// N tile width the GEMM uses for N (the producer's partial count is N / gemm_bn_for(M, N));
// 0 when (M, N) takes a kernel without the LN-fold epilogue.
int gemm_lnfold_bn(int M, int N);

// D = epilogue(A[M,K] · B[N,K]^T); lda/ldb in elements.
void gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const GemmEpilogue& ep,
               int mode, cudaStream_t st);

// Multi-head attention forward, head_dim 128, bf16.  For batch b, head h:
//   Q rows [b*q_rows_per_batch, +n_q) cols [q_col0 + h*128, +128) of q (row stride ldq)
//   K/V likewise with kv_rows_per_batch / n_kv; O -> o (row stride ldo) cols h*128.
struct AttnArgs {
    const void* q; int64_t ldq; int64_t q_col0; int64_t q_rows_per_batch; int64_t n_q; int64_t q_total_rows;
    const void* k; int64_t ldk; int64_t k_col0;
    const void* v; int64_t ldv; int64_t v_col0;
    int64_t kv_rows_per_batch; int64_t n_kv; int64_t kv_total_rows;
    void* o; int64_t ldo;
    int batch, heads;
    float scale;
    // q RMSNorm folded into the softmax scale: row r's scores are scaled by
    // rsqrt(sum(q_rms[r * rms_parts ...]) / rms_d + rms_eps) (the q rows are un-normalised and the
    // norm's per-channel weight is folded into K).  Null: off.
    const float* q_rms;
    int rms_parts;
    int rms_d;
    float rms_eps;
};
void attention_bf16(const AttnArgs& a, cudaStream_t st);

}  // namespace lpb200
