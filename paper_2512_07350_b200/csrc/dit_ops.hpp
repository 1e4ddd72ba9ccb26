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
};

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
};
void attention_bf16(const AttnArgs& a, cudaStream_t st);

}  // namespace lpb200
