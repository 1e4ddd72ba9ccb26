// dit_kernels.hpp — launchers of the DiT's memory-bound kernels (dit_kernels.cu).
#pragma once

#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"

namespace lpb200 {

struct TimeWeights {
    const __nv_bfloat16* w1; const float* b1;  // [dim, freq_dim]
    const __nv_bfloat16* w2; const float* b2;  // [dim, dim]
    const __nv_bfloat16* wp; const float* bp;  // [6*dim, dim]
    const float* block_mod;                     // [layers, 6, dim]
    const float* head_mod;                      // [2, dim]
};

void init_param(void* p, int64_t n, bool bf16, uint64_t seed, uint64_t stream, float scale, float offset,
                cudaStream_t st);
void text_context(__nv_bfloat16* out, int64_t n, uint64_t seed, cudaStream_t st);
void patchify(const void* z, int dtype, const int shape[4], const int patch[3], __nv_bfloat16* out, cudaStream_t st);
// scratch >= freq_dim + 8*dim floats; mod_out [layers, 6, dim]; head_mod_out [2, dim]
void time_embedding(const TimeWeights& w, const float* t_dev, int freq_dim, int dim, int layers, float* scratch,
                    float* mod_out, float* head_mod_out, cudaStream_t st);
// *p = v on the stream (a one-thread kernel: stream-ordered and independent of host memory)
void set_device_f32(float* p, float v, cudaStream_t st);
void layernorm_bf16(const float* x, __nv_bfloat16* y, int64_t rows, int d, const float* a, const float* b, bool affine,
                    float eps, cudaStream_t st);
// LayerNorm folded into the next GEMM (dit.cpp, knob dit_lnfold).  One job = one weight
// matrix W [N, K] bf16: cs[n] = sum_k W[n,k] (plus1 ? 1 + a[k] : a[k]) and
// bo[n] = sum_k W[n,k] b[k] + bias[n] (fp32), i.e. the column sums of diag(g) W^T and the
// folded shift/bias of LN(x) * g + b followed by W.
struct LnFoldJob {
    const __nv_bfloat16* W;
    const float* bias;
    const float* a;
    const float* b;
    float* cs;
    float* bo;
    int N, K, plus1, pad;
};
void lnfold_vectors(const LnFoldJob* jobs_dev, int njobs, int max_n, cudaStream_t st);
void rmsnorm_rope(__nv_bfloat16* buf, int64_t rows, int64_t ld, int64_t col0, int d, const float* g, float eps,
                  bool rope, int64_t rows_per_batch, int nh, int nw, cudaStream_t st);
// RoPE cos/sin table [nf*22 + nh*21 + nw*21] float2 of a shard grid (once per forward).
void rope_table(float2* tab, int nf, int nh, int nw, cudaStream_t st);
// out[r, c] = bf16(in[r, c] * g[c]) over rows x d (the q-norm weight folded into the text K)
void scale_cols_bf16(const __nv_bfloat16* in, int64_t rows, int d, const float* g, __nv_bfloat16* out, cudaStream_t st);
// Table-driven RMSNorm(+RoPE if tab) of nsec adjacent width-d sections (q | k), in place.
// Returns false when the width / alignment is not covered (callers use rmsnorm_rope).
bool rmsnorm_rope_tab(__nv_bfloat16* buf, int64_t rows, int64_t ld, int64_t col0, int d, int nsec, const float* g0,
                      const float* g1, float eps, const float2* tab, int64_t rows_per_batch, int nf, int nh, int nw,
                      cudaStream_t st);
// Peer copies of the ε̂ written by unpatchify_cfg: element i is also stored at
// (char*)(eps + i) + delta[j] (an IPC-mapped peer gather buffer), j < n.
struct EpsMirrors {
    int n = 0;
    int64_t delta[16] = {};
};
// single: `head` holds ONE pass (batch 1) and eps = quantize(prediction) (Denoiser::predict);
// else rows [0, ntok) are the uncond pass, [ntok, 2 ntok) the cond pass, combined as cfg_predict.
void unpatchify_cfg(const float* head, int dtype, const int shape[4], const int patch[3], double w, void* eps,
                    cudaStream_t st, const EpsMirrors& mr = EpsMirrors(), bool single = false);

}  // namespace lpb200
