// dit_kernels.cu — the DiT's non-GEMM kernels (memory-bound, fused):
//   patch gather (K2 prologue: sub-latent -> [tokens, 64] bf16 patches)
//   time embedding (sinusoid -> MLP -> 6-way modulation), GEMV on CUDA cores
//   LayerNorm + adaLN modulate -> bf16 (K4), affine LayerNorm -> bf16
//   q/k RMSNorm + 3-D RoPE in place on the QKV buffer
//   head unpatchify + CFG combine + quantize to the storage dtype (K8)
//   pinned weight / text-context generator
#include <cuda_bf16.h>

#include "dit_kernels.hpp"

namespace lpb200 {

// ---------------------------------------------------------------------------
// pinned generator: splitmix64(seed, stream, index) -> uniform [-1, 1)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ float hash_uniform(uint64_t seed, uint64_t stream, uint64_t i) {
    const uint64_t h = splitmix64(splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ull)) + i);
    return static_cast<float>(static_cast<double>(h >> 40) * (1.0 / 8388608.0) - 1.0);  // 24-bit, [-1, 1)
}

__global__ void k_init_param(void* p, int64_t n, int is_bf16, uint64_t seed, uint64_t stream, float scale,
                             float offset) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = offset + scale * hash_uniform(seed, stream, static_cast<uint64_t>(i));
        if (is_bf16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
        else static_cast<float*>(p)[i] = v;
    }
}

void init_param(void* p, int64_t n, bool bf16, uint64_t seed, uint64_t stream, float scale, float offset,
                cudaStream_t st) {
    k_init_param<<<592, 256, 0, st>>>(p, n, bf16 ? 1 : 0, seed, stream, scale, offset);
    LP_LAUNCH_CHECK();
}

// synthetic text context: N(0,1) via Box-Muller on two hash uniforms -> bf16
__global__ void k_text_context(__nv_bfloat16* out, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float u1 = 0.5f * (hash_uniform(seed, 0x7e47, 2 * i) + 1.f);
        const float u2 = 0.5f * (hash_uniform(seed, 0x7e47, 2 * i + 1) + 1.f);
        const float r = sqrtf(-2.f * logf(fmaxf(u1, 1e-7f)));
        out[i] = __float2bfloat16_rn(r * cosf(6.283185307179586f * u2));
    }
}
void text_context(__nv_bfloat16* out, int64_t n, uint64_t seed, cudaStream_t st) {
    k_text_context<<<592, 256, 0, st>>>(out, n, seed);
    LP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// patch gather: sub-latent [C, F, H, W] (storage dtype) -> patches [tok, C*pt*ph*pw]
// bf16, token = (f, y, x) row-major, feature = ((c*pt + kt)*ph + kh)*pw + kw
// (Conv3d weight flattening); positions past the extent are zero (padding).
// ---------------------------------------------------------------------------
template <int D>
__global__ void k_patchify(const typename Store<D>::T* __restrict__ z, __nv_bfloat16* __restrict__ out, int C, int F,
                           int H, int W, int pt, int ph, int pw, int nf, int nh, int nw) {
    const int feat = C * pt * ph * pw;
    const int64_t total = static_cast<int64_t>(nf) * nh * nw * feat;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int fe = static_cast<int>(i % feat);
        const int64_t tok = i / feat;
        const int xw = static_cast<int>(tok % nw), yh = static_cast<int>((tok / nw) % nh), tf = static_cast<int>(tok / (static_cast<int64_t>(nw) * nh));
        const int kw = fe % pw, kh = (fe / pw) % ph, kt = (fe / (pw * ph)) % pt, c = fe / (pw * ph * pt);
        const int t = tf * pt + kt, y = yh * ph + kh, x = xw * pw + kw;
        float v = 0.f;
        if (t < F && y < H && x < W) v = static_cast<float>(load_val<D>(z, ((static_cast<int64_t>(c) * F + t) * H + y) * W + x));
        out[i] = __float2bfloat16_rn(v);
    }
}

void patchify(const void* z, int dtype, const int shape[4], const int patch[3], __nv_bfloat16* out, cudaStream_t st) {
    const int nf = (shape[1] + patch[0] - 1) / patch[0], nh = (shape[2] + patch[1] - 1) / patch[1],
              nw = (shape[3] + patch[2] - 1) / patch[2];
    const int64_t total = static_cast<int64_t>(nf) * nh * nw * shape[0] * patch[0] * patch[1] * patch[2];
    const int g = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
#define LP_PATCH(DD) k_patchify<DD><<<g, 256, 0, st>>>(static_cast<const typename Store<DD>::T*>(z), out, shape[0], shape[1], shape[2], shape[3], patch[0], patch[1], patch[2], nf, nh, nw)
    if (dtype == 2) LP_PATCH(2);
    else if (dtype == 4) LP_PATCH(4);
    else LP_PATCH(8);
#undef LP_PATCH
    LP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// GEMV for the time path: y[o] = act_out( W[o,:] · act_in(x) + b[o] ) (+ add[o])
// W bf16 row-major [out, in]; one warp per output.  act: 0 none, 1 SiLU
// ---------------------------------------------------------------------------
__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

__global__ void k_gemv(const __nv_bfloat16* __restrict__ W, const float* __restrict__ bias,
                       const float* __restrict__ x, float* __restrict__ y, int in, int out, int act_in) {
    const int o = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (o >= out) return;
    float acc = 0.f;
    for (int i = lane; i < in; i += 32) {
        float v = x[i];
        if (act_in) v = silu(v);
        acc += __bfloat162float(W[static_cast<int64_t>(o) * in + i]) * v;
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, s);
    if (lane == 0) y[o] = acc + (bias ? bias[o] : 0.f);
}

// sinusoid embedding: [cos(t*w_i), sin(t*w_i)], w_i = 10000^(-i/half)
__global__ void k_sinusoid(float* out, int dim, const float* __restrict__ t_dev) {
    const float t = *t_dev;  // device-resident: a captured step graph replays with a new t
    const int half = dim / 2;
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
        const double w = pow(10000.0, -static_cast<double>(i) / half);
        const double a = static_cast<double>(t) * w;
        out[i] = static_cast<float>(cos(a));
        out[i + half] = static_cast<float>(sin(a));
    }
}

// mod[l, j, :] = param[l, j, :] + e0[j, :]   (j < 6), head: hmod[j] = hparam[j] + e[:]
__global__ void k_add_mod(const float* __restrict__ param, const float* __restrict__ e0, float* __restrict__ out,
                          int64_t per_layer, int64_t layers) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_layer * layers;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = param[i] + e0[i % per_layer];
}

__global__ void k_set_f32(float* p, float v) { *p = v; }

void set_device_f32(float* p, float v, cudaStream_t st) {
    k_set_f32<<<1, 1, 0, st>>>(p, v);
    LP_LAUNCH_CHECK();
}

void time_embedding(const TimeWeights& w, const float* t_dev, int freq_dim, int dim, int layers, float* scratch,
                    float* mod_out, float* head_mod_out, cudaStream_t st) {
    float* sin_ = scratch;                 // [freq_dim]
    float* h1 = sin_ + freq_dim;           // [dim]
    float* e = h1 + dim;                   // [dim]
    float* e0 = e + dim;                   // [6*dim]
    k_sinusoid<<<1, 256, 0, st>>>(sin_, freq_dim, t_dev);
    LP_LAUNCH_CHECK();
    k_gemv<<<(dim + 7) / 8, 256, 0, st>>>(w.w1, w.b1, sin_, h1, freq_dim, dim, 0);
    LP_LAUNCH_CHECK();
    k_gemv<<<(dim + 7) / 8, 256, 0, st>>>(w.w2, w.b2, h1, e, dim, dim, 1);
    LP_LAUNCH_CHECK();
    k_gemv<<<(6 * dim + 7) / 8, 256, 0, st>>>(w.wp, w.bp, e, e0, dim, 6 * dim, 1);
    LP_LAUNCH_CHECK();
    k_add_mod<<<296, 256, 0, st>>>(w.block_mod, e0, mod_out, 6LL * dim, layers);
    LP_LAUNCH_CHECK();
    k_add_mod<<<8, 256, 0, st>>>(w.head_mod, e, head_mod_out, dim, 2);
    LP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// LayerNorm (+ modulate | + affine) fp32 -> bf16, one warp per row, d % 256 == 0
//   MOD:    y = LN(x) * (1 + scale) + shift
//   AFFINE: y = LN(x) * weight + bias
// ---------------------------------------------------------------------------
// Row order of the row-wise HBM passes (LayerNorm, q/k RMSNorm+RoPE; knob row_rev): the GEMM
// that wrote their input finished on its last rows, which are the ones still in L2, and the
// GEMM that reads their output starts on its first rows — so walking rows last-to-first lets
// both ends of each pass meet L2 instead of HBM.  Results are identical (rows independent).
static int row_order_rev() { return tune_get("row_rev", 0); }

template <int PER, bool AFFINE>
__global__ void __launch_bounds__(256) k_layernorm(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                                   int64_t rows, int d, const float* __restrict__ a,
                                                   const float* __restrict__ b, float eps, int rev) {
    int64_t row = blockIdx.x * 8LL + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    if (rev) row = rows - 1 - row;  // last-written rows first (see row_order_rev)
    const float4* xr = reinterpret_cast<const float4*>(x + row * d);
    float v[PER * 4];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const float4 q = xr[lane + 32 * i];
        v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
        s += q.x + q.y + q.z + q.w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    const float mean = s / d;
    float var = 0.f;
#pragma unroll
    for (int i = 0; i < PER * 4; ++i) {
        const float c = v[i] - mean;
        var += c * c;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) var += __shfl_xor_sync(0xffffffff, var, o);
    const float rstd = rsqrtf(var / d + eps);
    uint2* yr = reinterpret_cast<uint2*>(y + row * d);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int c0 = 4 * (lane + 32 * i);
        const float4 a4 = reinterpret_cast<const float4*>(a)[lane + 32 * i];
        const float4 b4 = reinterpret_cast<const float4*>(b)[lane + 32 * i];
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
        float o4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float n = (v[4 * i + u] - mean) * rstd;
            o4[u] = AFFINE ? n * av[u] + bv[u] : n * (1.f + av[u]) + bv[u];
        }
        (void)c0;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(o4[0], o4[1]), p1 = __floats2bfloat162_rn(o4[2], o4[3]);
        yr[lane + 32 * i] = make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
    }
}

void layernorm_bf16(const float* x, __nv_bfloat16* y, int64_t rows, int d, const float* a, const float* b, bool affine,
                    float eps, cudaStream_t st) {
    if (d % 128) fail(LP_ERR_INVALID_ARGUMENT, "layernorm: d must be a multiple of 128");
    const int per = d / 128;
    const int rev = row_order_rev();
    const unsigned g = static_cast<unsigned>((rows + 7) / 8);
#define LP_LN(P)                                                                                 \
    if (per == P) {                                                                              \
        if (affine) k_layernorm<P, true><<<g, 256, 0, st>>>(x, y, rows, d, a, b, eps, rev);      \
        else k_layernorm<P, false><<<g, 256, 0, st>>>(x, y, rows, d, a, b, eps, rev);            \
        LP_LAUNCH_CHECK();                                                                       \
        return;                                                                                  \
    }
    LP_LN(1) LP_LN(2) LP_LN(4) LP_LN(8) LP_LN(12) LP_LN(16) LP_LN(24) LP_LN(32) LP_LN(40)
#undef LP_LN
    fail(LP_ERR_INVALID_ARGUMENT, "layernorm: unsupported width");
}

// ---------------------------------------------------------------------------
// LayerNorm fold: per-matrix column sums / folded biases (one warp per output row n)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_lnfold_vec(const LnFoldJob* __restrict__ jobs) {
    const LnFoldJob j = jobs[blockIdx.y];
    const int n = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (n >= j.N) return;
    const __nv_bfloat16* w = j.W + static_cast<int64_t>(n) * j.K;
    float cs = 0.f, bo = 0.f;
    for (int k = 8 * lane; k < j.K; k += 256) {
        const uint4 u = *reinterpret_cast<const uint4*>(w + k);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float4 a0 = *reinterpret_cast<const float4*>(j.a + k), a1 = *reinterpret_cast<const float4*>(j.a + k + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(j.b + k), b1 = *reinterpret_cast<const float4*>(j.b + k + 4);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int u2 = 0; u2 < 4; ++u2) {
            const float2 wf = __bfloat1622float2(h[u2]);
            cs = fmaf(wf.x, j.plus1 ? 1.f + av[2 * u2] : av[2 * u2], cs);
            cs = fmaf(wf.y, j.plus1 ? 1.f + av[2 * u2 + 1] : av[2 * u2 + 1], cs);
            bo = fmaf(wf.x, bv[2 * u2], bo);
            bo = fmaf(wf.y, bv[2 * u2 + 1], bo);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        cs += __shfl_xor_sync(0xffffffff, cs, o);
        bo += __shfl_xor_sync(0xffffffff, bo, o);
    }
    if (lane == 0) {
        j.cs[n] = cs;
        j.bo[n] = bo + (j.bias ? j.bias[n] : 0.f);
    }
}

void lnfold_vectors(const LnFoldJob* jobs_dev, int njobs, int max_n, cudaStream_t st) {
    if (njobs <= 0) return;
    k_lnfold_vec<<<dim3(static_cast<unsigned>((max_n + 7) / 8), static_cast<unsigned>(njobs)), 256, 0, st>>>(jobs_dev);
    LP_LAUNCH_CHECK();
}

// One thread per (row, part): the part's columns in 32-value chunks, through the same
// operations as the GEMM producer epilogue (lnfold.cuh), so the partials are bit-identical.

// ---------------------------------------------------------------------------
// RMSNorm over the full width d of a [rows, ld] bf16 slice (cols [col0, col0+d)),
// times weight g, then (optionally) 3-D RoPE per 128-wide head, in place.
// RoPE (WAN2.1): head_dim 128 = 64 complex pairs; pairs [0,22) rotate with the
// frame index, [22,43) with the row, [43,64) with the column; pair j of a part
// with P pairs uses theta^(-j/P) (theta 10000), i.e. rope_params(1024, 2P).
// ---------------------------------------------------------------------------
template <int PER>
__global__ void __launch_bounds__(256) k_rmsnorm_rope(__nv_bfloat16* __restrict__ buf, int64_t rows, int64_t ld,
                                                      int64_t col0, int d, const float* __restrict__ g, float eps,
                                                      int rope, int64_t rows_per_batch, int nh, int nw) {
    const int64_t row = blockIdx.x * 8LL + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    __nv_bfloat16* p = buf + row * ld + col0;
    // lane owns pairs: element index e = 2*(lane + 32*i) for i < PER (d = 64*PER)
    float v[2 * PER];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const __nv_bfloat162 q = reinterpret_cast<const __nv_bfloat162*>(p)[lane + 32 * i];
        v[2 * i] = __bfloat162float(q.x);
        v[2 * i + 1] = __bfloat162float(q.y);
        ss += v[2 * i] * v[2 * i] + v[2 * i + 1] * v[2 * i + 1];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    const float r = rsqrtf(ss / d + eps);
    int pf = 0, py = 0, px = 0;
    if (rope) {
        const int64_t tok = row % rows_per_batch;
        px = static_cast<int>(tok % nw);
        py = static_cast<int>((tok / nw) % nh);
        pf = static_cast<int>(tok / (static_cast<int64_t>(nw) * nh));
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = 2 * (lane + 32 * i);
        float a = v[2 * i] * r * g[e], b = v[2 * i + 1] * r * g[e + 1];
        if (rope) {
            const int j = (e & 127) >> 1;  // pair within the head
            int pos, jj, P;
            if (j < 22) { pos = pf; jj = j; P = 22; }
            else if (j < 43) { pos = py; jj = j - 22; P = 21; }
            else { pos = px; jj = j - 43; P = 21; }
            const float freq = exp2f(-13.287712379549449f * static_cast<float>(jj) / static_cast<float>(P));  // 10000^(-jj/P)
            float sn, cs;
            sincosf(static_cast<float>(pos) * freq, &sn, &cs);
            const float a2 = a * cs - b * sn, b2 = a * sn + b * cs;
            a = a2;
            b = b2;
        }
        reinterpret_cast<__nv_bfloat162*>(p)[lane + 32 * i] = __floats2bfloat162_rn(a, b);
    }
}

// RoPE cos/sin table of one shard grid, computed once per forward with exactly the
// per-element formula above: [nf x 22 | nh x 21 | nw x 21] float2 (cos, sin).
__global__ void k_rope_table(float2* __restrict__ tab, int nf, int nh, int nw) {
    const int total = nf * 22 + nh * 21 + nw * 21;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        int pos, jj, P;
        if (i < nf * 22) {
            pos = i / 22, jj = i % 22, P = 22;
        } else if (i < nf * 22 + nh * 21) {
            const int k = i - nf * 22;
            pos = k / 21, jj = k % 21, P = 21;
        } else {
            const int k = i - nf * 22 - nh * 21;
            pos = k / 21, jj = k % 21, P = 21;
        }
        const float freq = exp2f(-13.287712379549449f * static_cast<float>(jj) / static_cast<float>(P));
        float sn, cs;
        sincosf(static_cast<float>(pos) * freq, &sn, &cs);
        tab[i] = make_float2(cs, sn);
    }
}

// q and k (NSEC = 2 sections of width d at col0 and col0 + d, gains g0 / g1) or one
// section: RMSNorm over d then 3-D RoPE from the table, in place.  One warp per
// (row, section); each lane moves 16-byte chunks (8 bf16 = 4 rotation pairs).
// x / d for 32-bit x < 2^31 by multiply-shift (Granlund-Montgomery; exact in that range)
struct RopeDiv {
    uint64_t mul;
    uint32_t shift, d;
};
struct RopeDivs {
    RopeDiv batch, w, h;
};
static RopeDiv make_rdiv(uint32_t d) {
    if (d == 0) d = 1;
    RopeDiv r;
    r.d = d;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    r.shift = 31 + l;
    r.mul = ((1ull << r.shift) + d - 1) / d;
    return r;
}
__device__ __forceinline__ uint32_t rdiv(uint32_t x, const RopeDiv& v) {
    return static_cast<uint32_t>((static_cast<uint64_t>(x) * v.mul) >> v.shift);
}

// RMSNorm over one (row, section) unit of d = 256 * PER8 bf16 held as PER8 16-byte chunks per
// lane (chunk i of lane l = elements 8 (l + 32 i) .. +7), then the 3-D RoPE from the table;
// transforms the chunks in place.
template <int PER8>
__device__ __forceinline__ void rms_rope_unit(uint4 (&raw)[PER8], uint32_t row, const float* __restrict__ g, float eps,
                                              const float2* __restrict__ tab, const RopeDivs& dv, int nf, int nh,
                                              int lane) {
    constexpr int d = PER8 * 256;
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < PER8; ++i) {
        const uint32_t w[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[u]));
            ss += f.x * f.x + f.y * f.y;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    const float r = rsqrtf(ss / d + eps);
    const uint32_t tok = row - rdiv(row, dv.batch) * dv.batch.d;
    const uint32_t tw_ = rdiv(tok, dv.w), pf = rdiv(tw_, dv.h);
    const int px = static_cast<int>(tok - tw_ * dv.w.d), py = static_cast<int>(tw_ - pf * dv.h.d);
    // Lane l's 8-element chunks start at 8 (l + 32 i): within a 128-wide head that is pair
    // 4 (l & 15) for every i, so the lane rotates the same 4 pairs in every head.  Their
    // (cos, sin) are loaded once per unit, with branch-free table offsets (the per-pair
    // conditional loads diverged three ways across the warp).
    float2 cs4[4] = {};
    if (tab) {
        const int j0 = 4 * (lane & 15);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u;
            const int idx = j < 22 ? static_cast<int>(pf) * 22 + j
                                   : (j < 43 ? nf * 22 + py * 21 + j - 22 : nf * 22 + nh * 21 + px * 21 + j - 43);
            cs4[u] = tab[idx];
        }
    }
#pragma unroll
    for (int i = 0; i < PER8; ++i) {
        const int e = 8 * (lane + 32 * i);
        const float4 ga = reinterpret_cast<const float4*>(g + e)[0], gb = reinterpret_cast<const float4*>(g + e)[1];
        const float gv[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        const uint32_t in[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&in[u]));
            float a = f.x * r * gv[2 * u], b = f.y * r * gv[2 * u + 1];
            if (tab) {
                const float2 cs = cs4[u];  // pair ((e & 127) >> 1) + u of the head
                const float a2 = a * cs.x - b * cs.y, b2 = a * cs.y + b * cs.x;
                a = a2;
                b = b2;
            }
            const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
            w[u] = *reinterpret_cast<const uint32_t*>(&h);
        }
        raw[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

#ifndef LP_RMS_MINB
#define LP_RMS_MINB 2  // blocks per SM of the persistent grid (ncu A/B: 2 -> 72.0 us, 3 -> 82.2, 4 -> 115.5)
#endif
template <int PER8>
__global__ void __launch_bounds__(256, LP_RMS_MINB) k_rmsnorm_rope_tab(__nv_bfloat16* __restrict__ buf, int64_t rows, int64_t ld,
                                                          int64_t col0, int nsec, const float* __restrict__ g0,
                                                          const float* __restrict__ g1, float eps,
                                                          const float2* __restrict__ tab, const RopeDivs dv,
                                                          int nf, int nh, int nw, int rev) {
    constexpr int d = PER8 * 256;
    // 32-bit index math with multiply-shift division (the host checks the ranges): the
    // former 64-bit div/mod sequences cost more issue slots than the row's arithmetic.
    // Persistent warps walk (row, section) units with a stride of all warps, and the next
    // unit's row is loaded before the current one is normalised and rotated.
    const uint32_t nwarps = gridDim.x * 8u, units = static_cast<uint32_t>(rows) * static_cast<uint32_t>(nsec);
    const int lane = threadIdx.x & 31;
    uint32_t wid = blockIdx.x * 8u + threadIdx.x / 32;
    auto unit_ptr = [&](uint32_t w) {
        if (rev) w = units - 1u - w;
        const uint32_t row = nsec == 2 ? w >> 1 : w;
        const int sec = nsec == 2 ? static_cast<int>(w & 1u) : 0;
        return reinterpret_cast<uint4*>(buf + static_cast<int64_t>(row) * ld + col0 + static_cast<int64_t>(sec) * d);
    };
    uint4 raw[PER8], nxt[PER8];
    if (wid < units) {
        const uint4* p0 = unit_ptr(wid);
#pragma unroll
        for (int i = 0; i < PER8; ++i) nxt[i] = p0[lane + 32 * i];
    }
    for (; wid < units; wid += nwarps) {
        const uint32_t u = rev ? units - 1u - wid : wid;
        const uint32_t row = nsec == 2 ? u >> 1 : u;
        const int sec = nsec == 2 ? static_cast<int>(u & 1u) : 0;
        uint4* p = unit_ptr(wid);
        const float* g = sec ? g1 : g0;
#pragma unroll
        for (int i = 0; i < PER8; ++i) raw[i] = nxt[i];
        if (wid + nwarps < units) {
            const uint4* pn = unit_ptr(wid + nwarps);
#pragma unroll
            for (int i = 0; i < PER8; ++i) nxt[i] = pn[lane + 32 * i];
        }
        rms_rope_unit<PER8>(raw, row, g, eps, tab, dv, nf, nh, lane);
#pragma unroll
        for (int i = 0; i < PER8; ++i) p[lane + 32 * i] = raw[i];
    }
}

// out[r, c] = bf16(in[r, c] * g[c]) — the cross-attention q RMSNorm's per-channel weight folded
// into the cached text K (dit.cpp, knob dit_xq_rms)
__global__ void __launch_bounds__(256) k_scale_cols_bf16(const __nv_bfloat16* __restrict__ in, int64_t n, int d,
                                                         const float* __restrict__ g, __nv_bfloat16* __restrict__ out) {
    for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * 256)
        out[i] = __float2bfloat16_rn(__bfloat162float(in[i]) * g[i % d]);
}
void scale_cols_bf16(const __nv_bfloat16* in, int64_t rows, int d, const float* g, __nv_bfloat16* out, cudaStream_t st) {
    const int64_t n = rows * d;
    k_scale_cols_bf16<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(in, n, d, g, out);
    LP_LAUNCH_CHECK();
}

void rope_table(float2* tab, int nf, int nh, int nw, cudaStream_t st) {
    const int total = nf * 22 + nh * 21 + nw * 21;
    k_rope_table<<<(total + 255) / 256, 256, 0, st>>>(tab, nf, nh, nw);
    LP_LAUNCH_CHECK();
}

bool rmsnorm_rope_tab(__nv_bfloat16* buf, int64_t rows, int64_t ld, int64_t col0, int d, int nsec, const float* g0,
                      const float* g1, float eps, const float2* tab, int64_t rows_per_batch, int nf, int nh, int nw,
                      cudaStream_t st) {
    if (d % 256 || (ld % 8) || (col0 % 8) || (nsec != 1 && nsec != 2)) return false;
    if (rows * nsec >= (1ll << 31) || rows_per_batch >= (1ll << 31)) return false;
    RopeDivs dv;
    dv.batch = make_rdiv(static_cast<uint32_t>(rows_per_batch));
    dv.w = make_rdiv(static_cast<uint32_t>(nw));
    dv.h = make_rdiv(static_cast<uint32_t>(nh));
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned gr = static_cast<unsigned>(std::min<int64_t>((rows * nsec + 7) / 8, static_cast<int64_t>(sms) * LP_RMS_MINB));
    const int rev = row_order_rev();
#define LP_RMT(P)                                                                                                   \
    if (d == 256 * P) {                                                                                             \
        k_rmsnorm_rope_tab<P><<<gr, 256, 0, st>>>(buf, rows, ld, col0, nsec, g0, g1, eps, tab, dv, nf, nh, nw, rev); \
        LP_LAUNCH_CHECK();                                                                                          \
        return true;                                                                                                \
    }
    LP_RMT(1) LP_RMT(2) LP_RMT(4) LP_RMT(6) LP_RMT(8) LP_RMT(20)
#undef LP_RMT
    return false;
}

void rmsnorm_rope(__nv_bfloat16* buf, int64_t rows, int64_t ld, int64_t col0, int d, const float* g, float eps,
                  bool rope, int64_t rows_per_batch, int nh, int nw, cudaStream_t st) {
    if (d % 64) fail(LP_ERR_INVALID_ARGUMENT, "rmsnorm: d must be a multiple of 64");
    const int per = d / 64;
    const unsigned gr = static_cast<unsigned>((rows + 7) / 8);
#define LP_RMS(P)                                                                                               \
    if (per == P) {                                                                                             \
        k_rmsnorm_rope<P><<<gr, 256, 0, st>>>(buf, rows, ld, col0, d, g, eps, rope ? 1 : 0, rows_per_batch, nh, nw); \
        LP_LAUNCH_CHECK();                                                                                      \
        return;                                                                                                 \
    }
    LP_RMS(1) LP_RMS(2) LP_RMS(4) LP_RMS(8) LP_RMS(16) LP_RMS(24) LP_RMS(32) LP_RMS(48) LP_RMS(64) LP_RMS(80)
#undef LP_RMS
    fail(LP_ERR_INVALID_ARGUMENT, "rmsnorm: unsupported width");
}

// ---------------------------------------------------------------------------
// head output [2*ntok, C*pt*ph*pw] fp32 (feature = ((kt*ph + kh)*pw + kw)*C + c)
// -> unpatchify, crop, CFG: eps = q(u + w (c - u)) with u, c quantized first
// (cfg_predict, src/denoise.cpp:24-39), fp64 combine, stored in the storage dtype.
// ---------------------------------------------------------------------------
template <int D>
__global__ void k_unpatchify_cfg(const float* __restrict__ head, typename Store<D>::T* __restrict__ eps, int C, int F,
                                 int H, int W, int pt, int ph, int pw, int nh, int nw, int64_t ntok, double w,
                                 int single, const __grid_constant__ EpsMirrors mr) {
    using T = typename Store<D>::T;
    const int64_t total = static_cast<int64_t>(C) * F * H * W;
    const int feat = C * pt * ph * pw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = static_cast<int>(i % W);
        const int y = static_cast<int>((i / W) % H);
        const int t = static_cast<int>((i / (static_cast<int64_t>(W) * H)) % F);
        const int c = static_cast<int>(i / (static_cast<int64_t>(W) * H * F));
        const int64_t tok = (static_cast<int64_t>(t / pt) * nh + y / ph) * nw + x / pw;
        const int fe = (((t % pt) * ph + (y % ph)) * pw + (x % pw)) * C + c;
        const double u = quantize_dev<D>(static_cast<double>(head[tok * feat + fe]));
        T q;
        if (single) {  // one CFG pass (Denoiser::predict): the prediction, quantized
            store_q<D>(&q, 0, u);
        } else {
            const double cc = quantize_dev<D>(static_cast<double>(head[(ntok + tok) * feat + fe]));
            store_q<D>(&q, 0, __dadd_rn(u, __dmul_rn(w, __dsub_rn(cc, u))));
        }
        eps[i] = q;
        // K8+K9 fused: the same ε̂ element stored straight into every peer's gather buffer
        // (CUDA-IPC mapped; remote stores over NVLink), at the same offset as the local slot
        for (int j = 0; j < mr.n; ++j) reinterpret_cast<T*>(reinterpret_cast<char*>(eps + i) + mr.delta[j])[0] = q;
    }
    if (mr.n) __threadfence_system();
}

void unpatchify_cfg(const float* head, int dtype, const int shape[4], const int patch[3], double w, void* eps,
                    cudaStream_t st, const EpsMirrors& mr, bool single) {
    const int nh = (shape[2] + patch[1] - 1) / patch[1], nw = (shape[3] + patch[2] - 1) / patch[2];
    const int nf = (shape[1] + patch[0] - 1) / patch[0];
    const int64_t ntok = static_cast<int64_t>(nf) * nh * nw;
    const int64_t total = static_cast<int64_t>(shape[0]) * shape[1] * shape[2] * shape[3];
    const int g = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
#define LP_UNP(DD) k_unpatchify_cfg<DD><<<g, 256, 0, st>>>(head, static_cast<typename Store<DD>::T*>(eps), shape[0], shape[1], shape[2], shape[3], patch[0], patch[1], patch[2], nh, nw, ntok, w, single ? 1 : 0, mr)
    if (dtype == 2) LP_UNP(2);
    else if (dtype == 4) LP_UNP(4);
    else LP_UNP(8);
#undef LP_UNP
    LP_LAUNCH_CHECK();
}

}  // namespace lpb200
