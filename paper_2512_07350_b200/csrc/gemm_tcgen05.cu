// gemm_tcgen05.cu — persistent, warp-specialized tcgen05 GEMM for sm_100a.
//
//   D[M,N] = epilogue( A[M,K] · B[N,K]^T )      A, B bf16, K-major (row-major, K contiguous)
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one lane),
// warps 2..5 = epilogue (TMEM -> registers -> global), warp 2 also owns TMEM.
// Tiles 128 x BN x 64 (BN = 256/128/64), 4-stage smem ring fed by TMA with
// 128-byte swizzle, accumulators double-buffered in TMEM (2 x BN columns) so
// the epilogue of tile i overlaps the MMAs of tile i+1.  Raster: consecutive
// tiles walk N first, so the 148 co-resident CTAs share A rows through L2 and
// the whole weight matrix stays L2-resident.
//
// Epilogues fused into the DiT's dense layers:
//   BF16       out_bf16 = acc + bias
//   BF16_GELU  out_bf16 = gelu_tanh(acc + bias)          (FFN1)
//   F32_RESID  x_f32   += (acc + bias) * gate[col]       (attn-O / FFN2 gated residual)
//   F32        out_f32  = acc + bias                      (head)
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dit_ops.hpp"
#include "lnfold.cuh"
#include "tc_ptx.cuh"

namespace lpb200 {

using namespace tc;

// ---------------------------------------------------------------------------
// TMA descriptors (host)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) fail(LP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                              uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LP_ERR_CUDA, "cuTensorMapEncodeTiled(2d) failed: " + std::to_string(r));
    return m;
}

// Output / residual map of the TMA-staged epilogue: [rows, cols] of fp32 or bf16 with a
// 32 x 32 box; the box's inner extent is 128 B (fp32, 128B swizzle) or 64 B (bf16, 64B swizzle).
static CUtensorMap make_tmap_epi(void* base, bool f32, uint64_t cols, uint64_t rows, uint64_t ld_elems) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {ld_elems * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base,
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LP_ERR_CUDA, "cuTensorMapEncodeTiled(epilogue) failed: " + std::to_string(r));
    return m;
}

CUtensorMap make_tmap_3d_bf16(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                              uint32_t b0, uint32_t b1, uint32_t b2) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {s1, s2};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LP_ERR_CUDA, "cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
    return m;
}

// Plain 2-D map of 2/4/8-byte elements (no swizzle, zero OOB fill): K1's TMA-staged gather.
// Returns false when the driver rejects the geometry (stride or box not 16-B multiples).
bool make_tmap_2d_raw(CUtensorMap* m, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                      uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                   : elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                                     : CU_TENSOR_MAP_DATA_TYPE_INT64;
    return encode_fn()(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------
// Kernel
// ---------------------------------------------------------------------------
constexpr int kBM = 128, kBK = 64, kStages = 4, kGemmThreads = 192;

template <int BN>
constexpr int gemm_smem_bytes() {
    return kStages * (kBM * kBK * 2 + BN * kBK * 2) + 1024 /*align*/ + 256 /*barriers*/;
}

// GELU-tanh of a pair with packed f32x2 math: gelu(x) = hx + hx * tanh(x * (k0 + k0 k1 x^2)),
// hx = x / 2 — three FMUL2/FFMA2 for the argument and one FFMA2 for the result per pair,
// against ~12 scalar operations (knob-free; A/B build flag LP_GELU_SCALAR)
__device__ __forceinline__ float2 gelu_tanh2(float2 x) {
    const float2 x2 = __fmul2_rn(x, x);
    const float2 in = __ffma2_rn(x2, make_float2(0.7978845608028654f * 0.044715f, 0.7978845608028654f * 0.044715f),
                                 make_float2(0.7978845608028654f, 0.7978845608028654f));
    const float2 u = __fmul2_rn(x, in);
    float2 t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t.x) : "f"(u.x));
    asm("tanh.approx.f32 %0, %1;" : "=f"(t.y) : "f"(u.y));
    const float2 hx = __fmul2_rn(x, make_float2(0.5f, 0.5f));
    return __ffma2_rn(hx, t, hx);
}
__device__ __forceinline__ float gelu_tanh(float x) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
    return 0.5f * x * (1.f + t);
}

// one thread's 32 accumulator columns of row `row` -> fused epilogue store
template <int MODE>
__device__ __forceinline__ void epilogue_store(const GemmEpilogue& ep, int row, int col0, const uint32_t (&r)[32]) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) + (ep.bias ? __ldg(ep.bias + col0 + j) : 0.f);
    if (MODE == EPI_BF16 || MODE == EPI_BF16_GELU) {
        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
        uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = MODE == EPI_BF16_GELU ? gelu_tanh(v[8 * j + u]) : v[8 * j + u];
            o4[j] = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
        }
    } else {
        float* o = static_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
        float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float4 x;
            if (MODE == EPI_F32_RESID) {
                x = o4[j];
                const float* g = ep.gate ? ep.gate + col0 + 4 * j : nullptr;
                x.x += v[4 * j + 0] * (g ? __ldg(g + 0) : 1.f);
                x.y += v[4 * j + 1] * (g ? __ldg(g + 1) : 1.f);
                x.z += v[4 * j + 2] * (g ? __ldg(g + 2) : 1.f);
                x.w += v[4 * j + 3] * (g ? __ldg(g + 3) : 1.f);
            } else {
                x = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            o4[j] = x;
        }
    }
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, GemmEpilogue ep, int M,
           int N, int K) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = kBM * kBK * 2, B_BYTES = BN * kBK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * B_BYTES);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int num_n = N / BN, num_m = (M + kBM - 1) / kBM, tiles = num_m * num_n;
    const int nk = (K + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma);
        tma_prefetch(&tmb);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512))));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int mb = t / num_n, nb = t % num_n;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
                    tma_load_2d(&tma, &full[s], sA + s * A_BYTES, kb * kBK, mb * kBM);
                    tma_load_2d(&tmb, &full[s], sB + s * B_BYTES, kb * kBK, nb * BN);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // converged MMA-issue warp, one elected lane issues (see k_gemm2)
        const bool leader = elect_one();
        constexpr uint32_t idesc = idesc_bf16(kBM, BN);
        const uint64_t dA = desc_sw128(smem_u32(sA)), dB = desc_sw128(smem_u32(sB));
        int s = 0;
        uint32_t ph = 0;
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            mbar_wait(&tempty[acc], aph ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            for (int kb = 0; kb < nk; ++kb) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                if (leader) {
                    const uint64_t a0 = dA + static_cast<uint64_t>(s * A_BYTES >> 4);
                    const uint64_t b0 = dB + static_cast<uint64_t>(s * B_BYTES >> 4);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) mma_ss(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
                    mma_commit(&empty[s]);
                }
                __syncwarp();
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
            if (leader) mma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else {
        // epilogue: warps 2..5 -> TMEM lane quadrant warp % 4
        const uint32_t q = warp & 3;
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            const int mb = t / num_n, nb = t % num_n;
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = mb * kBM + q * 32 + lane;
            const uint32_t taddr = tmem + ((q * 32) << 16) + acc * BN;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld32(taddr + c, r);
                tmem_ld_wait();
                if (row < M) epilogue_store<MODE>(ep, row, nb * BN + c, r);
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512))));
}

// ---------------------------------------------------------------------------
// TMA-staged epilogue (CTA-pair kernel).  Each epilogue warp owns 32 accumulator rows; per
// 32-column chunk it writes its 32 x 32 block into a swizzled shared-memory box and ONE
// lane issues a TMA tensor store of the box — full 128-B lines, no per-row LSU traffic.  The
// fp32 residual epilogue first TMA-loads the x box into the same buffer, one chunk AHEAD
// (double-buffered per warp, the chunk sequence runs across tiles), so the load overlaps
// the previous chunk.  Swizzle (matches the tensor maps): fp32 rows are 128 B, 16-B unit
// j of row r sits at unit j ^ (r & 7); bf16 rows are 64 B, unit j at j ^ ((r >> 1) & 3) —
// a lane-per-row access then spreads over all banks (4 wavefronts per 512 B).
// ---------------------------------------------------------------------------
constexpr int kEpiBox = 4096;  // one 32 x 32 fp32 box (bf16 uses the first 2 KB)
#ifndef LP_EPI_LSU
constexpr bool kEpiTma = true;
#else
constexpr bool kEpiTma = false;  // A/B build: thread-per-row LSU stores
#endif

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_u32(smem)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_cta(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(smem)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// Per-row LayerNorm state of the LN-fold epilogue (one lane = one row of the tile).
struct LnRow {
    float mean = 0.f, rstd = 1.f;  // consumer: the row's LayerNorm statistics
    LnAcc acc;                    // producer: partials over this tile's chunks
    float rms[4] = {0.f, 0.f, 0.f, 0.f};  // BF16 rms_out: sum of squares of the written bf16 values
};

template <int MODE, bool XQ = false>
__device__ __forceinline__ void epi_chunk_smem(const GemmEpilogue& ep, int col0, const uint32_t (&r)[32], uint8_t* box,
                                               LnRow& ln, int chunk, uint8_t* xqbox = nullptr) {
    const uint32_t lane = lane_id();
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        const float4 b = ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
        float a0 = __uint_as_float(r[j]), a1 = __uint_as_float(r[j + 1]), a2 = __uint_as_float(r[j + 2]),
              a3 = __uint_as_float(r[j + 3]);
        if ((MODE == EPI_BF16 || MODE == EPI_BF16_GELU) && ep.stats_in) {
            // LN folded into this GEMM: A was bf16(x * g), so acc - mean * cs = sum_k (x_k - mean) g_k W_nk
            const float4 c = __ldg(reinterpret_cast<const float4*>(ep.cs + col0 + j));
            a0 = ln.rstd * fmaf(-ln.mean, c.x, a0);
            a1 = ln.rstd * fmaf(-ln.mean, c.y, a1);
            a2 = ln.rstd * fmaf(-ln.mean, c.z, a2);
            a3 = ln.rstd * fmaf(-ln.mean, c.w, a3);
        }
        v[j] = a0 + b.x;
        v[j + 1] = a1 + b.y;
        v[j + 2] = a2 + b.z;
        v[j + 3] = a3 + b.w;
    }
    if (MODE == EPI_BF16 || MODE == EPI_BF16_GELU) {
        uint8_t* row = box + lane * 64;
        if (MODE == EPI_BF16 && ep.rms_out) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float q = __bfloat162float(__float2bfloat16_rn(v[j]));
                ln.rms[j & 3] = fmaf(q, q, ln.rms[j & 3]);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float a[8];
#ifndef LP_GELU_SCALAR
            if (MODE == EPI_BF16_GELU) {
#pragma unroll
                for (int u = 0; u < 8; u += 2) {
                    const float2 g = gelu_tanh2(make_float2(v[8 * j + u], v[8 * j + u + 1]));
                    a[u] = g.x;
                    a[u + 1] = g.y;
                }
            } else
#endif
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = MODE == EPI_BF16_GELU ? gelu_tanh(v[8 * j + u]) : v[8 * j + u];
            *reinterpret_cast<uint4*>(row + ((j ^ ((lane >> 1) & 3)) << 4)) =
                make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
        }
    } else {
        uint8_t* row = box + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float4* p = reinterpret_cast<float4*>(row + ((j ^ (lane & 7)) << 4));
            float4 x;
            if (MODE == EPI_F32_RESID) {
                x = *p;
                const float4 g = ep.gate ? __ldg(reinterpret_cast<const float4*>(ep.gate + col0 + 4 * j))
                                         : make_float4(1.f, 1.f, 1.f, 1.f);
                x.x += v[4 * j] * g.x;
                x.y += v[4 * j + 1] * g.y;
                x.z += v[4 * j + 2] * g.z;
                x.w += v[4 * j + 3] * g.w;
            } else {
                x = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            *p = x;
            v[4 * j] = x.x;  // v now holds the chunk's x (LN-fold producer below)
            v[4 * j + 1] = x.y;
            v[4 * j + 2] = x.z;
            v[4 * j + 3] = x.w;
        }
        if (XQ) {
            // LayerNorm partials of this chunk's 32 values (lnfold.cuh), and xq = bf16(x * g)
            // into this chunk's 32 x 32 bf16 staging box (64-byte rows, the bf16 output layout),
            // TMA-stored by the caller next to the x box
            ln_acc_chunk(v, chunk, ln.acc);
            uint8_t* row = xqbox + lane * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float g[8];
                *reinterpret_cast<float4*>(g) = __ldg(reinterpret_cast<const float4*>(ep.g + col0 + 8 * j));
                *reinterpret_cast<float4*>(g + 4) = __ldg(reinterpret_cast<const float4*>(ep.g + col0 + 8 * j + 4));
                *reinterpret_cast<uint4*>(row + ((j ^ ((lane >> 1) & 3)) << 4)) = ln_xq8(v + 8 * j, g, ep.g_plus1);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a 2-CTA cluster computes a 256 x BN tile with
// one UMMA_M = 256 instruction stream issued by the leader CTA.  Each CTA TMA-loads
// its own 128 rows of A and BN/2 rows of B (half the B bytes per SM of the 1-CTA
// kernel), both CTAs' loads complete on the leader's full barrier, and commits are
// multicast to both CTAs.  Each CTA's TMEM holds its 128 accumulator rows.
// ---------------------------------------------------------------------------
// Epilogue staging boxes per warp: the fp32 residual epilogue keeps NB = 4 (two residual
// loads in flight ahead of the chunk being combined) and gives up one mainloop stage for it.
#ifndef LP_EPI_RESID_BOXES
#define LP_EPI_RESID_BOXES 4
#endif
#ifndef LP_EPI_RESID_DIST
#define LP_EPI_RESID_DIST 2
#endif
// Accumulator-free handshake of the CTA-pair kernel: after its last TMEM read of a tile, each
// epilogue warp (LP_TEMPTY_WARP=1, default) arrives once on the leader's tempty barrier with
// the plain remote arrive; 0: every thread arrives with release.cluster semantics (a
// cluster-scope fence per thread and tile — ncu: "membar" stalls).
#ifndef LP_TEMPTY_WARP
#define LP_TEMPTY_WARP 1
#endif
constexpr bool kTemptyWarp = LP_TEMPTY_WARP != 0;
__device__ __forceinline__ void tempty_arrive(uint64_t* bar) {
    if (kTemptyWarp) {
        __syncwarp();
        if (lane_id() == 0) mbar_arrive_remote(bar, 0);
    } else {
        mbar_arrive_cluster(bar, 0);
    }
}
// CTA-pair kernel barrier waits: spinning try_wait (default) or try_wait with a suspend-time
// hint, which parks the waiting warp instead of spending issue slots of the SMSP it shares
// with an epilogue warp (A/B build flag LP_GEMM_WAIT_SLEEP)
#ifndef LP_GEMM_WAIT_SLEEP
#define LP_GEMM_WAIT_SLEEP 0
#endif
__device__ __forceinline__ void gwait(uint64_t* bar, uint32_t parity) {
    if (LP_GEMM_WAIT_SLEEP) mbar_wait_sleep(bar, parity);
    else mbar_wait(bar, parity);
}
template <int MODE>
constexpr int epi_boxes() { return kEpiTma ? (MODE == EPI_F32_RESID ? LP_EPI_RESID_BOXES : 2) : 0; }
// XQ (LayerNorm-fold producer): two extra 2 KB bf16 boxes per epilogue warp for xq, paid for
// with one mainloop stage
constexpr int kXqBox = 2048;
// KSUB: 64-wide K sub-blocks per pipeline stage.  KSUB = 2 halves the mainloop's barrier
// checks and commits per FLOP (8 MMAs per full-barrier wait instead of 4: every check is a
// tensor-pipe bubble, the issue being nearly synchronous) at the same bytes in flight
// (half as many stages of twice the size).  Knob gemm_ksub; bf16-output epilogues only.
template <int BN, int MODE = EPI_BF16, bool XQ = false, int KSUB = 1>
constexpr int gemm2_stages() {
    return ((BN == 256 ? 6 : 8) - (epi_boxes<MODE>() > 2 ? (BN == 256 ? 1 : 2) : 0) - (XQ ? 1 : 0)) / KSUB;
}
template <int BN, int MODE, bool XQ = false, int KSUB = 1>
constexpr int gemm2_smem_bytes() {
    return gemm2_stages<BN, MODE, XQ, KSUB>() * KSUB * (kBM * kBK * 2 + (BN / 2) * kBK * 2) + 1024 + 512 +
           4 * epi_boxes<MODE>() * kEpiBox + (XQ ? 4 * 2 * kXqBox : 0);
}

template <int BN, int MODE, bool XQ = false, int KSUB = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    k_gemm2(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
            const __grid_constant__ CUtensorMap tmo, const __grid_constant__ CUtensorMap tmq, GemmEpilogue ep, int M,
            int N, int K) {
    constexpr int S = gemm2_stages<BN, MODE, XQ, KSUB>();
    constexpr int NB = epi_boxes<MODE>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_SUB = kBM * kBK * 2, B_SUB = (BN / 2) * kBK * 2;
    constexpr int A_BYTES = KSUB * A_SUB, B_BYTES = KSUB * B_SUB;
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * A_BYTES;
    uint8_t* sE = sB + S * B_BYTES;  // [4 epilogue warps][NB][kEpiBox] (1024-aligned)
    uint8_t* sX = sE + 4 * NB * kEpiBox;  // [4 epilogue warps][2][kXqBox] (XQ)
    uint64_t* full = reinterpret_cast<uint64_t*>(sX + (XQ ? 4 * 2 * kXqBox : 0));
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* ebar = tempty + 2;  // [4 warps][4] residual-box loads
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + 16);

    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int num_n = N / BN, num_m = (M + 2 * kBM - 1) / (2 * kBM), tiles = num_m * num_n;
    const int nk = (K + KSUB * kBK - 1) / (KSUB * kBK);  // stages per tile (a ragged K tail is zero-filled)

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma);
        tma_prefetch(&tmb);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            // both CTAs' epilogue warps (LP_TEMPTY_WARP: one arrive per warp) or threads arrive
            // on the leader's
            mbar_init(&tempty[a], kTemptyWarp ? 8 : 256);
        }
        for (int b = 0; b < 16; ++b) mbar_init(&ebar[b], 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_2sm(tmem_slot, 2 * BN);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = cluster; t < tiles; t += nclusters) {
                const int mb = t / num_n, nb = t % num_n;
                for (int kb = 0; kb < nk; ++kb) {
                    gwait(&empty[s], ph ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
#pragma unroll
                    for (int u = 0; u < KSUB; ++u) {
                        const int kc = (kb * KSUB + u) * kBK;
                        tma_load_2d_2sm(&tma, &full[s], sA + s * A_BYTES + u * A_SUB, kc, mb * 2 * kBM + rank * kBM);
                        tma_load_2d_2sm(&tmb, &full[s], sB + s * B_BYTES + u * B_SUB, kc, nb * BN + rank * (BN / 2));
                    }
                    if (++s == S) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // MMA issuer (leader CTA): the whole warp runs the loop converged — barrier checks are
        // warp-wide, descriptors stay in uniform registers — and one elected lane issues.
        // tcgen05.mma issue is nearly synchronous with execution, so a check from a lone
        // divergent lane costs ~100 pipe cycles per k-block (scripts/micro/mma_bench.py).
        if (rank == 0) {
            const bool leader = elect_one();
            constexpr uint32_t idesc = idesc_bf16(2 * kBM, BN);
            const uint64_t dA = desc_sw128(smem_u32(sA)), dB = desc_sw128(smem_u32(sB));
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int t = cluster; t < tiles; t += nclusters, ++it) {
                const int acc = it & 1;
                const uint32_t aph = (it >> 1) & 1;
                gwait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    gwait(&full[s], ph);
                    tc_fence_after();
                    if (leader) {
                        const uint64_t a0 = dA + static_cast<uint64_t>(s * A_BYTES >> 4);
                        const uint64_t b0 = dB + static_cast<uint64_t>(s * B_BYTES >> 4);
#pragma unroll
                        for (int u = 0; u < KSUB; ++u)
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k)  // +32 B per K=16 inside a sub-block
                                mma_ss_2sm(d, a0 + (u * A_SUB >> 4) + 2 * k, b0 + (u * B_SUB >> 4) + 2 * k, idesc,
                                           (kb | u | k) != 0);
                        mma_commit_2sm(&empty[s], 0x3);
                    }
                    __syncwarp();
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                if (leader) mma_commit_2sm(&tfull[acc], 0x3);
                __syncwarp();
            }
        }
    } else if (kEpiTma) {
        const uint32_t q = warp & 3;
        uint8_t* boxes = sE + q * NB * kEpiBox;
        uint64_t* wbar = ebar + q * 4;
        constexpr int NCH = BN / 32;
        constexpr bool RESID = MODE == EPI_F32_RESID;
        constexpr int DIST = RESID ? LP_EPI_RESID_DIST : 0;  // residual loads in flight ahead of the chunk combined
        static_assert(!RESID || (DIST >= 1 && DIST < NB), "residual lookahead must fit the boxes");
        uint32_t lph[4] = {0, 0, 0, 0};
        // chunk sequence u = (tile, chunk) in processing order, buffer u % NB.  Residual boxes
        // are TMA-loaded DIST chunks ahead (the load cursor runs across tiles); a buffer is
        // reloaded once the store from it (chunk u - NB + DIST... = u-2) has been read.
        int lt = cluster, lc = 0, lu = 0;
        auto issue_next = [&]() {
            if (lt >= tiles) return;
            const int b = lu % NB;
            if (lane == 0) {
                bulk_wait_read<(NB - DIST - 1 > 0 ? NB - DIST - 1 : 0)>();  // the last store from buffer b has been read
                mbar_arrive_expect_tx(&wbar[b], kEpiBox);
                tma_load_2d_cta(&tmo, &wbar[b], boxes + b * kEpiBox, (lt % num_n) * BN + lc * 32,
                                (lt / num_n) * 2 * kBM + rank * kBM + q * 32);
            }
            if (++lc == NCH) {
                lc = 0;
                lt += nclusters;
            }
            ++lu;
        };
        if (RESID)
            for (int d = 0; d < DIST; ++d) issue_next();
        int u = 0;
        int it = 0;
        for (int t = cluster; t < tiles; t += nclusters, ++it) {
            const int mb = t / num_n, nb = t % num_n;
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            gwait(&tfull[acc], aph);
            tc_fence_after();
            const int row0 = mb * 2 * kBM + rank * kBM + q * 32;
            const uint32_t taddr = tmem + ((q * 32) << 16) + acc * BN;
            const int my_row = row0 + static_cast<int>(lane);
            LnRow ln;
            if ((MODE == EPI_BF16 || MODE == EPI_BF16_GELU) && ep.stats_in && my_row < M) {
                // the row's LayerNorm statistics from its producer partials (equal counts)
                const float2* sp = ep.stats_in + static_cast<int64_t>(my_row) * ep.parts;
                float ms = 0.f;
                for (int i = 0; i < ep.parts; ++i) ms += sp[i].x;
                const float mean = ms / static_cast<float>(ep.parts);
                float m2 = 0.f;
                for (int i = 0; i < ep.parts; ++i) {
                    const float2 pi = sp[i];
                    const float dlt = pi.x - mean;
                    m2 += pi.y + ep.cols_per_part * dlt * dlt;
                }
                ln.mean = mean;
                ln.rstd = rsqrtf(m2 / (ep.cols_per_part * static_cast<float>(ep.parts)) + ep.eps);
            }
#pragma unroll 1
            for (int c = 0; c < NCH; ++c, ++u) {
                const int b = u % NB;
                uint32_t r[32];
                tmem_ld32(taddr + c * 32, r);
                if (RESID) {
                    issue_next();  // chunk u + DIST
                    mbar_wait(&wbar[b], lph[b]);
                    lph[b] ^= 1;
                } else if (lane == 0) {
                    bulk_wait_read<1>();  // the store issued from this buffer two chunks ago has read it
                }
                // XQ: xq box u % 2 was last stored at chunk u - 2 (issue_next waits for that
                // except at the very tail, where it issues no load)
                if (XQ && RESID && lane == 0) bulk_wait_read<1>();
                __syncwarp();
                tmem_ld_wait();
                // xq box u % 2: its last store (chunk u - 2) has been read — the wait above
                // leaves at most one store group (chunk u - 1) in flight
                uint8_t* xqb = sX + (q * 2 + (u & 1)) * kXqBox;
                epi_chunk_smem<MODE, XQ>(ep, nb * BN + c * 32, r, boxes + b * kEpiBox, ln, c, xqb);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmo, boxes + b * kEpiBox, nb * BN + c * 32, row0);
                    if (XQ) tma_store_2d(&tmq, xqb, nb * BN + c * 32, row0);
                    bulk_commit();
                }
            }
            if (XQ && my_row < M)
                ep.stats_out[static_cast<int64_t>(my_row) * num_n + nb] = ln_acc_final(ln.acc, static_cast<float>(BN));
            if (MODE == EPI_BF16 && ep.rms_out && my_row < M)
                ep.rms_out[static_cast<int64_t>(my_row) * num_n + nb] = (ln.rms[0] + ln.rms[1]) + (ln.rms[2] + ln.rms[3]);
            tc_fence_before();
            tempty_arrive(&tempty[acc]);
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    } else {
        const uint32_t q = warp & 3;
        int it = 0;
        for (int t = cluster; t < tiles; t += nclusters, ++it) {
            const int mb = t / num_n, nb = t % num_n;
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = mb * 2 * kBM + rank * kBM + q * 32 + lane;
            const uint32_t taddr = tmem + ((q * 32) << 16) + acc * BN;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld32(taddr + c, r);
                tmem_ld_wait();
                if (row < M) epilogue_store<MODE>(ep, row, nb * BN + c, r);
            }
            tc_fence_before();
            tempty_arrive(&tempty[acc]);
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) tmem_dealloc_2sm(tmem, 2 * BN);
}

// ---------------------------------------------------------------------------
// Host launch
// ---------------------------------------------------------------------------
static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

template <int BN, int MODE>
static void launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmEpilogue& ep, int M, int N, int K,
                        cudaStream_t st) {
    constexpr int smem = gemm_smem_bytes<BN>();
    static bool attr = false;
    if (!attr) {
        LP_CUDA(cudaFuncSetAttribute(k_gemm<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    const int tiles = ((M + kBM - 1) / kBM) * (N / BN);
    const int grid = tiles < num_sms() ? tiles : num_sms();
    k_gemm<BN, MODE><<<grid, kGemmThreads, smem, st>>>(ta, tb, ep, M, N, K);
    LP_LAUNCH_CHECK();
}

template <int BN, int MODE, bool XQ, int KSUB = 1>
static void launch_gemm2_x(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& tq,
                           const GemmEpilogue& ep, int M, int N, int K, cudaStream_t st) {
    if constexpr (KSUB == 1 && BN == 256 && !XQ && (MODE == EPI_BF16 || MODE == EPI_BF16_GELU)) {
        if (tune_get("gemm_ksub", 1) == 2 && K % (2 * kBK) == 0) {
            launch_gemm2_x<BN, MODE, XQ, 2>(ta, tb, to, tq, ep, M, N, K, st);
            return;
        }
    }
    constexpr int smem = gemm2_smem_bytes<BN, MODE, XQ, KSUB>();
    static bool attr = false;
    if (!attr) {
        LP_CUDA(cudaFuncSetAttribute(k_gemm2<BN, MODE, XQ, KSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    const int tiles = ((M + 2 * kBM - 1) / (2 * kBM)) * (N / BN);
    const int clusters = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
    k_gemm2<BN, MODE, XQ, KSUB><<<2 * clusters, kGemmThreads, smem, st>>>(ta, tb, to, tq, ep, M, N, K);
    LP_LAUNCH_CHECK();
}

template <int BN, int MODE>
static void launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, const GemmEpilogue& ep, int M, int N, int K,
                         cudaStream_t st) {
    const CUtensorMap to = make_tmap_epi(ep.out, MODE >= EPI_F32_RESID, static_cast<uint64_t>(N), static_cast<uint64_t>(M),
                                         static_cast<uint64_t>(ep.ldo));
    if constexpr (MODE >= EPI_F32_RESID && kEpiTma) {
        if (ep.xq) {  // LayerNorm-fold producer: xq (bf16, 32 x 32 boxes) stored by TMA next to x
            const CUtensorMap tq = make_tmap_epi(ep.xq, false, static_cast<uint64_t>(N), static_cast<uint64_t>(M),
                                                 static_cast<uint64_t>(ep.ldq));
            launch_gemm2_x<BN, MODE, true>(ta, tb, to, tq, ep, M, N, K, st);
            return;
        }
    }
    launch_gemm2_x<BN, MODE, false>(ta, tb, to, to, ep, M, N, K, st);
}

static int gemm_variant() { return tune_get("gemm_2sm", 1); }

template <int MODE>
static void gemm_bn(const CUtensorMap& ta, const void* B, int64_t ldb, const GemmEpilogue& ep, int M, int N, int K,
                    cudaStream_t st) {
    if (gemm_variant() && M > kBM && (N % 256 == 0 || N % 128 == 0)) {
        if (N % 256 == 0) {
            const CUtensorMap tb = make_tmap_2d_bf16(B, K, N, ldb * 2, kBK, 128);
            launch_gemm2<256, MODE>(ta, tb, ep, M, N, K, st);
        } else {
            const CUtensorMap tb = make_tmap_2d_bf16(B, K, N, ldb * 2, kBK, 64);
            launch_gemm2<128, MODE>(ta, tb, ep, M, N, K, st);
        }
        return;
    }
    if (N % 256 == 0) {
        const CUtensorMap tb = make_tmap_2d_bf16(B, K, N, ldb * 2, kBK, 256);
        launch_gemm<256, MODE>(ta, tb, ep, M, N, K, st);
    } else if (N % 128 == 0) {
        const CUtensorMap tb = make_tmap_2d_bf16(B, K, N, ldb * 2, kBK, 128);
        launch_gemm<128, MODE>(ta, tb, ep, M, N, K, st);
    } else if (N % 64 == 0) {
        const CUtensorMap tb = make_tmap_2d_bf16(B, K, N, ldb * 2, kBK, 64);
        launch_gemm<64, MODE>(ta, tb, ep, M, N, K, st);
    } else {
        fail(LP_ERR_INVALID_ARGUMENT, "gemm: N must be a multiple of 64");
    }
}

int gemm_lnfold_bn(int M, int N) {
    if (!kEpiTma || !gemm_variant() || M <= kBM) return 0;
    return N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 0);
}

void gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const GemmEpilogue& ep,
               int mode, cudaStream_t st) {
    if (M <= 0) return;
    if ((ep.xq || ep.stats_in) && !gemm_lnfold_bn(M, N))
        fail(LP_ERR_INVALID_ARGUMENT, "gemm: the LN-fold epilogue needs the CTA-pair kernel (M > 128, N % 128 == 0)");
    if (ep.xq && (mode < EPI_F32_RESID || !ep.g || !ep.stats_out || ep.ldq % 8))
        fail(LP_ERR_INVALID_ARGUMENT, "gemm: LN-fold producer needs an f32 epilogue, g, stats_out and ldq % 8 == 0");
    if (ep.rms_out && (mode != EPI_BF16 || !gemm_lnfold_bn(M, N)))
        fail(LP_ERR_INVALID_ARGUMENT, "gemm: rms_out needs the bf16 epilogue of the CTA-pair kernel");
    if (ep.stats_in && (mode > EPI_BF16_GELU || !ep.cs || ep.parts < 1))
        fail(LP_ERR_INVALID_ARGUMENT, "gemm: LN-fold consumer needs a bf16 epilogue, cs and parts >= 1");
    if (K % 8 || lda % 8 || ldb % 8) fail(LP_ERR_INVALID_ARGUMENT, "gemm: K and strides must be multiples of 8");
    const CUtensorMap ta = make_tmap_2d_bf16(A, K, M, lda * 2, kBK, kBM);
    prof_begin(KC_GEMM, st);
    switch (mode) {
        case EPI_BF16: gemm_bn<EPI_BF16>(ta, B, ldb, ep, M, N, K, st); break;
        case EPI_BF16_GELU: gemm_bn<EPI_BF16_GELU>(ta, B, ldb, ep, M, N, K, st); break;
        case EPI_F32_RESID: gemm_bn<EPI_F32_RESID>(ta, B, ldb, ep, M, N, K, st); break;
        case EPI_F32: gemm_bn<EPI_F32>(ta, B, ldb, ep, M, N, K, st); break;
        default: fail(LP_ERR_INVALID_ARGUMENT, "gemm: bad epilogue");
    }
    prof_end(KC_GEMM, st, 2.0 * M * N * K, 2.0 * (static_cast<double>(M) * K + static_cast<double>(N) * K) +
                                               static_cast<double>(M) * N * (mode >= EPI_F32_RESID ? 4.0 : 2.0));
}

}  // namespace lpb200

using namespace lpb200;

extern "C" int lp_gemm_bf16_epi(const void* A, const void* B, const void* bias, const float* gate, void* D,
                                int64_t M, int64_t N, int64_t K, int32_t mode, void* stream) {
    return guard([&] {
        if (mode < EPI_BF16 || mode > EPI_F32) fail(LP_ERR_INVALID_ARGUMENT, "epilogue mode 0..3");
        GemmEpilogue ep{};
        ep.bias = static_cast<const float*>(bias);
        ep.out = D;
        ep.ldo = N;
        ep.gate = gate;
        gemm_bf16(A, K, B, K, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), ep, mode,
                  as_stream(stream));
    });
}

extern "C" int lp_gemm_bf16(const void* A, const void* B, const void* bias, void* D, int64_t M, int64_t N, int64_t K,
                            void* stream) {
    return guard([&] {
        GemmEpilogue ep{};
        ep.bias = static_cast<const float*>(bias);
        ep.out = D;
        ep.ldo = N;
        gemm_bf16(A, K, B, K, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), ep, EPI_BF16,
                  as_stream(stream));
    });
}
