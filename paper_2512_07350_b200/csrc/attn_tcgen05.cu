// attn_tcgen05.cu — FlashAttention-style forward on tcgen05 (sm_100a), head_dim 128.
//
// One CTA per (128-row Q tile, head, batch).  Roles (192 threads):
//   warp 0      TMA producer: Q once, then K_j/V_j into a 2-stage ring
//   warp 1      MMA issuer (one lane):  S_j = Q K_j^T  -> TMEM (double-buffered)
//                                       O  += P_j V_j  -> TMEM
//   warps 2..5  softmax: one thread per query row (its TMEM lane); online
//               softmax in the exp2 domain with lazy rescaling (O is only
//               rescaled when the running max grows by > 8, i.e. 2^8), P_j
//               written to shared memory in the UMMA K-major 128B-swizzle layout.
// V is consumed straight from its row-major [kv, d] tile as an MN-major B operand.
#include <cuda.h>

#include "dit_ops.hpp"
#include "tc_ptx.cuh"

namespace lpb200 {

using namespace tc;

constexpr int kAttnThreads = 192;
constexpr int kTile = 128;          // q rows and kv rows per block
constexpr int kHD = 128;            // head dim
constexpr int kAtom = 128 * 128;    // bytes of one [128 rows x 128 B] swizzle block
constexpr int kTileBytes = 2 * kAtom;  // [128 x 128] bf16 = 32 KB
constexpr int kKVStages = 2;
constexpr int kAttnSmem = kTileBytes /*Q*/ + kKVStages * 2 * kTileBytes /*K,V*/ + kTileBytes /*P*/ + 1024 + 256;

struct AttnKernelArgs {
    int64_t q_col0, k_col0, v_col0;
    int64_t q_rows_per_batch, n_q, kv_rows_per_batch, n_kv;
    void* o;
    int64_t ldo;
    float scale_log2;  // softmax scale * log2(e)
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(kAttnThreads, 1)
    k_attention(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tv, AttnKernelArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + kTileBytes;                  // [stage]
    uint8_t* sV = sK + kKVStages * kTileBytes;      // [stage]
    uint8_t* sP = sV + kKVStages * kTileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kTileBytes);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;   // [2]
    uint64_t* kv_empty = bars + 3;  // [2]
    uint64_t* s_full = bars + 5;    // [2]
    uint64_t* s_empty = bars + 7;   // [2]
    uint64_t* p_full = bars + 9;
    uint64_t* o_done = bars + 10;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int nkv = static_cast<int>((a.n_kv + kTile - 1) / kTile);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tv);
        mbar_init(q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], 128);
        }
        mbar_init(p_full, 128);
        mbar_init(o_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS[2] = {tmem, tmem + 128};
    const uint32_t tO = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            const int32_t qrow = static_cast<int32_t>(b * a.q_rows_per_batch + qt * kTile);
            const int32_t qc = static_cast<int32_t>(a.q_col0 + h * kHD);
            mbar_arrive_expect_tx(q_full, kTileBytes);
            tma_load_2d(&tq, q_full, sQ, qc, qrow);
            tma_load_2d(&tq, q_full, sQ + kAtom, qc + 64, qrow);
            const int32_t kc = static_cast<int32_t>(a.k_col0 + h * kHD), vc = static_cast<int32_t>(a.v_col0 + h * kHD);
            for (int j = 0; j < nkv; ++j) {
                const int s = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                mbar_wait(&kv_empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&kv_full[s], 2 * kTileBytes);
                const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile);
                tma_load_2d(&tk, &kv_full[s], sK + s * kTileBytes, kc, kr);
                tma_load_2d(&tk, &kv_full[s], sK + s * kTileBytes + kAtom, kc + 64, kr);
                tma_load_2d(&tv, &kv_full[s], sV + s * kTileBytes, vc, kr);
                tma_load_2d(&tv, &kv_full[s], sV + s * kTileBytes + kAtom, vc + 64, kr);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16(128, 128);
            constexpr uint32_t idO = idesc_bf16(128, 128, /*b_mn_major=*/true);
            const uint32_t q0 = smem_u32(sQ), p0 = smem_u32(sP);
            mbar_wait(q_full, 0);
            auto issue_s = [&](int j) {
                const int s = j & 1;
                mbar_wait(&kv_full[s], (j >> 1) & 1);
                if (j >= 2) mbar_wait(&s_empty[s], ((j - 2) >> 1) & 1);
                tc_fence_after();
                const uint32_t k0 = smem_u32(sK + s * kTileBytes);
#pragma unroll
                for (int k = 0; k < kHD / 16; ++k) {
                    const uint32_t off = (k >> 2) * kAtom + (k & 3) * 32;
                    mma_ss(tS[s], desc_sw128(q0 + off), desc_sw128(k0 + off), idS, k != 0);
                }
                mma_commit(&s_full[s]);
            };
            issue_s(0);
            for (int j = 0; j < nkv; ++j) {
                const int s = j & 1;
                if (j + 1 < nkv) issue_s(j + 1);
                mbar_wait(p_full, j & 1);
                tc_fence_after();
                const uint32_t v0 = smem_u32(sV + s * kTileBytes);
#pragma unroll
                for (int k = 0; k < kTile / 16; ++k) {
                    // A = P (K-major, 2 atoms of 64 kv); B = V [kv][d] MN-major:
                    // 16 kv rows per step (2048 B), the two 64-wide d halves LBO = 16 KB apart
                    const uint64_t pd = desc_sw128(p0 + (k >> 2) * kAtom + (k & 3) * 32);
                    const uint64_t vd = desc_sw128(v0 + k * 2048, /*sbo=*/1024, /*lbo=*/kAtom);
                    mma_ss(tO, pd, vd, idO, (j | k) != 0);
                }
                mma_commit(o_done);
                mma_commit(&kv_empty[s]);
            }
        }
    } else {
        // softmax warpgroup: thread <-> query row (TMEM lane)
        const uint32_t q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (q * 32) << 16;
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < nkv; ++j) {
            const int s = j & 1;
            mbar_wait(&s_full[s], (j >> 1) & 1);
            tc_fence_after();
            float sv[kTile];
#pragma unroll
            for (int c = 0; c < kTile; c += 32) {
                uint32_t r[32];
                tmem_ld32(tS[s] + lane_off + c, r);
                tmem_ld_wait();
#pragma unroll
                for (int u = 0; u < 32; ++u) sv[c + u] = __uint_as_float(r[u]) * a.scale_log2;
            }
            tc_fence_before();
            mbar_arrive(&s_empty[s]);
            const int valid = static_cast<int>(a.n_kv - static_cast<int64_t>(j) * kTile);
            if (valid < kTile) {
#pragma unroll
                for (int u = 0; u < kTile; ++u)
                    if (u >= valid) sv[u] = -INFINITY;
            }
            float mx = m_run;
#pragma unroll
            for (int u = 0; u < kTile; ++u) mx = fmaxf(mx, sv[u]);
            // lazy rescale: keep the stale max unless it grew by more than 8 (2^8 headroom)
            const bool need = (mx > m_run + 8.f) || (m_run == -INFINITY);
            float m_use = need ? mx : m_run;
            const float alpha = need ? (m_run == -INFINITY ? 0.f : ex2(m_run - mx)) : 1.f;
            // P_{j-1} consumed and O settled before P_j / rescale
            if (j > 0) {
                mbar_wait(o_done, (j - 1) & 1);
                tc_fence_after();
                if (__any_sync(0xffffffff, need && m_run != -INFINITY)) {
#pragma unroll 1
                    for (int c = 0; c < kHD; c += 16) {
                        uint32_t r[16];
                        tmem_ld16(tO + lane_off + c, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 16; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * alpha);
                        tmem_st16(tO + lane_off + c, r);
                    }
                    tmem_st_wait();
                }
            }
            l_run *= alpha;
            m_run = m_use;
            // P = exp2(s - m) -> bf16, swizzled into sP
            uint8_t* prow = sP + row * 128;
#pragma unroll
            for (int c = 0; c < kTile / 8; ++c) {
                float p[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    p[u] = ex2(sv[c * 8 + u] - m_use);
                    l_run += p[u];
                }
                const int atom = c >> 3, cc = c & 7;
                *reinterpret_cast<uint4*>(prow + atom * kAtom + ((cc ^ (row & 7)) << 4)) =
                    make_uint4(pack_bf16(p[0], p[1]), pack_bf16(p[2], p[3]), pack_bf16(p[4], p[5]), pack_bf16(p[6], p[7]));
            }
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        // epilogue: O / l -> bf16
        mbar_wait(o_done, (nkv - 1) & 1);
        tc_fence_after();
        const int64_t grow = static_cast<int64_t>(qt) * kTile + row;
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.o) + (b * a.q_rows_per_batch + grow) * a.ldo + h * kHD;
#pragma unroll 1
        for (int c = 0; c < kHD; c += 32) {
            uint32_t r[32];
            tmem_ld32(tO + lane_off + c, r);
            tmem_ld_wait();
            if (grow < a.n_q) {
                uint4* o4 = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    o4[u] = make_uint4(pack_bf16(__uint_as_float(r[8 * u + 0]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                                       pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                                       pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                                       pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 512);
}

void attention_bf16(const AttnArgs& x, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        LP_CUDA(cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        attr = true;
    }
    if ((x.ldq | x.ldk | x.ldv | x.ldo) % 8) fail(LP_ERR_INVALID_ARGUMENT, "attention: strides must be multiples of 8");
    // 2-D views [rows, row_stride] with 64-element (128 B) boxes, 128-byte swizzle
    const CUtensorMap tq = make_tmap_2d_bf16(x.q, x.ldq, x.q_total_rows, x.ldq * 2, 64, kTile);
    const CUtensorMap tk = make_tmap_2d_bf16(x.k, x.ldk, x.kv_total_rows, x.ldk * 2, 64, kTile);
    const CUtensorMap tv = make_tmap_2d_bf16(x.v, x.ldv, x.kv_total_rows, x.ldv * 2, 64, kTile);
    AttnKernelArgs a;
    a.q_col0 = x.q_col0;
    a.k_col0 = x.k_col0;
    a.v_col0 = x.v_col0;
    a.q_rows_per_batch = x.q_rows_per_batch;
    a.n_q = x.n_q;
    a.kv_rows_per_batch = x.kv_rows_per_batch;
    a.n_kv = x.n_kv;
    a.o = x.o;
    a.ldo = x.ldo;
    a.scale_log2 = x.scale * 1.4426950408889634f;
    const dim3 grid(static_cast<unsigned>((x.n_q + kTile - 1) / kTile), x.heads, x.batch);
    const int cls = x.n_kv == x.n_q && x.q == x.k ? KC_SELF_ATTN : KC_CROSS_ATTN;
    prof_begin(cls, st);
    k_attention<<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, a);
    LP_LAUNCH_CHECK();
    prof_end(cls, st, 4.0 * x.batch * x.heads * static_cast<double>(x.n_q) * static_cast<double>(x.n_kv) * kHD,
             2.0 * x.batch * x.heads * kHD * (2.0 * x.n_q + 2.0 * x.n_kv));
}

}  // namespace lpb200

using namespace lpb200;

// q,k,v,o: [B, S, H, 128] bf16 contiguous
extern "C" int lp_attention_bf16(const void* q, const void* k, const void* v, void* o, int64_t batch, int64_t seq_q,
                                 int64_t seq_kv, int64_t heads, double scale, void* stream) {
    return guard([&] {
        AttnArgs a{};
        const int64_t ld = heads * 128;
        a.q = q; a.ldq = ld; a.q_col0 = 0; a.q_rows_per_batch = seq_q; a.n_q = seq_q; a.q_total_rows = batch * seq_q;
        a.k = k; a.ldk = ld; a.k_col0 = 0;
        a.v = v; a.ldv = ld; a.v_col0 = 0;
        a.kv_rows_per_batch = seq_kv; a.n_kv = seq_kv; a.kv_total_rows = batch * seq_kv;
        a.o = o; a.ldo = ld;
        a.batch = static_cast<int>(batch);
        a.heads = static_cast<int>(heads);
        a.scale = static_cast<float>(scale);
        attention_bf16(a, as_stream(stream));
    });
}
