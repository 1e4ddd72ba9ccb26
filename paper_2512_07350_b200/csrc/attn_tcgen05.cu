// attn_tcgen05.cu — FlashAttention-style forward on tcgen05 (sm_100a), head_dim 128.
//
// One CTA per (256 query rows = two 128-row Q tiles, head, batch).  Roles (320 threads):
//   warp 0      TMA producer: Q0/Q1 once, then K_j/V_j into a 2-stage ring
//   warp 1      MMA issuer (one lane), per kv block j and tile t in {0,1}:
//                   S_t = Q_t K_j^T            (SS: both operands in smem)  -> TMEM
//                   O_t += P_t V_j             (TS: P read from TMEM, V as MN-major smem)
//               The two tiles ping-pong so the tensor pipe runs one tile's MMAs while
//               the other tile's softmax runs.
//   warps 2..5  softmax of tile 0, warps 6..9 softmax of tile 1: one thread per query
//               row (its TMEM lane).  Online softmax in the exp2 domain with lazy
//               rescaling (O only rescaled when the running max grows by more than 8,
//               i.e. 2^8 headroom).  P_j is written back as packed bf16 into the first
//               64 columns of S_t's own TMEM columns (no shared-memory round trip).
// TMEM (512 columns): S0 [0,128), S1 [128,256), O0 [256,384), O1 [384,512).
// Ordering: tcgen05 MMAs from one thread execute in issue order, so S_t(j+1), issued
// after O_t += P_t(j) V_j, never overwrites P_t(j) early, and the s_full commit of
// S_t(j+1) also certifies that O_t(j) is final before the softmax rescales it.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "dit_ops.hpp"
#include "tc_ptx.cuh"

namespace lpb200 {

using namespace tc;

constexpr int kAttnThreads = 320;
constexpr int kTile = 128;             // q rows per tile and kv rows per block
constexpr int kHD = 128;               // head dim
constexpr int kAtom = 128 * 128;       // one [128 rows x 128 B] swizzle block
constexpr int kTileBytes = 2 * kAtom;  // [128 x 128] bf16 = 32 KB
#ifndef LP_ATTN_KS
#define LP_ATTN_KS 3
#endif
#ifndef LP_ATTN_VS
#define LP_ATTN_VS 2
#endif
constexpr int kKStages = LP_ATTN_KS, kVStages = LP_ATTN_VS;  // K / V ring depths (self-attention)
constexpr int kAttnSmem = (2 /*Q0,Q1*/ + kKStages + kVStages) * kTileBytes + 1024 + 256;
// NT = Q tiles per CTA.  NT = 2 (self-attention): the two tiles ping-pong inside the CTA,
// K/V rings 3/2, 224 KB smem, all 512 TMEM columns, one CTA per SM.  NT = 1 (short key
// sequences, i.e. cross-attention over 512 text tokens): one tile, single-buffered K/V,
// 96 KB smem and 256 TMEM columns, so TWO CTAs share an SM and one CTA's fixed costs (Q/K
// fetch, pipeline ramp, drain, epilogue ~4.6 us, profiles/r2b) overlap the other's blocks.
template <int NT> struct AttnCfg {
    static constexpr int KS = NT == 2 ? kKStages : 1, VS = NT == 2 ? kVStages : 1;
    static constexpr int threads = 64 + 128 * NT;
    static constexpr int smem = (NT + KS + VS) * kTileBytes + 1024 + 256;
    static constexpr uint32_t tmem_cols = NT == 2 ? 512 : 256;
};
#ifndef LP_ATTN_O_LSU
constexpr bool kAttnOTma = true;  // O epilogue: staged in Q's smem, TMA tensor stores
#else
constexpr bool kAttnOTma = false;  // A/B build: thread-per-row 16-B stores
#endif
__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* smem, int32_t c0, int32_t c1, int32_t c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

struct AttnKernelArgs {
    int64_t q_col0, k_col0, v_col0;
    int64_t q_rows_per_batch, n_q, kv_rows_per_batch, n_kv;
    void* o;
    int64_t ldo;
    float scale_log2;  // softmax scale * log2(e)
    int heads, batch;
    int p_whole;  // MMA warp: wait for the whole P (p_full) before any PV instead of half by half
    const void* q;        // raw Q (the TMEM-resident-Q instance loads its rows directly)
    int64_t ldq, q_total_rows;
    const float* q_rms;   // q RMSNorm folded into the per-row softmax scale (null: off)
    int rms_parts;
    float rms_inv_d, rms_eps;
};

// Softmax scale of one query row: c, times the row's RMSNorm factor when the q norm is folded
// into attention (AttnArgs::q_rms; rows past n_q keep c).
__device__ __forceinline__ float row_scale(const AttnKernelArgs& a, float c, int b, int64_t grow) {
    if (!a.q_rms || grow >= a.n_q) return c;
    const float* pp = a.q_rms + (static_cast<int64_t>(b) * a.q_rows_per_batch + grow) * a.rms_parts;
    float ss = 0.f;
    for (int i = 0; i < a.rms_parts; ++i) ss += pp[i];
    return c * rsqrtf(ss * a.rms_inv_d + a.rms_eps);
}

// Waits of the TMA producer lane (K/V slot free) and of the softmax warps (S ready): spinning
// try_wait (default) or try_wait with a suspend-time hint, so a waiting warp does not take
// issue slots from the other tile's softmax warps on its SMSP (A/B build flags)
#ifndef LP_ATTN_MMA_SPIN
#define LP_ATTN_MMA_SPIN 0
#endif
#ifndef LP_ATTN_PROD_SLEEP
#define LP_ATTN_PROD_SLEEP 0
#endif
#ifndef LP_ATTN_SM_SLEEP
#define LP_ATTN_SM_SLEEP 0
#endif
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity) {
    if (LP_ATTN_PROD_SLEEP) mbar_wait_sleep(bar, parity);
    else mbar_wait(bar, parity);
}
__device__ __forceinline__ void swait(uint64_t* bar, uint32_t parity) {
    if (LP_ATTN_SM_SLEEP) mbar_wait_sleep(bar, parity);
    else mbar_wait(bar, parity);
}

// p_half / p_full: one arrive per softmax warp instead of per thread (A/B build flag; measured
// no gain in-step, 1120-1127 vs 1131-1132 TF/s, profiles/r3w)
#ifndef LP_ATTN_WARP_ARRIVE
#define LP_ATTN_WARP_ARRIVE 0
#endif
constexpr bool kWarpArrive = LP_ATTN_WARP_ARRIVE != 0;

#ifndef LP_ATTN_MAX2
constexpr bool kMax3 = true;
#else
constexpr bool kMax3 = false;  // A/B build: two-input max chain
#endif
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// exp2 of a PAIR on the FMA pipe (packed f32x2 ops, FA4-style): round-to-nearest via
// the 1.5*2^23 magic constant, f = x - round(x) in [-0.5, 0.5], degree-3 minimax
// polynomial for 2^f (max rel. error 8e-5, far below bf16's 3.9e-3), exponent added
// as an integer.  Per pair: 2 FMNMX (clamp, ALU) + 6 packed FADD2/FFMA2 + 2 integer
// adds, instead of 2 MUFU.EX2 — it relieves the MUFU pipe, which is co-critical with
// the tensor pipe (2 x 128 x 128 exp2 per CTA and key block = 2048 cycles at 16/clk/SM,
// the same as the block's four 128^3 MMAs).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -126.f);
    x.y = fmaxf(x.y, -126.f);
    const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
    const float2 t = __fadd2_rn(x, magic);                       // round(x) in the low mantissa bits
    const float2 fl = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(fl, make_float2(-1.f, -1.f), x);
    float2 p = __ffma2_rn(f, make_float2(0.05516013875603676f, 0.05516013875603676f),
                          make_float2(0.2425827533006668f, 0.2425827533006668f));
    p = __ffma2_rn(p, f, make_float2(0.6932605504989624f, 0.6932605504989624f));
    p = __ffma2_rn(p, f, make_float2(0.999930202960968f, 0.999930202960968f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Debug timeline (TR variant only): clock64() stamps of CTA (0,0,0), indexed
// [(j * 2 + tile) * 16 + event] for the first 64 key blocks.  Events: 0 S ready (softmax),
// 1 row max done, 2 p_half arrived, 3 p_full arrived, 4 MMA saw p_half, 5 MMA saw p_full,
// 6 MMA issued S(j+1).
__device__ unsigned long long* g_attn_trace = nullptr;

template <bool TR>
__device__ __forceinline__ void trace_ev(int j, int t, int ev) {
    if (TR && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < 64 && g_attn_trace)
        g_attn_trace[(j * 2 + t) * 16 + ev] = clock64();
}

// One 128-key block of the online softmax for one query row (the calling thread's TMEM
// lane): pass 1 row max over S (all 128 columns in flight), lazy O rescale, pass 2
// re-reads S 64 columns at a time (registers stay free for the exponentials' ILP) and
// writes P = exp2(s*c - m*c) as packed bf16 over S's first 64 columns, published in two
// halves (p_half after keys [0,64), p_full after [64,128)) so the MMA warp starts
// O += P[:, :64] V[:64] while the second half is computed.  POLY of every 16 pairs use
// the FMA-pipe polynomial, the rest MUFU.EX2.  MASK: keys >= valid get probability 0.
template <int POLY, bool MASK, bool TR, bool PAIR = false>
__device__ __forceinline__ void softmax_block(uint32_t tS, uint32_t tO, int valid, float c, float& m_run,
                                              float& l_run, uint64_t* p_half, uint64_t* p_full, int j, int t,
                                              bool tr0) {
    float mx;
    {
        uint32_t r[kTile];
#pragma unroll
        for (int cc = 0; cc < kTile; cc += 32) tmem_ld32(tS + cc, *reinterpret_cast<uint32_t(*)[32]>(r + cc));
        tmem_ld_wait();
        if (MASK) {
#pragma unroll
            for (int u = 0; u < kTile; ++u)
                if (u >= valid) r[u] = __float_as_uint(-INFINITY);
        }
        float m8[8];
        if (kMax3) {
            // three-input max (FMNMX3 on sm_100a): 64 + 4 instead of 127 max instructions per row
#pragma unroll
            for (int u = 0; u < 8; ++u) m8[u] = fmaxf(__uint_as_float(r[u]), __uint_as_float(r[u + 8]));
#pragma unroll
            for (int u = 16; u < kTile; u += 16)
#pragma unroll
                for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], __uint_as_float(r[u + k]), __uint_as_float(r[u + 8 + k]));
            mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) m8[u] = __uint_as_float(r[u]);
#pragma unroll
            for (int u = 8; u < kTile; ++u) m8[u & 7] = fmaxf(m8[u & 7], __uint_as_float(r[u]));
            mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        }
    }
    if (tr0) trace_ev<TR>(j, t, 1);
    // lazy rescale: keep the stale max unless it grew by more than 8 (log2 units)
    const bool need = m_run == -INFINITY || (mx - m_run) * c > 8.f;
    if (__any_sync(0xffffffff, need && m_run != -INFINITY)) {
        // O_t(j-1) is final: S_t(j) was issued after it and has completed
        const float alpha = need && m_run != -INFINITY ? ex2((m_run - mx) * c) : 1.f;
#pragma unroll 1
        for (int cc = 0; cc < kHD; cc += 32) {
            uint32_t r[32];
            tmem_ld32(tO + cc, r);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * alpha);
            tmem_st32(tO + cc, r);
        }
        l_run *= alpha;
    }
    if (need) m_run = mx;
    const float2 c2 = make_float2(c, c), nmc2 = make_float2(-m_run * c, -m_run * c);
    float2 lsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    // 32-column chunks, the next chunk's TMEM load in flight while this one is computed
    // (register double buffer; LDTM results are scoreboard-tracked)
    auto chunk = [&](const uint32_t (&r)[32], int cc) {
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            float2 sx = make_float2(__uint_as_float(r[2 * u]), __uint_as_float(r[2 * u + 1]));
            if (MASK) {
                if (cc + 2 * u >= valid) sx.x = -INFINITY;
                if (cc + 2 * u + 1 >= valid) sx.y = -INFINITY;
            }
            const float2 x = __ffma2_rn(sx, c2, nmc2);
            float2 p;
            if (POLY > 0 && ((u * 5) & 15) < POLY) {  // spread the polynomial pairs over the chunk
                p = ex2_poly2(x);
            } else {
                p.x = ex2(x.x);
                p.y = ex2(x.y);
            }
            lsum[u & 1] = __fadd2_rn(lsum[u & 1], p);
            pk[u] = pack_bf16(p.x, p.y);
        }
        tmem_st16(tS + cc / 2, pk);
    };
    auto publish = [&](uint64_t* bar, int half) {
        tmem_st_wait();
        tc_fence_before();
        if (PAIR) {
            // CTA pair: one remote arrive per warp on the leader's barrier (count 8 = 4 warps x
            // 2 CTAs) once all 32 lanes' TMEM stores are complete
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive_remote(bar, 0);
        } else if (kWarpArrive) {
            // one arrive per warp (count 4): 128 per-thread arrivals serialise on one shared-
            // memory word right on the softmax -> PV critical path
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
        } else {
            mbar_arrive(bar);
        }
        if (tr0) trace_ev<TR>(j, t, 2 + half);
        // per lane-quarter arrival (events 8..11 p_half, 12..15 p_full): the barrier completes
        // at the slowest of the four warps
        if (TR && (threadIdx.x & 31) == 0) trace_ev<TR>(j, t, 8 + 4 * half + ((threadIdx.x >> 5) & 3));
    };
    uint32_t ra[32], rb[32];
    tmem_ld32(tS, ra);
    tmem_ld_wait();
    tmem_ld32(tS + 32, rb);
    chunk(ra, 0);
    tmem_ld_wait();
    tmem_ld32(tS + 64, ra);
    chunk(rb, 32);
    publish(p_half, 0);
    tmem_ld_wait();
    tmem_ld32(tS + 96, rb);
    chunk(ra, 64);
    tmem_ld_wait();
    chunk(rb, 96);
    publish(p_full, 1);
    const float2 ls = __fadd2_rn(lsum[0], lsum[1]);
    l_run += ls.x + ls.y;
}

template <int POLY, bool TR = false, int NT = 2, bool PERS = false>
__global__ void __launch_bounds__(AttnCfg<NT>::threads, NT == 2 ? 1 : 2)
    k_attention(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to, AttnKernelArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int KS = AttnCfg<NT>::KS, VS = AttnCfg<NT>::VS;
    uint8_t* sQ = smem;                    // [tile][2 atoms]
    uint8_t* sK = sQ + NT * kTileBytes;    // [KS]
    uint8_t* sV = sK + KS * kTileBytes;    // [VS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VS * kTileBytes);
    uint64_t* q_full = bars + 0;
    uint64_t* k_full = q_full + 1;     // [KS]
    uint64_t* k_empty = k_full + KS;   // [KS]
    uint64_t* v_full = k_empty + KS;   // [VS]
    uint64_t* v_empty = v_full + VS;   // [VS]
    uint64_t* s_full = v_empty + VS;   // [tile]
    uint64_t* p_full = s_full + NT;    // [tile]
    uint64_t* p_half = p_full + NT;    // [tile]
    uint64_t* o_final = p_half + NT;   // [tile]
    uint32_t* tmem_slot;  // after the persistent-mode barriers below

    uint64_t* q_empty = o_final + NT;  // Q smem free (the item's last S MMAs retired)     [persistent]
    uint64_t* o_empty = q_empty + 1;   // [tile] O_t read out of TMEM by the epilogue     [persistent]
    uint64_t* epi_done = o_empty + NT; // staging (V slots) read by the epilogue's stores  [persistent]
    tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 1);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int nkv = static_cast<int>((a.n_kv + kTile - 1) / kTile);
    // work items (Q tile group, head, batch).  One per CTA, or a grid-stride walk when the grid
    // is persistent: item it+1's Q and K stream in while item it drains, its S MMAs queue
    // behind item it's last PVs, and the epilogue stages O in the (then idle) V slots.
    const int n_qt = static_cast<int>((a.n_q + NT * kTile - 1) / (NT * kTile));
    const int items = n_qt * a.heads * a.batch;
    const int first = PERS ? static_cast<int>(blockIdx.x)
                           : static_cast<int>(blockIdx.x + n_qt * (blockIdx.y + a.heads * blockIdx.z));
    const int stride = PERS ? static_cast<int>(gridDim.x) : items;
    auto item = [&](int w, int& qt, int& h, int& b) {
        if (!PERS) {  // one item per CTA: the grid is (Q tile group, head, batch)
            qt = static_cast<int>(blockIdx.x), h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
            return;
        }
        qt = w % n_qt;
        h = (w / n_qt) % a.heads;
        b = w / (n_qt * a.heads);
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tv);
        mbar_init(q_full, 1);
        for (int s = 0; s < KS; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < VS; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int s = 0; s < NT; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], kWarpArrive ? 4 : 128);
            mbar_init(&p_half[s], kWarpArrive ? 4 : 128);
            mbar_init(&o_final[s], 1);
            mbar_init(&o_empty[s], 128);
        }
        mbar_init(q_empty, 1);
        mbar_init(epi_done, 4 * NT);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, AttnCfg<NT>::tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // K runs ahead in a KS-deep ring (needed first, by S = Q K^T); V in a VS-deep ring.
            // Ring positions count blocks over all of this CTA's items (g = it * nkv + j).
            int it = 0;
            for (int w = first; w < items; w += stride, ++it) {
                int qt, h, b;
                item(w, qt, h, b);
                const uint32_t g0 = PERS ? static_cast<uint32_t>(it) * static_cast<uint32_t>(nkv) : 0u;  // ring position base
                if (it > 0) mbar_wait(q_empty, (it - 1) & 1);  // the previous item's S MMAs retired
                const int32_t qrow = static_cast<int32_t>(b * a.q_rows_per_batch + qt * NT * kTile);
                const int32_t qc = static_cast<int32_t>(a.q_col0 + h * kHD);
                mbar_arrive_expect_tx(q_full, NT * kTileBytes);
                for (int t = 0; t < NT; ++t) {
                    tma_load_2d(&tq, q_full, sQ + t * kTileBytes, qc, qrow + t * kTile);
                    tma_load_2d(&tq, q_full, sQ + t * kTileBytes + kAtom, qc + 64, qrow + t * kTile);
                }
                const int32_t kc = static_cast<int32_t>(a.k_col0 + h * kHD), vc = static_cast<int32_t>(a.v_col0 + h * kHD);
                auto load_k = [&](int j) {
                    const uint32_t g = g0 + static_cast<uint32_t>(j);
                    const int s = static_cast<int>(g % KS);
                    pwait(&k_empty[s], ((g / KS) & 1u) ^ 1);
                    if (POLY == -2 && g >= KS) {  // debug (attn_trace=3): no TMA once the ring is primed
                        mbar_arrive(&k_full[s]);
                        return;
                    }
                    mbar_arrive_expect_tx(&k_full[s], kTileBytes);
                    const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile);
                    tma_load_2d(&tk, &k_full[s], sK + s * kTileBytes, kc, kr);
                    tma_load_2d(&tk, &k_full[s], sK + s * kTileBytes + kAtom, kc + 64, kr);
                };
                auto load_v = [&](int j) {
                    const uint32_t g = g0 + static_cast<uint32_t>(j);
                    const int s = static_cast<int>(g % VS);
                    pwait(&v_empty[s], ((g / VS) & 1u) ^ 1);
                    if (POLY == -2 && g >= VS) {
                        mbar_arrive(&v_full[s]);
                        return;
                    }
                    mbar_arrive_expect_tx(&v_full[s], kTileBytes);
                    const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile);
                    tma_load_2d(&tv, &v_full[s], sV + s * kTileBytes, vc, kr);
                    tma_load_2d(&tv, &v_full[s], sV + s * kTileBytes + kAtom, vc + 64, kr);
                };
                int jk = 0;
                for (; jk < nkv && jk < KS - 1; ++jk) load_k(jk);
                for (int j = 0; j < nkv; ++j) {
                    // single-buffered K (NT = 1): K_j first — S_j needs it before PV_j needs V_j
                    if (KS == 1 && jk < nkv) load_k(jk++);
                    // the previous item's epilogue staged O in the V slots
                    if (j == 0 && it > 0) mbar_wait(epi_done, (it - 1) & 1);
                    load_v(j);
                    if (KS > 1 && jk < nkv) load_k(jk++);
                }
            }
        }
    } else if (warp == 1) {
        // The whole warp runs the issue loop (converged: the barrier checks are warp-wide and
        // the operands stay in uniform registers); one elected lane issues the MMAs and
        // commits.  tcgen05.mma issue is nearly synchronous with execution, so each check in
        // this loop is a pipe bubble: ~38 cycles converged vs ~106 from a lone divergent lane
        // (scripts/micro/mma_bench.py, profiles/r1n).
        const bool leader = elect_one();
        // warp-wide waits that suspend in hardware (try_wait with a time hint) instead of
        // spinning: 32 spinning lanes would steal issue slots from the softmax warps sharing
        // this SMSP
        auto wait1 = [&](uint64_t* bar, uint32_t parity) {
            if (LP_ATTN_MMA_SPIN) mbar_wait(bar, parity);  // A/B build flag: spinning try_wait
            else mbar_wait_sleep(bar, parity);
        };
        constexpr uint32_t idS = idesc_bf16(128, 128);
        constexpr uint32_t idO = idesc_bf16(128, 128, /*b_mn_major=*/true);
        // descriptors built once; per-k offsets go into the start-address field (addr >> 4)
        const uint64_t dQ = desc_sw128(smem_u32(sQ)), dK = desc_sw128(smem_u32(sK));
        const uint64_t dV = desc_sw128(smem_u32(sV), /*sbo=*/1024, /*lbo=*/kAtom);
        int it = 0;
        for (int w = first; w < items; w += stride, ++it) {
            const uint32_t g0 = PERS ? static_cast<uint32_t>(it) * static_cast<uint32_t>(nkv) : 0u;  // ring position base
            wait1(q_full, it & 1);
            auto issue_s = [&](int t, int j) {
                const uint32_t g = g0 + static_cast<uint32_t>(j);
                const int s = static_cast<int>(g % KS);
                if (t == 0) {
                    wait1(&k_full[s], ((g / KS) & 1u));
                    tc_fence_after();
                }
                if (leader) {
                    const uint64_t q0 = dQ + t * (kTileBytes >> 4), k0 = dK + s * (kTileBytes >> 4);
#pragma unroll
                    for (int k = 0; k < kHD / 16; ++k) {
                        const uint64_t off = static_cast<uint64_t>((k >> 2) * kAtom + (k & 3) * 32) >> 4;
                        mma_ss(tmem + t * 128, q0 + off, k0 + off, idS, k != 0);
                    }
                    mma_commit(&s_full[t]);
                    if (t == NT - 1) {
                        mma_commit(&k_empty[s]);  // every tile's S issued: K_j slot frees on completion
                        if (j == nkv - 1) mma_commit(q_empty);  // the item's last S: Q smem frees on completion
                    }
                }
                __syncwarp();
            };
            auto issue_pv = [&](int t, int j, int half) {
                if (leader) {
                    const uint64_t v0 = dV + ((g0 + static_cast<uint32_t>(j)) % VS) * (kTileBytes >> 4);
#pragma unroll
                    for (int k = half * 4; k < half * 4 + 4; ++k) {
                        // A = P_t (TMEM, bf16 pairs: 8 columns per 16 kv); B = V [kv][d] MN-major:
                        // 16 kv rows per step (2048 B), d halves LBO = 16 KB apart
                        mma_ts(tmem + NT * 128 + t * 128, tmem + t * 128 + k * 8, v0 + ((k * 2048) >> 4), idO,
                               (j | k) != 0);
                    }
                }
                __syncwarp();
            };
            for (int t = 0; t < NT; ++t) issue_s(t, 0);
            for (int j = 0; j < nkv; ++j) {
                const bool more = j + 1 < nkv;
                const uint32_t g = g0 + static_cast<uint32_t>(j);
                for (int t = 0; t < NT; ++t) {
                    // knob attn_pwhole: one barrier check per tile and block instead of two (every
                    // check is a tensor-pipe bubble: the issue is nearly synchronous)
                    wait1(a.p_whole ? &p_full[t] : &p_half[t], (g & 1u));
                    if (t == 0) wait1(&v_full[g % VS], ((g / VS) & 1u));
                    // O_t is overwritten by this item's first PV: the previous epilogue read it
                    if (j == 0 && it > 0) wait1(&o_empty[t], (it - 1) & 1);
                    if (lane == 0) trace_ev<TR>(j, t, 4);
                    tc_fence_after();
                    issue_pv(t, j, 0);
                    if (!a.p_whole) {
                        wait1(&p_full[t], (g & 1u));
                        if (lane == 0) trace_ev<TR>(j, t, 5);
                        tc_fence_after();
                    }
                    issue_pv(t, j, 1);
                    if (leader) {
                        if (!more) mma_commit(&o_final[t]);
                        if (t == NT - 1) mma_commit(&v_empty[g % VS]);
                    }
                    __syncwarp();
                    if (more) issue_s(t, j + 1);
                    if (lane == 0) trace_ev<TR>(j, t, 6);
                }
            }
        }
    } else {
        // softmax warpgroups: tile t = (warp - 2) / 4, thread <-> query row / TMEM lane
        const int t = (warp - 2) >> 2;
        const uint32_t q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (q * 32) << 16;
        const uint32_t tS = tmem + t * 128 + lane_off, tO = tmem + NT * 128 + t * 128 + lane_off;
        const float c = a.scale_log2;
        int it = 0;
        for (int w = first; w < items; w += stride, ++it) {
            int qt, h, b;
            item(w, qt, h, b);
            const uint32_t g0 = PERS ? static_cast<uint32_t>(it) * static_cast<uint32_t>(nkv) : 0u;  // ring position base
            float m_run = -INFINITY, l_run = 0.f;
            const float cr = row_scale(a, c, b, static_cast<int64_t>(qt) * NT * kTile + t * kTile + row);
            for (int j = 0; j < nkv; ++j) {
                swait(&s_full[t], ((g0 + static_cast<uint32_t>(j)) & 1u));
                const bool tr0 = TR && (warp & 3) == 2 && lane == 0;
                if (tr0) trace_ev<TR>(j, t, 0);
                tc_fence_after();
                const int valid = static_cast<int>(a.n_kv - static_cast<int64_t>(j) * kTile);
                // the ragged last key block takes a separately compiled masked copy, so full
                // blocks carry no per-element compare/select
                if (POLY < 0) {  // debug (attn_trace=2/3): no softmax work, only the handoffs -> the MMA/sync floor
                    tc_fence_before();
                    mbar_arrive(&p_half[t]);
                    if (tr0) trace_ev<TR>(j, t, 2);
                    mbar_arrive(&p_full[t]);
                    if (tr0) trace_ev<TR>(j, t, 3);
                } else if (valid >= kTile)
                    softmax_block<POLY, false, TR>(tS, tO, valid, cr, m_run, l_run, &p_half[t], &p_full[t], j, t, tr0);
                else
                    softmax_block<POLY, true, TR>(tS, tO, valid, cr, m_run, l_run, &p_half[t], &p_full[t], j, t, tr0);
            }
            // epilogue: O_t / l -> bf16 rows.  The staging below reuses V slots: wait for the
            // LAST tile's final PV as well (it is the item's last MMA), so no PV still reads V
            mbar_wait(&o_final[t], it & 1);
            if (PERS && kAttnOTma && t != NT - 1) mbar_wait(&o_final[NT - 1], it & 1);
            tc_fence_after();
            const int64_t grow = static_cast<int64_t>(qt) * NT * kTile + t * kTile + row;
            const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
            if (kAttnOTma) {
                // O_t staged in V slot t (idle: every PV of the item retired before o_final; the
                // producer holds the next item's V loads on epi_done) in 128B-swizzled
                // [128 rows x 64 col] atoms; each warp TMA-stores its 32 rows as two 64-column
                // boxes.  The 3-D O map clips rows >= n_q per batch.
                // non-persistent: Q_t's smem is dead (its last S MMA completed before the last PV)
                uint8_t* stage = PERS ? sV + (t % VS) * kTileBytes : sQ + t * kTileBytes;
#pragma unroll 1
                for (int cc = 0; cc < kHD; cc += 32) {
                    uint32_t r[32];
                    tmem_ld32(tO + cc, r);
                    tmem_ld_wait();
                    uint8_t* arow = stage + (cc >> 6) * kAtom + row * 128;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int unit = ((cc & 63) >> 3) + u;
                        *reinterpret_cast<uint4*>(arow + ((unit ^ (row & 7)) << 4)) =
                            make_uint4(pack_bf16(__uint_as_float(r[8 * u + 0]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                                       pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                                       pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                                       pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
                    }
                }
                tc_fence_before();
                mbar_arrive(&o_empty[t]);  // O_t has been read out: the next item's PV may overwrite it
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    const int32_t r0 = static_cast<int32_t>(qt * NT * kTile + t * kTile + q * 32);
                    for (int at = 0; at < 2; ++at)
                        tma_store_3d(&to, stage + at * kAtom + q * 32 * 128, static_cast<int32_t>(h * kHD + at * 64), r0, b);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    // the staging must be read before the V slot is reloaded (or the CTA retires);
                    // the global writes complete asynchronously and are visible at grid end
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    mbar_arrive(epi_done);
                }
                __syncwarp();
            } else {
#pragma unroll 1
                for (int cc = 0; cc < kHD; cc += 32) {
                    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.o) + (b * a.q_rows_per_batch + grow) * a.ldo + h * kHD;
                    uint32_t r[32];
                    tmem_ld32(tO + cc, r);
                    tmem_ld_wait();
                    if (grow < a.n_q) {
                        uint4* o4 = reinterpret_cast<uint4*>(orow + cc);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            o4[u] = make_uint4(pack_bf16(__uint_as_float(r[8 * u + 0]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                                               pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                                               pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                                               pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
                    }
                }
                tc_fence_before();
                mbar_arrive(&o_empty[t]);
                if (lane == 0) mbar_arrive(epi_done);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, AttnCfg<NT>::tmem_cols);
}

// ---------------------------------------------------------------------------
// Self-attention on CTA pairs (cta_group::2; knob attn_pair).  A 2-CTA cluster shares one
// (head, batch) and each CTA keeps its own two 128-row Q tiles (256 query rows per CTA, 512 per
// pair).  The leader issues every MMA for both: S_t = [Q_t(cta0); Q_t(cta1)] K_j^T is ONE
// M = 256 instruction stream whose B operand (K_j, 128 keys) is split by rows — each CTA
// TMA-loads and holds 64 keys — and O_t += P_t V_j reads P from each CTA's own TMEM and V split
// by columns (each CTA holds 64 of the 128 dims of all 128 keys).  Per SM and key block that
// halves the K/V bytes TMA writes into shared memory (64 -> 32 KB) and the B-operand bytes
// the tensor core reads from it (S: 64 -> 48 KB per tile, PV: 32 -> 16 KB), and one issued
// MMA covers both SMs.  Barriers: Q/K/V completions count both CTAs' bytes on the leader's
// barriers (2-SM TMA), the leader's commits are multicast to both CTAs (s_full, k/v_empty,
// o_final), and both CTAs' softmax warps arrive on the leader's p_half / p_full (count 8).
// The softmax and epilogue are the single-CTA kernel's.
// ---------------------------------------------------------------------------
#ifndef LP_PAIR_KS
#define LP_PAIR_KS 4
#endif
#ifndef LP_PAIR_VS
#define LP_PAIR_VS 4
#endif
constexpr int kPairKS = LP_PAIR_KS, kPairVS = LP_PAIR_VS;  // K / V ring depths of the pair kernel
constexpr int kHalfTile = 64 * 128 * 2;  // 16 KB: [64 keys x 128 dims] (K) or [128 keys x 64 dims] (V)
constexpr int kPairSmem = 2 * kTileBytes + (kPairKS + kPairVS) * kHalfTile + 1024 + 256;

__device__ __forceinline__ void mma_ts_2sm(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int POLY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kAttnThreads, 1)
    k_attention_pair(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
                     AttnKernelArgs a) {
    constexpr int NT = 2, KS = kPairKS, VS = kPairVS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                    // [tile][2 atoms of 128 rows x 128 B]
    uint8_t* sK = sQ + NT * kTileBytes;    // [KS][2 atoms of 64 rows x 128 B]  (this CTA's 64 keys)
    uint8_t* sV = sK + KS * kHalfTile;     // [VS][1 atom of 128 rows x 128 B]  (this CTA's 64 dims)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VS * kHalfTile);
    uint64_t* q_full = bars + 0;
    uint64_t* k_full = q_full + 1;
    uint64_t* k_empty = k_full + KS;
    uint64_t* v_full = k_empty + KS;
    uint64_t* v_empty = v_full + VS;
    uint64_t* s_full = v_empty + VS;
    uint64_t* p_full = s_full + NT;
    uint64_t* p_half = p_full + NT;
    uint64_t* o_final = p_half + NT;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + NT);

    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int nkv = static_cast<int>((a.n_kv + kTile - 1) / kTile);
    const int qt = static_cast<int>(blockIdx.x), h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tv);
        mbar_init(q_full, 1);
        for (int s = 0; s < KS; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < VS; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int t = 0; t < NT; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 8);
            mbar_init(&p_half[t], 8);
            mbar_init(&o_final[t], 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const int32_t qrow = static_cast<int32_t>(b * a.q_rows_per_batch + qt * NT * kTile);
            const int32_t qc = static_cast<int32_t>(a.q_col0 + h * kHD);
            if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * NT * kTileBytes);
            for (int t = 0; t < NT; ++t) {
                tma_load_2d_2sm(&tq, q_full, sQ + t * kTileBytes, qc, qrow + t * kTile);
                tma_load_2d_2sm(&tq, q_full, sQ + t * kTileBytes + kAtom, qc + 64, qrow + t * kTile);
            }
            const int32_t kc = static_cast<int32_t>(a.k_col0 + h * kHD);
            const int32_t vc = static_cast<int32_t>(a.v_col0 + h * kHD + rank * 64);
            auto load_k = [&](int j) {
                const int s = j % KS;
                mbar_wait(&k_empty[s], ((j / KS) & 1) ^ 1);
                if (rank == 0) mbar_arrive_expect_tx(&k_full[s], 2 * kHalfTile);
                const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile + rank * 64);
                tma_load_2d_2sm(&tk, &k_full[s], sK + s * kHalfTile, kc, kr);
                tma_load_2d_2sm(&tk, &k_full[s], sK + s * kHalfTile + kHalfTile / 2, kc + 64, kr);
            };
            auto load_v = [&](int j) {
                const int s = j % VS;
                mbar_wait(&v_empty[s], ((j / VS) & 1) ^ 1);
                if (rank == 0) mbar_arrive_expect_tx(&v_full[s], 2 * kHalfTile);
                const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile);
                tma_load_2d_2sm(&tv, &v_full[s], sV + s * kHalfTile, vc, kr);
            };
            int jk = 0;
            for (; jk < nkv && jk < KS - 1; ++jk) load_k(jk);
            for (int j = 0; j < nkv; ++j) {
                load_v(j);
                if (jk < nkv) load_k(jk++);
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // the leader issues for both CTAs (converged warp, one elected lane; see k_attention)
            const bool leader = elect_one();
            constexpr uint32_t idS = idesc_bf16(256, 128);
            constexpr uint32_t idO = idesc_bf16(256, 128, /*b_mn_major=*/true);
            const uint64_t dQ = desc_sw128(smem_u32(sQ)), dK = desc_sw128(smem_u32(sK));
            const uint64_t dV = desc_sw128(smem_u32(sV), /*sbo=*/1024, /*lbo=*/kAtom);
            mbar_wait_sleep(q_full, 0);
            auto issue_s = [&](int t, int j) {
                const int s = j % KS;
                if (t == 0) {
                    mbar_wait_sleep(&k_full[s], (j / KS) & 1);
                    tc_fence_after();
                }
                if (leader) {
                    const uint64_t q0 = dQ + t * (kTileBytes >> 4), k0 = dK + s * (kHalfTile >> 4);
#pragma unroll
                    for (int k = 0; k < kHD / 16; ++k) {
                        const uint64_t oq = static_cast<uint64_t>((k >> 2) * kAtom + (k & 3) * 32) >> 4;
                        const uint64_t ok = static_cast<uint64_t>((k >> 2) * (kHalfTile / 2) + (k & 3) * 32) >> 4;
                        mma_ss_2sm(tmem + t * 128, q0 + oq, k0 + ok, idS, k != 0);
                    }
                    mma_commit_2sm(&s_full[t], 0x3);
                    if (t == NT - 1) mma_commit_2sm(&k_empty[s], 0x3);
                }
                __syncwarp();
            };
            auto issue_pv = [&](int t, int j, int half) {
                if (leader) {
                    const uint64_t v0 = dV + (j % VS) * (kHalfTile >> 4);
#pragma unroll
                    for (int k = half * 4; k < half * 4 + 4; ++k)
                        mma_ts_2sm(tmem + NT * 128 + t * 128, tmem + t * 128 + k * 8, v0 + ((k * 2048) >> 4), idO,
                                   (j | k) != 0);
                }
                __syncwarp();
            };
            for (int t = 0; t < NT; ++t) issue_s(t, 0);
            for (int j = 0; j < nkv; ++j) {
                const bool more = j + 1 < nkv;
                for (int t = 0; t < NT; ++t) {
                    mbar_wait_sleep(&p_half[t], j & 1);
                    if (t == 0) mbar_wait_sleep(&v_full[j % VS], (j / VS) & 1);
                    tc_fence_after();
                    issue_pv(t, j, 0);
                    mbar_wait_sleep(&p_full[t], j & 1);
                    tc_fence_after();
                    issue_pv(t, j, 1);
                    if (leader) {
                        if (!more) mma_commit_2sm(&o_final[t], 0x3);
                        if (t == NT - 1) mma_commit_2sm(&v_empty[j % VS], 0x3);
                    }
                    __syncwarp();
                    if (more) issue_s(t, j + 1);
                }
            }
        }
    } else {
        const int t = (warp - 2) >> 2;
        const uint32_t q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (q * 32) << 16;
        const uint32_t tS = tmem + t * 128 + lane_off, tO = tmem + NT * 128 + t * 128 + lane_off;
        const float c = a.scale_log2;
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < nkv; ++j) {
            mbar_wait(&s_full[t], j & 1);
            tc_fence_after();
            const int valid = static_cast<int>(a.n_kv - static_cast<int64_t>(j) * kTile);
            if (valid >= kTile)
                softmax_block<POLY, false, false, true>(tS, tO, valid, c, m_run, l_run, &p_half[t], &p_full[t], j, t, false);
            else
                softmax_block<POLY, true, false, true>(tS, tO, valid, c, m_run, l_run, &p_half[t], &p_full[t], j, t, false);
        }
        mbar_wait(&o_final[t], 0);
        tc_fence_after();
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        // O_t staged in Q_t's dead smem (its last S MMA completed before the final PV), then two
        // TMA tensor stores per warp; the 3-D O map clips rows >= n_q of each batch
        uint8_t* stage = sQ + t * kTileBytes;
#pragma unroll 1
        for (int cc = 0; cc < kHD; cc += 32) {
            uint32_t r[32];
            tmem_ld32(tO + cc, r);
            tmem_ld_wait();
            uint8_t* arow = stage + (cc >> 6) * kAtom + row * 128;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int unit = ((cc & 63) >> 3) + u;
                *reinterpret_cast<uint4*>(arow + ((unit ^ (row & 7)) << 4)) =
                    make_uint4(pack_bf16(__uint_as_float(r[8 * u + 0]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                               pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                               pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                               pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
            }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            const int32_t r0 = static_cast<int32_t>(qt * NT * kTile + t * kTile + q * 32);
            for (int at = 0; at < 2; ++at)
                tma_store_3d(&to, stage + at * kAtom + q * 32 * 128, static_cast<int32_t>(h * kHD + at * 64), r0, b);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
    }
    // the peer's remote arrivals and the leader's MMAs into this CTA's TMEM / smem are done
    // before either CTA frees TMEM or exits
    tc_fence_before();
    cluster_sync();
    if (warp == 2) tmem_dealloc_2sm(tmem, 512);
}

// ---------------------------------------------------------------------------
// Self-attention, CTA pair with Q resident in TMEM and S double-buffered (knob attn_qtm).
// Each CTA of a 2-CTA cluster owns ONE 128-row Q tile (256 query rows per pair).  Q is loaded
// once into TMEM (in the A-operand layout P uses), so S = Q K^T is a TS MMA (M = 256, the pair)
// that reads only K from shared memory; two S buffers let S(j+1) run while the softmax of
// block j does.  Per SM and 128-key block: S reads 32 KB, PV 32 KB, TMA writes 32 KB (96 KB vs
// 256 KB for the two-tile kernel: its SS S-MMAs alone use the whole ~128 B/clk operand path,
// profiles/r4h), and the softmax -> PV -> S chain is off the critical path.
// TMEM per CTA: Q [0,64) | S0 [128,256) | S1 [256,384) | O [384,512).
// A rare O rescale waits for the previous PV (o_done[(j-1) & 1]): the next PV that can
// complete needs this block's P, so those barriers never run a full phase ahead.
// ---------------------------------------------------------------------------
constexpr int kQtKS = 6, kQtVS = 6;
constexpr int kQtThreads = 64 + 256;  // TMA, MMA, two softmax warpgroups
constexpr int kQtSmem = (kQtKS + kQtVS) * kHalfTile + 1024 + 512 + 4096 + 1024;

// One 128-key block for one query row, split over TWO softmax warpgroups: warpgroup h owns key
// columns [64h, 64h + 64) of the row.  The row max is exchanged through shared memory (xch,
// double-buffered by block parity; a 64-thread named barrier per TMEM lane quarter), so both
// halves keep the same running max and rescale decision; each half keeps its own partial row
// sum, rescales its 64 columns of O, and writes its P as packed bf16 over the first 32 columns of
// ITS OWN S half (already read: keys [64h, 64h+64) -> S columns [64h, 64h+32)), published on
// p_half (h = 0) or p_full (h = 1): PV's first four k-steps read P at +0, the last four at +64.
template <int POLY, bool MASK>
__device__ __forceinline__ void softmax_half_qt(uint32_t tS, uint32_t tO, int valid, float c, float& m_run,
                                                float& l_run, uint64_t* p_bar, uint64_t* o_bar, uint32_t o_par,
                                                bool have_prev, int h, float* xch, int row, uint32_t qbar) {
    const int k0 = 64 * h;  // this half's first key column
    float mx;
    {
        uint32_t r[64];
        tmem_ld32(tS + k0, *reinterpret_cast<uint32_t(*)[32]>(r));
        tmem_ld32(tS + k0 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        tmem_ld_wait();
        if (MASK) {
#pragma unroll
            for (int u = 0; u < 64; ++u)
                if (k0 + u >= valid) r[u] = __float_as_uint(-INFINITY);
        }
        float m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(__uint_as_float(r[u]), __uint_as_float(r[u + 8]));
#pragma unroll
        for (int u = 16; u < 64; u += 16)
#pragma unroll
            for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], __uint_as_float(r[u + k]), __uint_as_float(r[u + 8 + k]));
        mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
    }
    xch[h * 128 + row] = mx;
    named_bar_sync(qbar, 64);
    mx = fmaxf(mx, xch[(h ^ 1) * 128 + row]);
    const bool need = m_run == -INFINITY || (mx - m_run) * c > 8.f;
    if (__any_sync(0xffffffff, need && m_run != -INFINITY)) {
        if (have_prev) mbar_wait(o_bar, o_par);  // O holds PV(j-1) before it is rescaled
        tc_fence_after();
        const float alpha = need && m_run != -INFINITY ? ex2((m_run - mx) * c) : 1.f;
#pragma unroll 1
        for (int cc = 0; cc < 64; cc += 32) {
            uint32_t r[32];
            tmem_ld32(tO + k0 + cc, r);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * alpha);
            tmem_st32(tO + k0 + cc, r);
        }
        l_run *= alpha;
    }
    if (need) m_run = mx;
    const float2 c2 = make_float2(c, c), nmc2 = make_float2(-m_run * c, -m_run * c);
    float2 lsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    auto chunk = [&](const uint32_t (&r)[32], int cc) {
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            float2 sx = make_float2(__uint_as_float(r[2 * u]), __uint_as_float(r[2 * u + 1]));
            if (MASK) {
                if (k0 + cc + 2 * u >= valid) sx.x = -INFINITY;
                if (k0 + cc + 2 * u + 1 >= valid) sx.y = -INFINITY;
            }
            const float2 x = __ffma2_rn(sx, c2, nmc2);
            float2 pv;
            if (POLY > 0 && ((u * 5) & 15) < POLY) {
                pv = ex2_poly2(x);
            } else {
                pv.x = ex2(x.x);
                pv.y = ex2(x.y);
            }
            lsum[u & 1] = __fadd2_rn(lsum[u & 1], pv);
            pk[u] = pack_bf16(pv.x, pv.y);
        }
        tmem_st16(tS + k0 + cc / 2, pk);
    };
    uint32_t ra[32], rb[32];
    tmem_ld32(tS + k0, ra);
    tmem_ld_wait();
    tmem_ld32(tS + k0 + 32, rb);
    chunk(ra, 0);
    tmem_ld_wait();
    chunk(rb, 32);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive_remote(p_bar, 0);
    const float2 ls = __fadd2_rn(lsum[0], lsum[1]);
    l_run += ls.x + ls.y;
}

template <int POLY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kQtThreads, 1)
    k_attention_qt(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                   const __grid_constant__ CUtensorMap to, AttnKernelArgs a) {
    constexpr int KS = kQtKS, VS = kQtVS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;                    // [KS][2 atoms of 64 rows x 128 B]  (this CTA's 64 keys)
    uint8_t* sV = sK + KS * kHalfTile;     // [VS][1 atom of 128 rows x 128 B]  (this CTA's 64 dims)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VS * kHalfTile);
    uint64_t* q_ready = bars + 0;          // leader: both CTAs' Q rows in TMEM (8 warps)
    uint64_t* k_full = q_ready + 1;        // leader [KS]
    uint64_t* k_empty = k_full + KS;       // [KS]
    uint64_t* v_full = k_empty + KS;       // leader [VS]
    uint64_t* v_empty = v_full + VS;       // [VS]
    uint64_t* s_full = v_empty + VS;       // [2] S(j) in buffer j & 1
    uint64_t* p_half = s_full + 2;         // leader [2]
    uint64_t* p_full = p_half + 2;         // leader [2]
    uint64_t* o_done = p_full + 2;         // [2] PV(j) complete, j & 1
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
    float* xch = reinterpret_cast<float*>(bars + 64);   // [2 block parity][2 halves][128 rows] row maxima
    float* lxch = xch + 2 * 2 * 128;                   // [2 halves][128 rows] partial row sums

    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int nkv = static_cast<int>((a.n_kv + kTile - 1) / kTile);
    const int qt = static_cast<int>(blockIdx.x), h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tk);
        tma_prefetch(&tv);
        mbar_init(q_ready, 16);  // 8 softmax warps x 2 CTAs
        for (int s = 0; s < KS; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < VS; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_half[i], 8);  // warpgroup 0's 4 warps x 2 CTAs (keys 0..63)
            mbar_init(&p_full[i], 8);  // warpgroup 1's (keys 64..127)
            mbar_init(&o_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_2sm(tmem_slot, 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t kColQ = 0, kColS = 128, kColO = 384;

    if (warp == 0) {
        if (lane == 0) {
            const int32_t kc = static_cast<int32_t>(a.k_col0 + h * kHD);
            const int32_t vc = static_cast<int32_t>(a.v_col0 + h * kHD + rank * 64);
            auto load_k = [&](int j) {
                const int s = j % KS;
                mbar_wait(&k_empty[s], ((j / KS) & 1) ^ 1);
                if (rank == 0) mbar_arrive_expect_tx(&k_full[s], 2 * kHalfTile);
                const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile + rank * 64);
                tma_load_2d_2sm(&tk, &k_full[s], sK + s * kHalfTile, kc, kr);
                tma_load_2d_2sm(&tk, &k_full[s], sK + s * kHalfTile + kHalfTile / 2, kc + 64, kr);
            };
            auto load_v = [&](int j) {
                const int s = j % VS;
                mbar_wait(&v_empty[s], ((j / VS) & 1) ^ 1);
                if (rank == 0) mbar_arrive_expect_tx(&v_full[s], 2 * kHalfTile);
                const int32_t kr = static_cast<int32_t>(b * a.kv_rows_per_batch + j * kTile);
                tma_load_2d_2sm(&tv, &v_full[s], sV + s * kHalfTile, vc, kr);
            };
            int jk = 0;
            for (; jk < nkv && jk < KS - 1; ++jk) load_k(jk);
            for (int j = 0; j < nkv; ++j) {
                load_v(j);
                if (jk < nkv) load_k(jk++);
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            const bool leader = elect_one();
            constexpr uint32_t idS = idesc_bf16(256, 128);                      // A (Q) from TMEM, B = K K-major
            constexpr uint32_t idO = idesc_bf16(256, 128, /*b_mn_major=*/true);  // A (P) from TMEM, B = V MN-major
            const uint64_t dK = desc_sw128(smem_u32(sK));
            const uint64_t dV = desc_sw128(smem_u32(sV), /*sbo=*/1024, /*lbo=*/kAtom);
            mbar_wait_sleep(q_ready, 0);
            tc_fence_after();
            auto issue_s = [&](int j) {
                const int s = j % KS;
                mbar_wait_sleep(&k_full[s], (j / KS) & 1);
                tc_fence_after();
                if (leader) {
                    const uint64_t k0 = dK + s * (kHalfTile >> 4);
                    const uint32_t dS = tmem + kColS + (j & 1) * 128;
#pragma unroll
                    for (int k = 0; k < kHD / 16; ++k) {
                        const uint64_t ok = static_cast<uint64_t>((k >> 2) * (kHalfTile / 2) + (k & 3) * 32) >> 4;
                        mma_ts_2sm(dS, tmem + kColQ + k * 8, k0 + ok, idS, k != 0);
                    }
                    mma_commit_2sm(&s_full[j & 1], 0x3);
                    mma_commit_2sm(&k_empty[s], 0x3);
                }
                __syncwarp();
            };
            issue_s(0);
            if (nkv > 1) issue_s(1);
            for (int j = 0; j < nkv; ++j) {
                const int bb = j & 1;
                const uint32_t par = (j >> 1) & 1;
                const uint32_t tP = tmem + kColS + bb * 128;
                const uint64_t v0 = dV + (j % VS) * (kHalfTile >> 4);
                mbar_wait_sleep(&p_half[bb], par);
                mbar_wait_sleep(&v_full[j % VS], (j / VS) & 1);
                tc_fence_after();
                if (leader) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_ts_2sm(tmem + kColO, tP + k * 8, v0 + ((k * 2048) >> 4), idO, (j | k) != 0);
                }
                __syncwarp();
                mbar_wait_sleep(&p_full[bb], par);
                tc_fence_after();
                if (leader) {
#pragma unroll
                    for (int k = 4; k < 8; ++k)  // keys 64..127: P at +64 (the second half's own S columns)
                        mma_ts_2sm(tmem + kColO, tP + 64 + (k - 4) * 8, v0 + ((k * 2048) >> 4), idO, true);
                    mma_commit_2sm(&o_done[bb], 0x3);
                    mma_commit_2sm(&v_empty[j % VS], 0x3);
                }
                __syncwarp();
                if (j + 2 < nkv) issue_s(j + 2);  // into buffer bb, after PV(j) read its P (in order)
            }
        }
    } else {
        // two softmax warpgroups (warps 2..5: keys 0..63, 6..9: keys 64..127 of every block);
        // thread <-> query row / TMEM lane, the two warps of a lane quarter meet on named barrier 1+q
        const int hh = (static_cast<int>(warp) - 2) >> 2;
        const uint32_t q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (q * 32) << 16;
        const uint32_t qbar = 1 + q;
        // this half's 64 dims of the Q row -> TMEM columns [32 hh, 32 hh + 32) (packed bf16 pairs,
        // the A-operand layout of P)
        {
            const int64_t grow = static_cast<int64_t>(b) * a.q_rows_per_batch + static_cast<int64_t>(qt) * kTile + row;
            uint32_t w[32];
            if (grow < a.q_total_rows) {
                const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + grow * a.ldq +
                                                                  a.q_col0 + h * kHD + 64 * hh);
#pragma unroll
                for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(w + 4 * i) = src[i];
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) w[i] = 0u;
            }
            tmem_st32(tmem + lane_off + kColQ + 32 * hh, w);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(q_ready, 0);
        }
        const uint32_t tO = tmem + lane_off + kColO;
        const float c = a.scale_log2;
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < nkv; ++j) {
            const int bb = j & 1;
            swait(&s_full[bb], (j >> 1) & 1);
            tc_fence_after();
            const uint32_t tS = tmem + lane_off + kColS + bb * 128;
            const int valid = static_cast<int>(a.n_kv - static_cast<int64_t>(j) * kTile);
            uint64_t* ob = &o_done[(j - 1) & 1];
            const uint32_t opar = static_cast<uint32_t>(((j - 1) >> 1) & 1);
            uint64_t* pb = hh == 0 ? &p_half[bb] : &p_full[bb];
            float* xj = xch + bb * 256;
            if (valid >= kTile)
                softmax_half_qt<POLY, false>(tS, tO, valid, c, m_run, l_run, pb, ob, opar, j > 0, hh, xj, row, qbar);
            else
                softmax_half_qt<POLY, true>(tS, tO, valid, c, m_run, l_run, pb, ob, opar, j > 0, hh, xj, row, qbar);
        }
        // epilogue: the row sum over both halves, the last PV, then this half's 64 columns of
        // O / l -> bf16 staged as atom hh in K ring slots 0..1 (every S MMA, the last readers of
        // K, completed before the last PV), one TMA store per warp
        lxch[hh * 128 + row] = l_run;
        named_bar_sync(qbar, 64);
        l_run = l_run + lxch[(hh ^ 1) * 128 + row];  // commutative: the same total in both halves
        mbar_wait(&o_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
        tc_fence_after();
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        uint8_t* stage = sK;
#pragma unroll 1
        for (int cc = 0; cc < 64; cc += 32) {
            uint32_t r[32];
            tmem_ld32(tO + 64 * hh + cc, r);
            tmem_ld_wait();
            uint8_t* arow = stage + hh * kAtom + row * 128;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int unit = (cc >> 3) + u;
                *reinterpret_cast<uint4*>(arow + ((unit ^ (row & 7)) << 4)) =
                    make_uint4(pack_bf16(__uint_as_float(r[8 * u + 0]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                               pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                               pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                               pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
            }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            const int32_t r0 = static_cast<int32_t>(qt * kTile + q * 32);
            tma_store_3d(&to, stage + hh * kAtom + q * 32 * 128, static_cast<int32_t>(h * kHD + hh * 64), r0, b);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) tmem_dealloc_2sm(tmem, 512);
}

static int attn_poly() {
    // self-attention (NT = 2, one CTA per item): pairs out of every 16 whose exp2 runs on the FMA
    // pipe (0, 4, 6, 8 compiled).  4 since r4: +0.9% in-step over 6 in two interleaved A/Bs
    // (self-attention 1148-1156 vs 1135-1140 TF/s, profiles/r4t) once the GEMMs' handshake fix
    // shifted the power budget; r2j had measured 6 best.  The other instances use 6.
    const int v = tune_get("attn_poly", 4);
    return v == 0 || v == 6 || v == 8 ? v : 4;
}

CUtensorMap make_tmap_3d_bf16(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                              uint32_t b0, uint32_t b1, uint32_t b2);  // gemm_tcgen05.cu (128B swizzle)

void attention_bf16(const AttnArgs& x, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        LP_CUDA(cudaFuncSetAttribute(k_attention<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<-1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<-2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<6, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     AttnCfg<1>::smem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<6, false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     AttnCfg<1>::smem));
        LP_CUDA(cudaFuncSetAttribute(k_attention<6, false, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kAttnSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention_pair<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem));
        LP_CUDA(cudaFuncSetAttribute(k_attention_qt<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQtSmem));
        attr = true;
    }
    if ((x.ldq | x.ldk | x.ldv | x.ldo) % 8) fail(LP_ERR_INVALID_ARGUMENT, "attention: strides must be multiples of 8");
    // 2-D views [rows, row_stride] with 64-element (128 B) boxes, 128-byte swizzle
    const CUtensorMap tq = make_tmap_2d_bf16(x.q, x.ldq, x.q_total_rows, x.ldq * 2, 64, kTile);
    const CUtensorMap tk = make_tmap_2d_bf16(x.k, x.ldk, x.kv_total_rows, x.ldk * 2, 64, kTile);
    const CUtensorMap tv = make_tmap_2d_bf16(x.v, x.ldv, x.kv_total_rows, x.ldv * 2, 64, kTile);
    // O as [batch][n_q rows][ldo]: rows past n_q of a batch are clipped by the map
    const CUtensorMap to = make_tmap_3d_bf16(x.o, x.ldo, x.n_q, x.batch, x.ldo * 2, x.q_rows_per_batch * x.ldo * 2, 64, 32, 1);
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
    a.heads = x.heads;
    a.batch = x.batch;
    a.p_whole = tune_get("attn_pwhole", 0);
    a.q = x.q;
    a.ldq = x.ldq;
    a.q_total_rows = x.q_total_rows;
    a.q_rms = x.q_rms;
    a.rms_parts = x.rms_parts;
    a.rms_inv_d = x.rms_d > 0 ? 1.f / static_cast<float>(x.rms_d) : 0.f;
    a.rms_eps = x.rms_eps;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // persistent grids: CTAs walk the items (knob attn_persist: 0 never, 1 the NT=1 short-key
    // instance only — cross-attention 640 -> 779 TF/s in-step —, 2 also self-attention, where
    // it measured slower: 1148-1151 vs 1157-1167 TF/s in-step, profiles/r2b)
    const int pk = tune_get("attn_persist", 1);
    // the persistent / NT=1 / pair instances are compiled with POLY = 6 only; attn_poly selects
    // the self-attention (NT = 2, one CTA per item) instance
    const bool ok_p = !tune_get("attn_trace", 0);
    const dim3 grid(static_cast<unsigned>((x.n_q + 2 * kTile - 1) / (2 * kTile)), x.heads, x.batch);
    const int cls = x.n_kv == x.n_q && x.q == x.k ? KC_SELF_ATTN : KC_CROSS_ATTN;
    prof_begin(cls, st);
    // short key sequences (cross-attention over the text tokens): one Q tile per CTA, two CTAs
    // per SM (AttnCfg<1>)
    const int nt1_knob = tune_get("attn_nt1", 1);  // 0 never, 1 short key sequences, 2 always (experiments)
    const bool nt1 = (nt1_knob == 2 || (nt1_knob == 1 && x.n_kv <= 4 * kTile)) && !tune_get("attn_trace", 0);
    if (nt1 && ok_p && pk >= 1) {
        const int64_t items = ((x.n_q + kTile - 1) / kTile) * x.heads * x.batch;
        const unsigned gp = static_cast<unsigned>(std::min<int64_t>(items, 2LL * sms));
        k_attention<6, false, 1, true><<<gp, AttnCfg<1>::threads, AttnCfg<1>::smem, st>>>(tq, tk, tv, to, a);
    } else if (nt1) {
        const dim3 g1(static_cast<unsigned>((x.n_q + kTile - 1) / kTile), x.heads, x.batch);
        k_attention<6, false, 1><<<g1, AttnCfg<1>::threads, AttnCfg<1>::smem, st>>>(tq, tk, tv, to, a);
    } else if (ok_p && tune_get("attn_qtm", 0) && x.ldq % 8 == 0 && (x.q_col0 % 8) == 0) {
        // CTA pairs, one Q tile per CTA resident in TMEM, double-buffered S (self-attention)
        const CUtensorMap tk64 = make_tmap_2d_bf16(x.k, x.ldk, x.kv_total_rows, x.ldk * 2, 64, 64);
        const unsigned tiles = static_cast<unsigned>((x.n_q + kTile - 1) / kTile);
        const dim3 gq((tiles + 1) / 2 * 2, x.heads, x.batch);
        k_attention_qt<6><<<gq, kQtThreads, kQtSmem, st>>>(tk64, tv, to, a);
    } else if (ok_p && tune_get("attn_pair", 0)) {
        // CTA pairs (self-attention): the K map's box is 64 key rows (each CTA loads half a block)
        const CUtensorMap tk64 = make_tmap_2d_bf16(x.k, x.ldk, x.kv_total_rows, x.ldk * 2, 64, 64);
        const unsigned groups = static_cast<unsigned>((x.n_q + 2 * kTile - 1) / (2 * kTile));
        const dim3 gp((groups + 1) / 2 * 2, x.heads, x.batch);
        k_attention_pair<6><<<gp, kAttnThreads, kPairSmem, st>>>(tq, tk64, tv, to, a);
    } else if (ok_p && pk >= 2) {
        const int64_t items = ((x.n_q + 2 * kTile - 1) / (2 * kTile)) * x.heads * x.batch;
        const unsigned gp = static_cast<unsigned>(std::min<int64_t>(items, sms));
        k_attention<6, false, 2, true><<<gp, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a);
    } else
    switch (tune_get("attn_trace", 0) ? -tune_get("attn_trace", 0) : attn_poly()) {
        case -1: k_attention<0, true><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
        case -2: k_attention<-1, true><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
        case -3: k_attention<-2, true><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
        case 0: k_attention<0><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
        case 6: k_attention<6><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
        case 8: k_attention<8><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
        default: k_attention<4><<<grid, kAttnThreads, kAttnSmem, st>>>(tq, tk, tv, to, a); break;
    }
    LP_LAUNCH_CHECK();
    prof_end(cls, st, 4.0 * x.batch * x.heads * static_cast<double>(x.n_q) * static_cast<double>(x.n_kv) * kHD,
             2.0 * x.batch * x.heads * kHD * (2.0 * x.n_q + 2.0 * x.n_kv));
}

}  // namespace lpb200

using namespace lpb200;

// Debug: device buffer of 64*2*16 u64 receiving the TR variant's timeline (lp_tune("attn_trace", 1)).
extern "C" int lp_attention_set_trace(void* dev_buf) {
    return guard([&] { LP_CUDA(cudaMemcpyToSymbol(g_attn_trace, &dev_buf, sizeof(void*))); });
}

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
