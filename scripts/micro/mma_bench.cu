// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1) for the operand
// modes the attention kernel uses.  One CTA per SM, one thread issues `iters` x 8 MMAs
// back to back (K = 128 per group, like one S or PV tile product), commit, wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -I paper_2512_07350_b200/csrc -I include scripts/micro/mma_bench.cu -o scripts/micro/libmma_bench.so
#include <cuda.h>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace lpb200::tc;

// mode: 0 SS N128 (S=QK^T), 1 TS N128 B MN-major (PV), 2 SS N256, 3 SS N64, 4 TS N128 B K-major,
//       5 SS N128 B MN-major, 6 two SS N128 groups sharing B with different A (S0,S1 of one K tile)
// Descriptors are built once; the per-k offsets are added to the 64-bit descriptor's
// start-address field (addr >> 4) so the issue loop is only the MMA instructions.
__device__ __forceinline__ void mma_ss_acc(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void mma_ts_acc(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%4, %4, %4, %4}, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(0u));
}

template <int MODE, bool WARP, int CONTEND = 0>
__global__ void __launch_bounds__(384, 1) k_mma(int iters, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;              // 2 x 32 KB (two 128x128 bf16 tiles, SW128 atoms)
    uint8_t* sB = sm + 65536;      // 64 KB (up to 256 rows x 128)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 131072);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    const uint32_t warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 2, 1); fence_barrier_init(); slot[1] = 0u; slot[2] = 0u; }
    if (warp == 0) tmem_alloc(slot, 512);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    // WARP: the whole warp 0 runs the (converged) issue loop and one elected lane issues
    // each MMA, so descriptors and TMEM addresses stay in uniform registers; otherwise
    // lane 0 alone runs it (divergent code: R2UR.BROADCAST + elect loop per MMA).
    if (WARP ? warp == 0 : threadIdx.x == 0) {
        constexpr int kAtom = 128 * 128;
        const uint64_t dA = desc_sw128(smem_u32(sA)), dB = desc_sw128(smem_u32(sB));
        const uint64_t dBmn = desc_sw128(smem_u32(sB), 1024, kAtom);
        constexpr uint32_t id128 = idesc_bf16(128, 128), id256 = idesc_bf16(128, 256), id64 = idesc_bf16(128, 64);
        constexpr uint32_t id128mn = idesc_bf16(128, 128, true);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t off = ((k >> 2) * kAtom + (k & 3) * 32) >> 4;
                if (WARP && !elect_one()) continue;
                if (MODE == 0) mma_ss_acc(tmem, dA + off, dB + off, id128);
                if (MODE == 1) mma_ts_acc(tmem, tmem + 256 + k * 8, dBmn + ((k * 2048) >> 4), id128mn);
                if (MODE == 2) mma_ss_acc(tmem, dA + off, dB + (((k >> 2) * 2 * kAtom + (k & 3) * 32) >> 4), id256);
                if (MODE == 3) mma_ss_acc(tmem, dA + off, dB + off, id64);
                if (MODE == 4) mma_ts_acc(tmem, tmem + 256 + k * 8, dB + off, id128);
                if (MODE == 5) mma_ss_acc(tmem, dA + off, dBmn + ((k * 2048) >> 4), id128mn);
                if (MODE == 7 || MODE == 8) {
                    // attention-like: PV (TS, A = P in S's columns) then the next S writing D over
                    // those columns (7: WAR on TMEM) or over another region (8: no overlap)
                    if (k < 4) {
                        mma_ts_acc(tmem + 256, tmem + k * 8, dBmn + ((k * 2048) >> 4), id128mn);
                        mma_ts_acc(tmem + 256, tmem + 32 + k * 8, dBmn + (((k + 4) * 2048) >> 4), id128mn);
                    } else {
                        const uint64_t o2 = (((k - 4) >> 2) * kAtom + ((k - 4) & 3) * 32) >> 4;
                        const uint32_t dS = MODE == 7 ? tmem : tmem + 128;
                        mma_ss_acc(dS, dA + o2, dB + o2, id128);
                        mma_ss_acc(dS, dA + o2 + 2, dB + o2 + 2, id128);
                    }
                }
                if (MODE == 13 || MODE == 14 || MODE == 15) {
                    if ((k & 3) == 0) {
                        const uint32_t ba = smem_u32(bar + 2);
                        if (MODE == 13) {  // non-blocking test_wait
                            uint32_t ok;
                            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                                         "selp.u32 %0, 1, 0, P1;\n\t}\n" : "=r"(ok) : "r"(ba), "r"(1u) : "memory");
                            if (!ok) __trap();
                        } else if (MODE == 14) {  // try_wait without the tcgen05 fence
                            if (!mbar_try_wait(ba, 1)) __trap();
                        } else {  // volatile shared-memory flag poll
                            if (*reinterpret_cast<volatile uint32_t*>(slot + 2) != 0u) __trap();
                        }
                        tc_fence_after();
                    }
                    mma_ss_acc(tmem + (k & 1) * 128, dA + off, dB + off, id128);
                }
                if (MODE == 11 || MODE == 12) {
                    // tcgen05.fence::after_thread_sync every 4 MMAs (11), or an mbarrier try_wait on an
                    // already-completed phase + fence every 4 MMAs (12) — the attention issuer's pattern
                    if ((k & 3) == 0) {
                        if (MODE == 12) mbar_wait(bar + 2, 1);
                        tc_fence_after();
                    }
                    mma_ss_acc(tmem + (k & 1) * 128, dA + off, dB + off, id128);
                }
                if (MODE == 9 || MODE == 10) {
                    mma_ss_acc(tmem + (k & 1) * 128, dA + off, dB + off, id128);
                    if (MODE == 9 && k == 7) mma_commit(bar + 2);   // one commit per 8-MMA group
                    if (MODE == 10 && (k & 1)) mma_commit(bar + 2); // one per 2 MMAs
                }
                if (MODE == 6) {
                    mma_ss_acc(tmem, dA + off, dB + off, id128);
                    mma_ss_acc(tmem + 128, dA + ((2 * kAtom) >> 4) + off, dB + off, id128);
                }
            }
        }
        if (!WARP || elect_one()) mma_commit(bar);
        __syncwarp(WARP ? 0xffffffffu : 1u);
        mbar_wait(bar, 0);
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[0] = t1 - t0;
        *reinterpret_cast<volatile uint32_t*>(slot + 1) = 1u;
    }
    if (CONTEND && warp >= 4) {
        // softmax-like TMEM traffic: each warp streams 64 columns of its lane quarter (cols 384..447
        // of the accumulator-free region) in and 32 columns out, until the MMA thread is done
        volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(slot + 1);
        const uint32_t q = warp & 3;
        const uint32_t base = tmem + ((q * 32) << 16) + 384 + ((warp >> 2) & 1) * 64;
        uint32_t acc = 0;
        while (*flag == 0) {
            uint32_t r[32];
            tmem_ld32(base, r);
            tmem_ld_wait();
            uint32_t s[32];
            tmem_ld32(base + 32, s);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) pk[u] = r[2 * u] ^ s[2 * u + 1];
            if (CONTEND == 2) tmem_st16(base, pk);
            acc += pk[0];
        }
        if (acc == 0x12345678u) out[1] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int M>
static int launch(int iters, unsigned long long* o, cudaStream_t s, bool warp, int contend) {
    cudaFuncSetAttribute(k_mma<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    cudaFuncSetAttribute(k_mma<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    cudaFuncSetAttribute(k_mma<M, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    cudaFuncSetAttribute(k_mma<M, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    if (contend == 1) k_mma<M, false, 1><<<148, 384, 196608 + 2048, s>>>(iters, o);
    else if (contend == 2) k_mma<M, false, 2><<<148, 384, 196608 + 2048, s>>>(iters, o);
    else if (warp) k_mma<M, true><<<148, 128, 196608 + 2048, s>>>(iters, o);
    else k_mma<M, false><<<148, 128, 196608 + 2048, s>>>(iters, o);
    return (int)cudaGetLastError();
}

extern "C" int mma_bench(int mode, int iters, unsigned long long* dev_out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int contend = mode / 100;
    mode %= 100;
    const bool w = mode >= 20;
    mode %= 20;
    switch (mode) {
        case 0: return launch<0>(iters, dev_out, s, w, contend);
        case 1: return launch<1>(iters, dev_out, s, w, contend);
        case 2: return launch<2>(iters, dev_out, s, w, contend);
        case 3: return launch<3>(iters, dev_out, s, w, contend);
        case 4: return launch<4>(iters, dev_out, s, w, contend);
        case 5: return launch<5>(iters, dev_out, s, w, contend);
        case 6: return launch<6>(iters, dev_out, s, w, contend);
        case 7: return launch<7>(iters, dev_out, s, w, contend);
        case 8: return launch<8>(iters, dev_out, s, w, contend);
        case 9: return launch<9>(iters, dev_out, s, w, contend);
        case 10: return launch<10>(iters, dev_out, s, w, contend);
        case 11: return launch<11>(iters, dev_out, s, w, contend);
        case 12: return launch<12>(iters, dev_out, s, w, contend);
        case 13: return launch<13>(iters, dev_out, s, w, contend);
        case 14: return launch<14>(iters, dev_out, s, w, contend);
        default: return launch<15>(iters, dev_out, s, w, contend);
    }
}
