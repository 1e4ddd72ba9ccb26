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

template <int MODE, bool WARP>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;              // 2 x 32 KB (two 128x128 bf16 tiles, SW128 atoms)
    uint8_t* sB = sm + 65536;      // 64 KB (up to 256 rows x 128)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 131072);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const uint32_t warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
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
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int M>
static int launch(int iters, unsigned long long* o, cudaStream_t s, bool warp) {
    cudaFuncSetAttribute(k_mma<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    cudaFuncSetAttribute(k_mma<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    if (warp) k_mma<M, true><<<148, 128, 196608 + 2048, s>>>(iters, o);
    else k_mma<M, false><<<148, 128, 196608 + 2048, s>>>(iters, o);
    return (int)cudaGetLastError();
}

extern "C" int mma_bench(int mode, int iters, unsigned long long* dev_out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const bool w = mode >= 10;
    mode %= 10;
    switch (mode) {
        case 0: return launch<0>(iters, dev_out, s, w);
        case 1: return launch<1>(iters, dev_out, s, w);
        case 2: return launch<2>(iters, dev_out, s, w);
        case 3: return launch<3>(iters, dev_out, s, w);
        case 4: return launch<4>(iters, dev_out, s, w);
        case 5: return launch<5>(iters, dev_out, s, w);
        default: return launch<6>(iters, dev_out, s, w);
    }
}
