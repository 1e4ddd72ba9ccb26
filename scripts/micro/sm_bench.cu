// Microbenchmark of the attention softmax inner loop in isolation (no MMA): W warps per
// SMSP each loop over `iters` x {LDTM 64 fp32 columns of its TMEM lanes, 64 exp2 via
// FFMA2 + MUFU.EX2, row-sum FADD2, pack bf16, STTM 32 columns}.  Reports cycles per
// 64-key chunk per warp.  mode bit0: skip TMEM (registers only); bit1: skip MUFU (FFMA only);
// bit2: pack with PRMT (truncation) instead of F2FP; bits 4..7: POLY pairs of 16 on the FMA pipe
#include <cuda.h>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace lpb200::tc;

__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -126.f);
    x.y = fmaxf(x.y, -126.f);
    const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
    const float2 fl = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(fl, make_float2(-1.f, -1.f), x);
    float2 p = __ffma2_rn(f, make_float2(0.05516f, 0.05516f), make_float2(0.24258f, 0.24258f));
    p = __ffma2_rn(p, f, make_float2(0.69326f, 0.69326f));
    p = __ffma2_rn(p, f, make_float2(0.99993f, 0.99993f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
__device__ __forceinline__ float ex2f_(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MODE>
__global__ void k_sm(int iters, unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    __shared__ volatile uint32_t stop;
    __shared__ uint64_t mb;
    extern __shared__ __align__(1024) uint8_t ops[];  // MMA operands (bit 8 mode)
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        stop = 0;
        mbar_init(&mb, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if ((MODE & 256) && warp == blockDim.x / 32 - 1) {
        // background tensor-pipe load: one lane issues 128x128x16 MMAs into TMEM columns [256, 384)
        __syncthreads();  // pairs with the softmax warps' pre-timing barrier
        if ((threadIdx.x & 31) == 0) {
            const uint64_t dA = desc_sw128(smem_u32(ops)), dB = desc_sw128(smem_u32(ops + 32768));
            constexpr uint32_t id = idesc_bf16(128, 128);
            while (!stop)
#pragma unroll
                for (int k = 0; k < 8; ++k) mma_ss(tmem + 256, dA + 2 * (k & 3), dB + 2 * (k & 3), id, 1);
            mma_commit(&mb);
            mbar_wait(&mb, 0);
        }
        __syncwarp();
        tc_fence_before();
        __syncthreads();  // pairs with the final barrier
        return;
    }
    const uint32_t q = warp & 3, w = warp >> 2;
    const uint32_t tS = tmem + ((q * 32) << 16) + w * 64;
    float2 acc = make_float2(0.f, 0.f);
    uint32_t seed = threadIdx.x;
    uint32_t r[64];
#pragma unroll
    for (int u = 0; u < 64; ++u) r[u] = __float_as_uint(-(float)((seed + u) & 15));
    const float2 c2 = make_float2(0.125f, 0.125f), m2 = make_float2(-1.f, -1.f);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (!(MODE & 1)) {
            tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(r));
            tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            tmem_ld_wait();
        }
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
            uint32_t pk[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[cc + 2 * u]), __uint_as_float(r[cc + 2 * u + 1])), c2, m2);
                float2 p;
                constexpr int POLY = (MODE >> 4) & 15;
                if (MODE & 2) {
                    p = __ffma2_rn(x, x, c2);
                } else if (POLY > 0 && ((u * 5) & 15) < POLY) {
                    p = ex2_poly2(x);
                } else {
                    p.x = ex2f_(x.x);
                    p.y = ex2f_(x.y);
                }
                acc = __fadd2_rn(acc, p);
                if (MODE & 4) pk[u] = __byte_perm(__float_as_uint(p.x), __float_as_uint(p.y), 0x7632);
                else pk[u] = pack_bf16(p.x, p.y);
            }
            if (!(MODE & 1)) tmem_st16(tS + cc / 2, pk);
            else {
#pragma unroll
                for (int u = 0; u < 16; ++u) r[cc + u] ^= pk[u];
            }
        }
        if (!(MODE & 1)) tmem_st_wait();
    }
    const long long t1 = clock64();
    if (MODE & 256) {
        __syncwarp();
        if (threadIdx.x == 0) stop = 1;
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
    if (blockIdx.x == 0 && lane == 0 && warp == 0) out[0] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

extern "C" int sm_bench(int mode, int warps, int iters, unsigned long long* out, float* sink, void* st) {
    auto s = (cudaStream_t)st;
    switch (mode) {
#define C_(m) case m: cudaFuncSetAttribute(k_sm<m>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024); \
        k_sm<m><<<148, warps * 32 + ((m & 256) ? 32 : 0), 65536 + 1024, s>>>(iters, out, sink); break;
        C_(0) C_(1) C_(2) C_(3) C_(4) C_(5) C_(6) C_(7) C_(0x40) C_(0x60) C_(0x80) C_(0x44) C_(0x64) C_(0x41) C_(0x61)
        C_(0x100) C_(0x160) C_(0x101)
#undef C_
        default: return -1;
    }
    return (int)cudaGetLastError();
}
