// common.cuh — status/error plumbing, launch accounting and the storage-dtype
// codec shared by every translation unit of liblp_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "lp_b200.h"

namespace lpb200 {

// C++ mirror of lpsim::Error (include/lpsim/errors.hpp:26-39); status = kind+1.
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Status(code, msg); }

void set_last_error(const std::string& msg);
void emit_warning(const std::string& msg);

// Every kernel launch issued by this library goes through this counter so the
// bench can report `gpu_launches` from the library itself.
void count_launch(uint64_t n = 1);
uint64_t launch_count();

#define LP_CUDA(call)                                                                            \
    do {                                                                                         \
        cudaError_t _e = (call);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            ::lpb200::fail(LP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
    } while (0)

#define LP_LAUNCH_CHECK()                                                                        \
    do {                                                                                         \
        ::lpb200::count_launch();                                                                \
        cudaError_t _e = cudaGetLastError();                                                     \
        if (_e != cudaSuccess)                                                                   \
            ::lpb200::fail(LP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

// Wrap a C-ABI body: exceptions -> status codes + thread-local message.
template <class F>
int guard(F&& f) {
    try {
        f();
        return LP_OK;
    } catch (const Status& s) {
        set_last_error(s.what());
        return s.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return LP_ERR_INVALID_ARGUMENT;
    }
}

inline void check_dtype(int d) {
    if (d != 2 && d != 4 && d != 8) fail(LP_ERR_INVALID_ARGUMENT, "dtype_bytes must be 2, 4 or 8, got " + std::to_string(d));
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Optional per-kernel-class timing (CUDA events on the launching stream), used by
// bench.py to measure the dominant kernel's live duration inside the timed region.
enum KernelClass {
    KC_SELF_ATTN = 0, KC_CROSS_ATTN = 1, KC_GEMM = 2,
    KC_ALLGATHER = 3,  // K9 ncclAllGather (bytes = received by this rank)
    KC_GATHER = 4,     // K1 partition gather (bytes = read + write)
    KC_RECON = 5,      // K10 reconstruct + sampler update (bytes = shards + z read, z write)
    KC_COUNT = 6
};
bool prof_enabled();
void prof_begin(int cls, cudaStream_t st);
void prof_end(int cls, cudaStream_t st, double flops, double bytes);

// Tuning knobs (kernel variants), set via lp_tune() or LP_TUNE_<KEY> env vars.
int tune_get(const char* key, int dflt);

// Device-side sticky error word (NonFinite etc.), read by lp_device_flags().
enum : unsigned { LP_FLAG_NONFINITE = 1u, LP_FLAG_ZERO_WEIGHT = 2u };
unsigned* device_flags_ptr();  // current device's flag word

}  // namespace lpb200

// ---------------------------------------------------------------------------
// Storage codec (src/dtype.cpp:34-116), device side.  Bit-identical to the
// reference's quantize(): f32 saturates at ±FLT_MAX, f16 is RNE straight from
// the double with ±65504 saturation and never produces Inf.
// ---------------------------------------------------------------------------
namespace lpb200 {

__host__ __device__ __forceinline__ uint16_t f16_encode_exact(double v) {
    if (v != v) return 0x7e00;
    if (v > 65504.0) v = 65504.0;
    if (v < -65504.0) v = -65504.0;
#ifdef __CUDA_ARCH__
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
#else
    uint64_t u;
    __builtin_memcpy(&u, &v, 8);
#endif
    const uint16_t sign = static_cast<uint16_t>((u >> 48) & 0x8000u);
    const int e = static_cast<int>((u >> 52) & 0x7ff) - 1023;
    if ((u << 1) == 0 || e < -25) return sign;
    const uint64_t m = (u & 0xfffffffffffffull) | (1ull << 52);
    const int shift = e >= -14 ? 42 : 42 + (-14 - e);
    uint16_t h = e >= -14 ? static_cast<uint16_t>(((e + 15) << 10) | ((m >> 42) & 0x3ff))
                          : static_cast<uint16_t>(m >> shift);
    const uint64_t rem = m & ((1ull << shift) - 1), half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) h = static_cast<uint16_t>(h + 1);
    if ((h & 0x7fff) >= 0x7c00) h = 0x7bff;
    return static_cast<uint16_t>(sign | h);
}

__host__ __device__ __forceinline__ double f16_decode_exact(uint16_t b) {
    const int e = (b >> 10) & 0x1f;
    const int m = b & 0x3ff;
    const double s = (b & 0x8000) ? -1.0 : 1.0;
    // m * 2^-24 and (m|0x400) * 2^(e-25) are exact products in double.
    if (e == 0) return s * (static_cast<double>(m) * 5.9604644775390625e-08);
    if (e == 31) {
#ifdef __CUDA_ARCH__
        return m ? __longlong_as_double(0x7ff8000000000000ll) : s * __longlong_as_double(0x7ff0000000000000ll);
#else
        return m ? __builtin_nan("") : s * __builtin_inf();
#endif
    }
    double scale = 1.0;
    int ex = e - 25;
    // exact power of two in [2^-24, 2^5]
    if (ex >= 0) { for (int i = 0; i < ex; ++i) scale *= 2.0; }
    else { for (int i = 0; i < -ex; ++i) scale *= 0.5; }
    return s * (static_cast<double>(m | 0x400) * scale);
}

template <int D> struct Store;
template <> struct Store<2> { using T = uint16_t; };
template <> struct Store<4> { using T = float; };
template <> struct Store<8> { using T = double; };

template <int D>
__device__ __forceinline__ double load_val(const typename Store<D>::T* p, int64_t i);
template <> __device__ __forceinline__ double load_val<2>(const uint16_t* p, int64_t i) { return f16_decode_exact(p[i]); }
template <> __device__ __forceinline__ double load_val<4>(const float* p, int64_t i) { return static_cast<double>(p[i]); }
template <> __device__ __forceinline__ double load_val<8>(const double* p, int64_t i) { return p[i]; }

// quantize + store; returns false when the stored value is not finite
// (LatentTensor::from_doubles rejects it, src/latent.cpp:72-77).
template <int D>
__device__ __forceinline__ bool store_q(typename Store<D>::T* p, int64_t i, double v);
template <> __device__ __forceinline__ bool store_q<8>(double* p, int64_t i, double v) {
    p[i] = v;
    return isfinite(v);
}
template <> __device__ __forceinline__ bool store_q<4>(float* p, int64_t i, double v) {
    const double lim = 3.4028234663852886e+38;
    float f = v > lim ? 3.4028234663852886e+38f : (v < -lim ? -3.4028234663852886e+38f : __double2float_rn(v));
    p[i] = f;
    return isfinite(f);
}
template <> __device__ __forceinline__ bool store_q<2>(uint16_t* p, int64_t i, double v) {
    const uint16_t h = f16_encode_exact(v);
    p[i] = h;
    return (h & 0x7c00) != 0x7c00;
}

template <int D>
__device__ __forceinline__ double quantize_dev(double v) {
    if constexpr (D == 8) return v;
    if constexpr (D == 4) {
        const double lim = 3.4028234663852886e+38;
        return v > lim ? lim : (v < -lim ? -lim : static_cast<double>(__double2float_rn(v)));
    }
    return f16_decode_exact(f16_encode_exact(v));
}

}  // namespace lpb200
