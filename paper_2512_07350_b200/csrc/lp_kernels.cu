// lp_kernels.cu — HBM-bound LP kernels for sm_100a:
//   K1  partition gather       (extract_sublatents / slice_axis)
//   K10 reconstruct + sampler  (reconstruct, sampler_step), exact & fast modes
//   K11 toy denoisers + CFG    (Box / GlobalMix / Identity, cfg_predict)
//
// Compiled with -fmad=false and written with explicit __d*_rn intrinsics: the
// EXACT paths reproduce the reference's fp64 arithmetic (no FMA contraction,
// worker-ordered sums, true division) bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "recon.hpp"
#include "tc_ptx.cuh"

namespace lpb200 {

__device__ unsigned g_lp_flags;

namespace {
std::atomic<uint64_t> g_launches{0};
}
void count_launch(uint64_t n) { g_launches += n; }
uint64_t launch_count() { return g_launches.load(); }

unsigned* device_flags_ptr() {
    void* p = nullptr;
    LP_CUDA(cudaGetSymbolAddress(&p, g_lp_flags));
    return static_cast<unsigned*>(p);
}

__device__ __forceinline__ void raise_flag(unsigned f) { atomicOr(&g_lp_flags, f); }

static int grid_for(int64_t n, int threads, int per_sm = 8) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const int64_t need = (n + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(sms) * per_sm;
    return static_cast<int>(need < cap ? (need > 0 ? need : 1) : cap);
}

// ---------------------------------------------------------------------------
// K1: partition gather.  dst[o, j, i] = z[o, s + j, i] for o < outer, j < len,
// i < inner — a pure copy, moved as the widest vector (16/8/4/2 B) that the
// run length, source offset and alignment allow.  Coalesced on both sides.
// ---------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) k_slice_copy(const V* __restrict__ src, V* __restrict__ dst, int64_t outer,
                                                    int64_t run, int64_t src_stride, int64_t src_off) {
    // run = len*inner (in V units), src_stride = D*inner, src_off = s*inner
    const int64_t total = outer * run;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = idx / run;
        const int64_t r = idx - o * run;
        dst[idx] = __ldg(src + o * src_stride + src_off + r);
    }
}

// 32-bit variant (outer*run < 2^31): row/offset split by multiply-shift division, 4
// independent vectors in flight per thread per iteration.
template <typename V>
__global__ void __launch_bounds__(256) k_slice_copy32(const V* __restrict__ src, V* __restrict__ dst, uint32_t total,
                                                      uint32_t run, FastDiv div_run, uint32_t src_stride,
                                                      uint32_t src_off) {
    const uint32_t step = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < total; base += 4 * step) {
        V v[4];
        uint32_t at[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t idx = base + u * step;
            at[u] = idx;
            if (idx < total) {
                const uint32_t o = static_cast<uint32_t>((static_cast<uint64_t>(idx) * div_run.mul) >> div_run.shift);
                v[u] = __ldg(src + static_cast<uint64_t>(o) * src_stride + src_off + (idx - o * run));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (at[u] < total) dst[at[u]] = v[u];
    }
}

// K1 through the TMA engine: the window is `outer` contiguous runs of run_b bytes (src
// stride stride_b) packed back to back in dst.  Runs are cut into <= 16 KB chunks; each
// warp's lane 0 is an independent copy engine with two shared-memory stages: bulk-load a
// chunk (mbarrier complete_tx), bulk-store it, and load the next chunk into the other
// stage while the store drains.  Requires 16-byte alignment of addresses, run and stride.
constexpr int kSliceChunk = 16 * 1024, kSliceWarps = 4;
__global__ void __launch_bounds__(32 * kSliceWarps) k_slice_bulk(const uint8_t* __restrict__ src,
                                                                 uint8_t* __restrict__ dst, int64_t outer,
                                                                 int64_t run_b, int64_t stride_b, int64_t off_b) {
    extern __shared__ __align__(128) uint8_t sbuf[];  // [warps][2][chunk]
    __shared__ uint64_t bars[kSliceWarps][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane != 0) return;
    uint64_t* bar = bars[warp];
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_barrier_init();
    uint8_t* buf = sbuf + static_cast<size_t>(warp) * 2 * kSliceChunk;
    const int64_t cpr = (run_b + kSliceChunk - 1) / kSliceChunk, nchunks = outer * cpr;
    const int64_t engines = static_cast<int64_t>(gridDim.x) * kSliceWarps;
    uint32_t ph[2] = {0, 0};
    int it = 0;
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * kSliceWarps + warp; c < nchunks; c += engines, ++it) {
        const int b = it & 1;
        const int64_t o = c / cpr, piece = c - o * cpr;
        const int64_t at = piece * kSliceChunk;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kSliceChunk), run_b - at));
        if (it >= 2) tc::bulk_wait_read<1>();  // the store issued from this stage two chunks ago has read it
        tc::mbar_arrive_expect_tx(&bar[b], bytes);
        tc::bulk_load(buf + b * kSliceChunk, src + o * stride_b + off_b + at, bytes, &bar[b]);
        tc::mbar_wait(&bar[b], ph[b]);
        ph[b] ^= 1;
        tc::bulk_store(dst + o * run_b + at, buf + b * kSliceChunk, bytes);
        tc::bulk_commit();
    }
    tc::bulk_wait_all();
}

template <typename V>
static void launch_slice(const void* src, void* dst, int64_t outer, int64_t run, int64_t stride, int64_t off,
                         cudaStream_t st) {
    const int64_t total = outer * run;
    if (total < (1ll << 31) && outer * stride < (1ll << 32)) {
        k_slice_copy32<V><<<grid_for((total + 3) / 4, 256, 16), 256, 0, st>>>(
            static_cast<const V*>(src), static_cast<V*>(dst), static_cast<uint32_t>(total), static_cast<uint32_t>(run),
            make_fastdiv(static_cast<uint32_t>(run)), static_cast<uint32_t>(stride), static_cast<uint32_t>(off));
    } else {
        k_slice_copy<V><<<grid_for(total, 256), 256, 0, st>>>(static_cast<const V*>(src), static_cast<V*>(dst), outer,
                                                              run, stride, off);
    }
    LP_LAUNCH_CHECK();
}

void slice_to(const void* z, const Shape4& s, int axis, i64 begin, i64 end, int E, void* dst, cudaStream_t st) {
    i64 outer, inner;
    axis_view(s, axis, outer, inner);
    const i64 D = s.extent(axis);
    const i64 run_b = (end - begin) * inner * E, stride_b = D * inner * E, off_b = begin * inner * E;
    const uintptr_t al = reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(dst);
    prof_begin(KC_GATHER, st);
    if (run_b % 16 == 0 && stride_b % 16 == 0 && off_b % 16 == 0 && al % 16 == 0 && tune_get("slice_tma", 1)) {
        // TMA-staged path (T and H windows; W windows of 4 x 16-byte multiples)
        static bool attr = false;
        constexpr int smem = kSliceWarps * 2 * kSliceChunk;
        if (!attr) {
            LP_CUDA(cudaFuncSetAttribute(k_slice_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr = true;
        }
        const int64_t chunks = outer * ((run_b + kSliceChunk - 1) / kSliceChunk);
        const int grid = static_cast<int>(std::min<int64_t>((chunks + kSliceWarps - 1) / kSliceWarps, 148));
        k_slice_bulk<<<grid, 32 * kSliceWarps, smem, st>>>(static_cast<const uint8_t*>(z), static_cast<uint8_t*>(dst),
                                                            outer, run_b, stride_b, off_b);
        LP_LAUNCH_CHECK();
        prof_end(KC_GATHER, st, 0.0, 2.0 * static_cast<double>(outer) * static_cast<double>(run_b));
        return;
    }
    for (int vb : {16, 8, 4, 2, 1}) {
        if (run_b % vb || stride_b % vb || off_b % vb || al % vb) continue;
        switch (vb) {
            case 16: launch_slice<uint4>(z, dst, outer, run_b / 16, stride_b / 16, off_b / 16, st); break;
            case 8: launch_slice<uint2>(z, dst, outer, run_b / 8, stride_b / 8, off_b / 8, st); break;
            case 4: launch_slice<uint32_t>(z, dst, outer, run_b / 4, stride_b / 4, off_b / 4, st); break;
            case 2: launch_slice<uint16_t>(z, dst, outer, run_b / 2, stride_b / 2, off_b / 2, st); break;
            default: launch_slice<uint8_t>(z, dst, outer, run_b, stride_b, off_b, st); break;
        }
        break;
    }
    prof_end(KC_GATHER, st, 0.0, 2.0 * static_cast<double>(outer) * static_cast<double>(run_b));
}

// ---------------------------------------------------------------------------
// K11: toy denoisers (src/denoise.cpp:56-142), fp64 in the reference order.
// MODE 0: plain predict (affine a0) -> out.
// MODE 1: fused cfg_predict: u = q(m + a0), c = q(m + a1), out = q(u + w(c-u)).
// ---------------------------------------------------------------------------
template <int D, int MODE>
__global__ void __launch_bounds__(256) k_box(const typename Store<D>::T* __restrict__ z,
                                             typename Store<D>::T* __restrict__ out, int64_t C, int64_t T, int64_t H,
                                             int64_t W, int64_t rt, int64_t rh, int64_t rw, double a0, double a1,
                                             double w_cfg) {
    const int64_t total = C * T * H * W;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx;
        const int64_t x = r % W; r /= W;
        const int64_t y = r % H; r /= H;
        const int64_t t = r % T;
        const int64_t c = r / T;
        const int64_t t0 = max((int64_t)0, t - rt), t1 = min(T - 1, t + rt);
        const int64_t h0 = max((int64_t)0, y - rh), h1 = min(H - 1, y + rh);
        const int64_t w0 = max((int64_t)0, x - rw), w1 = min(W - 1, x + rw);
        double acc = 0.0;
        for (int64_t a = t0; a <= t1; ++a)
            for (int64_t b = h0; b <= h1; ++b) {
                const int64_t row = ((c * T + a) * H + b) * W;
                for (int64_t e = w0; e <= w1; ++e) acc = __dadd_rn(acc, load_val<D>(z, row + e));
            }
        const double n = static_cast<double>((t1 - t0 + 1) * (h1 - h0 + 1) * (w1 - w0 + 1));
        const double m = __ddiv_rn(acc, n);
        bool ok;
        if (MODE == 0) {
            ok = store_q<D>(out, idx, __dadd_rn(m, a0));
        } else {
            const double u = quantize_dev<D>(__dadd_rn(m, a0));
            const double cc = quantize_dev<D>(__dadd_rn(m, a1));
            ok = isfinite(u) && isfinite(cc);
            ok = store_q<D>(out, idx, __dadd_rn(u, __dmul_rn(w_cfg, __dsub_rn(cc, u)))) && ok;
        }
        if (!ok) raise_flag(LP_FLAG_NONFINITE);
    }
}

// GlobalMix channel sums: the reference sums each channel sequentially in
// index order (src/denoise.cpp:112-116); a parallel tree would round
// differently, so one thread per channel walks it in order.
template <int D>
__global__ void k_channel_sum(const typename Store<D>::T* __restrict__ z, int64_t C, int64_t per, double* sums) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C) return;
    double acc = 0.0;
    for (int64_t i = 0; i < per; ++i) acc = __dadd_rn(acc, load_val<D>(z, c * per + i));
    sums[c] = __ddiv_rn(acc, static_cast<double>(per));
}

template <int D, int MODE>
__global__ void __launch_bounds__(256) k_global(const typename Store<D>::T* __restrict__ z,
                                                typename Store<D>::T* __restrict__ out, int64_t total, int64_t per,
                                                const double* __restrict__ means, double a0, double a1, double w_cfg) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const double mean = means[idx / per];
        const double base = __dadd_rn(__dmul_rn(0.5, load_val<D>(z, idx)), __dmul_rn(0.5, mean));
        bool ok;
        if (MODE == 0) {
            ok = store_q<D>(out, idx, __dadd_rn(base, a0));
        } else {
            const double u = quantize_dev<D>(__dadd_rn(base, a0));
            const double cc = quantize_dev<D>(__dadd_rn(base, a1));
            ok = isfinite(u) && isfinite(cc);
            ok = store_q<D>(out, idx, __dadd_rn(u, __dmul_rn(w_cfg, __dsub_rn(cc, u)))) && ok;
        }
        if (!ok) raise_flag(LP_FLAG_NONFINITE);
    }
}

// Identity under CFG: u = c = z, out = q(z + w*(z - z)).
template <int D, int MODE>
__global__ void __launch_bounds__(256) k_identity(const typename Store<D>::T* __restrict__ z,
                                                  typename Store<D>::T* __restrict__ out, int64_t total, double w_cfg) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const double v = load_val<D>(z, idx);
        const double r = MODE == 0 ? v : __dadd_rn(v, __dmul_rn(w_cfg, __dsub_rn(v, v)));
        if (!store_q<D>(out, idx, r)) raise_flag(LP_FLAG_NONFINITE);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_cfg_combine(const typename Store<D>::T* __restrict__ u,
                                                     const typename Store<D>::T* __restrict__ c,
                                                     typename Store<D>::T* __restrict__ out, int64_t n, double w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double uu = load_val<D>(u, i);
        if (!store_q<D>(out, i, __dadd_rn(uu, __dmul_rn(w, __dsub_rn(load_val<D>(c, i), uu)))))
            raise_flag(LP_FLAG_NONFINITE);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_sampler(const typename Store<D>::T* __restrict__ z,
                                                 const typename Store<D>::T* __restrict__ eps,
                                                 typename Store<D>::T* __restrict__ out, int64_t n, double eta) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!store_q<D>(out, i, __dsub_rn(load_val<D>(z, i), __dmul_rn(eta, load_val<D>(eps, i)))))
            raise_flag(LP_FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------
// K10: reconstruct (+ sampler).  Gather form: every output element (o, x, i)
// visits the entries covering x in worker order.
//   Z = Σ_k w_k(x)            (all covering entries, src/reconstruct.cpp:70-74)
//   A = Σ_{k: w≠0} w_k·pred_k (src/reconstruct.cpp:93-107)
//   ε̂ = q(A / Z); UPDATE: z = q(z - η ε̂)
// Weights are recomputed on device with the host's exact formulas
// (j/Δs, (ℓ-j)/Δe, IEEE division) — identical doubles.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double entry_weight(const ReconEntry& e, int64_t j) {
    if (j >= e.len - e.de) return __ddiv_rn(static_cast<double>(e.len - j), static_cast<double>(e.de));
    if (j < e.ds) return __ddiv_rn(static_cast<double>(j), static_cast<double>(e.ds));
    return 1.0;
}

template <int D, bool UPDATE, bool FAST>
__global__ void __launch_bounds__(256) k_reconstruct(const __grid_constant__ ReconParams p,
                                                     const typename Store<D>::T* __restrict__ preds,
                                                     typename Store<D>::T* __restrict__ z,
                                                     typename Store<D>::T* __restrict__ eps_out) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < p.total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % p.inner;
        const int64_t ox = idx / p.inner;
        const int64_t x = ox % p.D;
        const int64_t o = ox / p.D;
        double eps;
        if (!FAST) {
            double zs = 0.0, a = 0.0;
            for (int k = 0; k < p.n; ++k) {
                const ReconEntry& e = p.e[k];
                const int64_t j = x - e.begin;
                if (j < 0) break;  // entries are sorted by begin
                if (j >= e.len) continue;
                const double w = entry_weight(e, j);
                zs = __dadd_rn(zs, w);
                if (w != 0.0) a = __dadd_rn(a, __dmul_rn(w, load_val<D>(preds, e.base + (o * e.len + j) * p.inner + i)));
            }
            eps = quantize_dev<D>(__ddiv_rn(a, zs));
        } else {
            float zs = 0.f, a = 0.f;
            for (int k = 0; k < p.n; ++k) {
                const ReconEntry& e = p.e[k];
                const int64_t j = x - e.begin;
                if (j < 0) break;
                if (j >= e.len) continue;
                const float w = static_cast<float>(entry_weight(e, j));
                zs += w;
                a = fmaf(w, static_cast<float>(load_val<D>(preds, e.base + (o * e.len + j) * p.inner + i)), a);
            }
            eps = quantize_dev<D>(static_cast<double>(a / zs));
        }
        bool ok = isfinite(eps);
        if (UPDATE) {
            const double zn = FAST ? static_cast<double>(fmaf(-static_cast<float>(p.eta), static_cast<float>(eps),
                                                              static_cast<float>(load_val<D>(z, idx))))
                                   : __dsub_rn(load_val<D>(z, idx), __dmul_rn(p.eta, eps));
            ok = store_q<D>(z, idx, zn) && ok;
        } else {
            ok = store_q<D>(eps_out, idx, eps) && ok;
        }
        if (!ok) raise_flag(LP_FLAG_NONFINITE);
    }
}

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
    return static_cast<uint32_t>((static_cast<uint64_t>(x) * f.mul) >> f.shift);
}

// K10, exact mode, 32-bit indexing: the per-position weights w_k(x) and their sum
// Z(x) = Σ_k w_k(x) (worker order, the same IEEE divisions and adds as entry_weight and
// the reference) are tabulated once per block in shared memory ([n+1][D] doubles); every
// element then costs its shard loads, Σ w·pred in worker order, one true division and
// the sampler update.  Index decomposition uses multiply-shift division (FastDiv).
template <int D, bool UPDATE>
__global__ void __launch_bounds__(256) k_reconstruct_tab(const __grid_constant__ ReconParams p,
                                                         const typename Store<D>::T* __restrict__ preds,
                                                         typename Store<D>::T* __restrict__ z,
                                                         typename Store<D>::T* __restrict__ eps_out) {
    extern __shared__ double wt[];  // [n][Dx] weights, then [Dx] sums
    const int Dx = static_cast<int>(p.D), n = p.n;
    double* zsum = wt + n * Dx;
    for (int x = threadIdx.x; x < Dx; x += blockDim.x) {
        double zs = 0.0;
        for (int k = 0; k < n; ++k) {
            const ReconEntry& e = p.e[k];
            const int64_t j = x - e.begin;
            const double w = (j < 0 || j >= e.len) ? 0.0 : entry_weight(e, j);
            if (j >= 0 && j < e.len) zs = __dadd_rn(zs, w);
            wt[k * Dx + x] = w;
        }
        zsum[x] = zs;
    }
    __syncthreads();
    const uint32_t total = static_cast<uint32_t>(p.total), inner = static_cast<uint32_t>(p.inner);
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const uint32_t ox = fdiv(idx, p.div_inner);
        const uint32_t i = idx - ox * inner;
        const uint32_t o = fdiv(ox, p.div_d);
        const int x = static_cast<int>(ox - o * static_cast<uint32_t>(Dx));
        double a = 0.0;
        for (int k = 0; k < n; ++k) {
            const ReconEntry& e = p.e[k];
            const int64_t j = x - e.begin;
            if (j < 0) break;  // entries are sorted by begin
            if (j >= e.len) continue;
            const double w = wt[k * Dx + x];
            if (w != 0.0)
                a = __dadd_rn(a, __dmul_rn(w, load_val<D>(preds, e.base + (static_cast<int64_t>(o) * e.len + j) * inner + i)));
        }
        const double eps = quantize_dev<D>(__ddiv_rn(a, zsum[x]));
        bool ok = isfinite(eps);
        if (UPDATE) ok = store_q<D>(z, idx, __dsub_rn(load_val<D>(z, idx), __dmul_rn(p.eta, eps))) && ok;
        else ok = store_q<D>(eps_out, idx, eps) && ok;
        if (!ok) raise_flag(LP_FLAG_NONFINITE);
    }
}

template <int D, bool UPDATE>
static void launch_recon(const ReconParams& p, const void* preds, void* z, void* eps, bool fast, cudaStream_t st) {
    using T = typename Store<D>::T;
    const int g = grid_for(p.total, 256);
    const size_t tab = sizeof(double) * static_cast<size_t>(p.n + 1) * static_cast<size_t>(p.D);
    if (!fast && p.use32 && tab <= 48 * 1024) {
        k_reconstruct_tab<D, UPDATE><<<g, 256, tab, st>>>(p, static_cast<const T*>(preds), static_cast<T*>(z),
                                                          static_cast<T*>(eps));
    } else if (fast)
        k_reconstruct<D, UPDATE, true><<<g, 256, 0, st>>>(p, static_cast<const T*>(preds), static_cast<T*>(z), static_cast<T*>(eps));
    else
        k_reconstruct<D, UPDATE, false><<<g, 256, 0, st>>>(p, static_cast<const T*>(preds), static_cast<T*>(z), static_cast<T*>(eps));
    LP_LAUNCH_CHECK();
}

FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    f.shift = 31 + l;
    f.mul = ((1ull << f.shift) + d - 1) / d;
    return f;
}

ReconParams make_recon_params(const lp_plan& plan, const Shape4& s, const std::vector<i64>& base, double eta) {
    validate_plan(plan);
    if (s.extent(plan.axis) != plan.axis_extent)
        fail(LP_ERR_SHAPE_MISMATCH, "plan axis extent does not match the latent shape");
    if (plan.n_entries > kMaxKernelEntries) fail(LP_ERR_INVALID_ARGUMENT, "more than 64 plan entries");
    weight_sums(plan);  // ZeroWeight check on host (plan-only property)
    ReconParams p;
    std::memset(&p, 0, sizeof(p));
    p.n = plan.n_entries;
    axis_view(s, plan.axis, p.outer, p.inner);
    p.D = plan.axis_extent;
    p.total = s.volume();
    p.eta = eta;
    p.use32 = p.total < (1ll << 31) ? 1 : 0;
    if (p.use32) {
        p.div_inner = make_fastdiv(static_cast<uint32_t>(p.inner));
        p.div_d = make_fastdiv(static_cast<uint32_t>(p.D));
    }
    for (int k = 0; k < plan.n_entries; ++k) {
        const lp_entry& e = plan.entries[k];
        p.e[k] = ReconEntry{e.latent_begin, e.latent_end - e.latent_begin, e.delta_start, e.delta_end, base[k]};
    }
    return p;
}

void reconstruct_dispatch(const ReconParams& p, int dtype, const void* preds, void* z, void* eps, bool update,
                          bool fast, cudaStream_t st) {
    // algorithmic bytes: every shard element read once, z read (update) and the result written
    double shard = 0.0;
    for (int k = 0; k < p.n; ++k) shard += static_cast<double>(p.e[k].len);
    const double per_pos = static_cast<double>(p.total) / static_cast<double>(p.D);
    prof_begin(KC_RECON, st);
    switch (dtype) {
        case 2: update ? launch_recon<2, true>(p, preds, z, eps, fast, st) : launch_recon<2, false>(p, preds, z, eps, fast, st); break;
        case 4: update ? launch_recon<4, true>(p, preds, z, eps, fast, st) : launch_recon<4, false>(p, preds, z, eps, fast, st); break;
        case 8: update ? launch_recon<8, true>(p, preds, z, eps, fast, st) : launch_recon<8, false>(p, preds, z, eps, fast, st); break;
        default: fail(LP_ERR_INVALID_ARGUMENT, "bad dtype");
    }
    prof_end(KC_RECON, st, 0.0, (shard * per_pos + (update ? 2.0 : 1.0) * static_cast<double>(p.total)) * dtype);
}

template <int D>
static void toy_dispatch_t(int kind, const i64 r[3], const void* z, const Shape4& s, double a0, double a1, double w,
                           bool cfg, void* out, double* ws, cudaStream_t st) {
    using T = typename Store<D>::T;
    const T* zi = static_cast<const T*>(z);
    T* o = static_cast<T*>(out);
    const int64_t n = s.volume();
    const int g = grid_for(n, 256);
    if (kind == LP_TOY_BOX) {
        for (int i = 0; i < 3; ++i)
            if (r[i] < 0) fail(LP_ERR_INVALID_ARGUMENT, "box radius must be >= 0");
        if (cfg) k_box<D, 1><<<g, 256, 0, st>>>(zi, o, s.c, s.t, s.h, s.w, r[0], r[1], r[2], a0, a1, w);
        else k_box<D, 0><<<g, 256, 0, st>>>(zi, o, s.c, s.t, s.h, s.w, r[0], r[1], r[2], a0, a1, w);
        LP_LAUNCH_CHECK();
    } else if (kind == LP_TOY_GLOBAL) {
        if (!ws) fail(LP_ERR_INVALID_ARGUMENT, "GlobalMix needs a workspace (lp_toy_workspace_bytes)");
        const int64_t per = s.t * s.h * s.w;
        k_channel_sum<D><<<(int)((s.c + 31) / 32), 32, 0, st>>>(zi, s.c, per, ws);
        LP_LAUNCH_CHECK();
        if (cfg) k_global<D, 1><<<g, 256, 0, st>>>(zi, o, n, per, ws, a0, a1, w);
        else k_global<D, 0><<<g, 256, 0, st>>>(zi, o, n, per, ws, a0, a1, w);
        LP_LAUNCH_CHECK();
    } else if (kind == LP_TOY_IDENTITY) {
        if (cfg) k_identity<D, 1><<<g, 256, 0, st>>>(zi, o, n, w);
        else k_identity<D, 0><<<g, 256, 0, st>>>(zi, o, n, w);
        LP_LAUNCH_CHECK();
    } else {
        fail(LP_ERR_INVALID_ARGUMENT, "unknown toy denoiser kind");
    }
}

void toy_dispatch(int kind, const i64 r[3], const void* z, const Shape4& s, int dtype, double a0, double a1, double w,
                  bool cfg, void* out, double* ws, cudaStream_t st) {
    switch (dtype) {
        case 2: toy_dispatch_t<2>(kind, r, z, s, a0, a1, w, cfg, out, ws, st); break;
        case 4: toy_dispatch_t<4>(kind, r, z, s, a0, a1, w, cfg, out, ws, st); break;
        case 8: toy_dispatch_t<8>(kind, r, z, s, a0, a1, w, cfg, out, ws, st); break;
        default: fail(LP_ERR_INVALID_ARGUMENT, "bad dtype");
    }
}

// affine = t_coeff * t + cond_coeff * mean, separately rounded (src/denoise.cpp:67).
double toy_affine(double t_coeff, int t, double cond_coeff, double mean) {
    volatile double a = t_coeff * static_cast<double>(t);
    volatile double b = cond_coeff * mean;
    return a + b;
}

}  // namespace lpb200

using namespace lpb200;

extern "C" {

int lp_device_check(int device) {
    return guard([&] {
        int n = 0;
        LP_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(LP_ERR_CUDA, "no such CUDA device");
        cudaDeviceProp prop;
        LP_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) fail(LP_ERR_CUDA, std::string("device is not sm_100: ") + prop.name);
    });
}

int lp_device_flags(uint32_t* flags_out, int reset) {
    return guard([&] {
        unsigned* d = device_flags_ptr();
        unsigned h = 0;
        LP_CUDA(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
        if (reset) LP_CUDA(cudaMemset(d, 0, sizeof(unsigned)));
        *flags_out = h;
    });
}

uint64_t lp_launch_count(void) { return launch_count(); }

int lp_extract(const lp_plan* plan, int32_t first, int32_t count, const void* z, const int64_t shape[4], int dtype,
               void* dst, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        validate_plan(*plan);
        const Shape4 s = Shape4::from(shape);
        if (s.extent(plan->axis) != plan->axis_extent)
            fail(LP_ERR_SHAPE_MISMATCH, "plan was built for extent " + std::to_string(plan->axis_extent) +
                                            ", tensor has " + std::to_string(s.extent(plan->axis)));
        if (first < 0 || count < 0 || first + count > plan->n_entries) fail(LP_ERR_OUT_OF_BOUNDS, "entry range");
        const auto n = entry_elems(*plan, s);
        char* d = static_cast<char*>(dst);
        for (int k = first; k < first + count; ++k) {
            slice_to(z, s, plan->axis, plan->entries[k].latent_begin, plan->entries[k].latent_end, dtype, d,
                     as_stream(stream));
            d += n[k] * dtype;
        }
    });
}

size_t lp_toy_workspace_bytes(const int64_t shape[4]) { return static_cast<size_t>(shape[0]) * sizeof(double); }

int lp_toy_predict(int32_t kind, const int64_t radius[3], double t_coeff, double cond_coeff, const void* z,
                   const int64_t shape[4], int dtype, int timestep, double cond_mean, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        const Shape4 s = Shape4::from(shape);
        double* ws = nullptr;
        if (kind == LP_TOY_GLOBAL) LP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), s.c * sizeof(double), as_stream(stream)));
        toy_dispatch(kind, radius, z, s, dtype, toy_affine(t_coeff, timestep, cond_coeff, cond_mean), 0.0, 0.0, false,
                     out, ws, as_stream(stream));
        if (ws) LP_CUDA(cudaFreeAsync(ws, as_stream(stream)));
    });
}

int lp_toy_cfg_predict(int32_t kind, const int64_t radius[3], double t_coeff, double cond_coeff, const void* z,
                       const int64_t shape[4], int dtype, int timestep, double cond_mean, double guidance,
                       void* eps_out, void* workspace, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        // uncond uses the null vector, whose mean is exactly 0.0 (src/denoise.cpp:10-22)
        toy_dispatch(kind, radius, z, Shape4::from(shape), dtype, toy_affine(t_coeff, timestep, cond_coeff, 0.0),
                     toy_affine(t_coeff, timestep, cond_coeff, cond_mean), guidance, true, eps_out,
                     static_cast<double*>(workspace), as_stream(stream));
    });
}

int lp_cfg_combine(const void* u, const void* c, int64_t n, int dtype, double w, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        const int g = grid_for(n, 256);
        cudaStream_t st = as_stream(stream);
        switch (dtype) {
            case 2: k_cfg_combine<2><<<g, 256, 0, st>>>((const uint16_t*)u, (const uint16_t*)c, (uint16_t*)out, n, w); break;
            case 4: k_cfg_combine<4><<<g, 256, 0, st>>>((const float*)u, (const float*)c, (float*)out, n, w); break;
            case 8: k_cfg_combine<8><<<g, 256, 0, st>>>((const double*)u, (const double*)c, (double*)out, n, w); break;
        }
        LP_LAUNCH_CHECK();
    });
}

int lp_sampler_step(const void* z, const void* eps, int64_t n, int dtype, double eta, void* z_out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        const int g = grid_for(n, 256);
        cudaStream_t st = as_stream(stream);
        switch (dtype) {
            case 2: k_sampler<2><<<g, 256, 0, st>>>((const uint16_t*)z, (const uint16_t*)eps, (uint16_t*)z_out, n, eta); break;
            case 4: k_sampler<4><<<g, 256, 0, st>>>((const float*)z, (const float*)eps, (float*)z_out, n, eta); break;
            case 8: k_sampler<8><<<g, 256, 0, st>>>((const double*)z, (const double*)eps, (double*)z_out, n, eta); break;
        }
        LP_LAUNCH_CHECK();
    });
}

static std::vector<i64> packed_base(const lp_plan& plan, const Shape4& s) {
    const auto n = entry_elems(plan, s);
    std::vector<i64> base(n.size(), 0);
    for (size_t k = 1; k < n.size(); ++k) base[k] = base[k - 1] + n[k - 1];
    return base;
}

int lp_reconstruct(const lp_plan* plan, const void* preds, const int64_t shape[4], int dtype, int32_t mode,
                   void* eps_out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        const Shape4 s = Shape4::from(shape);
        const ReconParams p = make_recon_params(*plan, s, packed_base(*plan, s), 0.0);
        reconstruct_dispatch(p, dtype, preds, nullptr, eps_out, false, mode == LP_MODE_FAST, as_stream(stream));
    });
}

int lp_reconstruct_update(const lp_plan* plan, const void* preds, const int64_t shape[4], int dtype, int32_t mode,
                          double eta, void* z, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        const Shape4 s = Shape4::from(shape);
        const ReconParams p = make_recon_params(*plan, s, packed_base(*plan, s), eta);
        reconstruct_dispatch(p, dtype, preds, z, nullptr, true, mode == LP_MODE_FAST, as_stream(stream));
    });
}

}  // extern "C"
