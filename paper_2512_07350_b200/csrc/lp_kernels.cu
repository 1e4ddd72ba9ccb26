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
#include <map>
#include <mutex>
#include <string>
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
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
    return static_cast<uint32_t>((static_cast<uint64_t>(x) * f.mul) >> f.shift);
}

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

// K1, multi-entry form (the default): ONE launch gathers a run of plan entries, packed back
// to back in dst.  The work is the flat space of V-vectors of all entries; a vector g
// belongs to entry k with start_k <= g < start_{k+1} (a scan over <= 64 starts, warp-uniform
// except at the boundaries), row o = (g - start_k) / run_k by multiply-shift division, and
// is read from z at o * stride + off_k + (g - start_k - o * run_k).  dst is written at g
// itself: the packing IS the flat index.  Each thread keeps U vectors in flight.
struct GatherEntry {
    uint32_t start, run, off;  // in V units
    FastDiv div;
};
struct GatherParams {
    int n;
    uint32_t total, stride;  // in V units
    GatherEntry e[kMaxKernelEntries];
};

template <typename V, int U>
__global__ void __launch_bounds__(256) k_gather_entries(const __grid_constant__ GatherParams p,
                                                        const V* __restrict__ src, V* __restrict__ dst) {
    const uint32_t step = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < p.total; base += U * step) {
        V v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t g = base + u * step;
            if (g < p.total) {
                int k = 0;
                while (k + 1 < p.n && g >= p.e[k + 1].start) ++k;
                const uint32_t r = g - p.e[k].start;
                const uint32_t o = static_cast<uint32_t>((static_cast<uint64_t>(r) * p.e[k].div.mul) >> p.e[k].div.shift);
                v[u] = __ldg(src + static_cast<uint64_t>(o) * p.stride + p.e[k].off + (r - o * p.e[k].run));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (base + u * step < p.total) dst[base + u * step] = v[u];
    }
}

// K1, TMA-staged form (the default where its alignment conditions hold; knob gather_tma=0
// falls back to the vector-copy kernel above).
//  * W-axis windows (inner == 1: every latent row (c, t, h) contributes one short run of len
//    elements): one 2-D tensor map per entry over z viewed as [rows = C*T*H][W] with box
//    {lb, R}: the box starts at the window's first column rounded DOWN to a 16-byte boundary
//    (sh = the skipped columns; measured on B200: a box whose start is not 16-byte aligned
//    faults with an illegal instruction for 2- and 4-byte elements) and lb = sh + len rounded
//    up to a 16-byte multiple.  Each CTA pulls R-row boxes through a
//    kGtStages-deep shared-memory ring (one thread issues cp.async.bulk.tensor, completion on an
//    mbarrier); R consecutive rows of one entry are ONE contiguous span of R*len elements in dst,
//    which the block writes out as 16-byte vectors (coalesced, no strided global access at all).
//  * T/H windows (inner > 1: each row contributes a contiguous run of len*inner elements):
//    1-D bulk copies through shared memory (TMA engine, no thread touches the data), all
//    entries in one launch.
constexpr int kGtMaxEntries = 8, kGtStages = 4, kGtThreads = 256;
struct GatherTmaEntry {
    uint32_t len, lb, s, items_begin;  // s: the box's first column (16-byte aligned)
    uint32_t sh;                       // columns of the box before the window
    uint64_t dst_off;  // elements
    FastDiv div_len;
};
struct GatherTmaParams {
    int n;
    uint32_t rows, R, items, stage_bytes;
    GatherTmaEntry e[kGtMaxEntries];
};
struct GatherTmaMaps {
    CUtensorMap m[kGtMaxEntries];
};
template <int E> struct ElemOf;
template <> struct ElemOf<2> { using T = uint16_t; };
template <> struct ElemOf<4> { using T = uint32_t; };
template <> struct ElemOf<8> { using T = unsigned long long; };

template <int E>
__global__ void __launch_bounds__(kGtThreads) k_gather_tma(const __grid_constant__ GatherTmaMaps maps,
                                                           const __grid_constant__ GatherTmaParams p,
                                                           typename ElemOf<E>::T* __restrict__ dst) {
    using T = typename ElemOf<E>::T;
    constexpr int V = 16 / E;  // elements per 16-byte vector
    extern __shared__ __align__(128) uint8_t sbuf_raw[];
    // tensor-copy destinations must be 128-byte aligned: the dynamic segment follows the static
    // barriers, so align by hand (the launch adds 128 bytes)
    uint8_t* sbuf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sbuf_raw) + 127) & ~uintptr_t(127));
    __shared__ uint64_t full[kGtStages];
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < kGtStages; ++s) tc::mbar_init(&full[s], 1);
        tc::fence_barrier_init();
    }
    __syncthreads();
    auto locate = [&](uint32_t it, int& k, uint32_t& row0) {
        k = 0;
        while (k + 1 < p.n && it >= p.e[k + 1].items_begin) ++k;
        row0 = (it - p.e[k].items_begin) * p.R;
    };
    auto issue = [&](uint32_t it, int s) {
        int k;
        uint32_t row0;
        locate(it, k, row0);
        // the transaction counts the whole box, rows past the tensor end included (zero-filled)
        tc::mbar_arrive_expect_tx(&full[s], p.e[k].lb * p.R * E);
        tc::tma_load_2d(&maps.m[k], &full[s], sbuf + s * p.stage_bytes, static_cast<int32_t>(p.e[k].s),
                        static_cast<int32_t>(row0));
    };
    const uint32_t first = blockIdx.x, step = gridDim.x;
    const uint32_t n_my = first < p.items ? (p.items - first + step - 1) / step : 0;
    if (tid == 0)
        for (uint32_t j = 0; j < n_my && j < kGtStages; ++j) issue(first + j * step, static_cast<int>(j));
    for (uint32_t j = 0; j < n_my; ++j) {
        const int s = static_cast<int>(j % kGtStages);
        int k;
        uint32_t row0;
        locate(first + j * step, k, row0);
        const GatherTmaEntry& e = p.e[k];
        const uint32_t span = min(p.R, p.rows - row0) * e.len;
        const T* box = reinterpret_cast<const T*>(sbuf + s * p.stage_bytes);
        T* out = dst + e.dst_off + static_cast<uint64_t>(row0) * e.len;
        tc::mbar_wait(&full[s], (j / kGtStages) & 1u);
        const uint32_t nv = span / V;
        for (uint32_t v = tid; v < nv; v += kGtThreads) {
            T tmp[V];
#pragma unroll
            for (int u = 0; u < V; ++u) {
                const uint32_t idx = v * V + u;
                const uint32_t r = fdiv(idx, e.div_len);
                tmp[u] = box[r * e.lb + e.sh + (idx - r * e.len)];
            }
            *reinterpret_cast<uint4*>(out + v * V) = *reinterpret_cast<const uint4*>(tmp);
        }
        for (uint32_t idx = nv * V + tid; idx < span; idx += kGtThreads) {
            const uint32_t r = fdiv(idx, e.div_len);
            out[idx] = box[r * e.lb + e.sh + (idx - r * e.len)];
        }
        __syncthreads();  // stage s has been read by every thread
        if (tid == 0 && j + kGtStages < n_my) issue(first + (j + kGtStages) * step, s);
    }
}

// T/H windows: every entry's rows are runs of run_b contiguous bytes (src stride stride_b),
// cut into <= kSliceChunk pieces; a warp's lane 0 is a copy engine with two stages (bulk load
// -> mbarrier -> bulk store), chunks dealt round robin over all warps of the grid.
struct GatherBulkEntry {
    uint64_t run_b, off_b, dst_b, chunks_begin, cpr;
};
struct GatherBulkParams {
    int n;
    uint64_t stride_b, chunks;
    GatherBulkEntry e[kGtMaxEntries];
};
__global__ void __launch_bounds__(32 * kSliceWarps) k_gather_bulk(const __grid_constant__ GatherBulkParams p,
                                                                  const uint8_t* __restrict__ src,
                                                                  uint8_t* __restrict__ dst) {
    extern __shared__ __align__(128) uint8_t sbuf[];  // [warps][2][chunk]
    __shared__ uint64_t bars[kSliceWarps][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane != 0) return;
    uint64_t* bar = bars[warp];
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_barrier_init();
    uint8_t* buf = sbuf + static_cast<size_t>(warp) * 2 * kSliceChunk;
    const uint64_t engines = static_cast<uint64_t>(gridDim.x) * kSliceWarps;
    uint32_t ph[2] = {0, 0};
    int it = 0;
    for (uint64_t c = static_cast<uint64_t>(blockIdx.x) * kSliceWarps + warp; c < p.chunks; c += engines, ++it) {
        int k = 0;
        while (k + 1 < p.n && c >= p.e[k + 1].chunks_begin) ++k;
        const GatherBulkEntry& e = p.e[k];
        const uint64_t r = c - e.chunks_begin, o = r / e.cpr, at = (r - o * e.cpr) * kSliceChunk;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<uint64_t>(kSliceChunk), e.run_b - at));
        const int b = it & 1;
        if (it >= 2) tc::bulk_wait_read<1>();  // the store issued from this stage two chunks ago has read it
        tc::mbar_arrive_expect_tx(&bar[b], bytes);
        tc::bulk_load(buf + b * kSliceChunk, src + o * p.stride_b + e.off_b + at, bytes, &bar[b]);
        tc::mbar_wait(&bar[b], ph[b]);
        ph[b] ^= 1;
        tc::bulk_store(dst + e.dst_b + o * e.run_b + at, buf + b * kSliceChunk, bytes);
        tc::bulk_commit();
    }
    tc::bulk_wait_all();
}

bool make_tmap_2d_raw(CUtensorMap* m, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                      uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);  // gemm_tcgen05.cu

static int num_sms_lp() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// The TMA-staged K1 of entries ks[0..count) (packed in that order); false when its alignment
// conditions do not hold (the caller then uses the vector-copy kernel).
static bool gather_tma(const void* z, const Shape4& s, const lp_plan& plan, const int* ks, int count, int E, void* dst,
                       cudaStream_t st) {
    if (count <= 0 || count > kGtMaxEntries || !tune_get("gather_tma", 1)) return false;
    i64 outer, inner;
    axis_view(s, plan.axis, outer, inner);
    const i64 D = s.extent(plan.axis);
    if (reinterpret_cast<uintptr_t>(z) % 16 || reinterpret_cast<uintptr_t>(dst) % 16) return false;
    if (inner > 1) {
        GatherBulkParams p;
        std::memset(&p, 0, sizeof(p));
        p.n = count;
        p.stride_b = static_cast<uint64_t>(D * inner * E);
        if (p.stride_b % 16) return false;
        uint64_t chunks = 0, dst_b = 0;
        for (int c = 0; c < count; ++c) {
            const lp_entry& en = plan.entries[ks[c]];
            GatherBulkEntry& g = p.e[c];
            g.run_b = static_cast<uint64_t>((en.latent_end - en.latent_begin) * inner * E);
            g.off_b = static_cast<uint64_t>(en.latent_begin * inner * E);
            g.dst_b = dst_b;
            if (g.run_b % 16 || g.off_b % 16 || g.dst_b % 16) return false;
            g.cpr = (g.run_b + kSliceChunk - 1) / kSliceChunk;
            g.chunks_begin = chunks;
            chunks += g.cpr * static_cast<uint64_t>(outer);
            dst_b += g.run_b * static_cast<uint64_t>(outer);
        }
        p.chunks = chunks;
        static bool attr = false;
        constexpr int smem = kSliceWarps * 2 * kSliceChunk;
        if (!attr) {
            LP_CUDA(cudaFuncSetAttribute(k_gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr = true;
        }
        const uint64_t want = (chunks + kSliceWarps - 1) / kSliceWarps;
        const int grid = static_cast<int>(std::min<uint64_t>(want, 3ull * num_sms_lp()));
        prof_begin(KC_GATHER, st);
        k_gather_bulk<<<grid, 32 * kSliceWarps, smem, st>>>(p, static_cast<const uint8_t*>(z), static_cast<uint8_t*>(dst));
        LP_LAUNCH_CHECK();
        prof_end(KC_GATHER, st, 0.0, 2.0 * static_cast<double>(dst_b));
        return true;
    }
    // inner == 1: W-axis boxes
    const int V = 16 / E;
    const uint64_t rows = static_cast<uint64_t>(outer);
    if (rows >= (1ull << 31) || (D * E) % 16) return false;
    uint32_t lbmax = 0;
    for (int c = 0; c < count; ++c) {
        const lp_entry& en = plan.entries[ks[c]];
        const uint32_t len = static_cast<uint32_t>(en.latent_end - en.latent_begin);
        const uint32_t sh = static_cast<uint32_t>(en.latent_begin % V);
        const uint32_t lb = ((sh + len) * E + 15) / 16 * 16 / E;
        if (lb > 256) return false;
        lbmax = std::max(lbmax, lb);
    }
    // R rows per box: ~16 KB stages, a multiple of V (so every box's span starts 16-B aligned)
    uint32_t R = std::min<uint32_t>(256, 16384u / (lbmax * E));
    R = R / V * V;
    if (R < static_cast<uint32_t>(V)) return false;
    GatherTmaParams p;
    std::memset(&p, 0, sizeof(p));
    GatherTmaMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    p.n = count;
    p.rows = static_cast<uint32_t>(rows);
    p.R = R;
    p.stage_bytes = (lbmax * R * E + 127) / 128 * 128;
    uint64_t off = 0;
    uint32_t items = 0;
    for (int c = 0; c < count; ++c) {
        const lp_entry& en = plan.entries[ks[c]];
        GatherTmaEntry& g = p.e[c];
        g.len = static_cast<uint32_t>(en.latent_end - en.latent_begin);
        g.sh = static_cast<uint32_t>(en.latent_begin % V);
        g.lb = ((g.sh + g.len) * E + 15) / 16 * 16 / E;
        g.s = static_cast<uint32_t>(en.latent_begin) - g.sh;
        g.items_begin = items;
        g.dst_off = off;
        g.div_len = make_fastdiv(g.len);
        if (off % V) return false;
        if (!make_tmap_2d_raw(&maps.m[c], z, E, static_cast<uint64_t>(D), rows, static_cast<uint64_t>(D * E), g.lb, R))
            return false;
        items += static_cast<uint32_t>((rows + R - 1) / R);
        off += rows * g.len;
    }
    p.items = items;
    const int smem = kGtStages * static_cast<int>(p.stage_bytes) + 128;
    static int attr_bytes[9] = {};
    if (attr_bytes[E] < smem) {
        switch (E) {
            case 2: LP_CUDA(cudaFuncSetAttribute(k_gather_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); break;
            case 4: LP_CUDA(cudaFuncSetAttribute(k_gather_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); break;
            default: LP_CUDA(cudaFuncSetAttribute(k_gather_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); break;
        }
        attr_bytes[E] = smem;
    }
    const int per_sm = std::max(1, std::min(4, (200 * 1024) / smem));
    const int grid = static_cast<int>(std::min<uint64_t>(items, static_cast<uint64_t>(per_sm) * num_sms_lp()));
    prof_begin(KC_GATHER, st);
    switch (E) {
        case 2: k_gather_tma<2><<<grid, kGtThreads, smem, st>>>(maps, p, static_cast<uint16_t*>(dst)); break;
        case 4: k_gather_tma<4><<<grid, kGtThreads, smem, st>>>(maps, p, static_cast<uint32_t*>(dst)); break;
        default: k_gather_tma<8><<<grid, kGtThreads, smem, st>>>(maps, p, static_cast<unsigned long long*>(dst)); break;
    }
    LP_LAUNCH_CHECK();
    prof_end(KC_GATHER, st, 0.0, 2.0 * static_cast<double>(off) * E);
    return true;
}

// Builds the one-launch gather of entries ks[0..count) of `plan` (packed in that order);
// false when 32-bit vector indexing does not fit (the caller then copies entry by entry).
static bool gather_params(const void* z, const Shape4& s, const lp_plan& plan, const int* ks, int count, int E,
                          const void* dst, GatherParams& p, int& vb) {
    if (count <= 0 || count > kMaxKernelEntries || !tune_get("gather_multi", 1)) return false;
    i64 outer, inner;
    axis_view(s, plan.axis, outer, inner);
    const i64 stride_b = s.extent(plan.axis) * inner * E;
    uint64_t al = reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(dst) | static_cast<uint64_t>(stride_b);
    i64 bytes = 0;
    for (int c = 0; c < count; ++c) {
        const lp_entry& en = plan.entries[ks[c]];
        al |= static_cast<uint64_t>(en.latent_begin * inner * E) |
              static_cast<uint64_t>((en.latent_end - en.latent_begin) * inner * E);
        bytes += outer * (en.latent_end - en.latent_begin) * inner * E;
    }
    vb = 16;
    while (vb > E && al % vb) vb >>= 1;
    if (bytes / vb >= (1ll << 31) || outer * stride_b / vb >= (1ll << 32)) return false;
    std::memset(&p, 0, sizeof(p));
    p.n = count;
    p.stride = static_cast<uint32_t>(stride_b / vb);
    uint32_t start = 0;
    for (int c = 0; c < count; ++c) {
        const lp_entry& en = plan.entries[ks[c]];
        const uint32_t run = static_cast<uint32_t>((en.latent_end - en.latent_begin) * inner * E / vb);
        p.e[c] = GatherEntry{start, run, static_cast<uint32_t>(en.latent_begin * inner * E / vb), make_fastdiv(run)};
        start += run * static_cast<uint32_t>(outer);
    }
    p.total = start;
    return true;
}

void gather_entries(const void* z, const Shape4& s, const lp_plan& plan, const int* ks, int count, int E, void* dst,
                    cudaStream_t st) {
    if (gather_tma(z, s, plan, ks, count, E, dst, st)) return;
    i64 outer, inner;
    axis_view(s, plan.axis, outer, inner);
    GatherParams p;
    int vb = 0;
    if (gather_params(z, s, plan, ks, count, E, dst, p, vb)) {
        constexpr int U = 4;
        const int g = grid_for((p.total + U - 1) / U, 256, 8);
        prof_begin(KC_GATHER, st);
        switch (vb) {
            case 16: k_gather_entries<uint4, U><<<g, 256, 0, st>>>(p, static_cast<const uint4*>(z), static_cast<uint4*>(dst)); break;
            case 8: k_gather_entries<uint2, U><<<g, 256, 0, st>>>(p, static_cast<const uint2*>(z), static_cast<uint2*>(dst)); break;
            case 4: k_gather_entries<uint32_t, U><<<g, 256, 0, st>>>(p, static_cast<const uint32_t*>(z), static_cast<uint32_t*>(dst)); break;
            default: k_gather_entries<uint16_t, U><<<g, 256, 0, st>>>(p, static_cast<const uint16_t*>(z), static_cast<uint16_t*>(dst)); break;
        }
        LP_LAUNCH_CHECK();
        prof_end(KC_GATHER, st, 0.0, 2.0 * static_cast<double>(p.total) * vb);
        return;
    }
    char* d = static_cast<char*>(dst);
    for (int c = 0; c < count; ++c) {
        const lp_entry& en = plan.entries[ks[c]];
        slice_to(z, s, plan.axis, en.latent_begin, en.latent_end, E, d, st);
        d += outer * (en.latent_end - en.latent_begin) * inner * E;
    }
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
// K9 over peer memory (the engine's NVLink exchange; CUDA-IPC-mapped gather buffers).
// k_peer_push: rank r copies its own slot [off, off+bytes) of the local gather buffer to the
// same offset of every peer's buffer with 16-B remote stores, then the last block to finish
// (a grid-wide arrival counter) publishes `epoch` into every peer's flag word for rank r
// with a system-scope release.  k_peer_wait: spins (system-scope acquire) until every peer's
// flag for this rank's buffer reaches `epoch`; a wall-time watchdog (peer_timeout_ms) raises
// LP_FLAG_PEER_TIMEOUT and records the missing ranks instead of hanging.  The gather buffer is double-buffered by epoch
// parity, so a push for step i+1 never lands in a buffer a peer's K10 of step i still reads.
// ---------------------------------------------------------------------------
constexpr unsigned LP_FLAG_PEER_TIMEOUT = 4u;

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(256) k_peer_push(const __grid_constant__ PeerPush pp, unsigned* counter) {
    const uint64_t nvec = pp.bytes / 16;
    const uint4* src = reinterpret_cast<const uint4*>(pp.local + pp.off);
    for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < nvec;
         v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint4 x = __ldg(src + v);
        for (int j = 0; j < pp.npeers; ++j) reinterpret_cast<uint4*>(pp.peer[j] + pp.off)[v] = x;
    }
    // tail bytes (slot sizes are element multiples, not always 16-B multiples)
    if (blockIdx.x == 0)
        for (uint64_t b = nvec * 16 + threadIdx.x; b < pp.bytes; b += blockDim.x)
            for (int j = 0; j < pp.npeers; ++j) pp.peer[j][pp.off + b] = pp.local[pp.off + b];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned done = atomicAdd(counter, 1u);
        if (done == gridDim.x - 1) {
            __threadfence_system();
            const unsigned long long ep = *pp.epoch + 1;
            for (int j = 0; j < pp.npeers; ++j) st_release_sys(pp.peer_flag[j], ep);
            *pp.epoch = ep;
            *counter = 0;
        }
    }
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_peer_wait(const unsigned long long* flags, int world, int rank, const unsigned long long* epoch_p,
                            unsigned* status, int step, unsigned long long timeout_ns) {
    const int j = threadIdx.x;
    if (j >= world || j == rank) return;
    const unsigned long long epoch = *epoch_p;
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flags + j) < epoch) {
        if (global_ns() - t0 > timeout_ns) {  // a dead or stalled peer, not a slow one
            raise_flag(LP_FLAG_PEER_TIMEOUT);
            atomicOr(status, 1u << j);
            status[1] = static_cast<unsigned>(step);
            __threadfence();
            return;
        }
        __nanosleep(200);
    }
}

void peer_push(const PeerPush& pp, unsigned* counter, cudaStream_t st) {
    const int g = grid_for(static_cast<int64_t>(pp.bytes / 16) + 1, 256, 4);
    k_peer_push<<<g, 256, 0, st>>>(pp, counter);
    LP_LAUNCH_CHECK();
}

void peer_wait(const unsigned long long* flags, int world, int rank, const unsigned long long* epoch,
               unsigned* status, int step, cudaStream_t st) {
    // watchdog in wall time (%globaltimer): knob peer_timeout_ms, default 20 s
    const unsigned long long ns = 1000000ull * static_cast<unsigned long long>(std::max(1, tune_get("peer_timeout_ms", 20000)));
    k_peer_wait<<<1, 32 * ((world + 31) / 32), 0, st>>>(flags, world, rank, epoch, status, step, ns);
    LP_LAUNCH_CHECK();
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

// A peer's shard never arrived (peer exchange watchdog): leave z as it was.
__device__ __forceinline__ bool recon_aborted(const ReconParams& p) {
    return p.abort != nullptr && *reinterpret_cast<const volatile unsigned*>(p.abort) != 0u;
}

template <int D, bool UPDATE, bool FAST>
__global__ void __launch_bounds__(256) k_reconstruct(const __grid_constant__ ReconParams p,
                                                     const typename Store<D>::T* __restrict__ preds,
                                                     typename Store<D>::T* __restrict__ z,
                                                     typename Store<D>::T* __restrict__ eps_out) {
    if (recon_aborted(p)) return;
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
    if (recon_aborted(p)) return;
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

// K10, coverage-table form (the default when every position is covered by at most
// kReconCover entries and indices fit 32 bits).  The block first tabulates, per position x,
// the covering entries with a non-zero weight in worker order: weight w, the element offset
// of (o=0, j) in the gathered buffer and the per-o stride (len*inner), plus Z(x) — the same
// IEEE operations as entry_weight and the reference.  Each thread then owns 4 consecutive
// elements: z moves as one 4-element vector, and when inner % 4 == 0 the 4 elements share
// (o, x), so every covering prediction is one 4-element vector load too.  All loads of an
// iteration are issued before any arithmetic (predicated on the coverage count), so an SM
// keeps ~48 B per thread in flight.  Z(x) == 1 (one covering entry of weight 1, the bulk of
// the latent) needs no division: A/1 is exact.
constexpr int kReconCover = 4;

template <int D> struct Vec4;
template <> struct Vec4<4> {
    using T = float4;
    static __device__ __forceinline__ double get(const T& v, int u) {
        return static_cast<double>(u == 0 ? v.x : u == 1 ? v.y : u == 2 ? v.z : v.w);
    }
};
template <> struct Vec4<8> {
    struct T { double2 a, b; };
    static __device__ __forceinline__ double get(const T& v, int u) { return u == 0 ? v.a.x : u == 1 ? v.a.y : u == 2 ? v.b.x : v.b.y; }
};
template <> struct Vec4<2> {
    using T = uint2;
    static __device__ __forceinline__ double get(const T& v, int u) {
        const uint32_t w = u < 2 ? v.x : v.y;
        return f16_decode_exact(static_cast<uint16_t>((u & 1) ? (w >> 16) : (w & 0xffffu)));
    }
};
template <int D>
__device__ __forceinline__ typename Vec4<D>::T vload4(const typename Store<D>::T* p) {
    return *reinterpret_cast<const typename Vec4<D>::T*>(p);
}

// a / Z, correctly rounded, from the tabulated y = RN(1/Z): q = a*y, r = a - q*Z (exact, one
// FMA), q' = q + r*y — Markstein's final step, which yields RN(a/Z) when y = RN(1/Z) and q is
// within an ulp of a/Z (no overflow/underflow; here Z in [1, 64] and |a| is tested against the
// subnormal range).  Checked against true division on 5.2e8 (Z, a) pairs of ramp-weight sums
// (scripts/micro/markstein.c) and by every bit-exact K10 test.  r == 0 keeps q (exact, and
// the sign of a zero quotient).  Saves MUFU.RCP64H + the Newton steps of __ddiv_rn.
__device__ __forceinline__ double div_z(double a, double Z, double y) {
    if (fabs(a) < 0x1p-900 || !isfinite(a)) return __ddiv_rn(a, Z);
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, Z, a);
    return r == 0.0 ? q : __fma_rn(r, y, q);
}

// The coverage table of a plan (layout below), built once on the device by one block with
// entry_weight's exact operations and cached per (plan, gather layout, device): K10 blocks
// then only copy ~2 KB into shared memory instead of each re-deriving it.
struct CovLayout {
    // structure of arrays [cover][x]: lanes on consecutive x (W axis) hit distinct banks
    double* wts;      // [4][Dx]
    double* zsum;     // [Dx]
    double* zinv;     // [Dx] RN(1 / Z) (the division's Markstein step, div_z)
    float* zsumf;     // [Dx] (FAST)
    uint32_t* offs;   // [4][Dx]
    uint32_t* ostr;   // [4][Dx]
    uint32_t* cnt;    // [Dx]
    uint8_t* kidx;    // [4][Dx] the plan entry of each cover (W-axis tile kernel)
    __host__ __device__ explicit CovLayout(void* base, int Dx) {
        wts = static_cast<double*>(base);
        zsum = wts + kReconCover * Dx;
        zinv = zsum + Dx;
        zsumf = reinterpret_cast<float*>(zinv + Dx);
        offs = reinterpret_cast<uint32_t*>(zsumf + Dx);
        ostr = offs + kReconCover * Dx;
        cnt = ostr + kReconCover * Dx;
        kidx = reinterpret_cast<uint8_t*>(cnt + Dx);
    }
};

__global__ void __launch_bounds__(256) k_recon_table(const __grid_constant__ ReconParams p, void* table) {
    const int Dx = static_cast<int>(p.D);
    CovLayout t(table, Dx);
    for (int x = threadIdx.x; x < Dx; x += blockDim.x) {
        double zs = 0.0;
        float zf = 0.f;
        int c = 0;
        for (int k = 0; k < p.n; ++k) {
            const ReconEntry& e = p.e[k];
            const int64_t j = x - e.begin;
            if (j < 0 || j >= e.len) continue;
            const double w = entry_weight(e, j);
            zs = __dadd_rn(zs, w);
            zf += static_cast<float>(w);
            if (w != 0.0 && c < kReconCover) {
                t.wts[c * Dx + x] = w;
                t.offs[c * Dx + x] = static_cast<uint32_t>(e.base + j * p.inner);
                t.ostr[c * Dx + x] = static_cast<uint32_t>(e.len * p.inner);
                t.kidx[c * Dx + x] = static_cast<uint8_t>(k);
                ++c;
            }
        }
        t.zsum[x] = zs;
        t.zinv[x] = __ddiv_rn(1.0, zs);
        t.zsumf[x] = zf;
        t.cnt[x] = static_cast<uint32_t>(c);
    }
}

// One K10 element with a compile-time cover count C (no predicated-off conversions for the
// covers a position does not have) and the Z == 1 test hoisted by the caller (Z1): the blend
// sum_k w_k pred_k in worker order, / Z (true division, or div_z), quantized; UPDATE: the
// sampler's z - eta * eps, quantized and stored.  Returns false for a non-finite result.
template <int D, bool UPDATE, bool FAST, int C, bool Z1>
__device__ __forceinline__ bool k10_elem(const double (&w)[kReconCover], double Z, double Zi, float Zf, bool mk,
                                         double eta, const typename Store<D>::T (&r)[kReconCover],
                                         typename Store<D>::T zraw, typename Store<D>::T& out) {
    double eps;
    if (!FAST) {
        double a = 0.0;  // from +0 like the reference's accumulator (a -0 product sums to +0)
#pragma unroll
        for (int cc = 0; cc < C; ++cc) a = __dadd_rn(a, __dmul_rn(w[cc], load_val<D>(r, cc)));
        eps = quantize_dev<D>(Z1 ? a : (mk ? div_z(a, Z, Zi) : __ddiv_rn(a, Z)));
    } else {
        float a = 0.f;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) a = fmaf(static_cast<float>(w[cc]), static_cast<float>(load_val<D>(r, cc)), a);
        eps = quantize_dev<D>(static_cast<double>(Z1 ? a : a / Zf));
    }
    const bool ok = isfinite(eps);
    double res = eps;
    if (UPDATE) {
        const double zo = load_val<D>(&zraw, 0);
        res = FAST ? static_cast<double>(fmaf(-static_cast<float>(eta), static_cast<float>(eps), static_cast<float>(zo)))
                   : __dsub_rn(zo, __dmul_rn(eta, eps));
    }
    return store_q<D>(&out, 0, res) && ok;
}

// Dispatch a group of n elements sharing one position x onto the compile-time cover count
// and Z == 1 forms (c and Z are warp-uniform except at coverage boundaries).
template <int D, bool UPDATE, bool FAST, int N>
__device__ __forceinline__ bool k10_group(uint32_t c, const double (&w)[kReconCover], double Z, double Zi, float Zf,
                                          bool mk, double eta, const typename Store<D>::T (&r)[N][kReconCover],
                                          const typename Store<D>::T* zr, typename Store<D>::T* q, uint32_t live) {
    bool ok = true;
#define LP_K10G(CC, ZZ)                                                                                         \
    for (int u = 0; u < N; ++u)                                                                                 \
        if (u < static_cast<int>(live))                                                                         \
            ok = k10_elem<D, UPDATE, FAST, CC, ZZ>(w, Z, Zi, Zf, mk, eta, r[u], UPDATE ? zr[u] : typename Store<D>::T{}, q[u]) && ok;
    const bool z1 = FAST ? Zf == 1.f : Z == 1.0;
    switch (c) {
        case 1:
            if (z1) { LP_K10G(1, true) } else { LP_K10G(1, false) }
            break;
        case 2:
            if (z1) { LP_K10G(2, true) } else { LP_K10G(2, false) }
            break;
        case 3:
            if (z1) { LP_K10G(3, true) } else { LP_K10G(3, false) }
            break;
        default:
            if (z1) { LP_K10G(4, true) } else { LP_K10G(4, false) }
            break;
    }
#undef LP_K10G
    return ok;
}

template <int D, bool UPDATE, bool FAST, bool VEC, int GV = 8>
__global__ void __launch_bounds__(256) k_reconstruct_cov(const __grid_constant__ ReconParams p,
                                                         const typename Store<D>::T* __restrict__ preds,
                                                         typename Store<D>::T* __restrict__ z,
                                                         typename Store<D>::T* __restrict__ eps_out,
                                                         const uint4* __restrict__ table, uint32_t table_vecs) {
    if (recon_aborted(p)) return;
    using T = typename Store<D>::T;
    extern __shared__ __align__(16) double cov[];
    const int Dx = static_cast<int>(p.D);
    for (uint32_t v = threadIdx.x; v < table_vecs; v += blockDim.x) reinterpret_cast<uint4*>(cov)[v] = __ldg(table + v);
    const CovLayout t(cov, Dx);
    const double* wts = t.wts;
    const double* zsum = t.zsum;
    const double* zinv = t.zinv;
    const float* zsumf = t.zsumf;
    const uint32_t* offs = t.offs;
    const uint32_t* ostr = t.ostr;
    const uint32_t* cnt = t.cnt;
    const uint32_t inner = static_cast<uint32_t>(p.inner);
    __syncthreads();
    // one element: Σ_k w·pred (worker order) / Z, quantized; UPDATE: z - η ε̂, quantized
    auto finish = [&](uint32_t x, uint32_t c, const T* r, T zraw, T& out) -> bool {
        double eps;
        if (!FAST) {
            double a = 0.0;
#pragma unroll
            for (int cc = 0; cc < kReconCover; ++cc)
                if (cc < c) a = __dadd_rn(a, __dmul_rn(wts[cc * Dx + x], load_val<D>(r, cc)));
            const double Z = zsum[x];
            eps = quantize_dev<D>(Z == 1.0 ? a : (p.mk ? div_z(a, Z, zinv[x]) : __ddiv_rn(a, Z)));
        } else {
            float a = 0.f;
#pragma unroll
            for (int cc = 0; cc < kReconCover; ++cc)
                if (cc < c) a = fmaf(static_cast<float>(wts[cc * Dx + x]), static_cast<float>(load_val<D>(r, cc)), a);
            eps = quantize_dev<D>(static_cast<double>(a / zsumf[x]));
        }
        bool ok = isfinite(eps);
        double res = eps;
        if (UPDATE) {
            const double zo = load_val<D>(&zraw, 0);
            res = FAST ? static_cast<double>(fmaf(-static_cast<float>(p.eta), static_cast<float>(eps), static_cast<float>(zo)))
                       : __dsub_rn(zo, __dmul_rn(p.eta, eps));
        }
        return store_q<D>(&out, 0, res) && ok;
    };
    constexpr int G = VEC ? GV : 8;  // elements per thread per iteration (VEC: knob recon_g, 8 or 4)
    const uint32_t total = static_cast<uint32_t>(p.total);
    bool ok = true;
    if (VEC) {
        // 8 consecutive elements share (o, x): two 4-element vectors per covering prediction
        for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < total / G; gi += gridDim.x * blockDim.x) {
            const uint32_t idx0 = gi * G;
            const uint32_t ox = fdiv(idx0, p.div_inner), i = idx0 - ox * inner;
            const uint32_t o = fdiv(ox, p.div_d), x = ox - o * static_cast<uint32_t>(Dx);
            const uint32_t c = cnt[x];
            T raw[G][kReconCover];
#pragma unroll
            for (int cc = 0; cc < kReconCover; ++cc) {
                if (cc < c) {
                    const T* src = preds + offs[cc * Dx + x] + static_cast<uint64_t>(o) * ostr[cc * Dx + x] + i;
#pragma unroll
                    for (int h = 0; h < G / 4; ++h) {
                        const typename Vec4<D>::T v = vload4<D>(src + 4 * h);
                        const T* vt = reinterpret_cast<const T*>(&v);
#pragma unroll
                        for (int u = 0; u < 4; ++u) raw[4 * h + u][cc] = vt[u];
                    }
                }
            }
            T zr[G], q[G];
            if (UPDATE) {
#pragma unroll
                for (int h = 0; h < G / 4; ++h)
                    *reinterpret_cast<typename Vec4<D>::T*>(zr + 4 * h) = vload4<D>(z + idx0 + 4 * h);
            }
            double w[kReconCover];
#pragma unroll
            for (int cc = 0; cc < kReconCover; ++cc) w[cc] = cc < static_cast<int>(c) ? wts[cc * Dx + x] : 0.0;
            ok = k10_group<D, UPDATE, FAST, G>(c, w, FAST ? 0.0 : zsum[x], FAST ? 0.0 : zinv[x], FAST ? zsumf[x] : 1.f,
                                               p.mk, p.eta, raw, zr, q, G) && ok;
            T* out = (UPDATE ? z : eps_out) + idx0;
#pragma unroll
            for (int h = 0; h < G / 4; ++h)
                *reinterpret_cast<typename Vec4<D>::T*>(out + 4 * h) = *reinterpret_cast<const typename Vec4<D>::T*>(q + 4 * h);
        }
    } else {
        // lane-strided: a warp owns 32*G consecutive elements, element u of a lane sits at
        // +32u — every load and store instruction of the warp is one contiguous run
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
        for (uint32_t wc = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wc * (32u * G) < total; wc += warps) {
            T raw[G][kReconCover], zr[G];
            uint32_t xs[G], cs[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const uint32_t idx = wc * (32u * G) + 32u * u + lane;
                cs[u] = 0;
                xs[u] = 0;
                if (idx < total) {
                    const uint32_t ox = fdiv(idx, p.div_inner), i = idx - ox * inner;
                    const uint32_t o = fdiv(ox, p.div_d), x = ox - o * static_cast<uint32_t>(Dx);
                    const uint32_t c = cnt[x];
                    xs[u] = x;
                    cs[u] = c;
#pragma unroll
                    for (int cc = 0; cc < kReconCover; ++cc)
                        if (cc < c) raw[u][cc] = preds[offs[cc * Dx + x] + static_cast<uint64_t>(o) * ostr[cc * Dx + x] + i];
                    if (UPDATE) zr[u] = z[idx];
                }
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const uint32_t idx = wc * (32u * G) + 32u * u + lane;
                if (idx < total) {
                    T qv;
                    ok = finish(xs[u], cs[u], raw[u], UPDATE ? zr[u] : T{}, qv) && ok;
                    (UPDATE ? z : eps_out)[idx] = qv;
                }
            }
        }
    }
    if (!ok) raise_flag(LP_FLAG_NONFINITE);
}

// K10 for inner == 1 (W-axis plans): x-stationary.  A thread keeps one position x for its
// whole life — grid threads are used in multiples of D, so thread g owns x = g % D and walks
// rows o = g / D, g / D + R, ... (R = threads / D) — which puts its coverage-table column
// (weights, offsets, Z) in registers, loaded once.  Lanes hold consecutive x, so every load and
// store instruction of a warp is one contiguous run; 4 rows are in flight per iteration.
template <int D, bool UPDATE, bool FAST>
__global__ void __launch_bounds__(256) k_reconstruct_xs(const __grid_constant__ ReconParams p,
                                                        const typename Store<D>::T* __restrict__ preds,
                                                        typename Store<D>::T* __restrict__ z,
                                                        typename Store<D>::T* __restrict__ eps_out,
                                                        const void* __restrict__ table, uint32_t live) {
    if (recon_aborted(p)) return;
    using T = typename Store<D>::T;
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= live) return;
    const uint32_t Dx = static_cast<uint32_t>(p.D), rows = static_cast<uint32_t>(p.outer);
    const uint32_t x = g % Dx, R = live / Dx;
    const CovLayout t(const_cast<void*>(table), static_cast<int>(Dx));
    const uint32_t c = __ldg(t.cnt + x);
    double w[kReconCover];
    uint32_t off[kReconCover], str[kReconCover];
#pragma unroll
    for (int cc = 0; cc < kReconCover; ++cc) {
        w[cc] = cc < c ? __ldg(t.wts + cc * Dx + x) : 0.0;
        off[cc] = cc < c ? __ldg(t.offs + cc * Dx + x) : 0u;
        str[cc] = cc < c ? __ldg(t.ostr + cc * Dx + x) : 0u;
    }
    const double Z = __ldg(t.zsum + x), Zi = __ldg(t.zinv + x);
    const float Zf = __ldg(t.zsumf + x);
    bool ok = true;
    constexpr int U = 4;
    for (uint32_t o0 = g / Dx; o0 < rows; o0 += U * R) {
        T raw[U][kReconCover], zr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t o = o0 + u * R;
            if (o < rows) {
#pragma unroll
                for (int cc = 0; cc < kReconCover; ++cc)
                    if (cc < c) raw[u][cc] = preds[off[cc] + static_cast<uint64_t>(o) * str[cc]];
                if (UPDATE) zr[u] = z[static_cast<uint64_t>(o) * Dx + x];
            }
        }
        const uint32_t live = rows > o0 ? min(static_cast<uint32_t>(U), (rows - o0 + R - 1) / R) : 0u;
        T q[U];
        ok = k10_group<D, UPDATE, FAST, U>(c, w, Z, Zi, Zf, p.mk, p.eta, raw, zr, q, live) && ok;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < static_cast<int>(live)) (UPDATE ? z : eps_out)[static_cast<uint64_t>(o0 + u * R) * Dx + x] = q[u];
    }
    if (!ok) raise_flag(LP_FLAG_NONFINITE);
}

// K10 for inner == 1, branch-free x-stationary form (knob recon_xsb, default): the threads
// of a warp hold consecutive positions x, so at every window edge the lanes of one warp have
// different cover counts and Z == 1 tests — the form above then runs each variant's fp64 code
// serially.  Here every lane evaluates CM covers (CM = the plan's maximum, a compile-time
// count): a cover the position does not have re-reads cover 0's (cached) element and is
// dropped by a select, so the worker-order sum is the reference's bit for bit, NaN / inf
// included; the division and the Z == 1 shortcut are both evaluated and selected.  No branch
// depends on x.
template <int D, bool UPDATE, bool FAST, int CM, int U = 4>
__global__ void __launch_bounds__(256) k_reconstruct_xsb(const __grid_constant__ ReconParams p,
                                                         const typename Store<D>::T* __restrict__ preds,
                                                         typename Store<D>::T* __restrict__ z,
                                                         typename Store<D>::T* __restrict__ eps_out,
                                                         const void* __restrict__ table, uint32_t live) {
    if (recon_aborted(p)) return;
    using T = typename Store<D>::T;
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= live) return;
    const uint32_t Dx = static_cast<uint32_t>(p.D), rows = static_cast<uint32_t>(p.outer);
    const uint32_t x = g % Dx, R = live / Dx;
    const CovLayout t(const_cast<void*>(table), static_cast<int>(Dx));
    const uint32_t c = __ldg(t.cnt + x);
    double w[CM];
    float wf[CM];
    bool has[CM];
    uint32_t off[CM], str[CM];
#pragma unroll
    for (int cc = 0; cc < CM; ++cc) {
        has[cc] = cc < static_cast<int>(c);
        const uint32_t sc = has[cc] ? cc : 0u;  // absent cover: cover 0's element (a valid address)
        w[cc] = __ldg(t.wts + sc * Dx + x);
        wf[cc] = static_cast<float>(w[cc]);
        off[cc] = __ldg(t.offs + sc * Dx + x);
        str[cc] = __ldg(t.ostr + sc * Dx + x);
    }
    const double Z = __ldg(t.zsum + x), Zi = __ldg(t.zinv + x);
    const float Zf = __ldg(t.zsumf + x);
    const bool z1 = FAST ? Zf == 1.f : Z == 1.0;
    const bool mk = p.mk != 0;
    bool ok = true;
    for (uint32_t o0 = g / Dx; o0 < rows; o0 += U * R) {
        T raw[U][CM], zr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t o = min(o0 + u * R, rows - 1);  // clamped: rows past the end are not stored
#pragma unroll
            for (int cc = 0; cc < CM; ++cc) raw[u][cc] = preds[off[cc] + static_cast<uint64_t>(o) * str[cc]];
            if (UPDATE) zr[u] = z[static_cast<uint64_t>(o) * Dx + x];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t o = o0 + u * R;
            double eps;
            if (!FAST) {
                double a = 0.0;  // from +0 like the reference's accumulator
#pragma unroll
                for (int cc = 0; cc < CM; ++cc) {
                    const double s = __dadd_rn(a, __dmul_rn(w[cc], load_val<D>(raw[u], cc)));
                    a = has[cc] ? s : a;
                }
                const double qd = mk ? div_z(a, Z, Zi) : __ddiv_rn(a, Z);
                eps = quantize_dev<D>(z1 ? a : qd);
            } else {
                float a = 0.f;
#pragma unroll
                for (int cc = 0; cc < CM; ++cc) {
                    const float s = fmaf(wf[cc], static_cast<float>(load_val<D>(raw[u], cc)), a);
                    a = has[cc] ? s : a;
                }
                eps = quantize_dev<D>(static_cast<double>(z1 ? a : a / Zf));
            }
            bool fin = isfinite(eps);
            double res = eps;
            if (UPDATE) {
                const double zo = load_val<D>(zr, u);
                res = FAST ? static_cast<double>(fmaf(-static_cast<float>(p.eta), static_cast<float>(eps), static_cast<float>(zo)))
                           : __dsub_rn(zo, __dmul_rn(p.eta, eps));
            }
            if (o < rows) {
                T qv;
                fin = store_q<D>(&qv, 0, res) && fin;
                (UPDATE ? z : eps_out)[static_cast<uint64_t>(o) * Dx + x] = qv;
                ok = ok && fin;
            }
        }
    }
    if (!ok) raise_flag(LP_FLAG_NONFINITE);
}

// the largest number of entries covering one position of p's axis
static int recon_max_cover(const ReconParams& p) {
    int m = 0;
    for (int64_t x = 0; x < p.D; ++x) {
        int c = 0;
        for (int k = 0; k < p.n; ++k) c += (x >= p.e[k].begin && x < p.e[k].begin + p.e[k].len);
        m = std::max(m, c);
    }
    return m;
}

// Coverage-table K10 applicability: 32-bit offsets, total % 4 == 0, every position covered
// by at most kReconCover entries, table in 48 KB.  Returns the table bytes, 0 if not usable.
static size_t recon_cov_bytes(const ReconParams& p, int dtype) {
    if (!p.use32) return 0;
    int64_t preds = 0;
    for (int k = 0; k < p.n; ++k) preds += p.e[k].len * p.outer * p.inner;
    if (preds >= (1ll << 31)) return 0;
    for (int64_t x = 0; x < p.D; ++x) {
        int c = 0;
        for (int k = 0; k < p.n; ++k) c += (x >= p.e[k].begin && x < p.e[k].begin + p.e[k].len);
        if (c > kReconCover) return 0;
    }
    (void)dtype;
    if (p.n > 255) return 0;  // kidx is a byte
    const size_t bytes =
        (static_cast<size_t>(p.D) * (kReconCover * 8 + 8 + 8 + 4 + kReconCover * 8 + 4 + kReconCover) + 15) / 16 * 16;
    return bytes <= 48 * 1024 ? bytes : 0;
}

// Device coverage tables, cached per (device, plan entries, gather bases, D, inner).  Built on
// first use (eagerly: the engine's first step of an axis precedes any graph capture).  The
// cache holds at most kReconTables tables; past that, or on lp_release_caches(), every table is
// freed (cudaFree waits for the device, so no in-flight K10 still reads one).
constexpr size_t kReconTables = 64;
static std::mutex g_table_mu;
static std::map<std::string, void*> g_tables;

static void release_tables_locked() {
    for (auto& kv : g_tables) cudaFree(kv.second);
    g_tables.clear();
}

static const void* recon_table(const ReconParams& p, size_t bytes, cudaStream_t st) {
    std::mutex& mu = g_table_mu;
    std::map<std::string, void*>& cache = g_tables;
    int dev = 0;
    LP_CUDA(cudaGetDevice(&dev));
    std::string key(reinterpret_cast<const char*>(&dev), sizeof(dev));
    key.append(reinterpret_cast<const char*>(&p.D), sizeof(p.D));
    key.append(reinterpret_cast<const char*>(&p.inner), sizeof(p.inner));
    key.append(reinterpret_cast<const char*>(p.e), sizeof(ReconEntry) * static_cast<size_t>(p.n));
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LP_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone)
        fail(LP_ERR_INVALID_ARGUMENT, "K10 coverage table must be built by an eager launch before graph capture");
    if (cache.size() >= kReconTables) release_tables_locked();
    void* t = nullptr;
    LP_CUDA(cudaMalloc(&t, bytes));
    k_recon_table<<<1, 256, 0, st>>>(p, t);
    LP_LAUNCH_CHECK();
    // published only once built: a caller on another stream may use it right away
    LP_CUDA(cudaStreamSynchronize(st));
    cache.emplace(std::move(key), t);
    return t;
}

void* recon_table_build(const ReconParams& p, cudaStream_t st) {
    const size_t bytes = recon_cov_bytes(p, 0);
    if (!bytes) return nullptr;
    void* t = nullptr;
    LP_CUDA(cudaMalloc(&t, bytes));
    k_recon_table<<<1, 256, 0, st>>>(p, t);
    LP_LAUNCH_CHECK();
    LP_CUDA(cudaStreamSynchronize(st));
    return t;
}

template <int D, bool UPDATE>
static void launch_recon(const ReconParams& p, const void* preds, void* z, void* eps, bool fast, cudaStream_t st) {
    using T = typename Store<D>::T;
    const int g = grid_for(p.total, 256);
    const size_t tab = sizeof(double) * static_cast<size_t>(p.n + 1) * static_cast<size_t>(p.D);
    const size_t cov = tune_get("recon_cov", 1) ? recon_cov_bytes(p, D) : 0;
    const uintptr_t al = reinterpret_cast<uintptr_t>(preds) | reinterpret_cast<uintptr_t>(UPDATE ? z : eps);
    if (cov) {
        bool vec = p.inner % 8 == 0 && al % (4 * D) == 0;  // 8 elements share (o, x); prediction vectors need 8-aligned bases
        for (int k = 0; k < p.n; ++k) vec = vec && p.e[k].base % 8 == 0;
        // one wave of resident blocks: each block builds its table once
        const void* table = p.table ? p.table : recon_table(p, cov, st);
        const uint32_t tv = static_cast<uint32_t>(cov / 16);
        int res = 0;
        const bool g4 = vec && tune_get("recon_g", 4) == 4;  // VEC: 4 elements (one vector per cover) per thread
        auto kfn = fast ? (vec ? (g4 ? k_reconstruct_cov<D, UPDATE, true, true, 4> : k_reconstruct_cov<D, UPDATE, true, true>)
                               : k_reconstruct_cov<D, UPDATE, true, false>)
                        : (vec ? (g4 ? k_reconstruct_cov<D, UPDATE, false, true, 4> : k_reconstruct_cov<D, UPDATE, false, true>)
                               : k_reconstruct_cov<D, UPDATE, false, false>);
        LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, kfn, 256, cov));
        res = std::max(1, res);
        const int gq = grid_for(p.total / (g4 ? 4 : 8), 256, res);
        auto* out_z = static_cast<T*>(z);
        auto* out_e = static_cast<T*>(eps);
        const auto* in = static_cast<const T*>(preds);
        const int cm = p.inner == 1 && tune_get("recon_xsb", 1) ? std::min(recon_max_cover(p), kReconCover) : 0;
        if (cm > 0) {
            // W axis, branch-free x-stationary form: threads in a multiple of D, one resident wave
            auto pick = [&](auto kf) {
                int rx = 0;
                LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rx, kf, 256, 0));
                const int64_t cap = static_cast<int64_t>(grid_for(INT32_MAX, 256, std::max(1, rx))) * 256;
                const int64_t want = std::min<int64_t>(cap, p.total);
                const uint32_t live = static_cast<uint32_t>(std::max<int64_t>(p.D, want / p.D * p.D));
                kf<<<static_cast<int>((live + 255) / 256), 256, 0, st>>>(p, in, out_z, out_e, table, live);
            };
            // rows in flight per thread (knob recon_u: 4 or 8)
            const bool u8 = tune_get("recon_u", 4) == 8;
            switch (cm * 2 + (fast ? 1 : 0)) {
                case 2: u8 ? pick(k_reconstruct_xsb<D, UPDATE, false, 1, 8>) : pick(k_reconstruct_xsb<D, UPDATE, false, 1>); break;
                case 3: u8 ? pick(k_reconstruct_xsb<D, UPDATE, true, 1, 8>) : pick(k_reconstruct_xsb<D, UPDATE, true, 1>); break;
                case 4: u8 ? pick(k_reconstruct_xsb<D, UPDATE, false, 2, 8>) : pick(k_reconstruct_xsb<D, UPDATE, false, 2>); break;
                case 5: u8 ? pick(k_reconstruct_xsb<D, UPDATE, true, 2, 8>) : pick(k_reconstruct_xsb<D, UPDATE, true, 2>); break;
                case 6: u8 ? pick(k_reconstruct_xsb<D, UPDATE, false, 3, 8>) : pick(k_reconstruct_xsb<D, UPDATE, false, 3>); break;
                case 7: u8 ? pick(k_reconstruct_xsb<D, UPDATE, true, 3, 8>) : pick(k_reconstruct_xsb<D, UPDATE, true, 3>); break;
                case 8: u8 ? pick(k_reconstruct_xsb<D, UPDATE, false, 4, 8>) : pick(k_reconstruct_xsb<D, UPDATE, false, 4>); break;
                default: u8 ? pick(k_reconstruct_xsb<D, UPDATE, true, 4, 8>) : pick(k_reconstruct_xsb<D, UPDATE, true, 4>); break;
            }
        } else if (p.inner == 1 && tune_get("recon_xs", 1)) {
            // x-stationary: threads in a multiple of D, one resident wave
            int rx = 0;
            LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rx, fast ? k_reconstruct_xs<D, UPDATE, true>
                                                                              : k_reconstruct_xs<D, UPDATE, false>, 256, 0));
            const int64_t cap = static_cast<int64_t>(grid_for(INT32_MAX, 256, std::max(1, rx))) * 256;
            const int64_t want = std::min<int64_t>(cap, p.total);
            const uint32_t live = static_cast<uint32_t>(std::max<int64_t>(p.D, want / p.D * p.D));
            const int gx = static_cast<int>((live + 255) / 256);
            if (fast) k_reconstruct_xs<D, UPDATE, true><<<gx, 256, 0, st>>>(p, in, out_z, out_e, table, live);
            else k_reconstruct_xs<D, UPDATE, false><<<gx, 256, 0, st>>>(p, in, out_z, out_e, table, live);
        } else {
            kfn<<<gq, 256, cov, st>>>(p, in, out_z, out_e, static_cast<const uint4*>(table), tv);
        }
    } else if (!fast && p.use32 && tab <= 48 * 1024) {
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
    p.mk = tune_get("recon_mk", 1);
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

int lp_release_caches(void) {
    return guard([&] {
        std::lock_guard<std::mutex> lock(g_table_mu);
        release_tables_locked();
    });
}

// Device memory plumbing for hosts that bind only this header (the reference-side shim in
// integration/): no cuda_runtime.h needed on the caller's side.
int lp_device_alloc(size_t bytes, void** out) {
    return guard([&] {
        *out = nullptr;
        if (bytes) LP_CUDA(cudaMalloc(out, bytes));
    });
}
int lp_device_free(void* p) {
    return guard([&] { LP_CUDA(cudaFree(p)); });
}
int lp_copy_to_device(void* dst, const void* src, size_t bytes) {
    return guard([&] {
        if (bytes) LP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    });
}
int lp_copy_to_host(void* dst, const void* src, size_t bytes) {
    return guard([&] {
        if (bytes) LP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    });
}

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
        std::vector<int> ks(count);
        for (int c = 0; c < count; ++c) ks[c] = first + c;
        gather_entries(z, s, *plan, ks.data(), count, dtype, dst, as_stream(stream));  // K1, one launch
    });
}

size_t lp_toy_workspace_bytes(const int64_t shape[4]) { return static_cast<size_t>(shape[0]) * sizeof(double); }

int lp_toy_predict(int32_t kind, const int64_t radius[3], double t_coeff, double cond_coeff, const void* z,
                   const int64_t shape[4], int dtype, int timestep, double cond_mean, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        const Shape4 s = Shape4::from(shape);
        double* ws = nullptr;
        if (kind == LP_TOY_GLOBAL) {
            // C doubles of per-channel means: stream-ordered from the device's default pool, which
            // keeps freed blocks (release threshold raised once), so after the first call this is
            // a pool hit — no cudaMalloc, no device synchronisation
            static std::once_flag pool_once;
            std::call_once(pool_once, [] {
                int dev = 0;
                cudaMemPool_t pool = nullptr;
                if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                    uint64_t keep = UINT64_MAX;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
                }
            });
            LP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), s.c * sizeof(double), as_stream(stream)));
        }
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
