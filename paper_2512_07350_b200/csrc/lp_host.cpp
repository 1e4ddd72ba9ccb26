// lp_host.cpp — host LP core + its C-ABI (plan builder, weights, layouts,
// accounting, quantizer, synthetic inputs).  Compiled with -ffp-contract=off so
// every double op rounds separately, as in the reference build.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <random>

#include "lp_host.hpp"

namespace lpb200 {

namespace {
thread_local std::string g_last_error;
std::mutex g_warn_mu;
lp_warning_fn g_warn_fn = nullptr;
void* g_warn_user = nullptr;
bool g_warn_default = true;
const char* kAxisName[3] = {"T", "H", "W"};
}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

void emit_warning(const std::string& m) {
    std::lock_guard<std::mutex> lk(g_warn_mu);
    if (g_warn_fn) g_warn_fn(m.c_str(), g_warn_user);
    else if (g_warn_default) std::fprintf(stderr, "lp_b200: warning: %s\n", m.c_str());
}

int rotation_axis(int step_index) {
    if (step_index < 1) fail(LP_ERR_INVALID_ARGUMENT, "step index must be >= 1, got " + std::to_string(step_index));
    return (step_index - 1) % 3;
}

std::vector<Range> core_bounds(i64 patches, int workers) {
    if (patches < 1) fail(LP_ERR_INVALID_ARGUMENT, "patch count must be >= 1");
    if (workers < 1) fail(LP_ERR_INVALID_ARGUMENT, "worker count must be >= 1");
    const i64 per = (patches + workers - 1) / workers;
    std::vector<Range> out;
    for (i64 a = 0; a < patches && static_cast<i64>(out.size()) < workers; a += per)
        out.push_back({a, a + per < patches ? a + per : patches});
    return out;
}

std::vector<Range> extend_overlap(const std::vector<Range>& cores, i64 patches, i64 per_core, double r, int workers) {
    if (!(r >= 0.0 && r <= static_cast<double>(workers - 1)))
        fail(LP_ERR_INVALID_OVERLAP_RATIO,
             "overlap ratio " + std::to_string(r) + " outside [0, " + std::to_string(workers - 1) + "]");
    const i64 o = static_cast<i64>(static_cast<double>(per_core) * r);
    std::vector<Range> out;
    out.reserve(cores.size());
    for (const Range& c : cores) out.push_back({c.begin - o > 0 ? c.begin - o : 0, c.end + o < patches ? c.end + o : patches});
    return out;
}

lp_plan build_axis_plan(int axis, i64 extent, i64 patch, int step, int workers, double r) {
    if (axis < 0 || axis > 2) fail(LP_ERR_INVALID_ARGUMENT, "axis must be 0..2");
    if (patch < 1 || extent < patch)
        fail(LP_ERR_DEGENERATE_AXIS, std::string("axis ") + kAxisName[axis] + " extent " + std::to_string(extent) +
                                         " cannot hold patch size " + std::to_string(patch));
    if (workers > LP_MAX_WORKERS) fail(LP_ERR_INVALID_ARGUMENT, "workers > LP_MAX_WORKERS");
    const i64 n = extent / patch;
    const std::vector<Range> cores = core_bounds(n, workers);
    if (static_cast<int>(cores.size()) < workers)
        emit_warning(std::string("axis ") + kAxisName[axis] + " has " + std::to_string(n) + " patches for " +
                     std::to_string(workers) + " workers; " + std::to_string(workers - static_cast<int>(cores.size())) +
                     " idle this step");
    const i64 per = (n + workers - 1) / workers;
    const std::vector<Range> ext = extend_overlap(cores, n, per, r, workers);
    lp_plan p;
    std::memset(&p, 0, sizeof(p));
    p.axis = axis;
    p.step_index = step;
    p.overlap_ratio = r;
    p.patches_per_core = per;
    p.overlap_patches = static_cast<i64>(static_cast<double>(per) * r);
    p.axis_patches = n;
    p.axis_extent = extent;
    p.patch_size = patch;
    p.n_entries = static_cast<int32_t>(cores.size());
    for (size_t i = 0; i < cores.size(); ++i) {
        lp_entry& e = p.entries[i];
        e.worker_id = static_cast<int32_t>(i + 1);
        e.core_begin = cores[i].begin;
        e.core_end = cores[i].end;
        e.ext_begin = ext[i].begin;
        e.ext_end = ext[i].end;
        e.latent_begin = ext[i].begin * patch;
        // remainder rows past N*p belong to the final partition (partition.cpp:113-117)
        e.latent_end = (i + 1 == cores.size()) ? extent : ext[i].end * patch;
        e.delta_start = (cores[i].begin - ext[i].begin) * patch;
        e.delta_end = (ext[i].end - cores[i].end) * patch;
    }
    return p;
}

lp_plan build_plan_for_shape(const Shape4& s, const i64 patch[3], int step, int workers, double r) {
    const int a = rotation_axis(step);
    return build_axis_plan(a, s.extent(a), patch[a], step, workers, r);
}

std::vector<double> weight_profile(const lp_entry& e) {
    const i64 len = e.latent_end - e.latent_begin;
    std::vector<double> w(static_cast<size_t>(len > 0 ? len : 0), 1.0);
    for (i64 j = 0; j < e.delta_start && j < len; ++j) w[j] = static_cast<double>(j) / static_cast<double>(e.delta_start);
    for (i64 j = len - e.delta_end; j < len; ++j)
        if (j >= 0) w[j] = static_cast<double>(len - j) / static_cast<double>(e.delta_end);
    return w;
}

void validate_plan(const lp_plan& p) {
    if (p.axis < 0 || p.axis > 2) fail(LP_ERR_INVALID_ARGUMENT, "plan axis out of range");
    if (p.n_entries < 1 || p.n_entries > LP_MAX_WORKERS) fail(LP_ERR_INVALID_ARGUMENT, "plan has no entries");
    for (int k = 0; k < p.n_entries; ++k) {
        const lp_entry& e = p.entries[k];
        if (e.latent_begin == e.latent_end) fail(LP_ERR_EMPTY_RANGE, "empty slice in plan entry " + std::to_string(k + 1));
        if (e.latent_begin < 0 || e.latent_end > p.axis_extent || e.latent_begin > e.latent_end)
            fail(LP_ERR_OUT_OF_BOUNDS, "plan entry " + std::to_string(k + 1) + " outside [0," + std::to_string(p.axis_extent) + ")");
    }
}

std::vector<i64> entry_elems(const lp_plan& p, const Shape4& s) {
    i64 outer, inner;
    axis_view(s, p.axis, outer, inner);
    std::vector<i64> n(static_cast<size_t>(p.n_entries));
    for (int k = 0; k < p.n_entries; ++k) n[k] = outer * inner * (p.entries[k].latent_end - p.entries[k].latent_begin);
    return n;
}

std::vector<double> weight_sums(const lp_plan& p) {
    std::vector<double> z(static_cast<size_t>(p.axis_extent), 0.0);
    for (int k = 0; k < p.n_entries; ++k) {
        const std::vector<double> w = weight_profile(p.entries[k]);
        for (i64 j = 0; j < static_cast<i64>(w.size()); ++j) z[p.entries[k].latent_begin + j] += w[j];
    }
    for (i64 x = 0; x < p.axis_extent; ++x)
        if (z[x] < 1.0 - 1e-12)
            fail(LP_ERR_ZERO_WEIGHT, "weight sum " + std::to_string(z[x]) + " < 1 at axis position " + std::to_string(x));
    return z;
}

ShardLayout shard_layout(const lp_plan& p, const Shape4& s, int world, int rank, const AssignCost* cost) {
    if (world < 1 || rank < 0 || rank >= world) fail(LP_ERR_INVALID_ARGUMENT, "bad world/rank");
    const std::vector<i64> n = entry_elems(p, s);
    std::vector<int> owner(n.size(), 0);
    for (int k = 0; k < p.n_entries; ++k) owner[k] = k % world;  // round-robin (the default)
    if (cost && p.n_entries > world) {
        // balanced: longest-processing-time greedy over the per-entry cost model (the
        // reference leaves the worker -> device mapping open; its workers are threads)
        std::vector<int> order(n.size());
        for (int k = 0; k < p.n_entries; ++k) order[k] = k;
        auto c = [&](int k) { return cost->lin * static_cast<double>(n[k]) + cost->quad * static_cast<double>(n[k]) * static_cast<double>(n[k]); };
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return c(a) > c(b); });
        std::vector<double> load(static_cast<size_t>(world), 0.0);
        for (int k : order) {
            int best = 0;
            for (int r = 1; r < world; ++r)
                if (load[r] < load[best]) best = r;
            owner[k] = best;
            load[best] += c(k);
        }
    }
    std::vector<i64> per_rank(static_cast<size_t>(world), 0), within(n.size(), 0);
    for (int k = 0; k < p.n_entries; ++k) {  // each rank's slot packs its entries in worker order
        within[k] = per_rank[owner[k]];
        per_rank[owner[k]] += n[k];
    }
    ShardLayout L;
    for (int r = 0; r < world; ++r) L.slot_elems = std::max(L.slot_elems, per_rank[r]);
    // slots start on 16-byte boundaries for every storage width (8 elements >= 16 B), so the
    // peer exchange's 16-B vector copies of rank r's slot [r*slot, (r+1)*slot) are aligned
    L.slot_elems = (L.slot_elems + 7) / 8 * 8;
    for (int k = 0; k < p.n_entries; ++k) {
        if (owner[k] == rank) L.owned.push_back(k);
        L.base.push_back(static_cast<i64>(owner[k]) * L.slot_elems + within[k]);
        L.owner.push_back(owner[k]);
    }
    return L;
}

double host_quantize(double v, int d) {
    if (d == 8) return v;
    if (d == 4) {
        const double lim = std::numeric_limits<float>::max();
        if (v > lim) return lim;
        if (v < -lim) return -lim;
        return static_cast<double>(static_cast<float>(v));
    }
    return f16_decode_exact(f16_encode_exact(v));
}

namespace {
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
    double flops, bytes;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_ev_pool;
cudaEvent_t g_pending[KC_COUNT];
cudaEvent_t take_event() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    LP_CUDA(cudaEventCreate(&e));
    return e;
}
}  // namespace

namespace {
std::mutex g_tune_mu;
std::vector<std::pair<std::string, int>> g_tune;
}  // namespace

int tune_get(const char* key, int dflt) {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    for (auto& kv : g_tune)
        if (kv.first == key) return kv.second;
    std::string env = "LP_TUNE_";
    for (const char* c = key; *c; ++c) env += static_cast<char>(toupper(*c));
    const char* e = getenv(env.c_str());
    const int v = e ? atoi(e) : dflt;
    g_tune.emplace_back(key, v);
    return v;
}

bool prof_enabled() { return g_prof_on; }
void prof_begin(int cls, cudaStream_t st) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_pending[cls] = take_event();
    LP_CUDA(cudaEventRecord(g_pending[cls], st));
}
void prof_end(int cls, cudaStream_t st, double flops, double bytes) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t e = take_event();
    LP_CUDA(cudaEventRecord(e, st));
    g_prof.push_back({cls, g_pending[cls], e, flops, bytes});
}

}  // namespace lpb200

using namespace lpb200;

extern "C" int lp_tune(const char* key, int value) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_tune_mu);
        for (auto& kv : g_tune)
            if (kv.first == key) {
                kv.second = value;
                return;
            }
        g_tune.emplace_back(key, value);
    });
}

extern "C" int lp_profile_enable(int on) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof_on = on != 0;
    });
}

// Per class: launches, summed device ms, summed algorithmic flops and bytes; clears.
extern "C" int lp_profile_collect(uint64_t* launches, double* ms, double* flops, double* bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        for (int c = 0; c < KC_COUNT; ++c) launches[c] = 0, ms[c] = 0, flops[c] = 0, bytes[c] = 0;
        for (auto& r : g_prof) {
            LP_CUDA(cudaEventSynchronize(r.b));
            float t = 0.f;
            LP_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            launches[r.cls] += 1;
            ms[r.cls] += t;
            flops[r.cls] += r.flops;
            bytes[r.cls] += r.bytes;
            g_ev_pool.push_back(r.a);
            g_ev_pool.push_back(r.b);
        }
        g_prof.clear();
    });
}

extern "C" {

const char* lp_last_error(void) { return g_last_error.c_str(); }
const char* lp_version(void) { return "lp_b200 0.1.0 (sm_100a)"; }

void lp_set_warning_handler(lp_warning_fn fn, void* user) {
    std::lock_guard<std::mutex> lk(g_warn_mu);
    g_warn_fn = fn;
    g_warn_user = user;
    g_warn_default = false;  // an explicit NULL silences
}

int lp_rotation_axis(int step_index, int32_t* axis_out) {
    return guard([&] { *axis_out = rotation_axis(step_index); });
}

int lp_core_bounds(int64_t patches, int workers, int64_t* ranges_out, int32_t* n_out) {
    return guard([&] {
        const auto c = core_bounds(patches, workers);
        for (size_t i = 0; i < c.size(); ++i) {
            ranges_out[2 * i] = c[i].begin;
            ranges_out[2 * i + 1] = c[i].end;
        }
        *n_out = static_cast<int32_t>(c.size());
    });
}

int lp_extend_overlap(const int64_t* cores, int32_t n_cores, int64_t patches, int64_t per_core, double r, int workers,
                      int64_t* ext_out) {
    return guard([&] {
        std::vector<Range> c;
        for (int i = 0; i < n_cores; ++i) c.push_back({cores[2 * i], cores[2 * i + 1]});
        const auto e = extend_overlap(c, patches, per_core, r, workers);
        for (size_t i = 0; i < e.size(); ++i) {
            ext_out[2 * i] = e[i].begin;
            ext_out[2 * i + 1] = e[i].end;
        }
    });
}

int lp_build_axis_plan(int32_t axis, int64_t extent, int64_t patch, int step, int workers, double r, lp_plan* out) {
    return guard([&] { *out = build_axis_plan(axis, extent, patch, step, workers, r); });
}

int lp_build_plan(const int64_t shape[4], const int64_t patch[3], int step, int workers, double r, lp_plan* out) {
    return guard([&] { *out = build_plan_for_shape(Shape4::from(shape), patch, step, workers, r); });
}

int lp_weight_profile(const lp_plan* plan, int32_t entry, double* out) {
    return guard([&] {
        if (entry < 0 || entry >= plan->n_entries) fail(LP_ERR_OUT_OF_BOUNDS, "entry out of range");
        const auto w = weight_profile(plan->entries[entry]);
        std::memcpy(out, w.data(), w.size() * sizeof(double));
    });
}

int lp_plan_offsets(const lp_plan* plan, const int64_t shape[4], int64_t* offsets_out) {
    return guard([&] {
        const auto n = entry_elems(*plan, Shape4::from(shape));
        offsets_out[0] = 0;
        for (size_t k = 0; k < n.size(); ++k) offsets_out[k + 1] = offsets_out[k] + n[k];
    });
}

int lp_shard_layout(const lp_plan* plan, const int64_t shape[4], int world, int rank, int32_t* owned_out,
                    int32_t* n_owned_out, int64_t* slot_elems_out) {
    return guard([&] {
        const ShardLayout L = shard_layout(*plan, Shape4::from(shape), world, rank);
        for (size_t i = 0; i < L.owned.size(); ++i) owned_out[i] = L.owned[i];
        *n_owned_out = static_cast<int32_t>(L.owned.size());
        *slot_elems_out = L.slot_elems;
    });
}

int lp_shard_bases(const lp_plan* plan, const int64_t shape[4], int world, int64_t* base_out) {
    return guard([&] {
        const ShardLayout L = shard_layout(*plan, Shape4::from(shape), world, 0);
        for (size_t k = 0; k < L.base.size(); ++k) base_out[k] = L.base[k];
    });
}

int lp_shard_layout_ex(const lp_plan* plan, const int64_t shape[4], int world, int rank, int32_t policy, double lin,
                       double quad, int32_t* owned_out, int32_t* n_owned_out, int64_t* slot_elems_out,
                       int32_t* owner_out, int64_t* base_out) {
    return guard([&] {
        if (policy != LP_ASSIGN_ROUND_ROBIN && policy != LP_ASSIGN_BALANCED)
            fail(LP_ERR_INVALID_ARGUMENT, "assignment policy must be 0 (round-robin) or 1 (balanced)");
        const AssignCost cost{lin, quad};
        const ShardLayout L = shard_layout(*plan, Shape4::from(shape), world, rank, policy ? &cost : nullptr);
        if (owned_out)
            for (size_t i = 0; i < L.owned.size(); ++i) owned_out[i] = L.owned[i];
        if (n_owned_out) *n_owned_out = static_cast<int32_t>(L.owned.size());
        if (slot_elems_out) *slot_elems_out = L.slot_elems;
        for (size_t k = 0; k < L.base.size(); ++k) {
            if (owner_out) owner_out[k] = L.owner[k];
            if (base_out) base_out[k] = L.base[k];
        }
    });
}

int lp_step_comm_bytes(const lp_plan* plan, const int64_t shape[4], int wire_bytes, int world, int dtype_bytes,
                       uint64_t* ledger_out, uint64_t* allgather_out) {
    return guard([&] {
        const Shape4 s = Shape4::from(shape);
        const auto n = entry_elems(*plan, s);
        uint64_t sum = 0;
        for (size_t k = 1; k < n.size(); ++k) sum += static_cast<uint64_t>(n[k]);
        *ledger_out = 4ull * sum * static_cast<uint64_t>(wire_bytes);
        const ShardLayout L = shard_layout(*plan, s, world, 0);
        *allgather_out = static_cast<uint64_t>(world) * static_cast<uint64_t>(world - 1) *
                         static_cast<uint64_t>(L.slot_elems) * static_cast<uint64_t>(dtype_bytes);
    });
}

uint16_t lp_f16_encode(double v) { return f16_encode_exact(v); }
double lp_f16_decode(uint16_t b) { return f16_decode_exact(b); }
double lp_quantize(double v, int d) { return host_quantize(v, d); }

// synthetic_inputs (src/run_config.cpp:258-301): standard mt19937_64 words,
// Box-Muller with u1 in (0,1], u2 in [0,1), cosine first and the sine kept as
// the spare; latent (quantized) first, then 8 conditioning values.
int lp_synthetic_inputs(const int64_t shape[4], int dtype_bytes, uint64_t seed, double* latent_out, double* cond_out8) {
    return guard([&] {
        check_dtype(dtype_bytes);
        std::mt19937_64 rng(seed);
        bool have = false;
        double spare = 0.0;
        auto next = [&]() {
            if (have) {
                have = false;
                return spare;
            }
            const double u1 = (static_cast<double>(rng() >> 11) + 1.0) * 0x1.0p-53;
            const double u2 = static_cast<double>(rng() >> 11) * 0x1.0p-53;
            const double rad = std::sqrt(-2.0 * std::log(u1));
            const double ang = 6.283185307179586476925286766559 * u2;
            spare = rad * std::sin(ang);
            have = true;
            return rad * std::cos(ang);
        };
        const i64 n = Shape4::from(shape).volume();
        for (i64 i = 0; i < n; ++i) {
            const double q = host_quantize(next(), dtype_bytes);
            if (!std::isfinite(q)) fail(LP_ERR_NON_FINITE, "tensor element is not finite");
            latent_out[i] = q;
        }
        for (int i = 0; i < 8; ++i) cond_out8[i] = next();
    });
}

}  // extern "C"
