// b200_backend.cpp — the reference's hot path, replaced at link time by the B200 engine.
//
// Every function below has the exact signature of the reference function it replaces (cited);
// integration/Makefile links the reference's own archive with those symbols weakened, so the
// reference's callers (simulate/compare commands, the pybind module, its tests) run here.
// Value semantics, validation order and error kinds/messages follow the reference; the math
// runs in the engine's kernels (K1 gather, K11 toy denoisers, CFG combine, K10 blend +
// sampler), bit-identical to the reference's fp64 path.
#include <atomic>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

#include "b200.hpp"
#include "lpsim/cluster.hpp"
#include "lpsim/reconstruct.hpp"

namespace lpsim {
namespace {

using b200::check;
using b200::check_device_flags;
using b200::DeviceBuffer;

// The engine's own plan builder reports dropped idle workers as well; the shim keeps the
// reference's warnings (emitted by its build_plan) and mutes the engine's duplicates.
thread_local bool g_mute_engine_warnings = false;
void forward_warning(const char* msg, void*) {
    if (!g_mute_engine_warnings) emit_warning(msg);
}
struct WarningBridge {
    WarningBridge() { lp_set_warning_handler(forward_warning, nullptr); }
} g_warning_bridge;

void shape_arr(const Shape& s, int64_t out[4]) {
    out[0] = s.c;
    out[1] = s.t;
    out[2] = s.h;
    out[3] = s.w;
}

size_t bytes_of(const Shape& s, Dtype d) { return static_cast<size_t>(s.volume()) * dtype_bytes(d); }

void validate_cluster(const ClusterConfig& cluster) {  // src/cluster.cpp:100-111
    if (cluster.workers < 1) fail(ErrorKind::InvalidArgument, "cluster needs at least one worker");
    if (cluster.master_id != 1) fail(ErrorKind::InvalidArgument, "worker 1 is the master orchestrator");
    if (cluster.preset.dtype_bytes != 2 && cluster.preset.dtype_bytes != 4 && cluster.preset.dtype_bytes != 8)
        fail(ErrorKind::InvalidArgument, "preset dtype_bytes must be 2, 4 or 8");
}

// The per-step ledger records of run_lp (src/cluster.cpp:186-191, 204-209): scatter of every
// non-master sub-latent, then gather of every non-master prediction, each once per CFG pass.
void meter_step(CommLedger& ledger, int i, const PartitionPlan& plan, const Shape& s) {
    const int k_eff = plan.workers();
    auto elems = [&](int k) {
        return static_cast<std::uint64_t>(s.with_extent(plan.axis, plan.entries[static_cast<size_t>(k - 1)].latent.length()).volume());
    };
    for (Pass pass : {Pass::Cond, Pass::Uncond})
        for (int k = 2; k <= k_eff; ++k) ledger.add(i, pass, TransferKind::Scatter, 1, k, elems(k));
    for (Pass pass : {Pass::Cond, Pass::Uncond})
        for (int k = 2; k <= k_eff; ++k) ledger.add(i, pass, TransferKind::Gather, k, 1, elems(k));
}

// Engine config for a B200 denoiser (toy kinds or the DiT).
bool engine_config(const Denoiser& f, const LatentTensor& z, const SamplerConfig& cfg, const PatchGeometry& g,
                   int workers, double r, int wire_bytes, lp_engine_config& c) {
    const auto* toy = dynamic_cast<const b200::ToyDenoiser*>(&f);
    const auto* dit = dynamic_cast<const b200::DiTDenoiser*>(&f);
    if (!toy && !dit) return false;
    std::memset(&c, 0, sizeof(c));
    shape_arr(z.shape(), c.shape);
    c.patch[0] = g.p_t;
    c.patch[1] = g.p_h;
    c.patch[2] = g.p_w;
    c.dtype_bytes = dtype_bytes(z.dtype());
    c.workers = workers;
    c.overlap_ratio = r;
    c.total_steps = cfg.total_steps;
    c.mode = LP_MODE_EXACT;
    c.eta = cfg.step_size;
    c.guidance = cfg.guidance_scale;
    c.wire_bytes = wire_bytes;
    c.world = 1;
    c.rank = 0;
    if (toy) {
        c.denoiser = toy->kind();
        for (int a = 0; a < 3; ++a) c.radius[a] = toy->radius()[a];
        c.t_coeff = toy->t_coeff();
        c.cond_coeff = toy->cond_coeff();
    } else {
        c.denoiser = -1;
        c.dit = dit->handle();
    }
    return true;
}

struct Engine {
    lp_engine* e = nullptr;
    Engine(const lp_engine_config& c, const ConditioningVector& cond) {
        g_mute_engine_warnings = true;
        const int st = lp_engine_create(&c, nullptr, cond.values.data(), static_cast<int32_t>(cond.values.size()), &e);
        g_mute_engine_warnings = false;
        check(st);
    }
    ~Engine() { lp_engine_destroy(e); }
    void* latent() const {
        void* z = nullptr;
        check(lp_engine_latent(e, &z));
        return z;
    }
};

// The worker pool of run_lp (src/cluster.cpp:115-162) for a host-side Denoiser: up to `cap`
// threads, any exception reported for the lowest failing worker id.
void run_workers(const std::vector<SimWorker>& workers, const std::vector<ScatterMessage>& inbox,
                 std::vector<GatherMessage>& outbox, int cap, int step) {
    const int n = static_cast<int>(workers.size());
    std::vector<std::exception_ptr> failures(static_cast<size_t>(n));
    auto one = [&](int i) {
        try {
            outbox[static_cast<size_t>(i)] = workers[static_cast<size_t>(i)].process(inbox[static_cast<size_t>(i)]);
        } catch (...) {
            failures[static_cast<size_t>(i)] = std::current_exception();
        }
    };
    const int threads = std::min(cap, n);
    if (threads <= 1) {
        for (int i = 0; i < n; ++i) one(i);
    } else {
        std::atomic<int> next{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&] {
                for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) one(i);
            });
        for (auto& th : pool) th.join();
    }
    for (int i = 0; i < n; ++i)
        if (failures[static_cast<size_t>(i)]) {
            std::string detail = "unknown error";
            try {
                std::rethrow_exception(failures[static_cast<size_t>(i)]);
            } catch (const std::exception& ex) {
                detail = ex.what();
            } catch (...) {
            }
            fail(ErrorKind::WorkerFailure, "worker " + std::to_string(workers[static_cast<size_t>(i)].id()) +
                                               " failed at step " + std::to_string(step) + ": " + detail);
        }
}

}  // namespace

// ---- extract_sublatents — src/partition.cpp:136-148 (K1) ----
std::vector<LatentTensor> extract_sublatents(const LatentTensor& z, const PartitionPlan& plan) {
    if (z.extent(plan.axis) != plan.axis_extent) {
        fail(ErrorKind::ShapeMismatch, "plan was built for extent " + std::to_string(plan.axis_extent) + " on axis " +
                                           axis_name(plan.axis) + ", tensor has " + std::to_string(z.extent(plan.axis)));
    }
    const i64 d = z.extent(plan.axis);
    for (const PartitionEntry& e : plan.entries) {  // slice_axis's checks (src/latent.cpp:81-92)
        if (e.latent.begin == e.latent.end)
            fail(ErrorKind::EmptyRange, "empty slice [" + std::to_string(e.latent.begin) + "," +
                                            std::to_string(e.latent.end) + ") on axis " + axis_name(plan.axis));
        if (e.latent.begin < 0 || e.latent.end > d || e.latent.begin > e.latent.end)
            fail(ErrorKind::OutOfBounds, "slice [" + std::to_string(e.latent.begin) + "," +
                                             std::to_string(e.latent.end) + ") outside [0," + std::to_string(d) +
                                             ") on axis " + axis_name(plan.axis));
    }
    std::vector<LatentTensor> subs;
    if (plan.entries.empty()) return subs;
    const lp_plan pod = b200::to_pod(plan);
    int64_t sh[4];
    shape_arr(z.shape(), sh);
    std::vector<int64_t> off(plan.entries.size() + 1);
    check(lp_plan_offsets(&pod, sh, off.data()));
    const int E = dtype_bytes(z.dtype());
    DeviceBuffer zd(bytes_of(z.shape(), z.dtype())), out(static_cast<size_t>(off.back()) * E);
    b200::upload(z, zd.get());
    check(lp_extract(&pod, 0, pod.n_entries, zd.get(), sh, E, out.get(), nullptr));
    std::vector<uint8_t> bits(out.bytes());
    check(lp_copy_to_host(bits.data(), out.get(), bits.size()));
    subs.reserve(plan.entries.size());
    for (size_t k = 0; k < plan.entries.size(); ++k)
        subs.push_back(b200::from_bits(z.shape().with_extent(plan.axis, plan.entries[k].latent.length()), z.dtype(),
                                       bits.data() + static_cast<size_t>(off[k]) * E));
    return subs;
}

// ---- reconstruct — src/reconstruct.cpp:42-121 (K10, exact fp64) ----
LatentTensor reconstruct(const std::vector<LatentTensor>& predictions, const PartitionPlan& plan,
                         const Shape& full_shape) {
    if (predictions.size() != plan.entries.size()) {
        fail(ErrorKind::ShapeMismatch, "got " + std::to_string(predictions.size()) + " predictions for " +
                                           std::to_string(plan.entries.size()) + " partitions");
    }
    if (full_shape.extent(plan.axis) != plan.axis_extent) {
        fail(ErrorKind::ShapeMismatch, "plan axis extent " + std::to_string(plan.axis_extent) +
                                           " does not match output shape " + full_shape.str());
    }
    const Dtype dtype = predictions.empty() ? Dtype::F32 : predictions[0].dtype();
    for (size_t k = 0; k < predictions.size(); ++k) {
        const Shape expect = full_shape.with_extent(plan.axis, plan.entries[k].latent.length());
        if (predictions[k].shape() != expect || predictions[k].dtype() != dtype) {
            fail(ErrorKind::ShapeMismatch, "prediction " + std::to_string(k + 1) + " has shape " +
                                               predictions[k].shape().str() + ", expected " + expect.str());
        }
    }
    if (plan.entries.empty()) {  // no contributor anywhere: the reference's weight-sum check
        if (full_shape.extent(plan.axis) > 0)
            fail(ErrorKind::ZeroWeight, "weight sum " + std::to_string(0.0) + " < 1 at axis position 0");
        return LatentTensor::zeros(full_shape, dtype);
    }
    const int E = dtype_bytes(dtype);
    std::vector<uint8_t> packed;
    for (const LatentTensor& p : predictions) {
        const std::vector<uint8_t> b = b200::to_bits(p);
        packed.insert(packed.end(), b.begin(), b.end());
    }
    const lp_plan pod = b200::to_pod(plan);
    int64_t sh[4];
    shape_arr(full_shape, sh);
    DeviceBuffer pd(packed.size()), out(bytes_of(full_shape, dtype));
    check(lp_copy_to_device(pd.get(), packed.data(), packed.size()));
    check(lp_reconstruct(&pod, pd.get(), sh, E, LP_MODE_EXACT, out.get(), nullptr));
    check_device_flags();
    return b200::download(full_shape, dtype, out.get());
}

// ---- cfg_predict — src/denoise.cpp:24-39 ----
LatentTensor cfg_predict(const Denoiser& f, const LatentTensor& z, int timestep, const ConditioningVector& cond,
                         double guidance_scale) {
    if (cond.is_null) fail(ErrorKind::InvalidArgument, "cfg_predict requires a non-null conditioning vector");
    const Shape& s = z.shape();
    const int E = dtype_bytes(z.dtype());
    int64_t sh[4];
    shape_arr(s, sh);
    DeviceBuffer zd(bytes_of(s, z.dtype())), out(bytes_of(s, z.dtype()));
    if (const auto* toy = dynamic_cast<const b200::ToyDenoiser*>(&f)) {  // fused K11: both passes + combine
        b200::upload(z, zd.get());
        DeviceBuffer ws(lp_toy_workspace_bytes(sh) + 64);
        const int64_t rad[3] = {toy->radius()[0], toy->radius()[1], toy->radius()[2]};
        check(lp_toy_cfg_predict(toy->kind(), rad, toy->t_coeff(), toy->cond_coeff(), zd.get(), sh, E, timestep,
                                 cond.mean(), guidance_scale, out.get(), ws.get(), nullptr));
        check_device_flags();
        return b200::download(s, z.dtype(), out.get());
    }
    if (const auto* dit = dynamic_cast<const b200::DiTDenoiser*>(&f)) {  // CFG batch 2 in one forward
        if (cond.values != dit->cond_values())
            fail(ErrorKind::InvalidArgument, "B200 DiT was created for another conditioning vector");
        lp_dit_config c;
        check(lp_dit_get_config(dit->handle(), &c));
        const int64_t tokens = ((s.t + c.patch[0] - 1) / c.patch[0]) * ((s.h + c.patch[1] - 1) / c.patch[1]) *
                               ((s.w + c.patch[2] - 1) / c.patch[2]);
        check(lp_dit_reserve(dit->handle(), tokens));
        b200::upload(z, zd.get());
        check(lp_dit_cfg_predict(dit->handle(), zd.get(), sh, E, timestep, guidance_scale, out.get(), nullptr));
        check_device_flags();
        return b200::download(s, z.dtype(), out.get());
    }
    // a host Denoiser: its two passes in the reference's order, the combine on the device
    const LatentTensor uncond = f.predict(z, timestep, ConditioningVector::null_like(cond));
    const LatentTensor conditioned = f.predict(z, timestep, cond);
    if (!uncond.same_layout(z) || !conditioned.same_layout(z)) {
        fail(ErrorKind::ShapeMismatch, "denoiser changed the tensor layout");
    }
    DeviceBuffer cd(bytes_of(s, z.dtype()));
    b200::upload(uncond, zd.get());
    b200::upload(conditioned, cd.get());
    check(lp_cfg_combine(zd.get(), cd.get(), s.volume(), E, guidance_scale, out.get(), nullptr));
    check_device_flags();
    return b200::download(s, z.dtype(), out.get());
}

// ---- sampler_step — src/denoise.cpp:41-52 ----
LatentTensor sampler_step(const LatentTensor& z, const LatentTensor& eps_hat, int /*timestep*/,
                          const SamplerConfig& cfg) {
    if (!z.same_layout(eps_hat)) {
        fail(ErrorKind::ShapeMismatch, "sampler_step: latent " + z.shape().str() + " vs prediction " +
                                           eps_hat.shape().str());
    }
    const Shape& s = z.shape();
    DeviceBuffer zd(bytes_of(s, z.dtype())), ed(bytes_of(s, z.dtype()));
    b200::upload(z, zd.get());
    b200::upload(eps_hat, ed.get());
    check(lp_sampler_step(zd.get(), ed.get(), s.volume(), dtype_bytes(z.dtype()), cfg.step_size, zd.get(), nullptr));
    check_device_flags();
    return b200::download(s, z.dtype(), zd.get());
}

// ---- the toy denoiser factories — src/denoise.cpp:144-154 ----
std::unique_ptr<Denoiser> make_box_denoiser(std::array<i64, 3> radius, double t_coeff, double cond_coeff) {
    return std::make_unique<b200::ToyDenoiser>(LP_TOY_BOX, radius, t_coeff, cond_coeff);
}
std::unique_ptr<Denoiser> make_global_mix_denoiser(double t_coeff, double cond_coeff) {
    return std::make_unique<b200::ToyDenoiser>(LP_TOY_GLOBAL, std::array<i64, 3>{0, 0, 0}, t_coeff, cond_coeff);
}
std::unique_ptr<Denoiser> make_identity_denoiser() {
    return std::make_unique<b200::ToyDenoiser>(LP_TOY_IDENTITY, std::array<i64, 3>{0, 0, 0}, 0.0, 0.0);
}

// ---- run_centralized — src/denoise.cpp:156-174 ----
DenoiseResult run_centralized(const Denoiser& f, const LatentTensor& z_init, const SamplerConfig& cfg,
                              const ConditioningVector& cond) {
    if (cfg.total_steps < 1) fail(ErrorKind::InvalidArgument, "total_steps must be >= 1");
    DenoiseResult result;
    result.trace.reserve(static_cast<size_t>(cfg.total_steps));
    lp_engine_config c;
    if (!cond.is_null && engine_config(f, z_init, cfg, PatchGeometry{1, 1, 1}, 1, 0.0, 2, c)) {
        // one worker over the whole latent (K=1, r=0): its plan is the identity, the loop is
        // cfg_predict + sampler_step (test_cluster.cpp:75-92 pins K=1 == centralized bitwise)
        Engine eng(c, cond);
        void* zd = eng.latent();
        b200::upload(z_init, zd);
        for (int i = 1; i <= cfg.total_steps; ++i) {
            check(lp_engine_run(eng.e, i, 1, nullptr));
            check_device_flags();
            result.trace.push_back(b200::download(z_init.shape(), z_init.dtype(), zd));
        }
        result.final_latent = result.trace.back();
        return result;
    }
    LatentTensor z = z_init;
    for (int i = 1; i <= cfg.total_steps; ++i) {
        const int t = cfg.total_steps + 1 - i;
        const LatentTensor eps = cfg_predict(f, z, t, cond, cfg.guidance_scale);
        z = sampler_step(z, eps, t, cfg);
        result.trace.push_back(z);
    }
    result.final_latent = std::move(z);
    return result;
}

// ---- run_lp — src/cluster.cpp:166-225 ----
LpRunResult run_lp(const Denoiser& f, const LatentTensor& z_init, const SamplerConfig& cfg,
                   const ConditioningVector& cond, const ClusterConfig& cluster) {
    validate_cluster(cluster);
    if (cfg.total_steps < 1) fail(ErrorKind::InvalidArgument, "total_steps must be >= 1");
    LpRunResult result{LatentTensor(), CommLedger(cluster.preset.dtype_bytes), {}};
    result.trace.reserve(static_cast<size_t>(cfg.total_steps));
    const Shape& shape = z_init.shape();
    const Dtype dtype = z_init.dtype();
    lp_engine_config c;
    if (engine_config(f, z_init, cfg, cluster.geometry, cluster.workers, cluster.overlap_ratio,
                      cluster.preset.dtype_bytes, c)) {
        // B200 denoisers: the whole step on the device (K1, fused CFG, K10 + sampler); the plan
        // and ledger of each step are the reference's own (build_plan, the run_lp metering)
        std::unique_ptr<Engine> eng;
        void* zd = nullptr;
        for (int i = 1; i <= cfg.total_steps; ++i) {
            const PartitionPlan plan = build_plan_for_shape(shape, cluster.geometry, i, cluster.workers,
                                                            cluster.overlap_ratio);
            meter_step(result.ledger, i, plan, shape);
            if (!eng) {
                if (cond.is_null)  // where the reference's first worker fails (src/denoise.cpp:26-28)
                    fail(ErrorKind::WorkerFailure,
                         "worker 1 failed at step 1: cfg_predict requires a non-null conditioning vector");
                eng = std::make_unique<Engine>(c, cond);
                zd = eng->latent();
                b200::upload(z_init, zd);
            }
            check(lp_engine_run(eng->e, i, 1, nullptr));
            check_device_flags();
            result.trace.push_back(b200::download(shape, dtype, zd));
        }
        uint64_t exchanged = 0, ledger_bytes = 0;
        check(lp_engine_comm(eng->e, &exchanged, &ledger_bytes));
        if (ledger_bytes != result.ledger.grand_total())
            fail(ErrorKind::InvalidArgument, "engine ledger disagrees with the reference metering");
        result.final_latent = result.trace.back();
        result.ledger.validate();
        return result;
    }
    // a host Denoiser: K1 and K10 on the device, the workers' cfg_predict on the host pool
    const int cap = worker_thread_cap();
    const int E = dtype_bytes(dtype);
    int64_t sh[4];
    shape_arr(shape, sh);
    DeviceBuffer zd(bytes_of(shape, dtype));
    b200::upload(z_init, zd.get());
    for (int i = 1; i <= cfg.total_steps; ++i) {
        const int t = cfg.total_steps + 1 - i;
        const PartitionPlan plan = build_plan_for_shape(shape, cluster.geometry, i, cluster.workers, cluster.overlap_ratio);
        const lp_plan pod = b200::to_pod(plan);
        const int k_eff = plan.workers();
        std::vector<int64_t> off(static_cast<size_t>(k_eff) + 1);
        check(lp_plan_offsets(&pod, sh, off.data()));
        DeviceBuffer subs_d(static_cast<size_t>(off.back()) * E);
        check(lp_extract(&pod, 0, k_eff, zd.get(), sh, E, subs_d.get(), nullptr));
        std::vector<uint8_t> bits(subs_d.bytes());
        check(lp_copy_to_host(bits.data(), subs_d.get(), bits.size()));
        std::vector<SimWorker> workers;
        std::vector<ScatterMessage> inbox;
        for (int k = 1; k <= k_eff; ++k) {
            workers.emplace_back(k, f);
            const Shape sk = shape.with_extent(plan.axis, plan.entries[static_cast<size_t>(k - 1)].latent.length());
            inbox.push_back(ScatterMessage{i, t, b200::from_bits(sk, dtype, bits.data() + off[static_cast<size_t>(k - 1)] * E),
                                           cond, cfg.guidance_scale});
        }
        for (Pass pass : {Pass::Cond, Pass::Uncond})
            for (int k = 2; k <= k_eff; ++k)
                result.ledger.add(i, pass, TransferKind::Scatter, 1, k,
                                  static_cast<std::uint64_t>(inbox[static_cast<size_t>(k - 1)].sub_latent.size()));
        std::vector<GatherMessage> outbox(static_cast<size_t>(k_eff));
        run_workers(workers, inbox, outbox, cap, i);
        for (Pass pass : {Pass::Cond, Pass::Uncond})
            for (int k = 2; k <= k_eff; ++k)
                result.ledger.add(i, pass, TransferKind::Gather, k, 1,
                                  static_cast<std::uint64_t>(outbox[static_cast<size_t>(k - 1)].prediction.size()));
        // contributions in worker order, blended and applied on the device (K10, exact)
        for (int k = 1; k <= k_eff; ++k) {
            const std::vector<uint8_t> b = b200::to_bits(outbox[static_cast<size_t>(k - 1)].prediction);
            std::copy(b.begin(), b.end(), bits.begin() + off[static_cast<size_t>(k - 1)] * E);
        }
        check(lp_copy_to_device(subs_d.get(), bits.data(), bits.size()));
        check(lp_reconstruct_update(&pod, subs_d.get(), sh, E, LP_MODE_EXACT, cfg.step_size, zd.get(), nullptr));
        check_device_flags();
        result.trace.push_back(b200::download(shape, dtype, zd.get()));
    }
    result.final_latent = result.trace.back();
    result.ledger.validate();
    return result;
}

}  // namespace lpsim
