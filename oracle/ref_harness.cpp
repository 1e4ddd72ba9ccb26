// ref_harness.cpp — TEST INFRASTRUCTURE (oracle side; never linked into the product).
//
// A thin extern "C" face over the UNMODIFIED reference library (lpsim, compiled by
// oracle/Makefile from /root/reference/proj/src/*.cpp into oracle/_ref/liblpsim_core.a)
// so that ctypes-based tests and the bench's `--impl reference` arm can call the
// reference's own per-stage functions: build_plan, build_weight_mask,
// extract_sublatents, Denoiser::predict, cfg_predict, reconstruct, sampler_step,
// run_lp, run_centralized, synthetic_inputs, quantize, cost_report.
// Nothing here re-implements the algorithm; it only marshals flat arrays.
//
// Plan flat encoding (shared with oracle/lp_oracle.h):
//   meta[8]     = {axis, step_index, L, O, N, D, p, n_entries}
//   entries[9n] = {k, core_b, core_e, ext_b, ext_e, lat_b, lat_e, delta_s, delta_e}

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "lpsim/cluster.hpp"
#include "lpsim/commands.hpp"
#include "lpsim/io.hpp"
#include "lpsim/completeness.hpp"
#include "lpsim/cost.hpp"
#include "lpsim/denoise.hpp"
#include "lpsim/dtype.hpp"
#include "lpsim/errors.hpp"
#include "lpsim/partition.hpp"
#include "lpsim/reconstruct.hpp"
#include "lpsim/run_config.hpp"

using namespace lpsim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return static_cast<int>(e.kind()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1000;
    }
}

Shape to_shape(const int64_t* s) { return Shape{s[0], s[1], s[2], s[3]}; }

LatentTensor to_tensor(const double* v, const int64_t* s, int dtype_bytes) {
    const Shape sh = to_shape(s);
    return LatentTensor::from_doubles(sh, dtype_from_bytes(dtype_bytes),
                                      std::vector<double>(v, v + sh.volume()));
}

void copy_out(const LatentTensor& z, double* out) {
    std::memcpy(out, z.data().data(), sizeof(double) * z.data().size());
}

void write_plan(const PartitionPlan& p, int64_t* meta, int64_t* entries) {
    meta[0] = static_cast<int64_t>(p.axis);
    meta[1] = p.step_index;
    meta[2] = p.patches_per_core;
    meta[3] = p.overlap_patches;
    meta[4] = p.axis_patches;
    meta[5] = p.axis_extent;
    meta[6] = p.patch_size;
    meta[7] = p.workers();
    for (size_t i = 0; i < p.entries.size(); ++i) {
        const PartitionEntry& e = p.entries[i];
        int64_t* o = entries + 9 * i;
        o[0] = e.worker_id;
        o[1] = e.core_patches.begin;
        o[2] = e.core_patches.end;
        o[3] = e.ext_patches.begin;
        o[4] = e.ext_patches.end;
        o[5] = e.latent.begin;
        o[6] = e.latent.end;
        o[7] = e.delta_start;
        o[8] = e.delta_end;
    }
}

std::unique_ptr<Denoiser> toy(int kind, const int64_t* radius) {
    switch (kind) {
        case 0: return make_box_denoiser({radius[0], radius[1], radius[2]});
        case 1: return make_global_mix_denoiser();
        case 2: return make_identity_denoiser();
    }
    fail(ErrorKind::InvalidArgument, "unknown toy kind");
}

ConditioningVector to_cond(const double* c, int n, int is_null) {
    ConditioningVector v;
    v.values.assign(c, c + n);
    v.is_null = is_null != 0;
    return v;
}

// A Denoiser whose predict is a C callback (used to wrap an external model,
// e.g. the fp32 DiT oracle, behind the reference's plugin slot).
typedef void (*ref_predict_fn)(const double* z, const int64_t* shape, int dtype_bytes, int timestep,
                               const double* cond, int n_cond, int is_null, double* out, void* user);

class CallbackDenoiser final : public Denoiser {
public:
    CallbackDenoiser(ref_predict_fn fn, void* user) : fn_(fn), user_(user) {}
    LatentTensor predict(const LatentTensor& z, int timestep, const ConditioningVector& cond) const override {
        const Shape& s = z.shape();
        const int64_t shape[4] = {s.c, s.t, s.h, s.w};
        std::vector<double> out(static_cast<size_t>(z.size()));
        fn_(z.data().data(), shape, dtype_bytes(z.dtype()), timestep, cond.values.data(),
            static_cast<int>(cond.values.size()), cond.is_null ? 1 : 0, out.data(), user_);
        return LatentTensor::from_doubles(s, z.dtype(), std::move(out));
    }
    ReceptiveRadius receptive_radius() const override { return std::nullopt; }

private:
    ref_predict_fn fn_;
    void* user_;
};

ClusterConfig make_cluster(const int64_t* patch, int workers, double r, int wire_bytes) {
    ClusterConfig c;
    c.workers = workers;
    c.overlap_ratio = r;
    c.geometry = PatchGeometry{patch[0], patch[1], patch[2]};
    c.preset = ModelPreset{"harness", 1536, wire_bytes, ""};
    return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_silence_warnings(int silence) {
    if (silence) set_warning_handler(nullptr);
}

int ref_rotation_axis(int step, int* axis) {
    return guarded([&] { *axis = static_cast<int>(rotation_axis(step)); });
}

int ref_core_bounds(int64_t n, int k, int64_t* out, int* count) {
    return guarded([&] {
        const auto c = core_bounds(n, k);
        *count = static_cast<int>(c.size());
        for (size_t i = 0; i < c.size(); ++i) {
            out[2 * i] = c[i].begin;
            out[2 * i + 1] = c[i].end;
        }
    });
}

int ref_extend_overlap(const int64_t* cores, int n_cores, int64_t patches, int64_t per_core, double r, int workers,
                       int64_t* out) {
    return guarded([&] {
        std::vector<Range> c;
        for (int i = 0; i < n_cores; ++i) c.push_back({cores[2 * i], cores[2 * i + 1]});
        const auto e = extend_overlap(c, patches, per_core, r, workers);
        for (size_t i = 0; i < e.size(); ++i) {
            out[2 * i] = e[i].begin;
            out[2 * i + 1] = e[i].end;
        }
    });
}

int ref_build_axis_plan(int axis, int64_t extent, int64_t patch, int step, int workers, double r, int64_t* meta,
                        int64_t* entries) {
    return guarded([&] {
        write_plan(build_axis_plan(static_cast<Axis>(axis), extent, patch, step, workers, r), meta, entries);
    });
}

int ref_build_plan(const int64_t* shape, const int64_t* patch, int step, int workers, double r, int64_t* meta,
                   int64_t* entries) {
    return guarded([&] {
        write_plan(build_plan_for_shape(to_shape(shape), PatchGeometry{patch[0], patch[1], patch[2]}, step,
                                        workers, r),
                   meta, entries);
    });
}

int ref_weight_profile(const int64_t* shape, const int64_t* patch, int step, int workers, double r, int entry,
                       double* out) {
    return guarded([&] {
        const auto p = build_plan_for_shape(to_shape(shape), PatchGeometry{patch[0], patch[1], patch[2]}, step,
                                            workers, r);
        const auto m = build_weight_mask(p.entries.at(static_cast<size_t>(entry)));
        std::memcpy(out, m.axis_profile.data(), sizeof(double) * m.axis_profile.size());
    });
}

// All sub-latents of the step's plan, packed in worker order.
int ref_extract(const double* z, const int64_t* shape, int dtype_bytes, const int64_t* patch, int step, int workers,
                double r, double* out) {
    return guarded([&] {
        const LatentTensor zt = to_tensor(z, shape, dtype_bytes);
        const auto p = build_plan(zt, PatchGeometry{patch[0], patch[1], patch[2]}, step, workers, r);
        size_t off = 0;
        for (const LatentTensor& s : extract_sublatents(zt, p)) {
            std::memcpy(out + off, s.data().data(), sizeof(double) * s.data().size());
            off += s.data().size();
        }
    });
}

int ref_toy_predict(int kind, const int64_t* radius, const double* z, const int64_t* shape, int dtype_bytes, int t,
                    const double* cond, int n_cond, int is_null, double* out) {
    return guarded([&] {
        copy_out(toy(kind, radius)->predict(to_tensor(z, shape, dtype_bytes), t, to_cond(cond, n_cond, is_null)),
                 out);
    });
}

int ref_cfg_predict(int kind, const int64_t* radius, const double* z, const int64_t* shape, int dtype_bytes, int t,
                    const double* cond, int n_cond, double w, double* out) {
    return guarded([&] {
        copy_out(cfg_predict(*toy(kind, radius), to_tensor(z, shape, dtype_bytes), t, to_cond(cond, n_cond, 0), w),
                 out);
    });
}

int ref_reconstruct(const double* preds, const int64_t* shape, int dtype_bytes, const int64_t* patch, int step,
                    int workers, double r, double* out) {
    return guarded([&] {
        const Shape full = to_shape(shape);
        const auto p = build_plan_for_shape(full, PatchGeometry{patch[0], patch[1], patch[2]}, step, workers, r);
        std::vector<LatentTensor> ps;
        size_t off = 0;
        for (const PartitionEntry& e : p.entries) {
            const Shape s = full.with_extent(p.axis, e.latent.length());
            ps.push_back(LatentTensor::from_doubles(s, dtype_from_bytes(dtype_bytes),
                                                    std::vector<double>(preds + off, preds + off + s.volume())));
            off += static_cast<size_t>(s.volume());
        }
        copy_out(reconstruct(ps, p, full), out);
    });
}

int ref_sampler_step(const double* z, const double* eps, const int64_t* shape, int dtype_bytes, double eta,
                     double* out) {
    return guarded([&] {
        SamplerConfig cfg{1, eta, 1.0};
        copy_out(sampler_step(to_tensor(z, shape, dtype_bytes), to_tensor(eps, shape, dtype_bytes), 1, cfg), out);
    });
}

// Full LP loop.  trace (optional) receives steps * volume doubles (z after each step).
static int run_lp_impl(const Denoiser& f, const double* z, const int64_t* shape, int dtype_bytes, int steps,
                       double eta, double w, const double* cond, int n_cond, const int64_t* patch, int workers,
                       double r, int wire_bytes, double* trace, double* final_out, uint64_t* ledger_total) {
    return guarded([&] {
        const SamplerConfig cfg{steps, eta, w};
        LpRunResult res = run_lp(f, to_tensor(z, shape, dtype_bytes), cfg, to_cond(cond, n_cond, 0),
                                 make_cluster(patch, workers, r, wire_bytes));
        copy_out(res.final_latent, final_out);
        if (trace) {
            size_t off = 0;
            for (const LatentTensor& s : res.trace) {
                copy_out(s, trace + off);
                off += s.data().size();
            }
        }
        if (ledger_total) *ledger_total = res.ledger.grand_total();
    });
}

int ref_run_lp(int kind, const int64_t* radius, const double* z, const int64_t* shape, int dtype_bytes, int steps,
               double eta, double w, const double* cond, int n_cond, const int64_t* patch, int workers, double r,
               int wire_bytes, double* trace, double* final_out, uint64_t* ledger_total) {
    std::unique_ptr<Denoiser> f;
    const int st = guarded([&] { f = toy(kind, radius); });
    if (st) return st;
    return run_lp_impl(*f, z, shape, dtype_bytes, steps, eta, w, cond, n_cond, patch, workers, r, wire_bytes, trace,
                       final_out, ledger_total);
}

int ref_run_lp_callback(ref_predict_fn fn, void* user, const double* z, const int64_t* shape, int dtype_bytes,
                        int steps, double eta, double w, const double* cond, int n_cond, const int64_t* patch,
                        int workers, double r, int wire_bytes, double* trace, double* final_out,
                        uint64_t* ledger_total) {
    CallbackDenoiser f(fn, user);
    return run_lp_impl(f, z, shape, dtype_bytes, steps, eta, w, cond, n_cond, patch, workers, r, wire_bytes, trace,
                       final_out, ledger_total);
}

int ref_run_centralized(int kind, const int64_t* radius, const double* z, const int64_t* shape, int dtype_bytes,
                        int steps, double eta, double w, const double* cond, int n_cond, double* trace,
                        double* final_out) {
    return guarded([&] {
        const SamplerConfig cfg{steps, eta, w};
        DenoiseResult res = run_centralized(*toy(kind, radius), to_tensor(z, shape, dtype_bytes), cfg,
                                            to_cond(cond, n_cond, 0));
        copy_out(res.final_latent, final_out);
        if (trace) {
            size_t off = 0;
            for (const LatentTensor& s : res.trace) {
                copy_out(s, trace + off);
                off += s.data().size();
            }
        }
    });
}

int ref_synthetic(const int64_t* shape, int dtype_bytes, uint64_t seed, double* z_out, double* cond_out) {
    return guarded([&] {
        SyntheticInputs in = synthetic_inputs(to_shape(shape), dtype_from_bytes(dtype_bytes), seed);
        copy_out(in.latent, z_out);
        std::memcpy(cond_out, in.cond.values.data(), sizeof(double) * in.cond.values.size());
    });
}

double ref_quantize(double v, int dtype_bytes) { return quantize(v, dtype_from_bytes(dtype_bytes)); }
uint16_t ref_f16_encode(double v) { return f16_encode(v); }
double ref_f16_decode(uint16_t b) { return f16_decode(b); }

// cost_report (src/cost.cpp:215-248): out[20] =
// {S_z, S_H, ext_mean, gamma, g_T, g_H, g_W, NMP, PP, LP_exact, LP_approx, ratio_exact, ratio_approx,
//  Sz/SH, has_hybrid, inter, intra, total, ratio_vs_nmp, bound, within}
int ref_cost(int steps, int workers, double r, const int64_t* shape, const int64_t* patch, int64_t hidden,
             int wire_bytes, int groups, const int* sizes, double* out) {
    return guarded([&] {
        CostInputs in;
        in.steps = steps;
        in.workers = workers;
        in.overlap_ratio = r;
        in.shape = to_shape(shape);
        in.geometry = PatchGeometry{patch[0], patch[1], patch[2]};
        in.preset = ModelPreset{"harness", hidden, wire_bytes, ""};
        if (groups > 0) in.hybrid = HybridSpec{groups, std::vector<int>(sizes, sizes + groups)};
        const CostReport rep = cost_report(in);
        const double v[] = {static_cast<double>(rep.latent_bytes), static_cast<double>(rep.activation_bytes),
                            rep.ext_bytes_mean, rep.gamma, rep.gamma_per_axis[0], rep.gamma_per_axis[1],
                            rep.gamma_per_axis[2], static_cast<double>(rep.nmp_bytes),
                            static_cast<double>(rep.pp_bytes), static_cast<double>(rep.lp_exact_bytes),
                            rep.lp_approx_bytes, rep.ratio_exact, rep.ratio_approx, rep.latent_activation_ratio,
                            rep.hybrid.has_value() ? 1.0 : 0.0,
                            rep.hybrid ? static_cast<double>(rep.hybrid->inter_bytes) : 0.0,
                            rep.hybrid ? static_cast<double>(rep.hybrid->intra_bytes) : 0.0,
                            rep.hybrid ? static_cast<double>(rep.hybrid->total_bytes) : 0.0,
                            rep.hybrid ? rep.hybrid->ratio_vs_nmp : 0.0, rep.hybrid ? rep.hybrid->bound : 0.0,
                            rep.hybrid ? (rep.hybrid->within_bound ? 1.0 : 0.0) : 0.0};
        std::memcpy(out, v, sizeof(v));
    });
}

// verify_n_complete (src/completeness.cpp:104-160) with an explicit axis schedule.
// out[5] = {complete, complete_at, worst_t, worst_h, worst_w}
int ref_verify_n_complete(const int64_t* grid, int workers, double r, const int* schedule, int len, int budget,
                          int64_t* out) {
    return guarded([&] {
        std::vector<Axis> sched;
        for (int i = 0; i < budget; ++i) sched.push_back(static_cast<Axis>(schedule[i % len]));
        const CompletenessResult res = verify_n_complete(GridDims{grid[0], grid[1], grid[2]}, workers, r, sched, budget);
        out[0] = res.complete ? 1 : 0;
        out[1] = res.complete_at;
        out[2] = res.worst.t;
        out[3] = res.worst.h;
        out[4] = res.worst.w;
    });
}

// The reference's command layer (src/commands.cpp:46-216) — what its CLI runs
// (tools/lpsim_main.cpp:95-104, which needs the absent CLI11): load_run_config + the
// command, artifacts written into out_dir, the returned summary as dump(2) into buf.
// seed < 0: keep the config's seed.  cmd: simulate | compare | cost | completeness | partition-plan.
int ref_command(const char* cmd, const char* config, const char* out_dir, int64_t seed, const char* schedule,
                int max_steps, int step, char* buf, int64_t cap) {
    return guarded([&] {
        RunConfig cfg = load_run_config(config);
        if (out_dir && *out_dir) cfg.output.dir = out_dir;
        if (seed >= 0) cfg.denoiser.seed = static_cast<std::uint64_t>(seed);
        const std::string c = cmd;
        nlohmann::json s;
        if (c == "simulate") s = simulate_run(cfg);
        else if (c == "compare") s = compare_run(cfg);
        else if (c == "cost") s = cost_run(cfg);
        else if (c == "completeness") s = completeness_run(cfg, schedule, max_steps);
        else s = partition_plan_run(cfg, step);
        const std::string d = s.dump(2);
        std::snprintf(buf, static_cast<size_t>(cap), "%s", d.c_str());
    });
}

// write_latent_dump / read_latent_dump (src/io.cpp:37-139) on doubles.
int ref_save_latent(const char* path, const double* v, const int64_t* shape, int dtype_bytes) {
    return guarded([&] { write_latent_dump(path, to_tensor(v, shape, dtype_bytes)); });
}
int ref_load_latent(const char* path, int64_t* shape_out, int* dtype_out, double* v_out) {
    return guarded([&] {
        const LatentTensor z = read_latent_dump(path);
        shape_out[0] = z.shape().c, shape_out[1] = z.shape().t, shape_out[2] = z.shape().h, shape_out[3] = z.shape().w;
        *dtype_out = dtype_bytes(z.dtype());
        if (v_out) copy_out(z, v_out);
    });
}

}  // extern "C"
