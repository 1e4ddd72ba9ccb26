// plugin_check.cpp — ctypes entry points for the integration tests (tests/test_integration_gpu.py).
//
// Linked two ways by integration/Makefile:
//   libb200_plugin.so — with the UNMODIFIED reference archive: the reference's own run_lp /
//                       run_centralized drive the B200 denoisers through the Denoiser slot;
//   libb200_dropin.so — with the weakened archive + b200_backend.cpp: the same calls land on the
//                       B200 hot path (the drop-in).
// Inputs/outputs are plain arrays of the reference's doubles.
#include <cstring>
#include <string>

#include "b200.hpp"
#include "lpsim/cluster.hpp"

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
        return 100;
    }
}

LatentTensor tensor(const double* z, const int64_t shape[4], int dtype_bytes_) {
    const Shape s{shape[0], shape[1], shape[2], shape[3]};
    return LatentTensor::from_doubles(s, dtype_from_bytes(dtype_bytes_),
                                      std::vector<double>(z, z + s.volume()));
}

ConditioningVector cond_of(const double* c, int n) {
    ConditioningVector v;
    v.values.assign(c, c + n);
    return v;
}

// denoiser: -1 = B200 DiT (dit_layers blocks), else box(radius)/global/identity via the
// reference's factories (overridden in the drop-in build).
std::unique_ptr<Denoiser> make(int denoiser, const int64_t radius[3], const ConditioningVector& cond, int dit_layers) {
    if (denoiser < 0) return b200::make_dit_denoiser(cond, dit_layers);
    if (denoiser == 0) return make_box_denoiser({radius[0], radius[1], radius[2]});
    if (denoiser == 1) return make_global_mix_denoiser();
    return make_identity_denoiser();
}
}  // namespace

extern "C" {

const char* check_last_error() { return g_err.c_str(); }

// run_lp (src/cluster.cpp:166-225) through whichever implementation this library links.
// trace_out: steps x volume doubles (or NULL); ledger_out: [grand_total, records];
// records_out: 7 x records uint64 (step, pass, kind, src, dst, elements, bytes) or NULL.
int check_run_lp(int denoiser, const int64_t radius[3], int dit_layers, const double* z, const int64_t shape[4],
                 int dtype_bytes_, int steps, double eta, double w, const double* cond, int n_cond,
                 const int64_t patch[3], int workers, double r, int wire_bytes, double* final_out, double* trace_out,
                 uint64_t* ledger_out, uint64_t* records_out, int64_t records_cap) {
    return guarded([&] {
        const ConditioningVector c = cond_of(cond, n_cond);
        const auto f = make(denoiser, radius, c, dit_layers);
        ClusterConfig cl;
        cl.workers = workers;
        cl.overlap_ratio = r;
        cl.geometry = PatchGeometry{patch[0], patch[1], patch[2]};
        cl.preset = ModelPreset{"check", 1536, wire_bytes, ""};
        const LpRunResult res = run_lp(*f, tensor(z, shape, dtype_bytes_), SamplerConfig{steps, eta, w}, c, cl);
        std::memcpy(final_out, res.final_latent.data().data(), res.final_latent.data().size() * sizeof(double));
        if (trace_out)
            for (size_t i = 0; i < res.trace.size(); ++i)
                std::memcpy(trace_out + i * res.final_latent.data().size(), res.trace[i].data().data(),
                            res.trace[i].data().size() * sizeof(double));
        const auto& recs = res.ledger.records();
        ledger_out[0] = res.ledger.grand_total();
        ledger_out[1] = recs.size();
        if (records_out)
            for (size_t i = 0; i < recs.size() && static_cast<int64_t>(i) < records_cap; ++i) {
                const CommRecord& q = recs[i];
                const uint64_t row[7] = {static_cast<uint64_t>(q.step), static_cast<uint64_t>(q.pass),
                                         static_cast<uint64_t>(q.kind), static_cast<uint64_t>(q.src),
                                         static_cast<uint64_t>(q.dst), q.elements, q.bytes};
                std::memcpy(records_out + 7 * i, row, sizeof(row));
            }
    });
}

// run_centralized (src/denoise.cpp:156-174).
int check_run_centralized(int denoiser, const int64_t radius[3], int dit_layers, const double* z,
                          const int64_t shape[4], int dtype_bytes_, int steps, double eta, double w, const double* cond,
                          int n_cond, double* final_out) {
    return guarded([&] {
        const ConditioningVector c = cond_of(cond, n_cond);
        const auto f = make(denoiser, radius, c, dit_layers);
        const DenoiseResult res = run_centralized(*f, tensor(z, shape, dtype_bytes_), SamplerConfig{steps, eta, w}, c);
        std::memcpy(final_out, res.final_latent.data().data(), res.final_latent.data().size() * sizeof(double));
    });
}

// One Denoiser::predict of the B200 DiT (null_text selects the uncond pass).
int check_dit_predict(int dit_layers, const double* z, const int64_t shape[4], int dtype_bytes_, int t,
                      const double* cond, int n_cond, int null_text, double* out) {
    return guarded([&] {
        const ConditioningVector c = cond_of(cond, n_cond);
        const auto f = b200::make_dit_denoiser(c, dit_layers);
        const LatentTensor p = f->predict(tensor(z, shape, dtype_bytes_), t,
                                          null_text ? ConditioningVector::null_like(c) : c);
        std::memcpy(out, p.data().data(), p.data().size() * sizeof(double));
    });
}

}  // extern "C"
