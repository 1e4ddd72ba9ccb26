// cost.cpp — the reference's communication cost model (src/cost.cpp:16-248),
// restated on top of this library's plan builder, so the engine can report its
// measured NCCL bytes beside the reference's LP / NMP / PP / hybrid accounting
// (BASELINE.json configs C2/C3: "comm bytes vs reference TP/PP accounting").
// Same formulas and the same order of double operations; compiled with
// -ffp-contract=off like the reference build.
#include <cmath>
#include <limits>

#include "lp_host.hpp"

namespace lpb200 {
namespace {

struct CostIn {
    int steps, workers;
    double r;
    Shape4 shape;
    i64 patch[3];
    i64 hidden;
    int wire;
};

i64 extent(const CostIn& in, int a) { return in.shape.extent(a); }
i64 patch_count(const CostIn& in, int a) {  // src/latent.cpp:148-159
    if (in.patch[a] < 1) fail(LP_ERR_INVALID_ARGUMENT, "patch size must be >= 1");
    if (extent(in, a) < in.patch[a]) fail(LP_ERR_DEGENERATE_AXIS, "axis extent < patch size");
    return extent(in, a) / in.patch[a];
}
uint64_t latent_bytes(const CostIn& in) { return static_cast<uint64_t>(in.shape.volume()) * in.wire; }
uint64_t activation_bytes(const CostIn& in) {
    i64 tok = 1;
    for (int a = 0; a < 3; ++a) tok *= patch_count(in, a);
    return static_cast<uint64_t>(tok) * static_cast<uint64_t>(in.hidden) * static_cast<uint64_t>(in.wire);
}
double expansion(const CostIn& in, int a, int workers) {  // src/cost.cpp:68-71
    const lp_plan p = build_axis_plan(a, extent(in, a), in.patch[a], 1, workers, in.r);
    i64 ext = 0;
    for (int k = 0; k < p.n_entries; ++k) ext += p.entries[k].latent_end - p.entries[k].latent_begin;
    return static_cast<double>(ext) / static_cast<double>(extent(in, a));
}
uint64_t lp_step_bytes(const CostIn& in, int a) {  // src/cost.cpp:46-55
    const lp_plan p = build_axis_plan(a, extent(in, a), in.patch[a], 1, in.workers, in.r);
    const i64 unit = in.shape.volume() / extent(in, a);
    uint64_t sum = 0;
    for (int k = 1; k < p.n_entries; ++k)
        sum += static_cast<uint64_t>((p.entries[k].latent_end - p.entries[k].latent_begin) * unit);
    return 4 * sum * static_cast<uint64_t>(in.wire);
}
uint64_t cost_nmp(const CostIn& in) {  // src/cost.cpp:73-77
    return 2ull * static_cast<uint64_t>(in.steps) * static_cast<uint64_t>(in.workers - 1) * activation_bytes(in);
}

}  // namespace
}  // namespace lpb200

using namespace lpb200;

extern "C" int lp_cost_report(int steps, int workers, double overlap_ratio, const int64_t shape[4],
                              const int64_t patch[3], int64_t hidden_dim, int wire_bytes, int hybrid_groups,
                              const int32_t* group_sizes, lp_cost_report_t* out) {
    return guard([&] {
        if (steps < 1) fail(LP_ERR_INVALID_ARGUMENT, "steps must be >= 1");
        if (workers < 1) fail(LP_ERR_INVALID_ARGUMENT, "workers must be >= 1");
        const CostIn in{steps, workers, overlap_ratio, Shape4::from(shape), {patch[0], patch[1], patch[2]}, hidden_dim,
                        wire_bytes};
        const double nan = std::numeric_limits<double>::quiet_NaN();
        lp_cost_report_t r{};
        r.latent_bytes = latent_bytes(in);
        r.activation_bytes = activation_bytes(in);
        double gmean = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double g = expansion(in, a, workers);
            r.gamma_per_axis[a] = g;
            gmean += g;
        }
        r.gamma = gmean / 3.0;
        r.ext_bytes_mean = r.gamma * static_cast<double>(r.latent_bytes);
        r.nmp_bytes = cost_nmp(in);
        r.pp_bytes = r.nmp_bytes;
        uint64_t per_axis[3];
        for (int a = 0; a < 3; ++a) per_axis[a] = lp_step_bytes(in, a);
        uint64_t exact = 0;
        for (int i = 1; i <= steps; ++i) exact += per_axis[rotation_axis(i)];
        r.lp_exact_bytes = exact;
        // cost_lp_approx (src/cost.cpp:96-110)
        const double s_z = static_cast<double>(r.latent_bytes);
        const double balance = static_cast<double>(workers - 1) / static_cast<double>(workers);
        double approx = 0.0;
        for (int i = 1; i <= steps; ++i) approx += 4.0 * balance * r.gamma_per_axis[rotation_axis(i)] * s_z;
        r.lp_approx_bytes = approx;
        r.latent_activation_ratio = static_cast<double>(r.latent_bytes) / static_cast<double>(r.activation_bytes);
        if (workers >= 2) {
            r.ratio_exact = static_cast<double>(r.lp_exact_bytes) / static_cast<double>(r.nmp_bytes);
            r.ratio_approx = (2.0 * r.gamma / static_cast<double>(workers)) * r.latent_activation_ratio;
        } else {
            r.ratio_exact = nan;
            r.ratio_approx = nan;
        }
        r.has_hybrid = hybrid_groups > 0;
        if (r.has_hybrid) {  // cost_hybrid (src/cost.cpp:133-213)
            const int M = hybrid_groups;
            if (M < 1 || M > workers) fail(LP_ERR_INVALID_GROUPING, "group count must be in [1, K]");
            int total = 0;
            for (int m = 0; m < M; ++m) {
                if (group_sizes[m] < 1) fail(LP_ERR_INVALID_GROUPING, "every group needs at least one worker");
                total += group_sizes[m];
            }
            if (total != workers) fail(LP_ERR_INVALID_GROUPING, "group sizes must sum to K");
            if (M == 1) {
                r.hybrid_inter_bytes = 0;
                r.hybrid_intra_bytes = 2ull * static_cast<uint64_t>(steps) * static_cast<uint64_t>(group_sizes[0] - 1) *
                                       activation_bytes(in);
            } else {
                uint64_t inter_step[3], intra_step[3];
                for (int a = 0; a < 3; ++a) {
                    const lp_plan p = build_axis_plan(a, extent(in, a), in.patch[a], 1, M, overlap_ratio);
                    const i64 unit = in.shape.volume() / extent(in, a);
                    uint64_t scatter = 0;
                    for (int m = 1; m < p.n_entries; ++m)
                        scatter += static_cast<uint64_t>((p.entries[m].latent_end - p.entries[m].latent_begin) * unit);
                    inter_step[a] = 4 * scatter * static_cast<uint64_t>(wire_bytes);
                    i64 other = 1;
                    for (int b = 0; b < 3; ++b)
                        if (b != a) other *= patch_count(in, b);
                    uint64_t intra = 0;
                    for (int m = 0; m < p.n_entries; ++m) {
                        const uint64_t tokens = static_cast<uint64_t>((p.entries[m].ext_end - p.entries[m].ext_begin) * other);
                        const uint64_t act = tokens * static_cast<uint64_t>(hidden_dim) * static_cast<uint64_t>(wire_bytes);
                        intra += 2ull * static_cast<uint64_t>(group_sizes[m] - 1) * act;
                    }
                    intra_step[a] = intra;
                }
                for (int i = 1; i <= steps; ++i) {
                    r.hybrid_inter_bytes += inter_step[rotation_axis(i)];
                    r.hybrid_intra_bytes += intra_step[rotation_axis(i)];
                }
            }
            r.hybrid_total_bytes = r.hybrid_inter_bytes + r.hybrid_intra_bytes;
            if (workers >= 2) {
                r.hybrid_ratio_vs_nmp = static_cast<double>(r.hybrid_total_bytes) / static_cast<double>(cost_nmp(in));
                r.hybrid_bound = M == 1 ? static_cast<double>(workers - 1) / static_cast<double>(workers - 1)
                                        : static_cast<double>(workers - M) / static_cast<double>(workers - 1);
                r.hybrid_within_bound = r.hybrid_ratio_vs_nmp < r.hybrid_bound;
            } else {
                r.hybrid_ratio_vs_nmp = nan;
                r.hybrid_bound = nan;
                r.hybrid_within_bound = 0;
            }
        }
        *out = r;
    });
}
