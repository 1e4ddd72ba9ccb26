// completeness.cpp — receptive-field (N-completeness) checker for axis schedules.
//
// Restates the reference's exhaustive reachability analysis
// (src/completeness.cpp:29-160, include/lpsim/completeness.hpp:8-92): every patch-grid
// position p carries the set R(p) of positions whose information has reached it; one
// denoising step under a plan fuses, for every partition block (its ext range along the
// plan axis, the full range elsewhere), the union of the PRE-step sets of the block's
// positions into every member.  A schedule is N-complete when every R(p) is the whole
// grid; min_steps[p] is the first step at which that happens.
//
// Layout: one bitset row of ceil(n/64) words per position.  A block's members are the
// positions whose plan-axis coordinate lies in [ext_begin, ext_end); since the grid is
// row-major (t, h, w), for the T axis they are one contiguous run of rows, for H they are
// nt runs of (ext_len * nw) rows, for W they are nt*nh runs of ext_len rows, so the
// union/broadcast walks runs instead of testing every position.
//
// The reference caps the analysis at 4096 positions (kMaxGridPositions) and rejects
// larger grids with InvalidArgument; `max_positions` = 0 keeps that cap, a larger value
// lifts it (the BASELINE C5 grid is 41 x 30 x 52 = 63,960 positions).
#include <cstring>
#include <vector>

#include "lp_host.hpp"

namespace lpb200 {

namespace {

constexpr i64 kRefMaxPositions = 4096;

struct Grid {
    i64 n[3];  // nt, nh, nw
    i64 size() const { return n[0] * n[1] * n[2]; }
};

// Calls f(first_row, count) for every contiguous run of grid rows whose `axis`
// coordinate lies in [b, e).
template <class F>
void for_runs(const Grid& g, int axis, i64 b, i64 e, F&& f) {
    const i64 nt = g.n[0], nh = g.n[1], nw = g.n[2];
    if (axis == 0) {
        f(b * nh * nw, (e - b) * nh * nw);
    } else if (axis == 1) {
        for (i64 t = 0; t < nt; ++t) f((t * nh + b) * nw, (e - b) * nw);
    } else {
        for (i64 t = 0; t < nt; ++t)
            for (i64 h = 0; h < nh; ++h) f((t * nh + h) * nw + b, e - b);
    }
}

struct Reach {
    Grid g;
    i64 words = 0;
    std::vector<uint64_t> bits;
    uint64_t* row(i64 p) { return bits.data() + p * words; }
    const uint64_t* row(i64 p) const { return bits.data() + p * words; }
    i64 count(i64 p) const {
        i64 c = 0;
        const uint64_t* r = row(p);
        for (i64 i = 0; i < words; ++i) c += __builtin_popcountll(r[i]);
        return c;
    }
};

Reach initial(const Grid& g, i64 cap) {
    if (g.n[0] < 1 || g.n[1] < 1 || g.n[2] < 1) fail(LP_ERR_INVALID_ARGUMENT, "grid dimensions must be >= 1");
    if (g.size() > cap)
        fail(LP_ERR_INVALID_ARGUMENT, "grid has " + std::to_string(g.size()) +
                                          " positions, exhaustive analysis is capped at " + std::to_string(cap));
    Reach r;
    r.g = g;
    const i64 n = g.size();
    r.words = (n + 63) / 64;
    r.bits.assign(static_cast<size_t>(n * r.words), 0);
    for (i64 p = 0; p < n; ++p) r.row(p)[p / 64] |= 1ull << (p % 64);
    return r;
}

// One propagation step (src/completeness.cpp:69-102): block unions over the pre-step sets.
Reach propagate(const Reach& r, const lp_plan& plan) {
    if (plan.axis_extent != r.g.n[plan.axis] || plan.patch_size != 1)
        fail(LP_ERR_SHAPE_MISMATCH, "plan is not at patch granularity for this grid");
    Reach out = r;
    std::vector<uint64_t> u(static_cast<size_t>(r.words));
    for (int k = 0; k < plan.n_entries; ++k) {
        const lp_entry& e = plan.entries[k];
        std::fill(u.begin(), u.end(), 0);
        for_runs(r.g, plan.axis, e.ext_begin, e.ext_end, [&](i64 p0, i64 cnt) {
            for (i64 p = p0; p < p0 + cnt; ++p) {
                const uint64_t* s = r.row(p);
                for (i64 i = 0; i < r.words; ++i) u[static_cast<size_t>(i)] |= s[i];
            }
        });
        for_runs(r.g, plan.axis, e.ext_begin, e.ext_end, [&](i64 p0, i64 cnt) {
            for (i64 p = p0; p < p0 + cnt; ++p) {
                uint64_t* d = out.row(p);
                for (i64 i = 0; i < r.words; ++i) d[i] |= u[static_cast<size_t>(i)];
            }
        });
    }
    return out;
}

}  // namespace

}  // namespace lpb200

using namespace lpb200;

extern "C" int lp_verify_n_complete(const int64_t grid[3], int32_t workers, double r, const int32_t* schedule,
                                    int32_t schedule_len, int32_t budget, int64_t max_positions, int32_t* complete,
                                    int32_t* complete_at, int64_t worst[3], int32_t* min_steps) {
    return guard([&] {
        if (budget < 1) fail(LP_ERR_INVALID_ARGUMENT, "step budget must be >= 1");
        if (schedule_len < budget) fail(LP_ERR_INVALID_ARGUMENT, "schedule is shorter than the step budget");
        for (int i = 0; i < budget; ++i)
            if (schedule[i] < 0 || schedule[i] > 2) fail(LP_ERR_INVALID_ARGUMENT, "schedule axes must be 0..2");
        const Grid g{{grid[0], grid[1], grid[2]}};
        Reach reach = initial(g, max_positions > 0 ? max_positions : kRefMaxPositions);
        const i64 n = g.size();
        std::vector<int32_t> ms(static_cast<size_t>(n), -1);
        if (n == 1) ms[0] = 0;
        for (int step = 1; step <= budget; ++step) {
            const int a = schedule[step - 1];
            const lp_plan plan = build_axis_plan(a, g.n[a], 1, step, workers, r);
            reach = propagate(reach, plan);
            bool pending = false;
            for (i64 p = 0; p < n; ++p) {
                if (ms[static_cast<size_t>(p)] >= 0) continue;
                if (reach.count(p) == n) ms[static_cast<size_t>(p)] = step;
                else pending = true;
            }
            if (!pending) break;
        }
        // worst position: the first never-complete one, else the first with the largest min_steps
        int worst_steps = -1;
        i64 wp = 0;
        bool all = true;
        for (i64 p = 0; p < n; ++p) {
            const int s = ms[static_cast<size_t>(p)];
            if (s < 0) {
                all = false;
                wp = p;
                break;
            }
            if (s > worst_steps) worst_steps = s, wp = p;
        }
        *complete = all ? 1 : 0;
        *complete_at = all ? worst_steps : -1;
        worst[0] = wp / (g.n[1] * g.n[2]);
        worst[1] = (wp / g.n[2]) % g.n[1];
        worst[2] = wp % g.n[2];
        if (min_steps) std::memcpy(min_steps, ms.data(), ms.size() * sizeof(int32_t));
    });
}

// Per-step coverage rows of the `completeness` command's coverage.csv
// (src/commands.cpp:169-195): step, min/mean/max reached, complete positions, total.
// Stops after the first step at which every position is complete.
extern "C" int lp_coverage_trace(const int64_t grid[3], int32_t workers, double r, const int32_t* schedule,
                                 int32_t schedule_len, int32_t budget, int64_t max_positions, int64_t* rows_i,
                                 double* rows_mean, int32_t* n_rows) {
    return guard([&] {
        if (schedule_len < budget) fail(LP_ERR_INVALID_ARGUMENT, "schedule is shorter than the step budget");
        const Grid g{{grid[0], grid[1], grid[2]}};
        Reach reach = initial(g, max_positions > 0 ? max_positions : kRefMaxPositions);
        const i64 n = g.size();
        int rows = 0;
        for (int step = 1; step <= budget; ++step) {
            const int a = schedule[step - 1];
            reach = propagate(reach, build_axis_plan(a, g.n[a], 1, step, workers, r));
            i64 mn = n, mx = 0, full = 0;
            double mean = 0.0;
            for (i64 p = 0; p < n; ++p) {
                const i64 c = reach.count(p);
                mn = std::min(mn, c);
                mx = std::max(mx, c);
                mean += static_cast<double>(c);
                if (c == n) ++full;
            }
            mean /= static_cast<double>(n);
            int64_t* row = rows_i + 5 * rows;
            row[0] = step, row[1] = mn, row[2] = mx, row[3] = full, row[4] = n;
            rows_mean[rows] = mean;
            ++rows;
            if (full == n) break;
        }
        *n_rows = rows;
    });
}
