// lp_host.hpp — host-side LP core (C++), the B200 engine's mirror of the
// reference's partition / reconstruct API (include/lpsim/partition.hpp:12-78,
// include/lpsim/reconstruct.hpp:12-33).  Same types and semantics; plans are
// PODs (lp_plan) so they can be handed to kernels by value.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "common.cuh"

namespace lpb200 {

using i64 = int64_t;

struct Range {
    i64 begin = 0, end = 0;
    i64 length() const { return end - begin; }
};

struct Shape4 {
    i64 c = 0, t = 0, h = 0, w = 0;
    i64 extent(int axis) const { return axis == 0 ? t : (axis == 1 ? h : w); }
    i64 volume() const { return c * t * h * w; }
    static Shape4 from(const int64_t s[4]) { return Shape4{s[0], s[1], s[2], s[3]}; }
    Shape4 with_extent(int axis, i64 v) const {
        Shape4 r = *this;
        (axis == 0 ? r.t : (axis == 1 ? r.h : r.w)) = v;
        return r;
    }
};

// outer x D x inner view of a latent along `axis` (src/latent.cpp:96-102).
inline void axis_view(const Shape4& s, int axis, i64& outer, i64& inner) {
    if (axis == 0) { outer = s.c; inner = s.h * s.w; }
    else if (axis == 1) { outer = s.c * s.t; inner = s.w; }
    else { outer = s.c * s.t * s.h; inner = 1; }
}

int rotation_axis(int step_index);                                        // partition.cpp:38-43
std::vector<Range> core_bounds(i64 patches, int workers);                  // partition.cpp:45-62
std::vector<Range> extend_overlap(const std::vector<Range>& cores, i64 patches, i64 per_core, double r,
                                  int workers);                            // partition.cpp:64-78
lp_plan build_axis_plan(int axis, i64 extent, i64 patch, int step, int workers, double r);  // :80-123
lp_plan build_plan_for_shape(const Shape4& s, const i64 patch[3], int step, int workers, double r);  // :125-129
std::vector<double> weight_profile(const lp_entry& e);                    // reconstruct.cpp:9-27

// Elements of each entry's sub-latent (worker order) and their prefix sums.
std::vector<i64> entry_elems(const lp_plan& p, const Shape4& s);
// Σ_k w_k(x) for every axis coordinate in worker order; ZeroWeight check
// (src/reconstruct.cpp:57-74).  Throws ZeroWeight.
std::vector<double> weight_sums(const lp_plan& p);

struct ShardLayout {
    std::vector<int> owned;      // entry ids (0-based) this rank computes, ascending
    i64 slot_elems = 0;          // padded per-rank slot of the all-gather buffer (multiple of 8 elements)
    std::vector<i64> base;       // per entry: element offset in the gathered buffer
    std::vector<int> owner;      // per entry: the rank that computes it
};
// Per-entry cost model of the balanced assignment: cost = lin*elems + quad*elems^2
// (the DiT: linear layers ~ tokens, self-attention ~ tokens^2).
struct AssignCost {
    double lin = 1.0, quad = 0.0;
};
// Entries -> ranks: round-robin (entry e -> rank e % world) when cost is null, else
// longest-processing-time greedy on the cost model (ties -> lowest rank).
ShardLayout shard_layout(const lp_plan& p, const Shape4& s, int world, int rank, const AssignCost* cost = nullptr);

void validate_plan(const lp_plan& p);
double host_quantize(double v, int dtype_bytes);

}  // namespace lpb200
