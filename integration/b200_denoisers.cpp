// b200_denoisers.cpp — B200 denoisers behind the reference's Denoiser slot
// (include/lpsim/denoise.hpp:31-39) and the host<->device plumbing of the drop-in.
// Uses only the engine's C-ABI (include/lp_b200.h).
#include <cstring>
#include <string>

#include "b200.hpp"

namespace lpsim::b200 {

void check(int status) {
    if (status == LP_OK) return;
    const char* m = lp_last_error();
    const std::string msg = m ? m : "";
    if (status >= 1 && status <= 13) fail(static_cast<ErrorKind>(status - 1), msg);
    fail(ErrorKind::WorkerFailure, "B200 engine: " + msg);
}

void check_device_flags() {
    uint32_t flags = 0;
    check(lp_device_flags(&flags, 1));
    if (flags & 1u) fail(ErrorKind::NonFinite, "tensor element is not finite");  // src/latent.cpp:72-77
    if (flags & 2u) fail(ErrorKind::ZeroWeight, "weight sum < 1");
}

DeviceBuffer::DeviceBuffer(size_t bytes) : n_(bytes) { check(lp_device_alloc(bytes, &p_)); }
DeviceBuffer::~DeviceBuffer() {
    if (p_) lp_device_free(p_);
}

std::vector<uint8_t> to_bits(const LatentTensor& z) {
    const int E = dtype_bytes(z.dtype());
    const std::vector<double>& v = z.data();
    std::vector<uint8_t> out(v.size() * static_cast<size_t>(E));
    if (E == 8) {
        std::memcpy(out.data(), v.data(), out.size());
    } else if (E == 4) {  // values are already quantized to f32: the cast is exact
        for (size_t i = 0; i < v.size(); ++i) {
            const float f = static_cast<float>(v[i]);
            std::memcpy(out.data() + 4 * i, &f, 4);
        }
    } else {
        for (size_t i = 0; i < v.size(); ++i) {
            const uint16_t h = lp_f16_encode(v[i]);
            std::memcpy(out.data() + 2 * i, &h, 2);
        }
    }
    return out;
}

LatentTensor from_bits(const Shape& shape, Dtype dtype, const void* bits) {
    const int E = dtype_bytes(dtype);
    const size_t n = static_cast<size_t>(shape.volume());
    std::vector<double> v(n);
    const auto* b = static_cast<const uint8_t*>(bits);
    if (E == 8) {
        std::memcpy(v.data(), b, n * 8);
    } else if (E == 4) {
        for (size_t i = 0; i < n; ++i) {
            float f;
            std::memcpy(&f, b + 4 * i, 4);
            v[i] = f;
        }
    } else {
        for (size_t i = 0; i < n; ++i) {
            uint16_t h;
            std::memcpy(&h, b + 2 * i, 2);
            v[i] = lp_f16_decode(h);
        }
    }
    return LatentTensor::from_doubles(shape, dtype, std::move(v));  // exact: values are representable
}

void upload(const LatentTensor& z, void* dst) {
    const std::vector<uint8_t> bits = to_bits(z);
    check(lp_copy_to_device(dst, bits.data(), bits.size()));
}

LatentTensor download(const Shape& shape, Dtype dtype, const void* src) {
    std::vector<uint8_t> bits(static_cast<size_t>(shape.volume()) * dtype_bytes(dtype));
    check(lp_copy_to_host(bits.data(), src, bits.size()));
    return from_bits(shape, dtype, bits.data());
}

lp_plan to_pod(const PartitionPlan& plan) {
    if (plan.entries.size() > LP_MAX_WORKERS) fail(ErrorKind::InvalidArgument, "more than 256 plan entries");
    lp_plan p;
    std::memset(&p, 0, sizeof(p));
    p.axis = static_cast<int32_t>(plan.axis);
    p.step_index = plan.step_index;
    p.overlap_ratio = plan.overlap_ratio;
    p.patches_per_core = plan.patches_per_core;
    p.overlap_patches = plan.overlap_patches;
    p.axis_patches = plan.axis_patches;
    p.axis_extent = plan.axis_extent;
    p.patch_size = plan.patch_size;
    p.n_entries = static_cast<int32_t>(plan.entries.size());
    for (size_t k = 0; k < plan.entries.size(); ++k) {
        const PartitionEntry& e = plan.entries[k];
        lp_entry& d = p.entries[k];
        d.worker_id = e.worker_id;
        d.core_begin = e.core_patches.begin;
        d.core_end = e.core_patches.end;
        d.ext_begin = e.ext_patches.begin;
        d.ext_end = e.ext_patches.end;
        d.latent_begin = e.latent.begin;
        d.latent_end = e.latent.end;
        d.delta_start = e.delta_start;
        d.delta_end = e.delta_end;
    }
    return p;
}

static void shape_arr(const Shape& s, int64_t out[4]) {
    out[0] = s.c;
    out[1] = s.t;
    out[2] = s.h;
    out[3] = s.w;
}

// ---- toy denoisers (K11) ----
ToyDenoiser::ToyDenoiser(int kind, std::array<i64, 3> radius, double t_coeff, double cond_coeff)
    : kind_(kind), radius_(radius), t_coeff_(t_coeff), cond_coeff_(cond_coeff) {
    if (kind == LP_TOY_BOX)
        for (i64 r : radius_)
            if (r < 0) fail(ErrorKind::InvalidArgument, "box radius must be >= 0");  // src/denoise.cpp:59-61
}

LatentTensor ToyDenoiser::predict(const LatentTensor& z, int timestep, const ConditioningVector& cond) const {
    const Shape& s = z.shape();
    const size_t bytes = static_cast<size_t>(s.volume()) * dtype_bytes(z.dtype());
    DeviceBuffer in(bytes), out(bytes);
    upload(z, in.get());
    int64_t sh[4];
    shape_arr(s, sh);
    const int64_t rad[3] = {radius_[0], radius_[1], radius_[2]};
    check(lp_toy_predict(kind_, rad, t_coeff_, cond_coeff_, in.get(), sh, dtype_bytes(z.dtype()), timestep,
                         cond.mean(), out.get(), nullptr));
    check_device_flags();
    return download(s, z.dtype(), out.get());
}

ReceptiveRadius ToyDenoiser::receptive_radius() const {
    if (kind_ == LP_TOY_GLOBAL) return std::nullopt;
    if (kind_ == LP_TOY_IDENTITY) return std::array<i64, 3>{0, 0, 0};
    return radius_;
}

// ---- the DiT ----
DiTDenoiser::DiTDenoiser(const ConditioningVector& cond, int num_layers) : cond_(cond.values) {
    lp_dit_config c;
    lp_dit_default_config(&c);
    c.num_layers = num_layers;
    check(lp_dit_create(&c, cond_.data(), static_cast<int32_t>(cond_.size()), &dit_));
}

DiTDenoiser::~DiTDenoiser() {
    if (dit_) lp_dit_destroy(dit_);
}

LatentTensor DiTDenoiser::predict(const LatentTensor& z, int timestep, const ConditioningVector& cond) const {
    if (!cond.is_null && cond.values != cond_)
        fail(ErrorKind::InvalidArgument, "B200 DiT was created for another conditioning vector");
    const Shape& s = z.shape();
    lp_dit_config c;
    check(lp_dit_get_config(dit_, &c));
    const int64_t tokens = ((s.t + c.patch[0] - 1) / c.patch[0]) * ((s.h + c.patch[1] - 1) / c.patch[1]) *
                           ((s.w + c.patch[2] - 1) / c.patch[2]);
    std::lock_guard<std::mutex> lock(mu_);
    if (tokens > reserved_) {
        check(lp_dit_reserve(dit_, tokens));
        reserved_ = tokens;
    }
    const size_t bytes = static_cast<size_t>(s.volume()) * dtype_bytes(z.dtype());
    DeviceBuffer in(bytes), out(bytes);
    upload(z, in.get());
    int64_t sh[4];
    shape_arr(s, sh);
    check(lp_dit_predict(dit_, in.get(), sh, dtype_bytes(z.dtype()), timestep, cond.is_null ? 1 : 0, out.get(),
                         nullptr));
    check_device_flags();
    return download(s, z.dtype(), out.get());
}

std::unique_ptr<Denoiser> make_dit_denoiser(const ConditioningVector& cond, int num_layers) {
    return std::make_unique<DiTDenoiser>(cond, num_layers);
}

}  // namespace lpsim::b200
