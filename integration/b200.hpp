// b200.hpp — the reference side of the drop-in (what a maintainer adds to lpsim).
//
// Compiled against the reference's own headers (/root/reference/proj/include) and the
// engine's C-ABI (include/lp_b200.h); nothing here includes CUDA headers.  Two link modes
// (integration/Makefile):
//   plugin  — b200_denoisers.cpp only: the B200 denoisers drop into the reference's Denoiser
//             slot (include/lpsim/denoise.hpp:31-39) and the UNMODIFIED reference run_lp /
//             run_centralized drive them;
//   drop-in — + b200_backend.cpp, whose definitions replace the reference's hot path at link
//             time (extract_sublatents, reconstruct, cfg_predict, sampler_step, the toy
//             denoiser factories, run_centralized, run_lp): the reference's archive is linked
//             with those symbols weakened, so every caller (commands, bindings, tests) runs
//             on the B200 engine.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "lp_b200.h"
#include "lpsim/denoise.hpp"
#include "lpsim/errors.hpp"
#include "lpsim/partition.hpp"

namespace lpsim::b200 {

// lp_status -> lpsim::Error (status = ErrorKind + 1; CUDA/NCCL failures are WorkerFailure).
void check(int status);
// Raises the reference's NonFinite / ZeroWeight for sticky device flags (synchronizes).
void check_device_flags();

// Owned device buffer (lp_device_alloc / lp_device_free).
class DeviceBuffer {
public:
    explicit DeviceBuffer(size_t bytes);
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    void* get() const { return p_; }
    size_t bytes() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

// LatentTensor (doubles holding storage-dtype values) <-> the storage bits the engine holds.
std::vector<uint8_t> to_bits(const LatentTensor& z);
LatentTensor from_bits(const Shape& shape, Dtype dtype, const void* bits);
void upload(const LatentTensor& z, void* dst);
LatentTensor download(const Shape& shape, Dtype dtype, const void* src);
// PartitionPlan (include/lpsim/partition.hpp:32-46) -> the engine's POD plan.
lp_plan to_pod(const PartitionPlan& plan);

// The reference's toy denoisers (src/denoise.cpp:56-142) computed by the engine's K11 kernels
// (fp64, the reference's summation order: bit-identical predictions).
class ToyDenoiser final : public Denoiser {
public:
    ToyDenoiser(int kind, std::array<i64, 3> radius, double t_coeff, double cond_coeff);
    LatentTensor predict(const LatentTensor& z, int timestep, const ConditioningVector& cond) const override;
    ReceptiveRadius receptive_radius() const override;
    int kind() const { return kind_; }
    const std::array<i64, 3>& radius() const { return radius_; }
    double t_coeff() const { return t_coeff_; }
    double cond_coeff() const { return cond_coeff_; }

private:
    int kind_;
    std::array<i64, 3> radius_;
    double t_coeff_, cond_coeff_;
};

// The WAN2.1-shaped tcgen05 DiT as a Denoiser.  predict() is ONE CFG pass on the GPU
// (lp_dit_predict): the null ConditioningVector selects the null text, any other must be the
// vector the DiT was created with (its synthetic text context is built from it).  Reentrant:
// concurrent predict() calls from the reference's worker pool are serialised on the device.
class DiTDenoiser final : public Denoiser {
public:
    explicit DiTDenoiser(const ConditioningVector& cond, int num_layers = 30);
    ~DiTDenoiser() override;
    LatentTensor predict(const LatentTensor& z, int timestep, const ConditioningVector& cond) const override;
    ReceptiveRadius receptive_radius() const override { return std::nullopt; }
    lp_dit* handle() const { return dit_; }
    const std::vector<double>& cond_values() const { return cond_; }

private:
    lp_dit* dit_ = nullptr;
    std::vector<double> cond_;
    mutable std::mutex mu_;
    mutable int64_t reserved_ = 0;
};

std::unique_ptr<Denoiser> make_dit_denoiser(const ConditioningVector& cond, int num_layers = 30);

}  // namespace lpsim::b200
