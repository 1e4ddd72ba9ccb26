// recon.hpp — K10 launch parameters (shared by lp_kernels.cu and engine.cpp).
#pragma once
#include <vector>

#include "lp_host.hpp"

namespace lpb200 {

constexpr int kMaxKernelEntries = 64;
// One plan entry as K10 sees it: latent window [begin, begin+len) with
// ramps (ds, de) and the element offset of its prediction in the gather buffer.
struct ReconEntry {
    int64_t begin, len, ds, de, base;
};
// Division by a runtime-constant divisor d < 2^31 for dividends x < 2^31:
// q = (x * mul) >> shift with mul = ceil(2^(31+l) / d), l = ceil(log2 d), shift = 31 + l
// (Granlund–Montgomery: exact for every x < 2^31; mul < 2^32 + 1 fits in 64 bits).
struct FastDiv {
    uint64_t mul = 1;
    uint32_t shift = 0, d = 1;
};
FastDiv make_fastdiv(uint32_t d);

struct ReconParams {
    int n;
    int64_t D, outer, inner, total;
    double eta;
    FastDiv div_inner, div_d;  // valid (use32) when total < 2^31
    int use32;
    int mk;  // K10 exact division via the tabulated reciprocal (div_z; knob recon_mk)
    // peer exchange: the engine's failure word (non-zero = a peer's shard never arrived);
    // K10 then leaves z untouched instead of blending stale shards.  nullptr = no check.
    const unsigned* abort;
    // K10 coverage table owned by the caller (an engine builds one per axis with
    // recon_table_build and frees it at destroy); nullptr = the library's bounded cache
    const void* table;
    ReconEntry e[kMaxKernelEntries];
};
// The coverage table of p as an owned device allocation (cudaFree it), or nullptr when K10's
// coverage-table form does not apply to p.  Synchronizes `st`.
void* recon_table_build(const ReconParams& p, cudaStream_t st);

ReconParams make_recon_params(const lp_plan& plan, const Shape4& s, const std::vector<i64>& base, double eta);
void reconstruct_dispatch(const ReconParams& p, int dtype, const void* preds, void* z, void* eps, bool update,
                          bool fast, cudaStream_t st);
void slice_to(const void* z, const Shape4& s, int axis, i64 begin, i64 end, int E, void* dst, cudaStream_t st);
// K1 for several entries of one plan in one launch, packed in the order of ks.
void gather_entries(const void* z, const Shape4& s, const lp_plan& plan, const int* ks, int count, int E, void* dst,
                    cudaStream_t st);

// K9 over CUDA-IPC peer memory (engine exchange mode "peer").
constexpr int kMaxPeers = 16;
struct PeerPush {
    const uint8_t* local;                      // this rank's gather buffer (current parity)
    uint8_t* peer[kMaxPeers];                  // the peers' gather buffers (same parity)
    unsigned long long* peer_flag[kMaxPeers];  // &flags_of_peer[rank]
    uint64_t off, bytes;                       // this rank's slot
    // the exchange epoch lives on the device (so a CUDA graph of the step can be replayed):
    // the push kernel publishes *epoch + 1 and stores it back; the wait kernel waits for it
    unsigned long long* epoch;
    int npeers;
};
void peer_push(const PeerPush& pp, unsigned* counter, cudaStream_t st);
// status[0] |= 1 << j for every peer j whose flag did not reach `epoch` within the watchdog,
// status[1] = step (the engine reports WorkerFailure from it, src/cluster.cpp:149-161).
void peer_wait(const unsigned long long* flags, int world, int rank, const unsigned long long* epoch,
               unsigned* status, int step, cudaStream_t st);

}  // namespace lpb200
