// engine.cpp — the run_lp step loop (src/cluster.cpp:166-225), B200-native.
//
// One engine per rank (one process per GPU).  Per step i (t = T+1-i):
//   1. plan for rotation_axis(i) — precomputed on the host at creation (the plan
//      depends only on the axis, src/partition.cpp:125-129), bit-exact;
//   2. K1 gathers each OWNED entry's window from the replicated latent z
//      (no scatter: every rank holds z);
//   3. the denoiser runs cfg_predict on it (DiT: CFG batch 2 in one forward),
//      writing ε̂_k straight into this rank's slot of the gather buffer;
//   4. world > 1: ONE ncclAllGather of the padded slots (latent shards only,
//      never DiT activations);
//   5. K10 blends all entries in worker order and applies the sampler update to
//      z in place, redundantly on every rank, so z stays replicated.
// Entries are assigned round-robin (entry e -> rank e % world), so world = 1
// runs all K workers' shards on one GPU ("K ranks on one GPU").
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "recon.hpp"

using namespace lpb200;

#define LP_NCCL(call)                                                                        \
    do {                                                                                     \
        ncclResult_t _r = (call);                                                            \
        if (_r != ncclSuccess) fail(LP_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(_r)); \
    } while (0)

struct lp_engine {
    lp_engine_config cfg{};
    Shape4 shape;
    std::vector<double> cond;
    double cond_mean = 0.0;
    lp_plan plans[3];
    ShardLayout layout[3];
    std::vector<i64> elems[3];
    ReconParams recon[3];
    void* z = nullptr;
    void* gather = nullptr;
    void* sub = nullptr;  // K1 output: the step's owned entries, packed in owned order
    double* ws = nullptr;
    // owned entries' DiT forwards overlap on nslots streams (world == 1: K shards on one GPU)
    int nslots = 1;
    cudaStream_t slot_stream[4] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[4] = {};
    ncclComm_t comm = nullptr;
    uint64_t nccl_bytes = 0, ledger_bytes = 0, launches = 0;
    // hybrid LP x model-parallel groups (group_size M > 1): this rank is pipeline stage
    // `stage` of LP group `group`, running DiT blocks [layer0, layer1)
    int M = 1, groups = 1, group = 0, stage = 0, layer0 = 0, layer1 = 0;
    uint64_t intra_bytes = 0;  // activation bytes this rank sent to the next stage
    // exchange over CUDA-IPC peer memory (lp_engine_ipc_attach): arena = 2 gather buffers
    // (epoch parity) + per-rank flag words + the push kernel's arrival counter
    uint8_t* arena = nullptr;
    // status block: {missing-peer mask, step} at +0, the device exchange epoch at +64
    size_t gather_bytes = 0, flags_off = 0, status_off = 0;
    bool peer = false;
    uint8_t* peer_arena[kMaxPeers + 1] = {};
    unsigned long long epoch = 0;
    uint64_t peer_bytes = 0;
    int last_step = 0;  // last step issued (failure attribution)
    // DiT engines replay each axis's step as a CUDA graph (captured the second time the
    // axis comes up, so every kernel's one-time setup has run eagerly first)
    // (peer-exchange engines: one graph per (axis, gather-buffer parity))
    cudaGraphExec_t graph[6] = {};
    uint64_t graph_kernels[6] = {};
    int seen[6] = {};
    cudaStream_t cap_stream = nullptr;  // capture happens here (the caller's stream may be the legacy default)
};

extern "C" {

int lp_nccl_unique_id(uint8_t id_out[128]) {
    return guard([&] {
        ncclUniqueId id;
        LP_NCCL(ncclGetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(id_out, &id, 128);
    });
}

int lp_engine_create(const lp_engine_config* c, const uint8_t* nccl_id, const double* cond, int32_t n_cond,
                     lp_engine** out) {
    return guard([&] {
        check_dtype(c->dtype_bytes);
        if (c->total_steps < 1) fail(LP_ERR_INVALID_ARGUMENT, "total_steps must be >= 1");
        if (c->workers < 1) fail(LP_ERR_INVALID_ARGUMENT, "cluster needs at least one worker");
        if (c->wire_bytes != 2 && c->wire_bytes != 4 && c->wire_bytes != 8)
            fail(LP_ERR_INVALID_ARGUMENT, "preset dtype_bytes must be 2, 4 or 8");
        if (c->world < 1 || c->rank < 0 || c->rank >= c->world) fail(LP_ERR_INVALID_ARGUMENT, "bad world/rank");
        if (c->denoiser < 0 && !c->dit) fail(LP_ERR_INVALID_ARGUMENT, "DiT engine without a DiT");
        if (c->schedule_len < 0 || c->schedule_len > 64) fail(LP_ERR_INVALID_ARGUMENT, "schedule_len must be 0..64");
        for (int i = 0; i < c->schedule_len; ++i)
            if (c->schedule[i] < 0 || c->schedule[i] > 2) fail(LP_ERR_INVALID_ARGUMENT, "schedule axes must be 0..2");
        auto* e = new lp_engine();
        e->cfg = *c;
        e->M = c->group_size > 1 ? c->group_size : 1;
        e->groups = c->world;  // plain LP: every rank is its own group
        if (e->M > 1) {
            if (c->world % e->M) { delete e; fail(LP_ERR_INVALID_GROUPING, "world must be a multiple of group_size"); }
            if (!c->dit) { delete e; fail(LP_ERR_INVALID_GROUPING, "hybrid groups need the DiT denoiser"); }
            int L = 0;
            {
                lp_dit_config dc;
                lp_dit_get_config(c->dit, &dc);
                L = dc.num_layers;
            }
            if (e->M > L) { delete e; fail(LP_ERR_INVALID_GROUPING, "more pipeline stages than DiT blocks"); }
            e->groups = c->world / e->M;
            e->group = c->rank / e->M;
            e->stage = c->rank % e->M;
            e->layer0 = static_cast<int>(static_cast<int64_t>(e->stage) * L / e->M);
            e->layer1 = static_cast<int>(static_cast<int64_t>(e->stage + 1) * L / e->M);
        }
        e->shape = Shape4::from(c->shape);
        e->cond.assign(cond, cond + n_cond);
        if (n_cond > 0) {  // ConditioningVector::mean (src/denoise.cpp:17-22)
            double acc = 0.0;
            for (double v : e->cond) acc += v;
            e->cond_mean = acc / static_cast<double>(n_cond);
        }
        try {
            if (c->assign != LP_ASSIGN_ROUND_ROBIN && c->assign != LP_ASSIGN_BALANCED)
                fail(LP_ERR_INVALID_ARGUMENT, "assign must be 0 (round-robin) or 1 (balanced)");
            AssignCost cost;  // toys: elements
            if (c->dit) {
                // DiT FLOPs per entry with n = elems / (C * patch volume) tokens, CFG batch 2:
                // linear 4 n (6 d^2 + 2 d F) + self-attention 8 n^2 d
                lp_dit_config dc;
                lp_dit_get_config(c->dit, &dc);
                const double per_tok = static_cast<double>(e->shape.c) * dc.patch[0] * dc.patch[1] * dc.patch[2];
                cost.lin = 4.0 * (6.0 * dc.dim * dc.dim + 2.0 * dc.dim * dc.ffn_dim) / per_tok;
                cost.quad = 8.0 * dc.dim / (per_tok * per_tok);
            }
            i64 max_slot = 0;
            for (int a = 0; a < 3; ++a) {
                // step index a+1 has axis a; step_index is cosmetic in the plan
                e->plans[a] = build_plan_for_shape(e->shape, c->patch, a + 1, c->workers, c->overlap_ratio);
                e->layout[a] = shard_layout(e->plans[a], e->shape, e->groups, e->M > 1 ? e->group : c->rank,
                                            c->assign == LP_ASSIGN_BALANCED ? &cost : nullptr);
                e->elems[a] = entry_elems(e->plans[a], e->shape);
                e->recon[a] = make_recon_params(e->plans[a], e->shape, e->layout[a].base, c->eta);
                e->recon[a].table = recon_table_build(e->recon[a], nullptr);  // owned: graphs embed it
                max_slot = std::max(max_slot, e->layout[a].slot_elems);
            }
            const size_t E = static_cast<size_t>(c->dtype_bytes);
            LP_CUDA(cudaMalloc(&e->z, static_cast<size_t>(e->shape.volume()) * E));
            e->gather_bytes = (static_cast<size_t>(max_slot) * e->groups * E + 255) / 256 * 256;
            e->flags_off = 2 * e->gather_bytes;
            e->status_off = e->flags_off + (static_cast<size_t>(c->world) * 8 + 8 + 255) / 256 * 256;
            const size_t arena = e->status_off + 256;
            LP_CUDA(cudaMalloc(&e->arena, arena));
            LP_CUDA(cudaMemset(e->arena, 0, arena));
            e->gather = e->arena;
            size_t max_owned = 1;
            for (int a = 0; a < 3; ++a) max_owned = std::max(max_owned, e->layout[a].owned.size());
            const int want_slots = std::max(1, std::min(4, tune_get("engine_slots", 2)));
            if (c->dit && max_owned > 1 && e->M == 1) e->nslots = static_cast<int>(std::min<size_t>(max_owned, want_slots));
            // K1 gathers every owned entry of a step in one launch, packed in owned order
            size_t max_owned_elems = 1;
            for (int a = 0; a < 3; ++a) {
                size_t tot = 0;
                for (int k : e->layout[a].owned) tot += static_cast<size_t>(e->elems[a][k]);
                max_owned_elems = std::max(max_owned_elems, tot);
            }
            LP_CUDA(cudaMalloc(&e->sub, max_owned_elems * E));
            LP_CUDA(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
            for (int s = 0; s < e->nslots; ++s) {
                LP_CUDA(cudaStreamCreateWithFlags(&e->slot_stream[s], cudaStreamNonBlocking));
                LP_CUDA(cudaEventCreateWithFlags(&e->ev_join[s], cudaEventDisableTiming));
            }
            LP_CUDA(cudaMalloc(&e->ws, lp_toy_workspace_bytes(c->shape) + 64));
            if (c->dit) {
                // workspace for the largest shard the DiT will see: tokens per entry with the DiT's
                // own patch and ceil division (remainder rows pad a partial patch), the count
                // lp_dit_cfg_predict_slot / lp_dit_forward_layers compute
                lp_dit_config dc;
                lp_dit_get_config(c->dit, &dc);
                i64 max_tokens = 0;
                for (int a = 0; a < 3; ++a)
                    for (int k = 0; k < e->plans[a].n_entries; ++k) {
                        const Shape4 s = e->shape.with_extent(a, e->plans[a].entries[k].latent_end -
                                                                     e->plans[a].entries[k].latent_begin);
                        const i64 nt = (s.t + dc.patch[0] - 1) / dc.patch[0], nh = (s.h + dc.patch[1] - 1) / dc.patch[1],
                                  nw = (s.w + dc.patch[2] - 1) / dc.patch[2];
                        max_tokens = std::max(max_tokens, nt * nh * nw);
                    }
                const int st = lp_dit_reserve_slots(c->dit, max_tokens, e->nslots);
                if (st) fail(st, lp_last_error());
            }
            // world > 1 always exchanges through NCCL; world == 1 does when an id is given
            // (a 1-rank communicator: exercises the exchange path on a single GPU)
            // world > 1 exchanges through NCCL when given an id (lp_engine_run), or through the
            // caller (lp_engine_step_phase + lp_engine_gather_buffer) without one; world == 1
            // with an id runs the NCCL exchange on a 1-rank communicator
            if (nccl_id) {
                ncclUniqueId id;
                std::memcpy(&id, nccl_id, 128);
                LP_NCCL(ncclCommInitRank(&e->comm, c->world, id, c->rank));
            }
        } catch (...) {
            lp_engine_destroy(e);
            throw;
        }
        *out = e;
    });
}

int lp_engine_destroy(lp_engine* e) {
    if (!e) return LP_OK;
    for (auto& g : e->graph)
        if (g) cudaGraphExecDestroy(g);
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
    if (e->comm) ncclCommDestroy(e->comm);
    cudaFree(e->z);
    for (auto* p : e->peer_arena)
        if (p) cudaIpcCloseMemHandle(p);
    cudaFree(e->arena);
    cudaFree(e->sub);
    for (int s = 0; s < 4; ++s) {
        if (e->slot_stream[s]) cudaStreamDestroy(e->slot_stream[s]);
        if (e->ev_join[s]) cudaEventDestroy(e->ev_join[s]);
    }
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    cudaFree(e->ws);
    for (auto& r : e->recon)
        if (r.table) cudaFree(const_cast<void*>(r.table));
    delete e;
    return LP_OK;
}

int lp_engine_latent(lp_engine* e, void** z) {
    *z = e->z;
    return LP_OK;
}

}  // extern "C"

namespace {

// Captured step graphs bake the exchange mode (peer stores, gather-buffer parity): drop them
// whenever the mode changes.
void reset_graphs(lp_engine* e) {
    for (int g = 0; g < 6; ++g) {
        if (e->graph[g]) cudaGraphExecDestroy(e->graph[g]);
        e->graph[g] = nullptr;
        e->graph_kernels[g] = 0;
        e->seen[g] = 0;
    }
}

int step_axis(const lp_engine* e, int i) {
    const lp_engine_config& c = e->cfg;
    if (i < 1 || i > c.total_steps) fail(LP_ERR_INVALID_ARGUMENT, "step out of range");
    return c.schedule_len > 0 ? c.schedule[(i - 1) % c.schedule_len] : rotation_axis(i);
}

// Phase 1 of step i (run_lp body, src/cluster.cpp:178-206): K1 + cfg_predict for every entry
// this rank owns, written into its slot of the gather buffer (owned shards overlap on the
// slot streams when there are several).
void hybrid_entry(lp_engine* e, int i, int idx, cudaStream_t st);

void step_compute(lp_engine* e, int i, cudaStream_t st) {
    if (e->M > 1) {
        const int n = static_cast<int>(e->layout[step_axis(e, i)].owned.size());
        for (int idx = 0; idx < n; ++idx) hybrid_entry(e, i, idx, st);
        return;
    }
    const lp_engine_config& c = e->cfg;
    const int E = c.dtype_bytes;
    char* gather = static_cast<char*>(e->gather);
    const int t = c.total_steps + 1 - i;
    const int a = step_axis(e, i);
    const lp_plan& plan = e->plans[a];
    const ShardLayout& L = e->layout[a];
    const bool fork = e->nslots > 1 && L.owned.size() > 1 && !tune_get("engine_serial", 0);
    // K1: one launch gathers all owned entries (packed in owned order) before the fork
    if (!L.owned.empty()) gather_entries(e->z, e->shape, plan, L.owned.data(), static_cast<int>(L.owned.size()), E, e->sub, st);
    if (fork) {
        LP_CUDA(cudaEventRecord(e->ev_fork, st));
        for (int s = 0; s < e->nslots; ++s) LP_CUDA(cudaStreamWaitEvent(e->slot_stream[s], e->ev_fork, 0));
    }
    size_t sub_off = 0;
    for (size_t idx = 0; idx < L.owned.size(); ++idx) {
        const int k = L.owned[idx];
        const int slot = fork ? static_cast<int>(idx % e->nslots) : 0;
        cudaStream_t ss = fork ? e->slot_stream[slot] : st;
        char* sub = static_cast<char*>(e->sub) + sub_off;
        sub_off += static_cast<size_t>(e->elems[a][k]) * E;
        const lp_entry& en = plan.entries[k];
        const Shape4 s = e->shape.with_extent(a, en.latent_end - en.latent_begin);
        void* eps = gather + static_cast<size_t>(L.base[k]) * E;
        const int64_t sh[4] = {s.c, s.t, s.h, s.w};
        int rc;
        if (c.denoiser < 0)
            rc = lp_dit_cfg_predict_slot(c.dit, slot, sub, sh, E, t, c.guidance, eps, ss);
        else
            rc = lp_toy_cfg_predict(c.denoiser, c.radius, c.t_coeff, c.cond_coeff, sub, sh, E, t, e->cond_mean,
                                    c.guidance, eps, e->ws, ss);
        if (rc)
            fail(LP_ERR_WORKER_FAILURE,
                 "worker " + std::to_string(k + 1) + " failed at step " + std::to_string(i) + ": " + lp_last_error());
    }
    if (fork) {
        for (int s = 0; s < e->nslots; ++s) {
            LP_CUDA(cudaEventRecord(e->ev_join[s], e->slot_stream[s]));
            LP_CUDA(cudaStreamWaitEvent(st, e->ev_join[s], 0));
        }
    }
}

// Hybrid LP x model-parallel groups: this rank's pipeline stage for the idx-th entry its
// group owns at step i.  Stage 0 gathers the group's entries (one K1 launch, at idx 0) and
// embeds; every stage runs its blocks; stages > 0 first receive the activation from rank-1,
// stages < M-1 send it to rank+1 afterwards (NCCL; without a communicator the caller moves
// it, lp_engine_stage_activation); the last stage writes ε̂ into the group's gather slot.
void hybrid_entry(lp_engine* e, int i, int idx, cudaStream_t st) {
    const lp_engine_config& c = e->cfg;
    const int E = c.dtype_bytes, t = c.total_steps + 1 - i, a = step_axis(e, i);
    const lp_plan& plan = e->plans[a];
    const ShardLayout& L = e->layout[a];
    if (idx < 0 || idx >= static_cast<int>(L.owned.size())) fail(LP_ERR_OUT_OF_BOUNDS, "owned entry index");
    if (e->stage == 0 && idx == 0)
        gather_entries(e->z, e->shape, plan, L.owned.data(), static_cast<int>(L.owned.size()), E, e->sub, st);  // K1
    size_t sub_off = 0;
    for (int j = 0; j < idx; ++j) sub_off += static_cast<size_t>(e->elems[a][L.owned[j]]) * E;
    const int k = L.owned[idx];
    const lp_entry& en = plan.entries[k];
    const Shape4 s = e->shape.with_extent(a, en.latent_end - en.latent_begin);
    const int64_t sh[4] = {s.c, s.t, s.h, s.w};
    void* x = nullptr;
    int64_t xb = 0;
    int rc = lp_dit_activation(c.dit, 0, sh, &x, &xb);
    if (rc) fail(rc, lp_last_error());
    if (e->stage > 0 && e->comm) {
        LP_NCCL(ncclRecv(x, static_cast<size_t>(xb), ncclUint8, c.rank - 1, e->comm, st));
        e->nccl_bytes += static_cast<uint64_t>(xb);
    }
    void* eps = static_cast<char*>(e->gather) + static_cast<size_t>(L.base[k]) * E;
    rc = lp_dit_forward_layers(c.dit, 0, e->stage == 0 ? static_cast<char*>(e->sub) + sub_off : nullptr, sh, E, t,
                               c.guidance, e->layer0, e->layer1, eps, st);
    if (rc)
        fail(LP_ERR_WORKER_FAILURE,
             "worker " + std::to_string(k + 1) + " failed at step " + std::to_string(i) + ": " + lp_last_error());
    if (e->stage < e->M - 1) {
        if (e->comm) LP_NCCL(ncclSend(x, static_cast<size_t>(xb), ncclUint8, c.rank + 1, e->comm, st));
        e->intra_bytes += static_cast<uint64_t>(xb);
    }
}

// Phase 2 (K9): one in-place ncclAllGather of the padded rank slots.
void step_exchange(lp_engine* e, int i, cudaStream_t st) {
    const lp_engine_config& c = e->cfg;
    const ShardLayout& L = e->layout[step_axis(e, i)];
    const size_t slot = static_cast<size_t>(L.slot_elems) * c.dtype_bytes;
    char* gather = static_cast<char*>(e->gather);
    prof_begin(KC_ALLGATHER, st);
    if (e->M == 1) {
        LP_NCCL(ncclAllGather(gather + slot * c.rank, gather, slot, ncclUint8, e->comm, st));
    } else {
        // hybrid: group g's ε̂ slot lives on its last stage (rank g*M + M-1)
        LP_NCCL(ncclGroupStart());
        for (int g = 0; g < e->groups; ++g)
            LP_NCCL(ncclBroadcast(gather + slot * g, gather + slot * g, slot, ncclUint8, g * e->M + e->M - 1, e->comm, st));
        LP_NCCL(ncclGroupEnd());
    }
    prof_end(KC_ALLGATHER, st, 0.0, static_cast<double>(slot) * (e->groups - 1));
}

// Phase 3 (K10): reconstruct + sampler update of the replicated z from the gathered shards,
// and the reference ledger's bytes for the step (src/cluster.cpp:186-209).
void step_reconstruct(lp_engine* e, int i, cudaStream_t st) {
    const lp_engine_config& c = e->cfg;
    const int a = step_axis(e, i);
    reconstruct_dispatch(e->recon[a], c.dtype_bytes, e->gather, e->z, nullptr, true, c.mode == LP_MODE_FAST, st);
}

// Host-side accounting of step i: NCCL bytes this rank receives and the reference ledger's
// bytes for the step (src/cluster.cpp:186-209).
void account_step(lp_engine* e, int i) {
    const lp_engine_config& c = e->cfg;
    const int a = step_axis(e, i);
    if (e->comm && !e->peer) {
        const int foreign = e->M == 1 ? c.world - 1 : e->groups - (e->stage == e->M - 1 ? 1 : 0);
        e->nccl_bytes += static_cast<size_t>(e->layout[a].slot_elems) * c.dtype_bytes * foreign;
    }
    uint64_t sum = 0;
    for (size_t k = 1; k < e->elems[a].size(); ++k) sum += static_cast<uint64_t>(e->elems[a][k]);
    e->ledger_bytes += 4ull * sum * static_cast<uint64_t>(c.wire_bytes);
}

// K9 over peer memory: push this rank's slot into every peer's buffer of the current parity,
// publish the epoch, wait for every peer's epoch (engine exchange mode "peer").
void step_exchange_peer(lp_engine* e, int i, cudaStream_t st, bool fused) {
    const lp_engine_config& c = e->cfg;
    const ShardLayout& L = e->layout[step_axis(e, i)];
    const size_t slot = static_cast<size_t>(L.slot_elems) * c.dtype_bytes;
    const size_t parity = static_cast<size_t>(e->epoch & 1) * e->gather_bytes;
    PeerPush pp{};
    pp.local = static_cast<const uint8_t*>(e->gather);
    for (int j = 0; j < c.world; ++j) {
        if (j == c.rank) continue;
        pp.peer[pp.npeers] = e->peer_arena[j] + parity;
        pp.peer_flag[pp.npeers] = reinterpret_cast<unsigned long long*>(e->peer_arena[j] + e->flags_off) + c.rank;
        ++pp.npeers;
    }
    pp.off = slot * static_cast<size_t>(c.rank);
    pp.bytes = fused ? 0 : slot;  // fused: the slot already went out with the DiT epilogue; signal only
    pp.epoch = reinterpret_cast<unsigned long long*>(e->arena + e->status_off + 64);
    prof_begin(KC_ALLGATHER, st);
    peer_push(pp, reinterpret_cast<unsigned*>(e->arena + e->flags_off + static_cast<size_t>(c.world) * 8), st);
    peer_wait(reinterpret_cast<const unsigned long long*>(e->arena + e->flags_off), c.world, c.rank, pp.epoch,
              reinterpret_cast<unsigned*>(e->arena + e->status_off), i, st);
    prof_end(KC_ALLGATHER, st, 0.0, static_cast<double>(slot) * (c.world - 1));
    e->peer_bytes += static_cast<uint64_t>(slot) * (c.world - 1);
}

void run_step_eager(lp_engine* e, int i, cudaStream_t st) {
    if (e->peer) {  // double-buffered gather by epoch parity
        ++e->epoch;
        e->gather = e->arena + static_cast<size_t>(e->epoch & 1) * e->gather_bytes;
    }
    const bool fused = e->peer && e->cfg.dit && tune_get("peer_fused", 1);
    if (fused) {  // K8+K9: the DiT epilogue stores ε̂ into every peer's buffer as it computes it
        std::vector<int64_t> deltas;
        for (int j = 0; j < e->cfg.world; ++j)
            if (j != e->cfg.rank) deltas.push_back(static_cast<int64_t>(e->peer_arena[j] - e->arena));
        const int rc = lp_dit_set_mirrors(e->cfg.dit, static_cast<int>(deltas.size()), deltas.data());
        if (rc) fail(rc, lp_last_error());
    }
    try {
        step_compute(e, i, st);
    } catch (...) {
        if (fused) lp_dit_set_mirrors(e->cfg.dit, 0, nullptr);
        throw;
    }
    if (fused) lp_dit_set_mirrors(e->cfg.dit, 0, nullptr);
    if (e->peer) step_exchange_peer(e, i, st, fused);
    else if (e->comm) step_exchange(e, i, st);
    step_reconstruct(e, i, st);
}

// One step of a DiT engine as a graph replay: write the timestep into every slot's device
// scalar, then launch the axis's graph (captured on the second occurrence of the axis).
void run_step_graph(lp_engine* e, int i, cudaStream_t st) {
    const lp_engine_config& c = e->cfg;
    const int a = step_axis(e, i);
    const int t = c.total_steps + 1 - i;
    const int par = e->peer ? static_cast<int>((e->epoch + 1) & 1) : 0;  // the parity this step will use
    const int g_ix = 2 * a + par;
    if (++e->seen[g_ix] < 2 && !e->graph[g_ix]) {
        run_step_eager(e, i, st);
        return;
    }
    for (int s = 0; s < e->nslots; ++s) {
        const int rc = lp_dit_set_time(c.dit, s, t, st);
        if (rc) fail(rc, lp_last_error());
    }
    if (!e->graph[g_ix]) {
        lp_dit_time_on_device(c.dit, 1);
        const uint64_t l0 = launch_count();
        cudaGraph_t g = nullptr;
        if (!e->cap_stream) LP_CUDA(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
        cudaStream_t cs = e->cap_stream;
        LP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        try {
            run_step_eager(e, i, cs);
        } catch (...) {
            cudaStreamEndCapture(cs, &g);
            if (g) cudaGraphDestroy(g);
            lp_dit_time_on_device(c.dit, 0);
            throw;
        }
        LP_CUDA(cudaStreamEndCapture(cs, &g));
        lp_dit_time_on_device(c.dit, 0);
        e->graph_kernels[g_ix] = launch_count() - l0;
        const cudaError_t err = cudaGraphInstantiate(&e->graph[g_ix], g, 0);
        cudaGraphDestroy(g);
        LP_CUDA(err);
    } else {
        count_launch(e->graph_kernels[g_ix]);  // the replay runs the captured kernels again
        if (e->peer) {  // the host side of run_step_eager / step_exchange_peer for the replayed step
            ++e->epoch;
            e->gather = e->arena + static_cast<size_t>(e->epoch & 1) * e->gather_bytes;
            e->peer_bytes += static_cast<uint64_t>(e->layout[a].slot_elems) * c.dtype_bytes * (c.world - 1);
        }
    }
    LP_CUDA(cudaGraphLaunch(e->graph[g_ix], st));
}

}  // namespace

extern "C" {

int lp_engine_run(lp_engine* e, int32_t first, int32_t count, void* stream) {
    return guard([&] {
        cudaStream_t st = as_stream(stream);
        if (e->cfg.world > 1 && !e->comm && !e->peer)
            fail(LP_ERR_INVALID_ARGUMENT,
                 "world > 1 without an NCCL id or peer attach: drive the steps with lp_engine_step_phase and an "
                 "external exchange");
        const uint64_t l0 = launch_count();
        // graphs: DiT engines, on a stream that can be captured, unless per-launch profiling
        // or the serialised debug mode is on (both need the eager launches)
        // (NCCL-exchange engines stay eager: their step holds an ncclAllGather; the peer
        // exchange is plain kernels on device memory, so its steps are captured too, one graph
        // per (axis, gather-buffer parity), with the exchange epoch kept on the device)
        const bool graphs = e->cfg.dit != nullptr && (e->peer || e->comm == nullptr) && e->M == 1 &&
                            tune_get("engine_graph", 1) && !prof_enabled() && !tune_get("engine_serial", 0);
        for (int i = first; i < first + count; ++i) {
            e->last_step = i;
            if (graphs) run_step_graph(e, i, st);
            else run_step_eager(e, i, st);
            account_step(e, i);
        }
        e->launches += launch_count() - l0;
    });
}

int lp_engine_step_phase(lp_engine* e, int32_t step, int32_t phase, void* stream) {
    return guard([&] {
        cudaStream_t st = as_stream(stream);
        const uint64_t l0 = launch_count();
        if (e->peer) fail(LP_ERR_INVALID_ARGUMENT, "peer-attached engines exchange inside lp_engine_run");
        if (phase == 1) {
            if (e->M > 1 && !e->comm)
                fail(LP_ERR_INVALID_GROUPING, "hybrid engine without NCCL: drive its stages with lp_engine_stage");
            step_compute(e, step, st);
        }
        else if (phase == 2) {
            if (e->comm) step_exchange(e, step, st);
        } else if (phase == 3) {
            step_reconstruct(e, step, st);
            account_step(e, step);
        }
        else fail(LP_ERR_INVALID_ARGUMENT, "phase must be 1 (compute), 2 (exchange) or 3 (reconstruct)");
        e->launches += launch_count() - l0;
    });
}

int lp_engine_stage(lp_engine* e, int32_t step, int32_t idx, void* stream) {
    return guard([&] {
        if (e->M < 2) fail(LP_ERR_INVALID_GROUPING, "lp_engine_stage needs group_size > 1");
        const uint64_t l0 = launch_count();
        hybrid_entry(e, step, idx, as_stream(stream));
        e->launches += launch_count() - l0;
    });
}

int lp_engine_stage_activation(lp_engine* e, int32_t step, int32_t idx, void** x, int64_t* bytes) {
    return guard([&] {
        const int a = step_axis(e, step);
        const ShardLayout& L = e->layout[a];
        if (idx < 0 || idx >= static_cast<int>(L.owned.size())) fail(LP_ERR_OUT_OF_BOUNDS, "owned entry index");
        const lp_entry& en = e->plans[a].entries[L.owned[idx]];
        const Shape4 s = e->shape.with_extent(a, en.latent_end - en.latent_begin);
        const int64_t sh[4] = {s.c, s.t, s.h, s.w};
        const int rc = lp_dit_activation(e->cfg.dit, 0, sh, x, bytes);
        if (rc) fail(rc, lp_last_error());
    });
}

int lp_engine_hybrid(const lp_engine* e, int32_t* group_size, int32_t* group, int32_t* stage, int32_t* layer_begin,
                     int32_t* layer_end, uint64_t* intra_bytes) {
    *group_size = e->M;
    *group = e->group;
    *stage = e->stage;
    *layer_begin = e->layer0;
    *layer_end = e->layer1;
    *intra_bytes = e->intra_bytes;
    return LP_OK;
}

int lp_engine_owned(const lp_engine* e, int32_t step, int32_t* n_owned) {
    *n_owned = static_cast<int32_t>(e->layout[step_axis(e, step)].owned.size());
    return LP_OK;
}

int lp_engine_gather_buffer(const lp_engine* e, int32_t step, void** buffer, int64_t* slot_elems) {
    return guard([&] {
        *buffer = e->gather;
        *slot_elems = e->layout[step_axis(e, step)].slot_elems;
    });
}

int lp_engine_ipc_handle(lp_engine* e, uint8_t handle_out[64]) {
    return guard([&] {
        cudaIpcMemHandle_t h;
        LP_CUDA(cudaIpcGetMemHandle(&h, e->arena));
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
        std::memcpy(handle_out, &h, 64);
    });
}

int lp_engine_ipc_attach(lp_engine* e, const uint8_t* handles) {
    return guard([&] {
        const lp_engine_config& c = e->cfg;
        if (e->M > 1) fail(LP_ERR_INVALID_GROUPING, "peer exchange is for plain LP engines (group_size 1)");
        if (c.world < 2 || c.world > kMaxPeers + 1) fail(LP_ERR_INVALID_ARGUMENT, "peer exchange needs 2..17 ranks");
        for (int j = 0; j < c.world; ++j) {
            if (j == c.rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + 64 * static_cast<size_t>(j), 64);
            void* p = nullptr;
            LP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            e->peer_arena[j] = static_cast<uint8_t*>(p);
        }
        reset_graphs(e);
        e->peer = true;  // takes precedence over an NCCL communicator for the ε̂ exchange
        for (auto& r : e->recon) r.abort = reinterpret_cast<const unsigned*>(e->arena + e->status_off);
    });
}

int lp_engine_ipc_detach(lp_engine* e) {
    return guard([&] {
        for (auto*& p : e->peer_arena)
            if (p) {
                LP_CUDA(cudaIpcCloseMemHandle(p));
                p = nullptr;
            }
        reset_graphs(e);
        e->peer = false;
        e->gather = e->arena;
        for (auto& r : e->recon) r.abort = nullptr;
    });
}

// Failure attribution in the reference's terms: "worker k failed at step i: ..." with k the
// lowest failing worker id (src/cluster.cpp:149-161); a dead rank fails every entry it owns.
static std::string failed_workers(const lp_engine* e, unsigned rank_mask, int step) {
    const int a = step >= 1 && step <= e->cfg.total_steps ? step_axis(e, step) : 0;
    const ShardLayout& L = e->layout[a];
    int worst = -1, rank = -1;
    for (size_t k = 0; k < L.owner.size(); ++k)
        if ((rank_mask >> L.owner[k]) & 1u) {
            worst = static_cast<int>(k) + 1;
            rank = L.owner[k];
            break;
        }
    if (worst < 0) {  // the rank owned no entry at this step
        for (int r = 0; r < 32; ++r)
            if ((rank_mask >> r) & 1u) { rank = r; break; }
        return "rank " + std::to_string(rank) + " failed at step " + std::to_string(step);
    }
    return "worker " + std::to_string(worst) + " failed at step " + std::to_string(step) + ": rank " +
           std::to_string(rank);
}

int lp_engine_sync(lp_engine* e, void* stream, int64_t timeout_ms) {
    return guard([&] {
        cudaStream_t st = as_stream(stream);
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t q = cudaStreamQuery(st);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) fail(LP_ERR_CUDA, std::string("step ") + std::to_string(e->last_step) + ": " + cudaGetErrorString(q));
            if (e->comm) {
                ncclResult_t r = ncclSuccess;
                ncclCommGetAsyncError(e->comm, &r);
                if (r != ncclSuccess && r != ncclInProgress) {
                    const std::string why = ncclGetErrorString(r);
                    ncclCommAbort(e->comm);
                    e->comm = nullptr;
                    fail(LP_ERR_WORKER_FAILURE, "step " + std::to_string(e->last_step) + ": NCCL exchange failed: " + why);
                }
            }
            const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
            if (timeout_ms > 0 && ms > timeout_ms) {
                if (e->comm) {  // unblocks the stuck collective so the stream can drain
                    ncclCommAbort(e->comm);
                    e->comm = nullptr;
                }
                fail(LP_ERR_WORKER_FAILURE, "step " + std::to_string(e->last_step) + ": the step did not complete within " +
                                                std::to_string(timeout_ms) + " ms (a peer rank is dead or stalled)");
            }
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
        if (e->peer) {
            unsigned status[2] = {0, 0};
            LP_CUDA(cudaMemcpy(status, e->arena + e->status_off, sizeof(status), cudaMemcpyDeviceToHost));
            if (status[0]) {
                LP_CUDA(cudaMemset(e->arena + e->status_off, 0, sizeof(status)));
                fail(LP_ERR_WORKER_FAILURE, failed_workers(e, status[0], static_cast<int>(status[1])) +
                                                ": its epsilon shard never arrived over the peer exchange (watchdog); "
                                                "z was left at the previous step");
            }
        }
    });
}

int lp_engine_exchange_bench(lp_engine* e, int32_t step, int32_t iters, void* stream, double* ms_out,
                             uint64_t* bytes_out) {
    return guard([&] {
        if (!e->peer && !e->comm) fail(LP_ERR_INVALID_ARGUMENT, "exchange bench needs a peer attach or an NCCL communicator");
        if (e->M > 1) fail(LP_ERR_INVALID_GROUPING, "exchange bench is for plain LP engines");
        if (iters < 1) fail(LP_ERR_INVALID_ARGUMENT, "iters must be >= 1");
        cudaStream_t st = as_stream(stream);
        const uint64_t pb = e->peer_bytes;
        cudaEvent_t a = nullptr, b = nullptr;
        LP_CUDA(cudaEventCreate(&a));
        LP_CUDA(cudaEventCreate(&b));
        LP_CUDA(cudaEventRecord(a, st));
        for (int it = 0; it < iters; ++it) {
            if (e->peer) {  // the unfused push (copy + signal + wait) of the step's full slot
                ++e->epoch;
                e->gather = e->arena + static_cast<size_t>(e->epoch & 1) * e->gather_bytes;
                step_exchange_peer(e, step, st, false);
            } else {
                step_exchange(e, step, st);
            }
        }
        LP_CUDA(cudaEventRecord(b, st));
        LP_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        LP_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        e->peer_bytes = pb;
        const ShardLayout& L = e->layout[step_axis(e, step)];
        *ms_out = ms;
        *bytes_out = static_cast<uint64_t>(L.slot_elems) * e->cfg.dtype_bytes * (e->cfg.world - 1) * iters;
    });
}

int lp_engine_hbm_bench(lp_engine* e, int32_t step, int32_t iters, int32_t sets, void* stream, double out[4]) {
    return guard([&] {
        if (iters < 1 || sets < 1) fail(LP_ERR_INVALID_ARGUMENT, "iters and sets must be >= 1");
        if (e->M > 1) fail(LP_ERR_INVALID_GROUPING, "hbm bench is for plain LP engines");
        cudaStream_t st = as_stream(stream);
        const lp_engine_config& c = e->cfg;
        const int a = step_axis(e, step), E = c.dtype_bytes;
        const lp_plan& plan = e->plans[a];
        const ShardLayout& L = e->layout[a];
        const size_t zb = static_cast<size_t>(e->shape.volume()) * E;
        size_t subb = 0, predb = 0;
        for (int k : L.owned) subb += static_cast<size_t>(e->elems[a][k]) * E;
        for (size_t k = 0; k < e->elems[a].size(); ++k) predb += static_cast<size_t>(e->elems[a][k]) * E;
        const size_t gb = static_cast<size_t>(L.slot_elems) * E * c.world;
        const size_t zs = (zb + 255) / 256 * 256, ss = (subb + 255) / 256 * 256, gs = (gb + 255) / 256 * 256;
        // `sets` private copies of (z, sub, gather), used round robin, so with enough sets the
        // working set of consecutive launches exceeds L2 and every launch streams from HBM
        uint8_t* buf = nullptr;
        LP_CUDA(cudaMalloc(&buf, (zs + ss + gs) * static_cast<size_t>(sets)));
        auto zp = [&](int s) { return buf + static_cast<size_t>(s) * (zs + ss + gs); };
        for (int s = 0; s < sets; ++s) {
            LP_CUDA(cudaMemcpyAsync(zp(s), e->z, zb, cudaMemcpyDeviceToDevice, st));
            LP_CUDA(cudaMemcpyAsync(zp(s) + zs + ss, e->gather, gb, cudaMemcpyDeviceToDevice, st));
        }
        cudaEvent_t ev[3] = {};
        for (auto& x : ev) LP_CUDA(cudaEventCreate(&x));
        auto k1 = [&](int s, cudaStream_t q) {
            if (!L.owned.empty())
                gather_entries(zp(s), e->shape, plan, L.owned.data(), static_cast<int>(L.owned.size()), E, zp(s) + zs, q);
        };
        auto k10 = [&](int s, cudaStream_t q) {
            reconstruct_dispatch(e->recon[a], E, zp(s) + zs + ss, zp(s), nullptr, true, c.mode == LP_MODE_FAST, q);
        };
        for (int s = 0; s < sets; ++s) { k1(s, st); k10(s, st); }  // warm-up (and K10's coverage table)
        LP_CUDA(cudaStreamSynchronize(st));
        // each loop of `iters` launches replays as ONE CUDA graph: no host launch gaps between
        // these few-us kernels (eager launches from the host loop would time the launch rate)
        cudaStream_t cs = nullptr;
        LP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        const bool prof = prof_enabled();
        if (prof) lp_profile_enable(0);  // no profiling events inside the captured loops
        auto capture = [&](auto body) {
            cudaGraph_t g = nullptr;
            cudaGraphExec_t x = nullptr;
            LP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            for (int it = 0; it < iters; ++it) body(it % sets, cs);
            LP_CUDA(cudaStreamEndCapture(cs, &g));
            LP_CUDA(cudaGraphInstantiate(&x, g, 0));
            cudaGraphDestroy(g);
            return x;
        };
        cudaGraphExec_t g1 = capture(k1), g10 = capture(k10);
        if (prof) lp_profile_enable(1);
        LP_CUDA(cudaGraphLaunch(g1, st));  // graph warm-up
        LP_CUDA(cudaGraphLaunch(g10, st));
        LP_CUDA(cudaEventRecord(ev[0], st));
        LP_CUDA(cudaGraphLaunch(g1, st));
        LP_CUDA(cudaEventRecord(ev[1], st));
        LP_CUDA(cudaGraphLaunch(g10, st));
        LP_CUDA(cudaEventRecord(ev[2], st));
        LP_CUDA(cudaEventSynchronize(ev[2]));
        float m1 = 0.f, m2 = 0.f;
        LP_CUDA(cudaEventElapsedTime(&m1, ev[0], ev[1]));
        LP_CUDA(cudaEventElapsedTime(&m2, ev[1], ev[2]));
        for (auto& x : ev) cudaEventDestroy(x);
        cudaGraphExecDestroy(g1);
        cudaGraphExecDestroy(g10);
        cudaStreamDestroy(cs);
        LP_CUDA(cudaFree(buf));
        out[0] = static_cast<double>(m1) / iters;
        out[1] = 2.0 * static_cast<double>(subb);                // K1: read the windows, write them packed
        out[2] = static_cast<double>(m2) / iters;
        out[3] = static_cast<double>(predb) + 2.0 * zb;        // K10: every prediction once, z read + written
    });
}

int lp_engine_comm(const lp_engine* e, uint64_t* nccl_bytes, uint64_t* ledger_bytes) {
    *nccl_bytes = e->nccl_bytes + e->peer_bytes;
    *ledger_bytes = e->ledger_bytes;
    return LP_OK;
}

int lp_engine_launches(const lp_engine* e, uint64_t* launches) {
    *launches = e->launches;
    return LP_OK;
}

}  // extern "C"
