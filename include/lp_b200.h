/*
 * lp_b200.h — C-ABI of the B200-native Latent Parallelism (LP) engine.
 *
 * This is the drop-in boundary for the reference's (lpsim) hot path: the
 * per-step partition / denoise / reconstruct / sampler loop of
 * /root/reference/proj/src/cluster.cpp:166-225.  Every entry point below names
 * the reference interface it replaces (file:line, paths relative to
 * /root/reference/proj).  Plain C types only: pointers, sizes, POD structs.
 *
 * Conventions
 *  - Return value is a status: 0 = OK, otherwise (lpsim::ErrorKind + 1), see
 *    lp_status (include/lpsim/errors.hpp:10-24), or LP_ERR_CUDA / LP_ERR_NCCL.
 *    lp_last_error() returns a thread-local message for the last failure.
 *  - Storage dtypes use the reference's byte codes (include/lpsim/dtype.hpp:10-14):
 *    2 = IEEE binary16, 4 = binary32, 8 = binary64.  Device buffers hold exactly
 *    the bits the reference's quantized doubles represent.
 *  - Latents are dense row-major (c, t, h, w), channel outermost
 *    (include/lpsim/latent.hpp:90-92).
 *  - All device pointers are caller-owned; stream-ordered calls never allocate
 *    and never synchronize the host.  `stream` is a cudaStream_t passed as void*.
 *  - There is no CPU fallback: device calls fail with LP_ERR_CUDA when no
 *    sm_100a device is present.
 */
#ifndef LP_B200_H
#define LP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: lpsim::ErrorKind + 1 (include/lpsim/errors.hpp:10-24) ---- */
enum lp_status {
    LP_OK = 0,
    LP_ERR_OUT_OF_BOUNDS = 1,
    LP_ERR_EMPTY_RANGE = 2,
    LP_ERR_DEGENERATE_AXIS = 3,
    LP_ERR_INVALID_OVERLAP_RATIO = 4,
    LP_ERR_OUTSIDE_EXTENT = 5,
    LP_ERR_ZERO_WEIGHT = 6,
    LP_ERR_SHAPE_MISMATCH = 7,
    LP_ERR_WORKER_FAILURE = 8,
    LP_ERR_INVALID_GROUPING = 9,
    LP_ERR_INVALID_ARGUMENT = 10,
    LP_ERR_NON_FINITE = 11,
    LP_ERR_CONFIG = 12,
    LP_ERR_IO = 13,
    LP_ERR_CUDA = 100,
    LP_ERR_NCCL = 101
};

/* Axis order = rotation order (include/lpsim/latent.hpp:17-24). */
enum lp_axis { LP_AXIS_T = 0, LP_AXIS_H = 1, LP_AXIS_W = 2 };

/* Reconstruct+update arithmetic (K10).  EXACT reproduces the reference's fp64,
 * worker-ordered, non-fused arithmetic bit for bit; FAST accumulates in fp32. */
enum lp_mode { LP_MODE_EXACT = 0, LP_MODE_FAST = 1 };

/* Toy denoisers (src/denoise.cpp:56-142), used as bit-exact parity fixtures. */
enum lp_toy_kind { LP_TOY_BOX = 0, LP_TOY_GLOBAL = 1, LP_TOY_IDENTITY = 2 };

#define LP_MAX_WORKERS 256

/* One worker's assignment — PartitionEntry (include/lpsim/partition.hpp:22-30). */
typedef struct lp_entry {
    int32_t worker_id; /* k, 1-based */
    int32_t reserved;
    int64_t core_begin, core_end;     /* core_patches   */
    int64_t ext_begin, ext_end;       /* ext_patches    */
    int64_t latent_begin, latent_end; /* latent [s, e) */
    int64_t delta_start, delta_end;   /* Δs, Δe (latent units) */
} lp_entry;

/* PartitionPlan (include/lpsim/partition.hpp:32-46). */
typedef struct lp_plan {
    int32_t axis;       /* lp_axis */
    int32_t step_index; /* i, 1-based */
    double overlap_ratio;
    int64_t patches_per_core; /* L */
    int64_t overlap_patches;  /* O */
    int64_t axis_patches;     /* N */
    int64_t axis_extent;      /* D */
    int64_t patch_size;       /* p */
    int32_t n_entries;        /* K_eff */
    int32_t reserved;
    lp_entry entries[LP_MAX_WORKERS];
} lp_plan;

/* ------------------------------------------------------------------------ */
/* Diagnostics                                                              */
/* ------------------------------------------------------------------------ */
const char* lp_last_error(void);
const char* lp_version(void);
/* Warning sink — set_warning_handler (include/lpsim/partition.hpp:48-52,
 * src/partition.cpp:13-28).  NULL handler silences; the default prints to stderr. */
typedef void (*lp_warning_fn)(const char* message, void* user);
void lp_set_warning_handler(lp_warning_fn fn, void* user);

/* ------------------------------------------------------------------------ */
/* Host-side plan builder (bit-exact with src/partition.cpp:38-134)         */
/* ------------------------------------------------------------------------ */
/* rotation_axis — src/partition.cpp:38-43 */
int lp_rotation_axis(int step_index, int32_t* axis_out);
/* core_bounds — src/partition.cpp:45-62; out = 2*K int64 [begin,end) pairs */
int lp_core_bounds(int64_t patches, int workers, int64_t* ranges_out, int32_t* n_out);
/* extend_overlap — src/partition.cpp:64-78 */
int lp_extend_overlap(const int64_t* cores, int32_t n_cores, int64_t patches, int64_t patches_per_core,
                      double overlap_ratio, int workers, int64_t* ext_out);
/* build_axis_plan — src/partition.cpp:80-123 */
int lp_build_axis_plan(int32_t axis, int64_t axis_extent, int64_t axis_patch, int step_index, int workers,
                       double overlap_ratio, lp_plan* plan_out);
/* build_plan_for_shape — src/partition.cpp:125-129; shape = {c,t,h,w}, patch = {p_t,p_h,p_w} */
int lp_build_plan(const int64_t shape[4], const int64_t patch[3], int step_index, int workers,
                  double overlap_ratio, lp_plan* plan_out);
/* build_weight_mask — src/reconstruct.cpp:9-27; out has latent_end-latent_begin doubles */
int lp_weight_profile(const lp_plan* plan, int32_t entry, double* profile_out);
/* Elements of entry k's sub-latent, and the packed (worker-ordered) offsets of all
 * entries: offsets_out has n_entries+1 values (the gather buffer layout). */
int lp_plan_offsets(const lp_plan* plan, const int64_t shape[4], int64_t* offsets_out);

/* Multi-rank shard layout: entries are assigned to ranks round-robin
 * (entry e -> rank e % world).  For `rank`, writes the entry ids it owns
 * (owned_out, up to LP_MAX_WORKERS) and their count; slot_elems_out = the
 * padded per-rank slot of the all-gather buffer (max over ranks of the summed
 * elements it owns, rounded up to a multiple of 8 elements so every slot starts
 * 16-byte aligned).  Rank r's slot holds its entries packed in worker order. */
int lp_shard_layout(const lp_plan* plan, const int64_t shape[4], int world, int rank, int32_t* owned_out,
                    int32_t* n_owned_out, int64_t* slot_elems_out);
/* Element offset of every entry's ε̂ shard inside the gathered buffer
 * (world slots of slot_elems): the layout K10 reads after the all-gather. */
int lp_shard_bases(const lp_plan* plan, const int64_t shape[4], int world, int64_t* base_out);
/* The same layout under an assignment policy: LP_ASSIGN_ROUND_ROBIN, or LP_ASSIGN_BALANCED =
 * longest-processing-time greedy on cost(entry) = lin*elems + quad*elems^2 (ties -> lowest
 * rank; with K <= world it equals round-robin).  The reference leaves the worker -> device
 * mapping open (its workers are threads, src/cluster.cpp:115-162).  owner_out / base_out:
 * one value per entry (NULL to skip). */
enum lp_assign { LP_ASSIGN_ROUND_ROBIN = 0, LP_ASSIGN_BALANCED = 1 };
int lp_shard_layout_ex(const lp_plan* plan, const int64_t shape[4], int world, int rank, int32_t policy, double lin,
                       double quad, int32_t* owned_out, int32_t* n_owned_out, int64_t* slot_elems_out,
                       int32_t* owner_out, int64_t* base_out);

/* Communication accounting — CommLedger + run_lp metering (src/cluster.cpp:27-73,
 * 186-209): the reference ledger bytes of step i (2 passes x (scatter+gather)
 * x sum_{k>=2} S_sub x wire_bytes), and the bytes this engine's padded all-gather
 * receives on all ranks together (world-1 foreign slots per rank x slot x dtype). */
int lp_step_comm_bytes(const lp_plan* plan, const int64_t shape[4], int wire_bytes, int world, int dtype_bytes,
                       uint64_t* ledger_bytes_out, uint64_t* allgather_bytes_out);

/* Communication cost model — cost_report (src/cost.cpp:215-248) incl. cost_nmp /
 * cost_pp / cost_lp_exact / cost_lp_approx / cost_hybrid (src/cost.cpp:46-213),
 * at the preset's hidden width and wire bytes.  hybrid_groups = 0: no hybrid. */
typedef struct lp_cost_report_t {
    uint64_t latent_bytes, activation_bytes;  /* S_z, S_H */
    double ext_bytes_mean, gamma, gamma_per_axis[3];
    uint64_t nmp_bytes, pp_bytes, lp_exact_bytes;
    double lp_approx_bytes, ratio_exact, ratio_approx, latent_activation_ratio;
    int32_t has_hybrid, hybrid_within_bound;
    uint64_t hybrid_inter_bytes, hybrid_intra_bytes, hybrid_total_bytes;
    double hybrid_ratio_vs_nmp, hybrid_bound;
} lp_cost_report_t;
int lp_cost_report(int steps, int workers, double overlap_ratio, const int64_t shape[4], const int64_t patch[3],
                   int64_t hidden_dim, int wire_bytes, int hybrid_groups, const int32_t* group_sizes,
                   lp_cost_report_t* out);

/* N-completeness checker — verify_n_complete (src/completeness.cpp:104-160,
 * include/lpsim/completeness.hpp:8-92), host side.  grid = patch-grid {nt, nh, nw};
 * schedule[i] = axis of step i+1 (lp_axis), schedule_len >= budget.  max_positions = 0
 * keeps the reference's 4096-position cap (InvalidArgument beyond it), > 0 lifts it.
 * min_steps_out (nt*nh*nw int32, or NULL): first step at which each position is complete, -1 never. */
int lp_verify_n_complete(const int64_t grid[3], int32_t workers, double overlap_ratio, const int32_t* schedule,
                         int32_t schedule_len, int32_t budget, int64_t max_positions, int32_t* complete_out,
                         int32_t* complete_at_out, int64_t worst_out[3], int32_t* min_steps_out);
/* Per-step coverage rows of the completeness command (src/commands.cpp:169-195):
 * rows_i[5*s..] = {step, min_reached, max_reached, complete_positions, total_positions},
 * rows_mean[s] = mean_reached; stops after the first all-complete step. */
int lp_coverage_trace(const int64_t grid[3], int32_t workers, double overlap_ratio, const int32_t* schedule,
                      int32_t schedule_len, int32_t budget, int64_t max_positions, int64_t* rows_i, double* rows_mean,
                      int32_t* n_rows_out);

/* LPLT latent dump — write_latent_dump / read_latent_dump (src/io.cpp:37-139).  `bits` are
 * the storage-dtype bits (f16 / f32 / f64, little-endian) of a row-major (c,t,h,w) latent —
 * exactly what the engine holds on the device.  read: bits = NULL parses the header only. */
int lp_latent_dump_write(const char* path, const void* bits, const int64_t shape[4], int32_t dtype_bytes);
int lp_latent_dump_read(const char* path, int64_t shape_out[4], int32_t* dtype_bytes_out, void* bits,
                        int64_t capacity_bytes);

/* The `lpsim` command line (tools/lpsim_main.cpp:42-113, src/commands.cpp:46-216) on this
 * engine: simulate | compare | cost | completeness | partition-plan, --config/--out/--seed/
 * --quiet (+ --backend b200).  Returns the process exit code: 0, 2 (config/usage), 3. */
int lp_cli_main(int argc, const char* const* argv);

/* Quantizer (src/dtype.cpp:34-116), host side, for tests and host shims. */
uint16_t lp_f16_encode(double v);
double lp_f16_decode(uint16_t bits);
double lp_quantize(double v, int dtype_bytes);

/* ------------------------------------------------------------------------ */
/* Device kernels (stream-ordered; sm_100a)                                  */
/* ------------------------------------------------------------------------ */
/* Device + context management.  A context binds one CUDA device. */
int lp_device_check(int device); /* LP_OK iff device exists and is sm_100 */
/* Sticky device flags raised by kernels (1 = a stored value was non-finite:
 * the reference's NonFinite, src/latent.cpp:72-77).  Synchronizes. */
int lp_device_flags(uint32_t* flags_out, int reset);
/* Device memory for hosts that bind only this header (integration/ shim): cudaMalloc /
 * cudaFree / synchronous cudaMemcpy on the current device.  Not for the hot path. */
int lp_device_alloc(size_t bytes, void** out);
int lp_device_free(void* p);
int lp_copy_to_device(void* dst, const void* src, size_t bytes);
int lp_copy_to_host(void* dst, const void* src, size_t bytes);
/* Kernel launches issued by this library since load. */
uint64_t lp_launch_count(void);
/* Frees the library's device-side caches (K10 coverage tables; rebuilt on next use).  Waits for
 * the device.  The cache is also bounded (64 tables) and flushed when full. */
int lp_release_caches(void);
/* Live per-kernel-class timing with CUDA events on the launching stream
 * (classes: 0 self-attention, 1 cross-attention, 2 GEMM, 3 K9 all-gather, 4 K1 gather,
 * 5 K10 reconstruct+update).  collect() fills 6 entries each: launches, device ms,
 * algorithmic FLOPs, algorithmic bytes. */
int lp_profile_enable(int on);
/* Kernel-variant knobs for A/B measurement (INTEGRATION.md lists all of them with their
 * defaults), e.g. "attn_poly" (exp2 pairs of every 16 on the FMA pipe: 0, 4, 6, 8),
 * "gemm_2sm" (0/1: CTA-pair GEMM).  A key's first read also checks LP_TUNE_<KEY>. */
int lp_tune(const char* key, int value);
int lp_profile_collect(uint64_t* launches, double* ms, double* flops, double* bytes);

/* K1: partition gather — extract_sublatents / slice_axis
 * (src/partition.cpp:136-148, src/latent.cpp:81-111).  Copies the entries
 * [first, first+count) of `plan` from z into `dst`, packed in worker order
 * (entry first at dst[0], next at dst[size(first)], ...).  Bit-exact copy. */
int lp_extract(const lp_plan* plan, int32_t first, int32_t count, const void* z, const int64_t shape[4],
               int dtype_bytes, void* dst, void* stream);

/* K11: toy denoisers — Denoiser::predict of Box/GlobalMix/Identity
 * (src/denoise.cpp:56-142).  `cond_mean` = ConditioningVector::mean()
 * (src/denoise.cpp:17-22).  fp64, the reference's summation order. */
int lp_toy_predict(int32_t kind, const int64_t radius[3], double t_coeff, double cond_coeff, const void* z,
                   const int64_t shape[4], int dtype_bytes, int timestep, double cond_mean, void* out,
                   void* stream);
/* cfg_predict with a toy denoiser (src/denoise.cpp:24-39), fused: one pass
 * computes uncond (null cond, mean 0) and cond predictions, each quantized,
 * then uncond + w*(cond-uncond) in fp64, quantized.  `workspace` needs
 * lp_toy_workspace_bytes(shape) bytes (GlobalMix channel sums), else NULL. */
int lp_toy_cfg_predict(int32_t kind, const int64_t radius[3], double t_coeff, double cond_coeff, const void* z,
                       const int64_t shape[4], int dtype_bytes, int timestep, double cond_mean, double guidance,
                       void* eps_out, void* workspace, void* stream);
size_t lp_toy_workspace_bytes(const int64_t shape[4]);

/* CFG combine of two already-quantized predictions (src/denoise.cpp:34-38). */
int lp_cfg_combine(const void* uncond, const void* cond, int64_t n, int dtype_bytes, double guidance, void* out,
                   void* stream);

/* reconstruct (src/reconstruct.cpp:42-121): `preds` = all entries' predictions
 * packed in worker order (layout of lp_plan_offsets).  Writes ε̂ (quantized). */
int lp_reconstruct(const lp_plan* plan, const void* preds, const int64_t shape[4], int dtype_bytes, int32_t mode,
                   void* eps_out, void* stream);
/* sampler_step (src/denoise.cpp:41-52): z_out = quantize(z - eta*eps). */
int lp_sampler_step(const void* z, const void* eps, int64_t n, int dtype_bytes, double eta, void* z_out,
                    void* stream);
/* K10: reconstruct + sampler_step fused, in place on z (one HBM pass):
 * z = quantize(z - eta * quantize(Σ_k w_k·pred_k / Σ_k w_k)). */
int lp_reconstruct_update(const lp_plan* plan, const void* preds, const int64_t shape[4], int dtype_bytes,
                          int32_t mode, double eta, void* z, void* stream);

/* Synthetic inputs — synthetic_inputs (src/run_config.cpp:258-301), host side:
 * mt19937_64 + pinned Box-Muller; latent quantized to dtype, 8 cond values. */
int lp_synthetic_inputs(const int64_t shape[4], int dtype_bytes, uint64_t seed, double* latent_out,
                        double* cond_out8);

/* ------------------------------------------------------------------------ */
/* DiT denoiser (the plugin slot Denoiser::predict, include/lpsim/denoise.hpp:31-39) */
/* ------------------------------------------------------------------------ */
typedef struct lp_dit_config {
    int32_t in_channels;  /* 16 */
    int32_t dim;          /* 1536 (1.3B) / 5120 (14B) */
    int32_t ffn_dim;      /* 8960 / 13824 */
    int32_t num_heads;    /* 12 / 40 ; head_dim = dim/num_heads = 128 */
    int32_t num_layers;   /* 30 / 40 */
    int32_t text_len;     /* 512 */
    int32_t text_dim;     /* 4096 */
    int32_t freq_dim;     /* 256 */
    int32_t patch[3];     /* 1,2,2 */
    int32_t reserved;
    double eps;           /* LayerNorm / RMSNorm eps, 1e-6 */
    double t_scale;       /* sinusoid input = t * t_scale (builder-pinned; 1000/T) */
    uint64_t seed;        /* weights + synthetic text context */
} lp_dit_config;

typedef struct lp_dit lp_dit;

void lp_dit_default_config(lp_dit_config* cfg); /* WAN2.1-1.3B shape */
/* Allocates weights (bf16) and the cond/uncond text K/V caches on the current
 * device, initialised from the pinned generator (see lp_dit_param). */
int lp_dit_create(const lp_dit_config* cfg, const double* cond_values, int32_t n_cond, lp_dit** out);
int lp_dit_destroy(lp_dit* dit);
int lp_dit_get_config(const lp_dit* dit, lp_dit_config* cfg_out);
/* Workspace for shards up to max_tokens tokens (allocates; call once). */
int lp_dit_reserve(lp_dit* dit, int64_t max_tokens);
/* Independent workspaces ("slots") so that several shards' forwards can be in
 * flight at once on different streams (the engine overlaps its owned entries). */
int lp_dit_reserve_slots(lp_dit* dit, int64_t max_tokens, int32_t nslots);
int lp_dit_cfg_predict_slot(lp_dit* dit, int32_t slot, const void* sub, const int64_t shape[4], int dtype_bytes,
                            int timestep, double guidance, void* eps_out, void* stream);
/* Pipeline stage of the same forward (hybrid LP x intra-group model parallelism,
 * src/cost.cpp:133-213 models its traffic): blocks [layer_begin, layer_end).  layer_begin == 0
 * embeds `sub`; otherwise the slot's activation must hold the residual stream after block
 * layer_begin-1.  layer_end == num_layers runs the head and writes ε̂ (eps_out); otherwise
 * the activation is left for the next stage.  Stages chained over any split give the
 * bit-identical ε̂ of lp_dit_cfg_predict_slot. */
int lp_dit_forward_layers(lp_dit* dit, int32_t slot, const void* sub, const int64_t shape[4], int dtype_bytes,
                          int timestep, double guidance, int32_t layer_begin, int32_t layer_end, void* eps_out,
                          void* stream);
/* The slot's activation (fp32 residual stream [2 * tokens, dim]) for a shard of `shape`:
 * what one pipeline stage hands the next (bytes = 2 * tokens * dim * 4). */
int lp_dit_activation(lp_dit* dit, int32_t slot, const int64_t shape[4], void** x_dptr, int64_t* bytes);
/* K8+K9 fusion for the engine's peer exchange: while n > 0 the CFG-combine epilogue stores
 * every ε̂ element also at eps_out + byte_deltas[j] (peer gather buffers mapped by CUDA IPC). */
int lp_dit_set_mirrors(lp_dit* dit, int32_t n, const int64_t* byte_deltas);
/* cfg_predict with the DiT: CFG batch 2 (uncond = null text, cond = synthetic
 * text), one forward, combine uncond + w*(cond-uncond), quantize to dtype. */
int lp_dit_cfg_predict(lp_dit* dit, const void* sub, const int64_t shape[4], int dtype_bytes, int timestep,
                       double guidance, void* eps_out, void* stream);
/* ONE CFG pass — Denoiser::predict (include/lpsim/denoise.hpp:35-36) of the DiT: null_text != 0
 * uses the null (zero) text context (the uncond pass cfg_predict makes with
 * ConditioningVector::null_like, src/denoise.cpp:29), else the synthetic cond text.  Writes
 * the prediction quantized to dtype.  Bit-identical to the matching half of the CFG-batched
 * forward, so the reference's own cfg_predict over two predict calls reproduces
 * lp_dit_cfg_predict bit for bit. */
int lp_dit_predict(lp_dit* dit, const void* sub, const int64_t shape[4], int dtype_bytes, int timestep,
                   int32_t null_text, void* eps_out, void* stream);
int lp_dit_predict_slot(lp_dit* dit, int32_t slot, const void* sub, const int64_t shape[4], int dtype_bytes,
                        int timestep, int32_t null_text, void* eps_out, void* stream);
/* For step loops captured into CUDA graphs: with time_on_device(1) the forwards read the
 * timestep from the slot's device scalar, which lp_dit_set_time writes (stream-ordered)
 * before each replay, instead of baking the host value into a kernel argument. */
int lp_dit_set_time(lp_dit* dit, int32_t slot, int timestep, void* stream);
int lp_dit_time_on_device(lp_dit* dit, int32_t on);
/* Parameter access for tests: index -> name, device pointer, element count, dtype (2=bf16,4=f32). */
int lp_dit_num_params(const lp_dit* dit);
int lp_dit_param(const lp_dit* dit, int32_t index, const char** name, void** dptr, int64_t* numel,
                 int32_t* elem_bytes);
/* Intermediate-tensor access for per-block tests (valid after a forward). */
int lp_dit_debug_tensor(const lp_dit* dit, const char* name, void** dptr, int64_t* numel);

/* ------------------------------------------------------------------------ */
/* Standalone GEMM (tcgen05) — exposed for unit tests and the bench roofline */
/* ------------------------------------------------------------------------ */
/* D[M,N] (bf16, row-major) = A[M,K] (bf16, row-major) · B[N,K]^T (bf16) + bias[N] (f32 or NULL). */
int lp_gemm_bf16(const void* A, const void* B, const void* bias, void* D, int64_t M, int64_t N, int64_t K,
                 void* stream);
/* The same GEMM with the DiT's fused epilogues (kernel tests / benches): mode 0 = bf16
 * D = AB^T + bias; 1 = bf16 GELU(tanh); 2 = fp32 residual D += gate ⊙ (AB^T + bias)
 * (gate may be NULL = 1); 3 = fp32 D = AB^T + bias.  D row stride = N. */
int lp_gemm_bf16_epi(const void* A, const void* B, const void* bias, const float* gate, void* D, int64_t M, int64_t N,
                     int64_t K, int32_t mode, void* stream);
/* Flash attention forward (tcgen05): q,k,v,o bf16 [B, S, H, 128] row-major. */
int lp_attention_bf16(const void* q, const void* k, const void* v, void* o, int64_t batch, int64_t seq_q,
                      int64_t seq_kv, int64_t heads, double scale, void* stream);

/* ------------------------------------------------------------------------ */
/* LP engine: the run_lp step loop (src/cluster.cpp:166-225)                */
/* ------------------------------------------------------------------------ */
typedef struct lp_engine_config {
    int64_t shape[4];
    int64_t patch[3];
    int32_t dtype_bytes;
    int32_t workers;       /* K */
    double overlap_ratio;  /* r */
    int32_t total_steps;   /* T */
    int32_t mode;          /* lp_mode for K10 */
    double eta;
    double guidance;
    int32_t denoiser;      /* -1 = DiT (dit != NULL), else lp_toy_kind */
    int32_t wire_bytes;    /* preset dtype_bytes for the reference ledger (2 = wan21-like) */
    int64_t radius[3];
    double t_coeff, cond_coeff;
    int32_t world, rank;   /* ranks sharing the plan; entries round-robin over ranks */
    lp_dit* dit;
    /* Axis schedule (BASELINE config C5): 0 = the reference's
     * T->H->W rotation (src/partition.cpp:38-43); else step i uses axis
     * schedule[(i-1) % schedule_len].  Plans per axis are build_axis_plan's. */
    int32_t schedule_len;
    int32_t schedule[64];
    /* Hybrid LP x intra-group model parallelism (src/cost.cpp:133-213):
     * group_size M > 1 splits the world into world/M LP groups of M ranks; rank r is
     * stage r % M of group r / M, running DiT blocks [s*L/M, (s+1)*L/M) and handing the
     * activation to the next stage (ncclSend/Recv).  Entries are assigned to groups.  0 or 1
     * = plain LP.  Requires the DiT denoiser. */
    int32_t group_size;
    /* Entry -> rank assignment (lp_assign).  LP_ASSIGN_BALANCED weighs entries by the
     * DiT's FLOPs (linear layers ~ tokens, self-attention ~ tokens^2), toys by elements. */
    int32_t assign;
} lp_engine_config;

typedef struct lp_engine lp_engine;

/* NCCL plumbing for world > 1: rank 0 gets an id, the caller broadcasts it.  With
 * world == 1 a non-NULL id makes a 1-rank communicator and runs the same exchange path. */
int lp_nccl_unique_id(uint8_t id_out[128]);
int lp_engine_create(const lp_engine_config* cfg, const uint8_t* nccl_id, const double* cond, int32_t n_cond,
                     lp_engine** out);
int lp_engine_destroy(lp_engine* e);
/* Device latent z (replicated on every rank), size shape volume * dtype. */
int lp_engine_latent(lp_engine* e, void** z_dptr);
/* Runs steps [first, first+count) (1-based i; t = T+1-i) on `stream`. */
int lp_engine_run(lp_engine* e, int32_t first_step, int32_t count, void* stream);
/* The same step in phases: 1 = K1 + cfg_predict of this rank's entries into its slot of the
 * gather buffer, 2 = K9 all-gather (no-op without an NCCL communicator), 3 = K10 from the
 * gathered buffer.  With world > 1 and no NCCL id the caller exchanges the slots itself
 * between phases 1 and 3 (world slots of slot_elems elements, rank r's slot at r*slot_elems). */
int lp_engine_step_phase(lp_engine* e, int32_t step, int32_t phase, void* stream);
int lp_engine_gather_buffer(const lp_engine* e, int32_t step, void** buffer, int64_t* slot_elems);
/* Hybrid engines (group_size M > 1), driven stage by stage without NCCL: runs this rank's
 * pipeline stage for the idx-th entry its group owns at `step` (idx < lp_engine_owned).
 * Stage 0 gathers (K1) and embeds; stages > 0 expect the previous stage's activation in
 * lp_engine_stage_activation's buffer; the last stage writes ε̂ into its group's slot of the
 * gather buffer (groups slots of slot_elems).  With NCCL, phase 1 runs every entry and the
 * activations move by ncclSend/Recv; phase 2 broadcasts each group's slot from its last
 * stage. */
int lp_engine_stage(lp_engine* e, int32_t step, int32_t idx, void* stream);
/* K9 over NVLink peer memory instead of NCCL (plain LP engines created without an NCCL id):
 * every rank exports its exchange arena (double-buffered gather buffer + flag words) with
 * lp_engine_ipc_handle, the caller all-gathers the 64-byte handles, and lp_engine_ipc_attach
 * maps the peers' arenas (CUDA IPC); with an NCCL communicator too, the peer path takes
 * precedence for the ε̂ exchange.  lp_engine_run then pushes this rank's ε̂ slot into every
 * peer with remote stores and a system-scope release flag per step, and K10 starts once every
 * peer's flag for the step has arrived. */
int lp_engine_ipc_handle(lp_engine* e, uint8_t handle_out[64]);
int lp_engine_ipc_attach(lp_engine* e, const uint8_t* handles /* world x 64 bytes, by rank */);
/* Unmaps the peers and returns the exchange to NCCL (or to the caller). */
int lp_engine_ipc_detach(lp_engine* e);
int lp_engine_stage_activation(lp_engine* e, int32_t step, int32_t idx, void** x_dptr, int64_t* bytes);
int lp_engine_owned(const lp_engine* e, int32_t step, int32_t* n_owned);
/* Group decomposition of this rank and the activation bytes it handed to the next stage. */
int lp_engine_hybrid(const lp_engine* e, int32_t* group_size, int32_t* group, int32_t* stage, int32_t* layer_begin,
                     int32_t* layer_end, uint64_t* intra_bytes);
/* Waits for everything enqueued on `stream` (the host side of run_workers' join,
 * src/cluster.cpp:149-161), polling instead of blocking: an NCCL asynchronous error
 * (ncclCommGetAsyncError) or `timeout_ms` (> 0) without completion aborts the
 * communicator and returns LP_ERR_WORKER_FAILURE naming the step; a peer whose ε̂ shard
 * never arrived over the NVLink exchange returns LP_ERR_WORKER_FAILURE naming the lowest
 * worker id that rank owns ("worker k failed at step i: rank r ..."), and K10 has left z
 * at the previous step instead of blending stale shards. */
int lp_engine_sync(lp_engine* e, void* stream, int64_t timeout_ms);
/* K9 alone, for its NVLink roofline: `iters` back-to-back exchanges of step's full ε̂ slots
 * (peer: the unfused remote-store push + flag + wait; NCCL: the all-gather), timed with CUDA
 * events on `stream`.  Every rank must call it with the same arguments.  bytes_out = bytes
 * this rank received (slot x (world-1) x iters). */
int lp_engine_exchange_bench(lp_engine* e, int32_t step, int32_t iters, void* stream, double* ms_out,
                             uint64_t* bytes_out);
/* K1 and K10 alone, for their HBM roofline: `iters` back-to-back launches each of step's K1
 * (gather of this rank's windows) and K10 (blend + sampler update of the full latent), on
 * `sets` private copies of (z, shards, gathered ε̂) used round robin so consecutive launches
 * stream from HBM, not L2.  Each loop of `iters` launches is captured once and replayed as a
 * CUDA graph, timed with events on `stream` (no host launch gaps between the few-µs kernels).
 * out = {K1 ms per launch, K1 algorithmic bytes per launch, K10 ms per launch, K10 algorithmic
 * bytes per launch}; the engine's own z is untouched. */
int lp_engine_hbm_bench(lp_engine* e, int32_t step, int32_t iters, int32_t sets, void* stream, double out[4]);
/* Bytes this engine moved over NCCL so far, and the reference ledger bytes. */
int lp_engine_comm(const lp_engine* e, uint64_t* nccl_bytes, uint64_t* ledger_bytes);
/* Kernel launches issued by the engine so far (this library's kernels only). */
int lp_engine_launches(const lp_engine* e, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* LP_B200_H */
