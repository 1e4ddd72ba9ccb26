/*
 * lp_oracle.h — CPU restatement of the reference LP algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker (or the timed CPU baseline) — never as the product path.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against the
 * reference's own known-answer tests and against the compiled,
 * unmodified reference (oracle/_ref/libref_harness.so) on randomized sweeps.
 *
 * Plan flat encoding (same as oracle/ref_harness.cpp):
 *   meta[8]     = {axis, step_index, L, O, N, D, p, n_entries}
 *   entries[9n] = {k, core_b, core_e, ext_b, ext_e, lat_b, lat_e, delta_s, delta_e}
 * Status returns: 0 ok, else lpsim::ErrorKind + 1 (include/lpsim/errors.hpp:10-24).
 */
#ifndef LP_ORACLE_H
#define LP_ORACLE_H
#include <stdint.h>

int orc_rotation_axis(int step, int* axis);
int orc_build_axis_plan(int axis, int64_t extent, int64_t patch, int step, int workers, double r, int64_t* meta,
                        int64_t* entries);
int orc_build_plan(const int64_t* shape, const int64_t* patch, int step, int workers, double r, int64_t* meta,
                   int64_t* entries);
int orc_weight_profile(const int64_t* entry9, double* out);

uint16_t orc_f16_encode(double v);
double orc_f16_decode(uint16_t bits);
double orc_quantize(double v, int dtype_bytes);

int orc_extract(const double* z, const int64_t* shape, const int64_t* meta, const int64_t* entries, double* out);
int orc_toy_predict(int kind, const int64_t* radius, double t_coeff, double cond_coeff, const double* z,
                    const int64_t* shape, int dtype_bytes, int t, double cond_mean, double* out);
int orc_cfg_predict(int kind, const int64_t* radius, const double* z, const int64_t* shape, int dtype_bytes, int t,
                    const double* cond, int n_cond, double w, double* out);
int orc_reconstruct(const double* preds, const int64_t* shape, int dtype_bytes, const int64_t* meta,
                    const int64_t* entries, double* out);
int orc_sampler_step(const double* z, const double* eps, int64_t n, int dtype_bytes, double eta, double* out);
int orc_synthetic(const int64_t* shape, int dtype_bytes, uint64_t seed, double* z_out, double* cond_out);
int orc_run_lp(int kind, const int64_t* radius, const double* z, const int64_t* shape, int dtype_bytes, int steps,
               double eta, double w, const double* cond, int n_cond, const int64_t* patch, int workers, double r,
               int wire_bytes, double* final_out, uint64_t* ledger_total);
#endif
