/*
 * lp_oracle.c — plain-C restatement of the reference LP hot path (lpsim).
 *
 * TEST INFRASTRUCTURE ONLY (see lp_oracle.h).  Written from the reference's
 * behaviour, not copied: the reconstruct is restated in per-output "gather"
 * form (each output element visits its contributors in worker order), which is
 * the form the GPU kernel K10 uses, and is bit-identical to the reference's
 * scatter form because each element sees the same ordered sequence of
 * separately-rounded additions.  Built with -ffp-contract=off (no FMA), as the
 * reference is.
 */
#include "lp_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { E_OOB = 1, E_EMPTY = 2, E_DEGEN = 3, E_RATIO = 4, E_OUTSIDE = 5, E_ZERO = 6, E_SHAPE = 7,
       E_WORKER = 8, E_GROUP = 9, E_ARG = 10, E_NONFINITE = 11 };

/* rotation_axis — src/partition.cpp:38-43: T,H,W cycle, i >= 1. */
int orc_rotation_axis(int step, int* axis) {
    if (step < 1) return E_ARG;
    *axis = (step - 1) % 3;
    return 0;
}

/* build_axis_plan — src/partition.cpp:45-123 (core_bounds, extend_overlap,
 * latent mapping with the remainder absorbed by the last entry). */
int orc_build_axis_plan(int axis, int64_t extent, int64_t p, int step, int workers, double r, int64_t* meta,
                        int64_t* entries) {
    if (p < 1 || extent < p) return E_DEGEN;                        /* partition.cpp:82-86 */
    const int64_t n = extent / p;                                   /* N = floor(D/p) */
    if (n < 1) return E_ARG;                                        /* partition.cpp:46-48 */
    if (workers < 1) return E_ARG;                                  /* partition.cpp:49-51 */
    const int64_t l = (n + workers - 1) / workers;                  /* L = ceil(N/K) */
    if (!(r >= 0.0 && r <= (double)(workers - 1))) return E_RATIO;  /* partition.cpp:66-70 */
    const int64_t o = (int64_t)((double)l * r);                     /* O = trunc(L*r), in double */
    int k_eff = 0;
    for (int k = 1; k <= workers; ++k) {
        if ((int64_t)(k - 1) * l >= n) break;                       /* trailing idle workers dropped */
        ++k_eff;
    }
    meta[0] = axis; meta[1] = step; meta[2] = l; meta[3] = o; meta[4] = n; meta[5] = extent; meta[6] = p;
    meta[7] = k_eff;
    for (int i = 0; i < k_eff; ++i) {
        const int64_t a = (int64_t)i * l;
        const int64_t b = a + l < n ? a + l : n;
        const int64_t ea = a - o > 0 ? a - o : 0;
        const int64_t eb = b + o < n ? b + o : n;
        int64_t* e = entries + 9 * i;
        e[0] = i + 1; e[1] = a; e[2] = b; e[3] = ea; e[4] = eb;
        e[5] = ea * p;
        e[6] = (i + 1 == k_eff) ? extent : eb * p;                  /* partition.cpp:113-117 */
        e[7] = (a - ea) * p;
        e[8] = (eb - b) * p;
    }
    return 0;
}

int orc_build_plan(const int64_t* shape, const int64_t* patch, int step, int workers, double r, int64_t* meta,
                   int64_t* entries) {
    int axis;
    int st = orc_rotation_axis(step, &axis);
    if (st) return st;
    return orc_build_axis_plan(axis, shape[1 + axis], patch[axis], step, workers, r, meta, entries);
}

/* build_weight_mask — src/reconstruct.cpp:9-27: j/Δs on the front ramp,
 * (ℓ-j)/Δe on the rear ramp, 1 on the core. */
int orc_weight_profile(const int64_t* e, double* out) {
    const int64_t len = e[6] - e[5], ds = e[7], de = e[8];
    for (int64_t j = 0; j < len; ++j) out[j] = 1.0;
    for (int64_t j = 0; j < ds; ++j) out[j] = (double)j / (double)ds;
    for (int64_t j = len - de; j < len; ++j) out[j] = (double)(len - j) / (double)de;
    return 0;
}

/* f16 encode — src/dtype.cpp:34-73: RNE straight from the double, saturating at
 * ±65504 (never Inf), NaN -> 0x7e00. Restated with integer arithmetic. */
uint16_t orc_f16_encode(double v) {
    if (v != v) return 0x7e00;
    if (v > 65504.0) v = 65504.0;
    if (v < -65504.0) v = -65504.0;
    uint64_t u;
    memcpy(&u, &v, 8);
    const uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
    const int e = (int)((u >> 52) & 0x7ff) - 1023;
    if ((u << 1) == 0 || e < -25) return sign;
    const uint64_t m = (u & 0xfffffffffffffull) | (1ull << 52);
    const int shift = e >= -14 ? 42 : 42 + (-14 - e);
    uint16_t h = e >= -14 ? (uint16_t)(((e + 15) << 10) | ((m >> 42) & 0x3ff)) : (uint16_t)(m >> shift);
    const uint64_t rem = m & ((1ull << shift) - 1), half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) h = (uint16_t)(h + 1);
    if ((h & 0x7fff) >= 0x7c00) h = 0x7bff;
    return (uint16_t)(sign | h);
}

/* f16 decode — src/dtype.cpp:75-100 (exact widening). */
double orc_f16_decode(uint16_t b) {
    const int e = (b >> 10) & 0x1f, m = b & 0x3ff;
    const double s = (b & 0x8000) ? -1.0 : 1.0;
    if (e == 0) return s * ldexp((double)m, -24);
    if (e == 31) return m ? NAN : s * INFINITY;
    return s * ldexp((double)(m | 0x400), e - 25);
}

/* quantize — src/dtype.cpp:102-116: f32 saturates at ±FLT_MAX. */
double orc_quantize(double v, int d) {
    if (d == 8) return v;
    if (d == 4) {
        if (v > FLT_MAX) return FLT_MAX;
        if (v < -FLT_MAX) return -FLT_MAX;
        return (double)(float)v;
    }
    return orc_f16_decode(orc_f16_encode(v));
}

static void axis_view(const int64_t* s, int axis, int64_t* outer, int64_t* inner) {
    /* latent.cpp:96-102: outer x axis x inner view */
    if (axis == 0) { *outer = s[0]; *inner = s[2] * s[3]; }
    else if (axis == 1) { *outer = s[0] * s[1]; *inner = s[3]; }
    else { *outer = s[0] * s[1] * s[2]; *inner = 1; }
}

/* extract_sublatents + slice_axis — src/partition.cpp:136-148, src/latent.cpp:81-111.
 * All entries packed in worker order.  A pure copy (values are already quantized). */
int orc_extract(const double* z, const int64_t* shape, const int64_t* meta, const int64_t* entries, double* out) {
    const int axis = (int)meta[0];
    const int64_t d = shape[1 + axis];
    if (d != meta[5]) return E_SHAPE;
    int64_t outer, inner;
    axis_view(shape, axis, &outer, &inner);
    int64_t off = 0;
    for (int k = 0; k < meta[7]; ++k) {
        const int64_t s = entries[9 * k + 5], e = entries[9 * k + 6], len = e - s;
        if (len == 0) return E_EMPTY;
        if (s < 0 || e > d || s > e) return E_OOB;
        for (int64_t o = 0; o < outer; ++o)
            memcpy(out + off + o * len * inner, z + (o * d + s) * inner, sizeof(double) * (size_t)(len * inner));
        off += outer * len * inner;
    }
    return 0;
}

/* Box / GlobalMix / Identity predict — src/denoise.cpp:56-142 (quantized like
 * LatentTensor::from_doubles, src/latent.cpp:66-79). */
int orc_toy_predict(int kind, const int64_t* radius, double t_coeff, double cond_coeff, const double* z,
                    const int64_t* s, int d, int t, double cond_mean, double* out) {
    const int64_t C = s[0], T = s[1], H = s[2], W = s[3];
    const double affine = t_coeff * (double)t + cond_coeff * cond_mean;
    if (kind == 2) {
        memcpy(out, z, sizeof(double) * (size_t)(C * T * H * W));
        return 0;
    }
    if (kind == 1) {
        const int64_t per = T * H * W;
        for (int64_t c = 0; c < C; ++c) {
            double acc = 0.0;
            for (int64_t i = 0; i < per; ++i) acc += z[c * per + i];
            const double mean = acc / (double)per;
            for (int64_t i = 0; i < per; ++i) {
                const double v = orc_quantize(0.5 * z[c * per + i] + 0.5 * mean + affine, d);
                if (!isfinite(v)) return E_NONFINITE;
                out[c * per + i] = v;
            }
        }
        return 0;
    }
    for (int i = 0; i < 3; ++i) if (radius[i] < 0) return E_ARG;
    for (int64_t c = 0; c < C; ++c)
        for (int64_t tt = 0; tt < T; ++tt) {
            const int64_t t0 = tt - radius[0] > 0 ? tt - radius[0] : 0;
            const int64_t t1 = tt + radius[0] < T - 1 ? tt + radius[0] : T - 1;
            for (int64_t h = 0; h < H; ++h) {
                const int64_t h0 = h - radius[1] > 0 ? h - radius[1] : 0;
                const int64_t h1 = h + radius[1] < H - 1 ? h + radius[1] : H - 1;
                for (int64_t w = 0; w < W; ++w) {
                    const int64_t w0 = w - radius[2] > 0 ? w - radius[2] : 0;
                    const int64_t w1 = w + radius[2] < W - 1 ? w + radius[2] : W - 1;
                    double acc = 0.0;
                    for (int64_t a = t0; a <= t1; ++a)
                        for (int64_t b = h0; b <= h1; ++b)
                            for (int64_t x = w0; x <= w1; ++x) acc += z[((c * T + a) * H + b) * W + x];
                    const double n = (double)((t1 - t0 + 1) * (h1 - h0 + 1) * (w1 - w0 + 1));
                    const double v = orc_quantize(acc / n + affine, d);
                    if (!isfinite(v)) return E_NONFINITE;
                    out[((c * T + tt) * H + h) * W + w] = v;
                }
            }
        }
    return 0;
}

static double cond_mean(const double* c, int n) {
    /* ConditioningVector::mean — src/denoise.cpp:17-22 */
    if (n == 0) return 0.0;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += c[i];
    return acc / (double)n;
}

/* cfg_predict — src/denoise.cpp:24-39: uncond (null = zeros) first, then cond;
 * u + w*(c-u) in double, quantized.  Toy defaults t_coeff 0.01, cond_coeff 0.1
 * (include/lpsim/denoise.hpp:56-61). */
int orc_cfg_predict(int kind, const int64_t* radius, const double* z, const int64_t* s, int d, int t,
                    const double* cond, int n_cond, double w, double* out) {
    const int64_t n = s[0] * s[1] * s[2] * s[3];
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    double* c = (double*)malloc(sizeof(double) * (size_t)n);
    double zero_mean = 0.0;
    if (n_cond > 0) {
        /* null_like: n_cond zeros; their mean is 0.0 (0+0+...)/n */
        double acc = 0.0;
        for (int i = 0; i < n_cond; ++i) acc += 0.0;
        zero_mean = acc / (double)n_cond;
    }
    int st = orc_toy_predict(kind, radius, 0.01, 0.1, z, s, d, t, zero_mean, u);
    if (!st) st = orc_toy_predict(kind, radius, 0.01, 0.1, z, s, d, t, cond_mean(cond, n_cond), c);
    for (int64_t i = 0; !st && i < n; ++i) {
        const double v = orc_quantize(u[i] + w * (c[i] - u[i]), d);
        if (!isfinite(v)) st = E_NONFINITE;
        out[i] = v;
    }
    free(u);
    free(c);
    return st;
}

/* reconstruct — src/reconstruct.cpp:42-121, restated per output element:
 * Z(x) = Σ_k W_k(x) and A = Σ_k W_k(x)·pred_k (W != 0 only), both in worker
 * order, out = quantize(A / Z).  ZeroWeight when Z < 1 - 1e-12. */
int orc_reconstruct(const double* preds, const int64_t* shape, int dt, const int64_t* meta, const int64_t* entries,
                    double* out) {
    const int axis = (int)meta[0];
    const int kn = (int)meta[7];
    const int64_t d = shape[1 + axis];
    if (d != meta[5]) return E_SHAPE;
    int64_t outer, inner;
    axis_view(shape, axis, &outer, &inner);
    double** prof = (double**)malloc(sizeof(double*) * (size_t)kn);
    int64_t* base = (int64_t*)malloc(sizeof(int64_t) * (size_t)kn);
    int64_t off = 0;
    for (int k = 0; k < kn; ++k) {
        const int64_t len = entries[9 * k + 6] - entries[9 * k + 5];
        prof[k] = (double*)malloc(sizeof(double) * (size_t)(len > 0 ? len : 1));
        orc_weight_profile(entries + 9 * k, prof[k]);
        base[k] = off;
        off += outer * len * inner;
    }
    int st = 0;
    for (int64_t x = 0; x < d && !st; ++x) {
        double z = 0.0;
        for (int k = 0; k < kn; ++k) {
            const int64_t s = entries[9 * k + 5], e = entries[9 * k + 6];
            if (x >= s && x < e) z += prof[k][x - s];
        }
        if (z < 1.0 - 1e-12) { st = E_ZERO; break; }
        for (int64_t o = 0; o < outer; ++o)
            for (int64_t i = 0; i < inner; ++i) {
                double a = 0.0;
                for (int k = 0; k < kn; ++k) {
                    const int64_t s = entries[9 * k + 5], e = entries[9 * k + 6], len = e - s;
                    if (x < s || x >= e) continue;
                    const double w = prof[k][x - s];
                    if (w == 0.0) continue;
                    a += w * preds[base[k] + (o * len + (x - s)) * inner + i];
                }
                const double v = orc_quantize(a / z, dt);
                if (!isfinite(v)) st = E_NONFINITE;
                out[(o * d + x) * inner + i] = v;
            }
    }
    for (int k = 0; k < kn; ++k) free(prof[k]);
    free(prof);
    free(base);
    return st;
}

/* sampler_step — src/denoise.cpp:41-52: quantize(z - eta*eps). */
int orc_sampler_step(const double* z, const double* eps, int64_t n, int d, double eta, double* out) {
    for (int64_t i = 0; i < n; ++i) {
        const double v = orc_quantize(z[i] - eta * eps[i], d);
        if (!isfinite(v)) return E_NONFINITE;
        out[i] = v;
    }
    return 0;
}

/* ---- mt19937_64 (the standard 64-bit Mersenne Twister) ---- */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* synthetic_inputs — src/run_config.cpp:258-301: pinned Box-Muller over raw
 * mt19937_64 words (u1 in (0,1], u2 in [0,1), cos first then the sin spare);
 * latent first (quantized), then 8 cond values (not quantized). */
int orc_synthetic(const int64_t* s, int d, uint64_t seed, double* z, double* cond) {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    const int64_t n = s[0] * s[1] * s[2] * s[3];
    int have = 0;
    double spare = 0.0;
    for (int64_t i = 0; i < n + 8; ++i) {
        double v;
        if (have) { have = 0; v = spare; }
        else {
            const double u1 = ((double)(mt64_next(g) >> 11) + 1.0) * 0x1.0p-53;
            const double u2 = (double)(mt64_next(g) >> 11) * 0x1.0p-53;
            const double rad = sqrt(-2.0 * log(u1));
            const double ang = 6.283185307179586476925286766559 * u2;
            spare = rad * sin(ang);
            have = 1;
            v = rad * cos(ang);
        }
        if (i < n) z[i] = orc_quantize(v, d);
        else cond[i - n] = v;
    }
    free(g);
    return 0;
}

/* run_lp — src/cluster.cpp:166-225 with the CommLedger metering of
 * src/cluster.cpp:186-209: per step 2 passes x (scatter + gather) x Σ_{k>=2} S_sub. */
int orc_run_lp(int kind, const int64_t* radius, const double* z0, const int64_t* s, int d, int steps, double eta,
               double w, const double* cond, int n_cond, const int64_t* patch, int workers, double r, int wire,
               double* final_out, uint64_t* ledger_total) {
    if (workers < 1 || steps < 1) return E_ARG;
    if (wire != 2 && wire != 4 && wire != 8) return E_ARG;
    const int64_t n = s[0] * s[1] * s[2] * s[3];
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    double* eps = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t meta[8];
    int64_t* ent = (int64_t*)malloc(sizeof(int64_t) * 9 * (size_t)workers);
    for (int64_t i = 0; i < n; ++i) z[i] = orc_quantize(z0[i], d);
    uint64_t ledger = 0;
    int st = 0;
    for (int i = 1; i <= steps && !st; ++i) {
        const int t = steps + 1 - i;
        st = orc_build_plan(s, patch, i, workers, r, meta, ent);
        if (st) break;
        int64_t outer, inner, total = 0;
        axis_view(s, (int)meta[0], &outer, &inner);
        for (int k = 0; k < meta[7]; ++k) total += outer * inner * (ent[9 * k + 6] - ent[9 * k + 5]);
        double* sub = (double*)malloc(sizeof(double) * (size_t)total);
        double* pred = (double*)malloc(sizeof(double) * (size_t)total);
        st = orc_extract(z, s, meta, ent, sub);
        int64_t off = 0;
        for (int k = 0; k < meta[7] && !st; ++k) {
            const int64_t len = ent[9 * k + 6] - ent[9 * k + 5];
            int64_t ss[4] = {s[0], s[1], s[2], s[3]};
            ss[1 + meta[0]] = len;
            st = orc_cfg_predict(kind, radius, sub + off, ss, d, t, cond, n_cond, w, pred + off);
            if (st) st = E_WORKER; /* run_workers wraps worker errors, cluster.cpp:149-161 */
            if (k >= 1) ledger += 4ull * (uint64_t)(outer * inner * len) * (uint64_t)wire;
            off += outer * inner * len;
        }
        if (!st) st = orc_reconstruct(pred, s, d, meta, ent, eps);
        if (!st) st = orc_sampler_step(z, eps, n, d, eta, z);
        free(sub);
        free(pred);
    }
    if (!st) memcpy(final_out, z, sizeof(double) * (size_t)n);
    if (ledger_total) *ledger_total = ledger;
    free(z);
    free(eps);
    free(ent);
    return st;
}
