// Markstein final-step division check (K10 exact, div_z in lp_kernels.cu): q = a*y, r = fma(-q, Z, a),
// q2 = fma(r, y, q) with y = RN(1/Z) against true division a/Z over ramp-weight sums Z and varied a.
// gcc -O2 -ffp-contract=off markstein.c -lm && ./a.out   (expect "bad 0")
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s = 88172645463325252ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rd(void) { return (double)(rnd() >> 11) * 0x1.0p-53; }
int main(void) {
    long bad = 0, tot = 0;
    // Z values: sums of ramp weights j/D (+1) for D up to 40, and random doubles in [1, 2)
    for (int D = 1; D <= 40; ++D)
        for (int j = 0; j <= D; ++j)
            for (int kind = 0; kind < 3; ++kind) {
                double Z;
                if (kind == 0) Z = 1.0 + (double)j / D;
                else if (kind == 1) Z = (double)j / D + (double)(D - j) / D;
                else Z = (double)j / D + (double)(D - j + 1) / (D + 1);
                if (Z < 1.0 - 1e-12) continue;
                const double y = 1.0 / Z;
                for (int i = 0; i < 200000; ++i) {
                    double a;
                    switch (i % 4) {
                        case 0: a = (rd() * 2 - 1) * ldexp(1.0, (int)(rnd() % 40) - 20); break;
                        case 1: a = (float)((rd() * 2 - 1) * 8.0) * ((double)(rnd() % (D + 1)) / D) + (float)((rd() * 2 - 1) * 8.0); break;
                        case 2: { uint64_t b = rnd() & 0x000FFFFFFFFFFFFFull; b |= (uint64_t)(1023 + (int)(rnd()%20) - 10) << 52; memcpy(&a, &b, 8); } break;
                        default: a = (double)(float)(rd() * 4 - 2); break;
                    }
                    const double q = a * y;
                    const double r = fma(-q, Z, a);
                    const double q2 = fma(r, y, q);
                    const double want = a / Z;
                    ++tot;
                    if (q2 != want) { if (bad < 5) printf("mismatch Z=%.17g a=%.17g got %.17g want %.17g\n", Z, a, q2, want); ++bad; }
                }
            }
    printf("total %ld bad %ld\n", tot, bad);
    return 0;
}
