/* CPU check of paper_2304_11165_b200/csrc/pd_libm_exp.h against the host
 * libm's exp() (the function the reference's D(phi) calls,
 * geometry.hpp:182-187) and of pd_smooth_diffusion against the reference
 * expression. Prints "<checked> <mismatches>" and the first mismatches.
 * Build: gcc -O2 -ffp-contract=off [-mfma] -I<csrc> libm_exp_check.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pd_libm_exp.h"

static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t rnd(void) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    return s;
}
static double uni(double a, double b) { return a + (b - a) * ((rnd() >> 11) * 0x1p-53); }

static long long bad = 0, n = 0;
static void check(double x) {
    volatile double xv = x;
    double want = exp(xv);
    double got = pd_libm_exp(xv);
    n++;
    if (memcmp(&want, &got, 8) != 0 && !(isnan(want) && isnan(got))) {
        if (bad < 10) printf("exp(%a): libm %a mine %a\n", x, want, got);
        bad++;
    }
}
static void check_d(double phi, double dmin, double dmax, double g1, double g2) {
    volatile double p = phi;
    double want = dmin + dmax / (1.0 + exp(-(g1 + g2 * p)));
    double got = pd_smooth_diffusion(p, dmin, dmax, g1, g2);
    n++;
    if (memcmp(&want, &got, 8) != 0) {
        if (bad < 10) printf("D(%a): ref %a mine %a\n", phi, want, got);
        bad++;
    }
}

int main(int argc, char** argv) {
    long long m = argc > 1 ? atoll(argv[1]) : 1000000;
    for (long long i = 0; i < m; i++) {
        uint64_t u = rnd();
        double x;
        memcpy(&x, &u, 8);
        check(x);                        /* every exponent / sign / nan / inf */
        check(uni(-750.0, 750.0));       /* normal + both special-case scalings */
        check(uni(-40.0, 40.0));         /* where D is not saturated */
        check(uni(-745.2, -700.0));      /* subnormal results */
        check(uni(700.0, 709.8));        /* near overflow */
        check(uni(-1e-3, 1e-3));
        check(ldexp(uni(-1.0, 1.0), -(int)(rnd() % 80)));  /* tiny |x| */
        /* D(phi) as the bench builds it: d_min 0, d_max 1, gamma1 0,
         * gamma2 = 4 n for n = 64..2048 (SDF values in box units) */
        double g2 = 4.0 * (double)(64 << (rnd() % 6));
        check_d(uni(-0.6, 0.6), 0.0, 1.0, 0.0, g2);
        check_d(uni(-0.02, 0.02), 0.05, 0.95, 1.5, g2);
    }
    const double edges[] = {0.0, -0.0, INFINITY, -INFINITY, NAN, 0x1p-54, -0x1p-54, 0x1.fffffffffffffp-55, 512.0,
                            -512.0, 1024.0, -1024.0, 709.782712893384, 709.7827128933841, -708.3964185322641,
                            -745.1332191019411, -745.1332191019412, -744.4400719213812, 0x1p-1074, 1.0, -1.0};
    for (unsigned i = 0; i < sizeof edges / sizeof edges[0]; i++)
        for (int k = -64; k <= 64; k++) check(nextafter(edges[i], k < 0 ? -INFINITY : INFINITY) * 0 + edges[i] + 0 * k),
            check(edges[i] == 0 || isinf(edges[i]) || isnan(edges[i]) ? edges[i] : edges[i] + k * ldexp(1.0, ilogb(edges[i]) - 52));
    printf("%lld %lld\n", n, bad);
    return bad != 0;
}
