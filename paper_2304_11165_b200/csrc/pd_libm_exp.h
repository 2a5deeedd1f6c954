// Bit-exact restatement of the double-precision exp() the reference's D(phi)
// calls (std::exp in smooth_diffusion_coefficient, geometry.hpp:182-187).
//
// The reference links glibc (>= 2.28), whose exp is the table-driven
// algorithm exp(x) = 2^(k/128) * exp(r), |r| <= ln2/256, with a 5th-order
// polynomial for exp(r) - 1 and the special cases below. On x86-64 hosts with
// FMA + AVX2 (every B200 host) the ifunc selects the FMA build, whose operation
// sequence -- which products are fused, in which order sums are formed -- was
// read from the image's libm (glibc 2.39) and is reproduced here operation by
// operation. Every step is one IEEE-754 double operation (fma, add, sub, mul,
// integer bit manipulation), so the result is the same bits on the host and
// on the device. Verified against the host libm on ~10^8 arguments spanning
// every branch (tests/test_libm_exp.py) and through the device D channel
// against the reference builder (tests/test_gpu_parity.py).
//
// Usable from host C/C++ (gcc, for the CPU check) and from CUDA device code.
#pragma once
#include <stdint.h>
#include <string.h>

#include "pd_exp_table.h"

#if defined(__CUDACC__)
#define PD_LX_HD __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define PD_LX_FMA(a, b, c) __fma_rn((a), (b), (c))
#define PD_LX_ADD(a, b) __dadd_rn((a), (b))
#define PD_LX_SUB(a, b) __dsub_rn((a), (b))
#define PD_LX_MUL(a, b) __dmul_rn((a), (b))
#endif
#else
#include <math.h>
#define PD_LX_HD static inline
#endif
#ifndef PD_LX_FMA
// host: compile with -ffp-contract=off so these stay single operations
#define PD_LX_FMA(a, b, c) fma((a), (b), (c))
#define PD_LX_ADD(a, b) ((a) + (b))
#define PD_LX_SUB(a, b) ((a) - (b))
#define PD_LX_MUL(a, b) ((a) * (b))
#endif

#if defined(__CUDACC__)
__device__ static const uint64_t pd_lx_tab_d[256] = PD_EXP_TABLE_INIT;
#endif
static const uint64_t pd_lx_tab_h[256] = PD_EXP_TABLE_INIT;

PD_LX_HD double pd_lx_d(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}
PD_LX_HD uint64_t pd_lx_u(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}

// Table entry j (0..255). On the device the table lives in global memory and
// is read through the read-only data path (the index varies per lane, so a
// __constant__ table would serialise the warp).
PD_LX_HD uint64_t pd_lx_tab(uint32_t j) {
#if defined(__CUDA_ARCH__)
    return __ldg((const unsigned long long*)pd_lx_tab_d + j);
#else
    return pd_lx_tab_h[j];
#endif
}

PD_LX_HD double pd_libm_exp(double x) {
    const double InvLn2N = 0x1.71547652b82fep7;  // 128 / ln 2
    const double Shift = 0x1.8p52;
    const double NegLn2hiN = -0x1.62e42fefa0000p-8;
    const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;

    const uint64_t ux = pd_lx_u(x);
    uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
    if (abstop - 0x3c9u > 0x3eu) {  // |x| < 2^-54, or |x| >= 512, or inf / nan
        if ((int32_t)(abstop - 0x3c9u) < 0) return PD_LX_ADD(x, 1.0);
        if (abstop > 0x408u) {  // |x| >= 1024
            if (ux == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ffu) return PD_LX_ADD(x, 1.0);
            if (ux >> 63) return 0.0;               // __math_uflow: 0x1p-767 * 0x1p-767
            return pd_lx_d(0x7ff0000000000000ull);  // __math_oflow: +inf
        }
        abstop = 0;  // 512 <= |x| < 1024: scaled below
    }
    const double z = PD_LX_FMA(x, InvLn2N, Shift);
    const uint64_t ki = pd_lx_u(z);
    const double kd = PD_LX_SUB(z, Shift);
    double r = PD_LX_FMA(kd, NegLn2hiN, x);
    r = PD_LX_FMA(kd, NegLn2loN, r);
    const uint32_t idx = 2u * (uint32_t)(ki & 127u);
    const uint64_t top = ki << 45;
    const double tail = pd_lx_d(pd_lx_tab(idx));
    uint64_t sbits = pd_lx_tab(idx + 1) + top;
    const double p23 = PD_LX_FMA(r, C3, C2);
    const double rt = PD_LX_ADD(r, tail);
    const double r2 = PD_LX_MUL(r, r);
    const double p45 = PD_LX_FMA(r, C5, C4);
    const double t = PD_LX_FMA(p23, r2, rt);
    const double r4 = PD_LX_MUL(r2, r2);
    const double tmp = PD_LX_FMA(r4, p45, t);
    if (abstop != 0) {
        const double scale = pd_lx_d(sbits);
        return PD_LX_FMA(scale, tmp, scale);
    }
    // specialcase: the scale 2^(k/128) is not a normal double
    if ((ki & 0x80000000ull) == 0) {  // k > 0: result may overflow
        sbits -= 1009ull << 52;
        const double scale = pd_lx_d(sbits);
        return PD_LX_MUL(PD_LX_FMA(scale, tmp, scale), 0x1p1009);
    }
    // k < 0: result may be subnormal; round once, in the final scaling
    sbits += 1022ull << 52;
    const double scale = pd_lx_d(sbits);
    const double st = PD_LX_MUL(tmp, scale);
    double y = PD_LX_ADD(scale, st);
    if (1.0 > y) {
        const double hi = PD_LX_ADD(y, 1.0);
        double lo = PD_LX_SUB(scale, y);
        lo = PD_LX_ADD(lo, st);
        double s = PD_LX_SUB(1.0, hi);
        s = PD_LX_ADD(s, y);
        s = PD_LX_ADD(s, lo);
        s = PD_LX_ADD(s, hi);
        y = PD_LX_SUB(s, 1.0);
        if (y == 0.0) return 0.0;  // +0 in round-to-nearest (never -0)
    }
    return PD_LX_MUL(y, 0x1p-1022);
}

// smooth_diffusion_coefficient (geometry.hpp:182-187), validation aside:
// d_min + d_max / (1 + exp(-(gamma1 + gamma2 * phi))), each operation
// rounded once (the reference builds with -ffp-contract=off).
PD_LX_HD double pd_smooth_diffusion(double phi, double d_min, double d_max, double g1, double g2) {
    const double a = PD_LX_ADD(g1, PD_LX_MUL(g2, phi));
    const double e = pd_libm_exp(-a);
    return PD_LX_ADD(d_min, d_max / PD_LX_ADD(1.0, e));
}
