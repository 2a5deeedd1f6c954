// Plane-marching FTCS step for 3-D FP32 grids (the reference's T = float
// instantiation, solver.hpp:385-455 in float arithmetic). Same design as the
// FP64 ftcs_march14_kernel (pd_march.cu) — persistent warps, one chunk per
// warp marching its 8 z-planes, cp.async ring of plane tiles 5 loads ahead,
// D_eff = fluid ? D : -inf, face fluxes computed once, interior-plane fast
// path, exact generic rare path — with every datum half as wide: a lane's
// x-pair is 8 B (cp.async.ca 8, LDS.64), x-halo cells 4 B, a tile 768 B, so
// 6 CTAs x 4 warps fit per SM. Bit-identical to the reference's float path
// (no contraction: --fmad=false; same expression order; the fast path's
// zero flux for a substituted face equals the reference's
// ((d_c+d_c)*0.5f)*(u_c-u_c) = +-0 for finite operands).
#include <cstdlib>

#include "pd_internal.cuh"

namespace pdb {

namespace {

constexpr int kW32 = 4;                 // warps per CTA
constexpr int kT32 = 32 * kW32;
#ifndef PD_M32_CTAS
#define PD_M32_CTAS 6
#endif
constexpr int kCtas32 = PD_M32_CTAS;    // CTAs per SM
constexpr int kRing32 = 8;
constexpr int kAhead32 = kRing32 - 3;   // planes z-1, z, z+1 resident
constexpr unsigned kSent32 = 0xFF800000u;  // -inf
constexpr int kFlagDir32 = 2;           // desc flags (pd_march.cu desc_kernel)
constexpr int kFlagUnif32 = 1 << 18;    // uniform chunk (pd_march.cu mark_uniform): no D_eff loads
constexpr uint32_t kCtx32 = 176;        // lm[32] | desc[8] | id | uniform D (at 164)

__device__ __forceinline__ bool sent32(float d) { return __float_as_uint(d) == kSent32; }
// non-finite (exponent all ones): the fast result needs the exact re-derivation
__device__ __forceinline__ bool nonfinite32(float x) { return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u; }

struct Tile32 {
    float u[80], hxu[2][8];
    float d[80], hxd[2][8];
};
constexpr uint32_t kTile32 = sizeof(Tile32);                // 768
constexpr uint32_t kDOff32 = (uint32_t)offsetof(Tile32, d);  // u -> D_eff (bytes)
constexpr uint32_t kHx32 = (uint32_t)offsetof(Tile32, hxu);
constexpr uint32_t kWarpBytes32 = kRing32 * kTile32 + 3 * kCtx32;

struct Args32 {
    StepArgs<float> A;
    const int32_t* __restrict__ sched;
    int64_t n;
    const int32_t* __restrict__ desc;
    const uint32_t* __restrict__ lm;
    const float* __restrict__ deff;
    const float* __restrict__ dv;  // per chunk: uniform D_eff of kFlagUnif32 chunks
    int* counter;
    int zero;
    int64_t n_all;
};

struct Slow32 {
    int64_t size[3];
    float inv_dx2[3];
    float bcv[6];
    float dt, neg_k, src_factor;
    int dirichlet;
};

struct Geo32 {
    int y, xp;
    bool xface, yface;
    uint32_t s_c, s_l, s_r, s_hx, s_hy, bp;
};

__device__ __forceinline__ Geo32 geo32(int lane) {
    Geo32 G;
    G.y = lane >> 2;
    G.xp = lane & 3;
    const int x0 = 2 * G.xp;
    G.xface = G.xp == 0 || G.xp == 3;
    G.yface = G.y == 0 || G.y == 7;
    G.s_c = (uint32_t)(x0 + 8 * (G.y + 1)) * 4u;
    G.s_l = G.xp == 0 ? kHx32 + (uint32_t)G.y * 4u : G.s_c - 4u;
    G.s_r = G.xp == 3 ? kHx32 + (uint32_t)(8 + G.y) * 4u : G.s_c + 8u;
    G.s_hx = kHx32 + (uint32_t)((G.xp == 3 ? 8 : 0) + G.y) * 4u;
    G.s_hy = G.y == 0 ? G.s_c - 32u : G.s_c + 32u;
    G.bp = (uint32_t)(G.y * 8 + x0);
    return G;
}

__device__ __forceinline__ void cp_commit32() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait32() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cpa(uint32_t sa, const void* g, int bytes_is8, bool pred) {
    if (bytes_is8)
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
            " @p cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(sa),
            "l"(g), "r"((int)pred));
    else
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
            " @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(sa),
            "l"(g), "r"((int)pred));
}
__device__ __forceinline__ float2 lds2f(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds1f(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t ldsu(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void stsu(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(a), "r"(v)); }
__device__ __forceinline__ void stg2f(float* p, float a, float b, bool a0, bool a1) {
    asm volatile(
        "{\n .reg .pred p, q, r;\n setp.ne.b32 p, %3, 0;\n setp.ne.b32 q, %4, 0;\n"
        " and.pred r, p, q;\n"
        " @r st.global.cs.v2.f32 [%0], {%1, %2};\n"
        " xor.pred p, p, r;\n xor.pred q, q, r;\n"
        " @p st.global.cs.f32 [%0], %1;\n"
        " @q st.global.cs.f32 [%0+4], %2;\n}\n" ::"l"(p),
        "f"(a), "f"(b), "r"((int)a0), "r"((int)a1)
        : "memory");
}

// HALF: the ring holds D_eff / 2 (see face<HALF> in pd_march.cu)
template <bool HALF>
__device__ __forceinline__ float face32(float da, float db, float ua, float ub) {
    const float s = da + db;
    const float f = (HALF ? s : s * 0.5f) * (ub - ua);
    return sent32(s) ? 0.0f : f;
}
template <bool HALF>
__device__ __forceinline__ float fface32(float da, float db, float ua, float ub) {
    return (HALF ? (da + db) : (da + db) * 0.5f) * (ub - ua);
}

// Exact generic node update (solver.hpp:360-441) in float.
template <int REACTION>
__device__ __noinline__ float slow_node32(const Slow32& K, float u_c, float d_c, const float* nu, const float* nd,
                                         int64_t gx, int64_t gy, int64_t gz, bool sink, float src) {
    const int64_t g[3] = {gx, gy, gz};
    float lap = 0.0f;
    for (int ax = 0; ax < 3; ++ax) {
        float u2[2], d2[2];
        for (int side = 0; side < 2; ++side) {
            const int f = ax * 2 + side;
            const int64_t gg = g[ax] + (side ? 1 : -1);
            if (gg < 0 || gg >= K.size[ax]) {
                u2[side] = (K.dirichlet >> f) & 1 ? K.bcv[f] : u_c;
                d2[side] = d_c;
            } else if (sent32(nd[f])) {
                u2[side] = u_c;
                d2[side] = d_c;
            } else {
                u2[side] = nu[f];
                d2[side] = nd[f];
            }
        }
        const float dh_m = (d_c + d2[0]) * 0.5f;
        const float dh_p = (d_c + d2[1]) * 0.5f;
        lap += (dh_p * (u2[1] - u_c) - dh_m * (u_c - u2[0])) * K.inv_dx2[ax];
    }
    float rate = 0.0f;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        if (sink) rate = K.neg_k * u_c;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        rate = src * K.src_factor;
    }
    return u_c + K.dt * lap + K.dt * rate;
}

struct Ctx32 {
    int c, key, flags;
    uint32_t lm;
    float dv;
};

struct Load32 {
    uint32_t own, zl, zh, xo, yo, lm;
    bool zlok, zhok, xok, yok;
    bool dl;  // load D_eff (false for uniform chunks)
};

__device__ __forceinline__ Load32 load_ctx32(int c, uint32_t lm, int dv, const Geo32& G) {
    int nb[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) nb[f] = __shfl_sync(0xffffffffu, dv, 24 + f);
    Load32 L;
    const bool ok = c >= 0;
    L.dl = !(__shfl_sync(0xffffffffu, dv, 31) & kFlagUnif32);
    L.own = ok ? (uint32_t)c * 512u + G.bp : 0u;
    L.lm = ok ? lm : 0u;
    L.zlok = ok && nb[4] >= 0;
    L.zhok = ok && nb[5] >= 0;
    L.zl = L.zlok ? (uint32_t)nb[4] * 512u + 448u + G.bp : 0u;
    L.zh = L.zhok ? (uint32_t)nb[5] * 512u + G.bp : 0u;
    const int jx = G.xp == 0 ? nb[0] : nb[1];
    L.xok = ok && G.xface && jx >= 0;
    L.xo = L.xok ? (uint32_t)jx * 512u + (uint32_t)G.y * 8u + (G.xp == 0 ? 7u : 0u) : 0u;
    const int jy = G.y == 0 ? nb[2] : nb[3];
    L.yok = ok && G.yface && jy >= 0;
    L.yo = L.yok ? (uint32_t)jy * 512u + (G.y == 0 ? 56u : 0u) + 2u * (uint32_t)G.xp : 0u;
    return L;
}

// load i (0..9) of a chunk into the tile at st (see issue14 in pd_march.cu)
__device__ __forceinline__ void issue32(uint32_t st, const float* __restrict__ u, const float* __restrict__ de,
                                        const Load32& L, int i, const Geo32& G, uint32_t sent_off) {
    if (i == 0 || i == 9) {
        const bool ok = i == 0 ? L.zlok : L.zhok;
        const uint32_t o = i == 0 ? L.zl : L.zh;
        cpa(st + G.s_c, u + o, 1, ok);
        cpa(st + kDOff32 + G.s_c, de + (ok ? o : sent_off + G.bp), 1, L.dl);
        return;
    }
    const uint32_t p64 = (uint32_t)(i - 1) * 64u;
    const bool ok = ((L.lm >> (2 * (i - 1))) & 3u) != 0u;
    const uint32_t o = L.own + p64;
    cpa(st + G.s_c, u + o, 1, ok);
    cpa(st + kDOff32 + G.s_c, de + (ok ? o : sent_off + G.bp + p64), 1, L.dl);
    const uint32_t ox = L.xo + p64;
    cpa(st + G.s_hx, u + ox, 0, L.xok);
    cpa(st + kDOff32 + G.s_hx, de + (L.xok ? ox : sent_off + G.bp + p64), 0, G.xface && L.dl);
    const uint32_t oy = L.yo + p64;
    cpa(st + G.s_hy, u + oy, 1, L.yok);
    cpa(st + kDOff32 + G.s_hy, de + (L.yok ? oy : sent_off + G.bp + p64), 1, G.yface && L.dl);
}

// Rare path: Dirichlet-exposed chunk (whole chunk exact) or a non-finite fast
// result (re-derived exactly), then the reference's error flags.
template <int REACTION, bool HALF>
__device__ __noinline__ float2 slow_pair32(const Args32& M, const Slow32& K, Ctx32 C, int z, uint32_t tm, uint32_t t0,
                                           uint32_t tp, Geo32 G, float out0, float out1) {
    const bool un = (C.flags & kFlagUnif32) != 0;  // no D_eff in the ring: every d is dv
    const float2 vv = make_float2(C.dv, C.dv);
    const float2 uc = lds2f(t0 + G.s_c), dc0 = un ? vv : lds2f(t0 + kDOff32 + G.s_c);
    const float uL = lds1f(t0 + G.s_l), dL0 = un ? C.dv : lds1f(t0 + kDOff32 + G.s_l);
    const float uR = lds1f(t0 + G.s_r), dR0 = un ? C.dv : lds1f(t0 + kDOff32 + G.s_r);
    const float2 uym = lds2f(t0 + G.s_c - 32), dym0 = un ? vv : lds2f(t0 + kDOff32 + G.s_c - 32);
    const float2 uyp = lds2f(t0 + G.s_c + 32), dyp0 = un ? vv : lds2f(t0 + kDOff32 + G.s_c + 32);
    const float2 uzm = lds2f(tm + G.s_c), dzm0 = un ? vv : lds2f(tm + kDOff32 + G.s_c);
    const float2 uzp = lds2f(tp + G.s_c), dzp0 = un ? vv : lds2f(tp + kDOff32 + G.s_c);
    auto dd = [](float h) { return HALF ? h + h : h; };  // D from D/2 (exact)
    auto dd2 = [&](float2 h) { return make_float2(dd(h.x), dd(h.y)); };
    const float2 dc = dd2(dc0), dym = dd2(dym0), dyp = dd2(dyp0), dzm = dd2(dzm0), dzp = dd2(dzp0);
    const float dL = dd(dL0), dR = dd(dR0);
    const bool s0 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (16 + 2 * z)) & 1u);
    const bool s1 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (17 + 2 * z)) & 1u);
    float src0 = 0.0f, src1 = 0.0f;
    if (REACTION == PD_REACTION_VOLUMETRIC) {
        const float* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + G.bp;
        src0 = sp[0];
        src1 = sp[1];
    }
    const float nu0[6] = {uL, uc.y, uym.x, uyp.x, uzm.x, uzp.x};
    const float nd0[6] = {dL, dc.y, dym.x, dyp.x, dzm.x, dzp.x};
    const float nu1[6] = {uc.x, uR, uym.y, uyp.y, uzm.y, uzp.y};
    const float nd1[6] = {dc.x, dR, dym.y, dyp.y, dzm.y, dzp.y};
    const bool dirichlet = (C.flags & kFlagDir32) != 0;
    const int x0 = 2 * G.xp;
    const int kx = C.key & 1023, ky = (C.key >> 10) & 1023, kz = (C.key >> 20) & 1023;
    const int64_t gx = (int64_t)kx * 8 + x0, gy = (int64_t)ky * 8 + G.y, gz = (int64_t)kz * 8 + z;
    const bool a0 = (C.lm >> (2 * z)) & 1u, a1 = (C.lm >> (2 * z + 1)) & 1u;
    if (dirichlet) {
        if (!sent32(dc.x)) out0 = slow_node32<REACTION>(K, uc.x, dc.x, nu0, nd0, gx, gy, gz, s0, src0);
        if (!sent32(dc.y)) out1 = slow_node32<REACTION>(K, uc.y, dc.y, nu1, nd1, gx + 1, gy, gz, s1, src1);
    } else {
        if (a0 && nonfinite32(out0) && !sent32(dc.x))
            out0 = slow_node32<REACTION>(K, uc.x, dc.x, nu0, nd0, gx, gy, gz, s0, src0);
        if (a1 && nonfinite32(out1) && !sent32(dc.y))
            out1 = slow_node32<REACTION>(K, uc.y, dc.y, nu1, nd1, gx + 1, gy, gz, s1, src1);
    }
    const bool bad0 = a0 && nonfinite32(out0), bad1 = a1 && nonfinite32(out1);
    if (bad0 | bad1) {
        const int o = z * 64 + G.y * 8 + x0;
        atomicMin(M.A.bad_key, ((unsigned long long)C.c << 10) | (unsigned long long)(o + (bad0 ? 0 : 1)));
        atomicOr(M.A.flags + M.A.k, 1);
    }
    return make_float2(out0, out1);
}

// Uniform chunk: every face coefficient is (dv + dv) * 0.5f (compute14u in
// pd_march.cu, in float).
template <int REACTION, bool HALF>
__device__ __forceinline__ void compute32u(const Args32& M, const Slow32& K, const Ctx32& C, int z, uint32_t tm,
                                           uint32_t t0, uint32_t tp, const Geo32& G, float* __restrict__ un) {
    const uint32_t lz = C.lm >> (2 * z);
    const float2 uc = lds2f(t0 + G.s_c);
    const float uL = lds1f(t0 + G.s_l), uR = lds1f(t0 + G.s_r);
    const float2 uym = lds2f(t0 + G.s_c - 32), uyp = lds2f(t0 + G.s_c + 32);
    const float2 uzm = lds2f(tm + G.s_c), uzp = lds2f(tp + G.s_c);
    const float dh = HALF ? C.dv + C.dv : (C.dv + C.dv) * 0.5f;
    const float fxl = dh * (uc.x - uL), fxi = dh * (uc.y - uc.x), fxr = dh * (uR - uc.y);
    const float fy0m = dh * (uc.x - uym.x), fy0p = dh * (uyp.x - uc.x);
    const float fz0m = dh * (uc.x - uzm.x), fz0p = dh * (uzp.x - uc.x);
    const float fy1m = dh * (uc.y - uym.y), fy1p = dh * (uyp.y - uc.y);
    const float fz1m = dh * (uc.y - uzm.y), fz1p = dh * (uzp.y - uc.y);
    const float ix = M.A.inv_dx2[0], iy = M.A.inv_dx2[1], iz = M.A.inv_dx2[2];
    float lap0 = 0.0f;
    lap0 += (fxi - fxl) * ix;
    lap0 += (fy0p - fy0m) * iy;
    lap0 += (fz0p - fz0m) * iz;
    float lap1 = 0.0f;
    lap1 += (fxr - fxi) * ix;
    lap1 += (fy1p - fy1m) * iy;
    lap1 += (fz1p - fz1m) * iz;
    float r0 = 0.0f, r1 = 0.0f;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        r0 = ((lz >> 16) & 1u) ? M.A.neg_k * uc.x : 0.0f;
        r1 = ((lz >> 17) & 1u) ? M.A.neg_k * uc.y : 0.0f;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        const float* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + G.bp;
        r0 = sp[0] * M.A.src_factor;
        r1 = sp[1] * M.A.src_factor;
    }
    const float dt = M.A.dt;
    float out0 = uc.x + dt * lap0 + dt * r0;
    float out1 = uc.y + dt * lap1 + dt * r1;
    if (nonfinite32(out0) | nonfinite32(out1)) {
        const float2 r = slow_pair32<REACTION, HALF>(M, K, C, z, tm, t0, tp, G, out0, out1);
        out0 = r.x;
        out1 = r.y;
    }
    stg2f(un + ((uint32_t)C.c * 512u + (uint32_t)z * 64u + G.bp), out0, out1, true, true);
}

template <int REACTION, bool HALF>
__device__ __forceinline__ void compute32(const Args32& M, const Slow32& K, const Ctx32& C, int z, uint32_t tm,
                                          uint32_t t0, uint32_t tp, const Geo32& G, float* __restrict__ un) {
    if (C.flags & kFlagUnif32) {  // warp-uniform
        compute32u<REACTION, HALF>(M, K, C, z, tm, t0, tp, G, un);
        return;
    }
    const uint32_t lz = C.lm >> (2 * z);
    const bool a0 = lz & 1u, a1 = (lz >> 1) & 1u;
    const float2 uc = lds2f(t0 + G.s_c), dc = lds2f(t0 + kDOff32 + G.s_c);
    const float uL = lds1f(t0 + G.s_l), dL = lds1f(t0 + kDOff32 + G.s_l);
    const float uR = lds1f(t0 + G.s_r), dR = lds1f(t0 + kDOff32 + G.s_r);
    const float2 uym = lds2f(t0 + G.s_c - 32), dym = lds2f(t0 + kDOff32 + G.s_c - 32);
    const float2 uyp = lds2f(t0 + G.s_c + 32), dyp = lds2f(t0 + kDOff32 + G.s_c + 32);
    const float2 uzm = lds2f(tm + G.s_c), dzm = lds2f(tm + kDOff32 + G.s_c);
    const float2 uzp = lds2f(tp + G.s_c), dzp = lds2f(tp + kDOff32 + G.s_c);
    float fxl, fxi, fxr, fy0m, fy0p, fz0m, fz0p, fy1m, fy1p, fz1m, fz1p;
    const bool interior = (C.flags >> (8 + z)) & 1;
    if (interior) {
        fxl = fface32<HALF>(dL, dc.x, uL, uc.x);
        fxi = fface32<HALF>(dc.x, dc.y, uc.x, uc.y);
        fxr = fface32<HALF>(dc.y, dR, uc.y, uR);
        fy0m = fface32<HALF>(dym.x, dc.x, uym.x, uc.x);
        fy0p = fface32<HALF>(dc.x, dyp.x, uc.x, uyp.x);
        fz0m = fface32<HALF>(dzm.x, dc.x, uzm.x, uc.x);
        fz0p = fface32<HALF>(dc.x, dzp.x, uc.x, uzp.x);
        fy1m = fface32<HALF>(dym.y, dc.y, uym.y, uc.y);
        fy1p = fface32<HALF>(dc.y, dyp.y, uc.y, uyp.y);
        fz1m = fface32<HALF>(dzm.y, dc.y, uzm.y, uc.y);
        fz1p = fface32<HALF>(dc.y, dzp.y, uc.y, uzp.y);
    } else {
        fxl = face32<HALF>(dL, dc.x, uL, uc.x);
        fxi = face32<HALF>(dc.x, dc.y, uc.x, uc.y);
        fxr = face32<HALF>(dc.y, dR, uc.y, uR);
        fy0m = face32<HALF>(dym.x, dc.x, uym.x, uc.x);
        fy0p = face32<HALF>(dc.x, dyp.x, uc.x, uyp.x);
        fz0m = face32<HALF>(dzm.x, dc.x, uzm.x, uc.x);
        fz0p = face32<HALF>(dc.x, dzp.x, uc.x, uzp.x);
        fy1m = face32<HALF>(dym.y, dc.y, uym.y, uc.y);
        fy1p = face32<HALF>(dc.y, dyp.y, uc.y, uyp.y);
        fz1m = face32<HALF>(dzm.y, dc.y, uzm.y, uc.y);
        fz1p = face32<HALF>(dc.y, dzp.y, uc.y, uzp.y);
    }
    const float ix = M.A.inv_dx2[0], iy = M.A.inv_dx2[1], iz = M.A.inv_dx2[2];
    float lap0 = 0.0f;  // T lap = T(0) (solver.hpp:420)
    lap0 += (fxi - fxl) * ix;
    lap0 += (fy0p - fy0m) * iy;
    lap0 += (fz0p - fz0m) * iz;
    float lap1 = 0.0f;
    lap1 += (fxr - fxi) * ix;
    lap1 += (fy1p - fy1m) * iy;
    lap1 += (fz1p - fz1m) * iz;
    float r0 = 0.0f, r1 = 0.0f;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        r0 = ((lz >> 16) & 1u) ? M.A.neg_k * uc.x : 0.0f;
        r1 = ((lz >> 17) & 1u) ? M.A.neg_k * uc.y : 0.0f;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        const float* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + G.bp;
        r0 = sp[0] * M.A.src_factor;
        r1 = sp[1] * M.A.src_factor;
    }
    const float dt = M.A.dt;
    float out0 = uc.x + dt * lap0 + dt * r0;
    float out1 = uc.y + dt * lap1 + dt * r1;
    if (!interior) {  // walls stay frozen (solver.hpp:413-417)
        if (sent32(dc.x)) out0 = uc.x;
        if (sent32(dc.y)) out1 = uc.y;
    }
    if ((C.flags & kFlagDir32) || ((a0 && nonfinite32(out0)) | (a1 && nonfinite32(out1)))) {
        const float2 r = slow_pair32<REACTION, HALF>(M, K, C, z, tm, t0, tp, G, out0, out1);
        out0 = r.x;
        out1 = r.y;
    }
    stg2f(un + ((uint32_t)C.c * 512u + (uint32_t)z * 64u + G.bp), out0, out1, a0, a1);
}

template <int REACTION, bool HALF>
__global__ void __launch_bounds__(kT32, kCtas32) ftcs_march32_kernel(Args32 M) {
    extern __shared__ __align__(16) unsigned char smem32[];
    __shared__ Slow32 K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<float>& A = M.A;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    if (t == 0) {
        for (int a = 0; a < 3; ++a) {
            K.size[a] = A.size[a];
            K.inv_dx2[a] = A.inv_dx2[a];
        }
        for (int f = 0; f < 6; ++f) K.bcv[f] = A.bcv[f];
        K.dt = A.dt;
        K.neg_k = A.neg_k;
        K.src_factor = A.src_factor;
        K.dirichlet = A.dirichlet;
    }
    __syncthreads();
    Geo32 G = geo32(lane);
#ifndef PD_M32_NOPIN
    // opaque copies: ptxas cannot rematerialise a shuffle result inside the
    // plane loop, so the lane constants stay in registers
    G.s_c = __shfl_sync(0xffffffffu, G.s_c, lane);
    G.s_l = __shfl_sync(0xffffffffu, G.s_l, lane);
    G.s_r = __shfl_sync(0xffffffffu, G.s_r, lane);
    G.s_hx = __shfl_sync(0xffffffffu, G.s_hx, lane);
    G.s_hy = __shfl_sync(0xffffffffu, G.s_hy, lane);
    G.bp = __shfl_sync(0xffffffffu, G.bp, lane);
#endif
    uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem32) + (uint32_t)warp * kWarpBytes32;
#ifndef PD_NOPIN2
    sb = __shfl_sync(0xffffffffu, sb, lane);
    G.xface = __shfl_sync(0xffffffffu, (int)G.xface, lane) != 0;
    G.yface = __shfl_sync(0xffffffffu, (int)G.yface, lane) != 0;
#endif
    const float* __restrict__ u = A.u;
    const float* __restrict__ de = M.deff;
    float* __restrict__ un = A.un;
    const uint32_t sent_off = (uint32_t)M.n_all * 512u;

    // claim -> id -> masks / descriptor pipeline through a 3-entry context
    // ring in shared memory (ftcs_march14_kernel)
    int* ctr_l = M.counter + ((t >> 5) & M.zero);
    const int n = (int)M.n;
    const uint32_t cb = sb + kRing32 * kTile32;
    auto cent = [&](int e) -> uint32_t { return cb + (uint32_t)e * kCtx32; };
    int raw = 0;
    auto claim = [&]() {
        if (lane == 0) asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(raw) : "l"(ctr_l) : "memory");
    };
    auto sched_sync = [&]() -> int {
        claim();
        const int p = __shfl_sync(0xffffffffu, raw, 0);
        return p < n ? __ldg(&M.sched[p]) : -1;
    };
    auto fetch = [&](uint32_t e, int c) {
        const int64_t cc = c < 0 ? 0 : c;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(
                e + 4u * (uint32_t)lane),
            "l"(M.lm + cc * 32 + lane), "r"((int)(c >= 0)));
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(
                e + 128u + 4u * (uint32_t)(lane & 7)),
            "l"(M.desc + cc * 8 + (lane & 7)), "r"((int)(c >= 0 && lane < 8)));
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(
                e + 164u),
            "l"(M.dv + cc), "r"((int)(c >= 0 && lane == 0)));
    };
    {
        const int id0 = sched_sync();
        if (id0 < 0) return;
        const int id1 = sched_sync();
        if (lane == 0) {
            stsu(cent(0) + 160u, (uint32_t)id0);
            stsu(cent(1) + 160u, (uint32_t)id1);
        }
        fetch(cent(0), id0);
        cp_commit32();
        cp_wait32<0>();
        __syncwarp();
        claim();
    }
    int ek = 0;
    Ctx32 Cld;
    Load32 Lld;
    auto advance = [&]() {
        const uint32_t e0 = cent(ek);
        const int e1i = ek == 2 ? 0 : ek + 1, e2i = e1i == 2 ? 0 : e1i + 1;
        const uint32_t e1 = cent(e1i), e2 = cent(e2i);
        const int c = (int)ldsu(e0 + 160u);
        const uint32_t lm = c >= 0 ? ldsu(e0 + 4u * (uint32_t)lane) : 0u;
        const int dv = (int)ldsu(e0 + 128u + 4u * (uint32_t)(lane >= 24 ? lane - 24 : 0));
        Cld = Ctx32{c, __shfl_sync(0xffffffffu, dv, 30), __shfl_sync(0xffffffffu, dv, 31), lm, lds1f(e0 + 164u)};
        Lld = load_ctx32(c, lm, c >= 0 ? dv : -1, G);
        fetch(e1, (int)ldsu(e1 + 160u));
        if (lane == 0) {
            const bool ok = raw < n;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(
                    e2 + 160u),
                "l"(M.sched + (ok ? raw : 0)), "r"((int)ok));
            if (!ok) stsu(e2 + 160u, 0xFFFFFFFFu);
        }
        claim();
        ek = e1i;
    };
    advance();
    int p_ld = 0;
    uint32_t Lc = 0;
    auto issue_next = [&]() {
        issue32(sb + (Lc & (kRing32 - 1)) * kTile32, u, de, Lld, p_ld, G, sent_off);
        if (++p_ld == 10) {
            p_ld = 0;
            advance();
        }
        cp_commit32();
        ++Lc;
    };
    Ctx32 Cc = Cld;
    uint32_t base = 0;
#pragma unroll 1
    for (int k = 0; k < 3 + kAhead32; ++k) issue_next();
#pragma unroll 1
    while (Cc.c >= 0) {
#pragma unroll 1
        for (int z = 0; z < 8; ++z) {
            cp_wait32<kAhead32>();
            __syncwarp();
            const uint32_t b = base + (uint32_t)z;
            compute32<REACTION, HALF>(M, K, Cc, z, sb + (b & 7u) * kTile32, sb + ((b + 1u) & 7u) * kTile32,
                                sb + ((b + 2u) & 7u) * kTile32, G, un);
            __syncwarp();
            issue_next();
            if (z == 7) {
                issue_next();
                issue_next();
            }
        }
        base += 10u;
        Cc = Cld;
    }
    cp_wait32<0>();
}

__global__ void deff32_kernel(const float* __restrict__ dcol, const uint64_t* __restrict__ fluid, int64_t n_slots,
                              float* __restrict__ deff, unsigned long long* bad, int half) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_slots + 512) return;
    if (i >= n_slots) {  // the sentinel chunk after the last one
        deff[i] = __uint_as_float(kSent32);
        return;
    }
    const bool fl = (fluid[i >> 6] >> (i & 63)) & 1ull;
    const float v = dcol[i];
    deff[i] = fl ? (half ? v * 0.5f : v) : __uint_as_float(kSent32);
    if (fl && !isfinite(v)) atomicAdd(bad, 1ull);
    // halving would not be exact (tiny D), or the reference's d_a + d_b could
    // overflow where h_a + h_b does not (huge D)
    if (fl && (fabsf(v) < 0x1p-125f || fabsf(v) >= 0x1p126f)) atomicAdd(bad + 1, 1ull);
}

}  // namespace

// D_eff of a float grid (+ trailing sentinel chunk); returns false if a fluid
// node has a non-finite D (the exact tile kernel is kept then).
bool march32_deff(pd_grid* g, const void* d_dcol, const uint64_t* d_fluid, void** out, bool* half) {
    const int64_t slots = g->n_chunks * 512;
    float* p = nullptr;
    PD_CUDA(pd_malloc(&p, sizeof(float) * (size_t)(slots + 512)));
    unsigned long long* d_bad = nullptr;
    PD_CUDA(pd_malloc(&d_bad, 2 * sizeof(unsigned long long)));
    static const int half_env = [] {
        const char* e = getenv("PD_MARCH_HALF");
        return e ? atoi(e) : 1;
    }();
    unsigned long long bad[2] = {0, 0};
    for (int pass = 0; pass < 2; ++pass) {  // second pass only when a tiny D forbids halving
        const int h = pass == 0 ? half_env : 0;
        PD_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(unsigned long long), g->stream));
        deff32_kernel<<<(unsigned)((slots + 512 + 255) / 256), 256, 0, g->stream>>>((const float*)d_dcol, d_fluid,
                                                                                   slots, p, d_bad, h);
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cudaMemcpyAsync(bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        *half = h && !bad[1];
        if (bad[0] || !h || !bad[1]) break;
    }
    pd_free(d_bad);
    if (bad[0]) {
        pd_free(p);
        return false;
    }
    *out = p;
    return true;
}

void march32_launch_sched(pd_grid* g, MarchPlan& p, const StepArgs<float>& a, int reaction, const int32_t* sched,
                          int64_t n, int* counter) {
    Args32 M;
    M.A = a;
    M.sched = sched;
    M.n = n;
    M.desc = p.d_desc;
    M.lm = p.d_lm;
    M.deff = static_cast<const float*>(p.d_deff);
    M.dv = static_cast<const float*>(p.d_dv);
    M.counter = counter;
    M.zero = 0;
    M.n_all = g->n_chunks;
    using KernT = void (*)(Args32);
    static const KernT table[2][3] = {
        {ftcs_march32_kernel<0, false>, ftcs_march32_kernel<1, false>, ftcs_march32_kernel<2, false>},
        {ftcs_march32_kernel<0, true>, ftcs_march32_kernel<1, true>, ftcs_march32_kernel<2, true>}};
    constexpr size_t bytes = (size_t)kWarpBytes32 * kW32;
    // the dynamic shared-memory opt-in is per device: set it once per device
    static uint64_t attr_done = 0;
    if (g->device < 0 || g->device >= 64) fail(PD_E_INPUT, "device index out of range");
    if (!((attr_done >> g->device) & 1u)) {
        for (auto& row : table)
            for (auto k : row) PD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        attr_done |= 1ull << g->device;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    const int r = reaction == PD_REACTION_SURFACE_SINK ? 1 : reaction == PD_REACTION_VOLUMETRIC ? 2 : 0;
    table[p.half ? 1 : 0][r]<<<sms * kCtas32, kT32, bytes, g->stream>>>(M);
    PD_CUDA(cudaGetLastError());
}

void march32_launch(pd_grid* g, MarchPlan& p, const StepArgs<float>& a, int reaction) {
    march32_launch_sched(g, p, a, reaction, p.d_stream, p.n, p.d_counter + (a.k & 1023));
}

}  // namespace pdb
