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
#include "pd_async.cuh"

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
    int dbg;  // measurement only (PD_MARCH_DBG): 8 = compute warps release every stage unread
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
// shared-memory addresses (u side; D_eff at +DH) of a pair's operands
struct Addr32 {
    uint32_t c, l, r, ym, yp, zm, zp;
};

template <int REACTION, bool HALF, uint32_t DH>
__device__ __noinline__ float2 slow_pair32a(const Args32& M, const Slow32& K, const Ctx32& C, int z, const Geo32& G,
                                            Addr32 a, float out0, float out1) {
    const bool un = (C.flags & kFlagUnif32) != 0;  // no D_eff staged: every d is dv
    const float2 vv = make_float2(C.dv, C.dv);
    const float2 uc = lds2f(a.c), dc0 = un ? vv : lds2f(a.c + DH);
    const float uL = lds1f(a.l), dL0 = un ? C.dv : lds1f(a.l + DH);
    const float uR = lds1f(a.r), dR0 = un ? C.dv : lds1f(a.r + DH);
    const float2 uym = lds2f(a.ym), dym0 = un ? vv : lds2f(a.ym + DH);
    const float2 uyp = lds2f(a.yp), dyp0 = un ? vv : lds2f(a.yp + DH);
    const float2 uzm = lds2f(a.zm), dzm0 = un ? vv : lds2f(a.zm + DH);
    const float2 uzp = lds2f(a.zp), dzp0 = un ? vv : lds2f(a.zp + DH);
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

// the ring-tile rare path of ftcs_march32_kernel
template <int REACTION, bool HALF>
__device__ __forceinline__ float2 slow_pair32(const Args32& M, const Slow32& K, const Ctx32& C, int z, uint32_t tm,
                                              uint32_t t0, uint32_t tp, const Geo32& G, float out0, float out1) {
    Addr32 a;
    a.c = t0 + G.s_c;
    a.l = t0 + G.s_l;
    a.r = t0 + G.s_r;
    a.ym = t0 + G.s_c - 32;
    a.yp = t0 + G.s_c + 32;
    a.zm = tm + G.s_c;
    a.zp = tp + G.s_c;
    return slow_pair32a<REACTION, HALF, kDOff32>(M, K, C, z, G, a, out0, out1);
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

// ---------------------------------------------------------------------------
// FP32 v43: the FP64 march v43 design (pd_march.cu) in float.
// * CTA = 4 compute warps + 1 producer warp; the producer claims chunks four
//   at a time and moves each chunk with per-lane cp.async into a padded stage
//   (u half; D_eff at +kHalf32b): 10 planes z = -1..8 at a 320-B pitch (rows
//   y = -1..8 of 32 B), then the x- halo block [z][y] (4-B cells) and, 32 B
//   further (other banks), the x+ block; the 176-B chunk record is one bulk
//   copy. Completion: lane 0's expect_tx + 32 cp.async arrivals on the
//   stage's "full" mbarrier; the compute warps release it on "empty".
// * Compute warp w: planes 2w, 2w+1; lane (y, xp): the x pair (2xp, 2xp+1)
//   of row y as one 8-B word. z / y neighbours at -+320 / -+32 from the own
//   pair, x neighbours by shuffle (face lanes: the halo cell); both planes in
//   one straight-line block on a warp-uniform path (uniform chunk /
//   interior-fluid planes / generic); one vote for the rare path
//   (Dirichlet-exposed chunk or a non-finite result).
// * float arithmetic in the reference's order (ftcs_march32_kernel's
//   expressions): bitwise equal to the reference's T = float path.
// ---------------------------------------------------------------------------
constexpr uint32_t kPP32b = 320;                              // plane pitch
constexpr uint32_t kXL32b = 10 * kPP32b, kXH32b = kXL32b + 288;  // x-halo blocks [z][y]
constexpr uint32_t kHalf32b = kXH32b + 256;                   // D_eff half (3744)
constexpr uint32_t kCtx32b = 2 * kHalf32b;                    // record; chunk id at +176
constexpr uint32_t kStage32b = kCtx32b + 256;                 // 7744
constexpr int kW32b = 4, kB32b = 4;
constexpr int kThreads32b = 32 * (kW32b + 1);
// configurations: CTAs per SM and stages per CTA
__host__ __device__ constexpr int ctas32b(int cfg) { return cfg == 1 ? 5 : cfg == 2 ? 4 : 6; }
__host__ __device__ constexpr int nst32b(int cfg) { return cfg == 0 ? 3 : 4; }
__host__ __device__ constexpr int maxreg32b(int cfg) {
    return 16384 / (32 * ((kThreads32b / 32 * ctas32b(cfg) + 3) / 4)) / 8 * 8;
}
__host__ __device__ constexpr uint32_t smem32b(int cfg) { return nst32b(cfg) * kStage32b + 16u * nst32b(cfg); }

template <int REACTION, bool HALF>
__device__ __noinline__ float2 pair_slow32b(const Args32& M, const Slow32& K, uint32_t st, int lane, int z, float out0,
                                            float out1) {
    Ctx32 C;
    C.c = (int)ldsu(st + kCtx32b + 176u);
    C.lm = ldsu(st + kCtx32b + 4u * (uint32_t)lane);
    C.key = (int)ldsu(st + kCtx32b + 152u);
    C.flags = (int)ldsu(st + kCtx32b + 156u);
    C.dv = lds1f(st + kCtx32b + 160u);
    Geo32 G = geo32(lane);
    const uint32_t zz = (uint32_t)z, pz = st + (zz + 1u) * kPP32b;
    Addr32 a;
    a.c = pz + (uint32_t)(G.y + 1) * 32u + 8u * (uint32_t)G.xp;
    a.zm = a.c - kPP32b;
    a.zp = a.c + kPP32b;
    a.ym = a.c - 32u;
    a.yp = a.c + 32u;
    a.l = G.xp > 0 ? a.c - 4u : st + kXL32b + zz * 32u + 4u * (uint32_t)G.y;
    a.r = G.xp < 3 ? a.c + 8u : st + kXH32b + zz * 32u + 4u * (uint32_t)G.y;
    return slow_pair32a<REACTION, HALF, kHalf32b>(M, K, C, z, G, a, out0, out1);
}

template <int REACTION>
__device__ __forceinline__ float node32b(float dt, float neg_k, float sfac, float ix, float iy, float iz, float uc,
                                         float fxm, float fxp, float fym, float fyp, float fzm, float fzp, bool sink,
                                         float src) {
    float lap = 0.0f;  // T lap = T(0) (solver.hpp:420)
    lap += (fxp - fxm) * ix;
    lap += (fyp - fym) * iy;
    lap += (fzp - fzm) * iz;
    float r = 0.0f;
    if (REACTION == PD_REACTION_SURFACE_SINK) r = sink ? neg_k * uc : 0.0f;
    else if (REACTION == PD_REACTION_VOLUMETRIC) r = src * sfac;
    return uc + dt * lap + dt * r;
}

// u + dt * lap of one node in float (the reaction term is added per warp)
__device__ __forceinline__ float node32bx(float dt, float ix, float iy, float iz, float uc, float fxm, float fxp,
                                          float fym, float fyp, float fzm, float fzp) {
    float lap = 0.0f;  // T lap = T(0) (solver.hpp:420)
    lap += (fxp - fxm) * ix;
    lap += (fyp - fym) * iy;
    lap += (fzp - fzm) * iz;
    return uc + dt * lap;
}

template <int REACTION, bool HALF, int CFG>
__global__ void __maxnreg__(maxreg32b(CFG)) ftcs_march32b_kernel(const __grid_constant__ Args32 M,
                                                                  const uint32_t* __restrict__ ctxa) {
    extern __shared__ __align__(128) unsigned char smem32b_raw[];
    __shared__ Slow32 K;
    constexpr int kSt = nst32b(CFG);
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
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem32b_raw);
    const uint32_t full0 = sm0 + kSt * kStage32b, empty0 = full0 + 8u * kSt;
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
        for (int s = 0; s < kSt; ++s) {
            mbar_init(full0 + 8u * s, 33u);  // lane 0's expect_tx arrive + 32 cp.async arrivals
            mbar_init(empty0 + 8u * s, (uint32_t)kW32b);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const float* __restrict__ u = A.u;
    const float* __restrict__ de = M.deff;
    const int n = (int)M.n;

    if (warp == kW32b) {  // ---------------- producer warp ----------------
        int* ctr = M.counter;
        const int4* desc4 = reinterpret_cast<const int4*>(M.desc);
        const uint32_t sent_off = (uint32_t)M.n_all * 512u;  // D_eff sentinel chunk (elements)
        auto claim = [&]() -> int {
            int r = 0;
            if (lane == 0)
                asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(ctr), "r"(kB32b) : "memory");
            return r;
        };
        auto entries = [&](int p0) -> int {
            const int p = __shfl_sync(0xffffffffu, p0, 0) + lane;
            return lane < kB32b && p < n ? __ldg(&M.sched[p]) : -1;
        };
        auto chunk_of = [](int e) { return e == -1 ? -1 : (int)((uint32_t)e & 0x7FFFFFFFu); };
        auto descs = [&](int e, int4& d0, int4& d1) {
            const int c = chunk_of(e);
            if (lane < kB32b && c >= 0) {
                d0 = __ldg(desc4 + 2 * (int64_t)c);
                d1 = __ldg(desc4 + 2 * (int64_t)c + 1);
            }
        };
        auto prefetch = [&](int e) {  // the batch's u slabs and records into L2
            const int64_t c = (int64_t)chunk_of(e);
            if (lane < kB32b && c >= 0) {
                prefetch_l2(u + c * 512, 2048u);
                prefetch_l2(ctxa + c * 44, 176u);
            }
        };
        int e_c = entries(claim());
        int e_n = entries(claim());
        int p_nn = claim();
        int4 d0c = make_int4(0, 0, 0, 0), d1c = d0c;
        descs(e_c, d0c, d1c);
        prefetch(e_c);
        const uint32_t L = (uint32_t)lane;
        // own slab: 16-B pieces p = L + 32 i -> plane 2 i + L / 16, row (L % 16) / 2, half L % 2
        const uint32_t d_own = ((L >> 4) + 1u) * kPP32b + (((L & 15u) >> 1) + 1u) * 32u + 16u * (L & 1u);
        // z halos: lanes 0-15 the z- neighbour's plane 7 -> plane -1, lanes 16-31 the z+ one's plane 0 -> plane 8
        const bool zh = L >= 16u;
        const uint32_t Lq = L & 15u;
        const uint32_t d_z = (zh ? 9u * kPP32b : 0u) + 32u + 16u * Lq, s_z = (zh ? 0u : 448u) + 4u * Lq;
        // y halos: lanes 0-15 row 7 of the y- neighbour -> row -1, lanes 16-31 row 0 of the y+ one -> row 8
        const uint32_t d_y = ((Lq >> 1) + 1u) * kPP32b + (zh ? 288u : 0u) + 16u * (L & 1u);
        const uint32_t s_y = (Lq >> 1) * 64u + (zh ? 0u : 56u) + 4u * (L & 1u);
        uint32_t s = 0, ph = 0, k = 0;
#pragma unroll 1
        for (;;) {
            int4 d0n = make_int4(0, 0, 0, 0), d1n = d0n;
            descs(e_n, d0n, d1n);
            prefetch(e_n);
            const int e_nn = entries(p_nn);
            p_nn = claim();
            bool done = false;
#pragma unroll 1
            for (int j = 0; j < kB32b; ++j, ++k) {
                const int c_cur = chunk_of(__shfl_sync(0xffffffffu, e_c, j));
                const uint32_t st = sm0 + s * kStage32b, full = full0 + 8u * s;
                if (k >= (uint32_t)kSt) mbar_wait(empty0 + 8u * s, ph ^ 1u);
                if (c_cur < 0) {  // end marker
                    if (lane == 0) {
                        sts_u32(st + kCtx32b + 176u, 0xFFFFFFFFu);
                        mbar_arrive(full);
                    }
                    cp_mbar_arrive_noinc(full);
                    done = true;
                    break;
                }
                const int nb0 = __shfl_sync(0xffffffffu, d0c.x, j), nb1 = __shfl_sync(0xffffffffu, d0c.y, j);
                const int nb2 = __shfl_sync(0xffffffffu, d0c.z, j), nb3 = __shfl_sync(0xffffffffu, d0c.w, j);
                const int nb4 = __shfl_sync(0xffffffffu, d1c.x, j), nb5 = __shfl_sync(0xffffffffu, d1c.y, j);
                const bool dl = !(__shfl_sync(0xffffffffu, d1c.w, j) & kFlagUnif32);
                if (lane == 0) {
                    sts_u32(st + kCtx32b + 176u, (uint32_t)c_cur);
                    mbar_arrive_tx(full, 176u);
                    bulk_g2s(st + kCtx32b, ctxa + (int64_t)c_cur * 44, 176u, full);
                }
                const uint32_t so = (uint32_t)c_cur * 512u + 4u * L;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    cp16(st + d_own + 640u * (uint32_t)i, u + so + 128 * i, true);
                    cp16(st + kHalf32b + d_own + 640u * (uint32_t)i, de + so + 128 * i, dl);
                }
                {
                    const int nz = zh ? nb5 : nb4;
                    const uint32_t oz = (uint32_t)nz * 512u + s_z;
                    cp16(st + d_z, u + (nz >= 0 ? oz : 0u), nz >= 0);
                    cp16(st + kHalf32b + d_z, de + (nz >= 0 ? oz : sent_off + s_z), dl);
                    const int ny = zh ? nb3 : nb2;
                    const uint32_t oy = (uint32_t)ny * 512u + s_y;
                    cp16(st + d_y, u + (ny >= 0 ? oy : 0u), ny >= 0);
                    cp16(st + kHalf32b + d_y, de + (ny >= 0 ? oy : sent_off + s_y), dl);
                }
                {  // x halos: cells (z, y) = L, L + 32 of column 7 of the x- / column 0 of the x+ neighbour
                    const uint32_t xl = (uint32_t)nb0 * 512u + 8u * L + 7u, xh = (uint32_t)nb1 * 512u + 8u * L;
                    const uint32_t xs = sent_off + 8u * L;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const uint32_t o = 256u * (uint32_t)jj;  // +32 cells: 8 elements each
                        cpa(st + kXL32b + 4u * L + 128u * (uint32_t)jj, u + (nb0 >= 0 ? xl + o : 0u), 0, nb0 >= 0);
                        cpa(st + kXH32b + 4u * L + 128u * (uint32_t)jj, u + (nb1 >= 0 ? xh + o : 0u), 0, nb1 >= 0);
                        cpa(st + kHalf32b + kXL32b + 4u * L + 128u * (uint32_t)jj, de + (nb0 >= 0 ? xl + o : xs + o), 0, dl);
                        cpa(st + kHalf32b + kXH32b + 4u * L + 128u * (uint32_t)jj, de + (nb1 >= 0 ? xh + o : xs + o), 0, dl);
                    }
                }
                cp_mbar_arrive_noinc(full);
                if (++s == (uint32_t)kSt) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (done) break;
            e_c = e_n;
            d0c = d0n;
            d1c = d1n;
            e_n = e_nn;
        }
        return;
    }

    // ---------------- compute warps ----------------
    if (M.dbg & 8) {  // measurement only: the copy pipeline alone
        uint32_t s = 0, ph = 0;
        for (;;) {
            mbar_wait(full0 + 8u * s, ph);
            if ((int)ldsu(sm0 + s * kStage32b + kCtx32b + 176u) < 0) break;
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8u * s);
            if (++s == (uint32_t)kSt) {
                s = 0;
                ph ^= 1u;
            }
        }
        return;
    }
    const float dt = A.dt, neg_k = A.neg_k, sfac = A.src_factor;
    const bool dt_fin = isfinite(dt);  // the float dt (positive; inf only if the double dt exceeds FLT_MAX)
    const float ix = A.inv_dx2[0], iy = A.inv_dx2[1], iz = A.inv_dx2[2];
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t z0 = 2u * (uint32_t)warp;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp);
    const uint32_t o_c = pin((z0 + 1u) * kPP32b + (uint32_t)(y + 1) * 32u + 8u * (uint32_t)xp, lane);
    const uint32_t o_x = pin((xp == 3 ? kXH32b : kXL32b) + z0 * 32u + 4u * (uint32_t)y, lane);
    const bool xlo = xp == 0, xhi = xp == 3;
    const uint32_t zsh = 2u * z0;
    float* __restrict__ un = A.un;
    uint32_t s = 0, ph = 0;
#pragma unroll 1
    for (;;) {
        mbar_wait(full0 + 8u * s, ph);
        const uint32_t st = sm0 + s * kStage32b;
        const int c = (int)ldsu(st + kCtx32b + 176u);
        if (c < 0) break;
        const uint32_t lm = ldsu(st + kCtx32b + 4u * (uint32_t)lane);
        const int flags = (int)ldsu(st + kCtx32b + 156u);
        const uint32_t ab = (lm >> zsh) & 0xFu;
        const uint32_t sk = (lm >> (16u + zsh)) & 0xFu;
        const uint32_t g_off = z0 * 64u + bp;
        float src[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (REACTION == PD_REACTION_VOLUMETRIC) {
            const float* sp = A.src + (int64_t)c * 512 + g_off;
            src[0] = sp[0];
            src[1] = sp[1];
            src[2] = sp[64];
            src[3] = sp[65];
        }
        const uint32_t a = st + o_c, ax = st + o_x;
        const float2 uc0 = lds2f(a), uc1 = lds2f(a + kPP32b);
        const float2 uzm = lds2f(a - kPP32b), uzp = lds2f(a + 2u * kPP32b);
        const float2 uym0 = lds2f(a - 32u), uyp0 = lds2f(a + 32u);
        const float2 uym1 = lds2f(a + kPP32b - 32u), uyp1 = lds2f(a + kPP32b + 32u);
        const float uh0 = lds1f(ax), uh1 = lds1f(ax + 32u);
        const float su0 = __shfl_up_sync(0xffffffffu, uc0.y, 1), sd0 = __shfl_down_sync(0xffffffffu, uc0.x, 1);
        const float su1 = __shfl_up_sync(0xffffffffu, uc1.y, 1), sd1 = __shfl_down_sync(0xffffffffu, uc1.x, 1);
        const float uL0 = xlo ? uh0 : su0, uR0 = xhi ? uh0 : sd0;
        const float uL1 = xlo ? uh1 : su1, uR1 = xhi ? uh1 : sd1;
        float o00, o01, o10, o11;  // u + dt * lap first, the reaction term below
        bool w00 = false, w01 = false, w10 = false, w11 = false;
        const uint32_t ib = ((uint32_t)flags >> (8u + z0)) & 3u;
        if (flags & kFlagUnif32) {
            const float dv = lds1f(st + kCtx32b + 160u);
            const float dh = HALF ? dv + dv : (dv + dv) * 0.5f;
            const float fzx = dh * (uc1.x - uc0.x), fzy = dh * (uc1.y - uc0.y);
            const float f0i = dh * (uc0.y - uc0.x), f1i = dh * (uc1.y - uc1.x);
            o00 = node32bx(dt, ix, iy, iz, uc0.x, dh * (uc0.x - uL0), f0i, dh * (uc0.x - uym0.x),
                                    dh * (uyp0.x - uc0.x), dh * (uc0.x - uzm.x), fzx);
            o01 = node32bx(dt, ix, iy, iz, uc0.y, f0i, dh * (uR0 - uc0.y), dh * (uc0.y - uym0.y),
                                    dh * (uyp0.y - uc0.y), dh * (uc0.y - uzm.y), fzy);
            o10 = node32bx(dt, ix, iy, iz, uc1.x, dh * (uc1.x - uL1), f1i, dh * (uc1.x - uym1.x),
                                    dh * (uyp1.x - uc1.x), fzx, dh * (uzp.x - uc1.x));
            o11 = node32bx(dt, ix, iy, iz, uc1.y, f1i, dh * (uR1 - uc1.y), dh * (uc1.y - uym1.y),
                                    dh * (uyp1.y - uc1.y), fzy, dh * (uzp.y - uc1.y));
        } else {
            const uint32_t b = a + kHalf32b, bx = ax + kHalf32b;
            const float2 dc0 = lds2f(b), dc1 = lds2f(b + kPP32b);
            const float2 dzm = lds2f(b - kPP32b), dzp = lds2f(b + 2u * kPP32b);
            const float2 dym0 = lds2f(b - 32u), dyp0 = lds2f(b + 32u);
            const float2 dym1 = lds2f(b + kPP32b - 32u), dyp1 = lds2f(b + kPP32b + 32u);
            const float dh0 = lds1f(bx), dh1 = lds1f(bx + 32u);
            const float tu0 = __shfl_up_sync(0xffffffffu, dc0.y, 1), td0 = __shfl_down_sync(0xffffffffu, dc0.x, 1);
            const float tu1 = __shfl_up_sync(0xffffffffu, dc1.y, 1), td1 = __shfl_down_sync(0xffffffffu, dc1.x, 1);
            const float dL0 = xlo ? dh0 : tu0, dR0 = xhi ? dh0 : td0;
            const float dL1 = xlo ? dh1 : tu1, dR1 = xhi ? dh1 : td1;
#define PD_F32B(F)                                                                                                  \
    {                                                                                                               \
        const float fzx = F(dc0.x, dc1.x, uc0.x, uc1.x), fzy = F(dc0.y, dc1.y, uc0.y, uc1.y);                       \
        const float f0i = F(dc0.x, dc0.y, uc0.x, uc0.y), f1i = F(dc1.x, dc1.y, uc1.x, uc1.y);                       \
        o00 = node32bx(dt, ix, iy, iz, uc0.x, F(dL0, dc0.x, uL0, uc0.x), f0i,                  \
                                F(dym0.x, dc0.x, uym0.x, uc0.x), F(dc0.x, dyp0.x, uc0.x, uyp0.x),                    \
                                F(dzm.x, dc0.x, uzm.x, uc0.x), fzx);                                \
        o01 = node32bx(dt, ix, iy, iz, uc0.y, f0i, F(dc0.y, dR0, uc0.y, uR0),                  \
                                F(dym0.y, dc0.y, uym0.y, uc0.y), F(dc0.y, dyp0.y, uc0.y, uyp0.y),                    \
                                F(dzm.y, dc0.y, uzm.y, uc0.y), fzy);                                \
        o10 = node32bx(dt, ix, iy, iz, uc1.x, F(dL1, dc1.x, uL1, uc1.x), f1i,                  \
                                F(dym1.x, dc1.x, uym1.x, uc1.x), F(dc1.x, dyp1.x, uc1.x, uyp1.x), fzx,               \
                                F(dc1.x, dzp.x, uc1.x, uzp.x));                                     \
        o11 = node32bx(dt, ix, iy, iz, uc1.y, f1i, F(dc1.y, dR1, uc1.y, uR1),                  \
                                F(dym1.y, dc1.y, uym1.y, uc1.y), F(dc1.y, dyp1.y, uc1.y, uyp1.y), fzy,               \
                                F(dc1.y, dzp.y, uc1.y, uzp.y));                                     \
    }
            if (ib == 3u) {
                PD_F32B(fface32<HALF>)
            } else {
                PD_F32B(face32<HALF>)
                w00 = sent32(dc0.x);  // walls (solver.hpp:413-417), applied after the reaction term
                w01 = sent32(dc0.y);
                w10 = sent32(dc1.x);
                w11 = sent32(dc1.y);
            }
#undef PD_F32B
        }
        // + dt * r (solver.hpp:437-441); dt * 0 = +0 when the float dt is
        // finite, so warps without a sink node then add +0 and skip the products
        if (REACTION == PD_REACTION_SURFACE_SINK && (!dt_fin || __any_sync(0xffffffffu, sk != 0u))) {
            o00 = o00 + dt * ((sk & 1u) ? neg_k * uc0.x : 0.0f);
            o01 = o01 + dt * ((sk & 2u) ? neg_k * uc0.y : 0.0f);
            o10 = o10 + dt * ((sk & 4u) ? neg_k * uc1.x : 0.0f);
            o11 = o11 + dt * ((sk & 8u) ? neg_k * uc1.y : 0.0f);
        } else if (REACTION == PD_REACTION_VOLUMETRIC) {
            o00 = o00 + dt * (src[0] * sfac);
            o01 = o01 + dt * (src[1] * sfac);
            o10 = o10 + dt * (src[2] * sfac);
            o11 = o11 + dt * (src[3] * sfac);
        } else if (dt_fin) {
            o00 = o00 + 0.0f;
            o01 = o01 + 0.0f;
            o10 = o10 + 0.0f;
            o11 = o11 + 0.0f;
        } else {
            o00 = o00 + dt * 0.0f;
            o01 = o01 + dt * 0.0f;
            o10 = o10 + dt * 0.0f;
            o11 = o11 + dt * 0.0f;
        }
        if (w00) o00 = uc0.x;
        if (w01) o01 = uc0.y;
        if (w10) o10 = uc1.x;
        if (w11) o11 = uc1.y;
        // rare path: Dirichlet-exposed chunk or a non-finite result (inactive
        // slots keep u there: a non-finite one only costs the re-check)
        const uint32_t em = max(max(__float_as_uint(o00) & 0x7f800000u, __float_as_uint(o01) & 0x7f800000u),
                                max(__float_as_uint(o10) & 0x7f800000u, __float_as_uint(o11) & 0x7f800000u));
        const bool slow = (flags & kFlagDir32) || em == 0x7f800000u;
        if (__any_sync(0xffffffffu, slow)) {
            if (slow) {
                const float2 r0 = pair_slow32b<REACTION, HALF>(M, K, st, lane, (int)z0, o00, o01);
                const float2 r1 = pair_slow32b<REACTION, HALF>(M, K, st, lane, (int)z0 + 1, o10, o11);
                o00 = r0.x;
                o01 = r0.y;
                o10 = r1.x;
                o11 = r1.y;
            }
        }
        float* gp = un + ((uint32_t)c * 512u + g_off);
        stg2f(gp, o00, o01, ab & 1u, ab & 2u);
        stg2f(gp + 64, o10, o11, ab & 4u, ab & 8u);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * s);
        if (++s == (uint32_t)kSt) {
            s = 0;
            ph ^= 1u;
        }
    }
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

void march32b_launch(pd_grid* g, MarchPlan& p, const Args32& M, int r) {
    using KB = void (*)(const Args32, const uint32_t*);
#define PD_T(C)                                                                                                  \
    {{ftcs_march32b_kernel<0, false, C>, ftcs_march32b_kernel<1, false, C>, ftcs_march32b_kernel<2, false, C>},  \
     {ftcs_march32b_kernel<0, true, C>, ftcs_march32b_kernel<1, true, C>, ftcs_march32b_kernel<2, true, C>}}
    static const KB tabs[3][2][3] = {PD_T(0), PD_T(1), PD_T(2)};
#undef PD_T
    static const int cfg = [] {
        const char* e = getenv("PD_M32B_CFG");
        const int v = e ? atoi(e) : 0;
        return v >= 0 && v <= 2 ? v : 0;
    }();
    const uint32_t smem = cfg == 1 ? smem32b(1) : cfg == 2 ? smem32b(2) : smem32b(0);
    const int ctas = cfg == 1 ? ctas32b(1) : cfg == 2 ? ctas32b(2) : ctas32b(0);
    static uint64_t attr_done[3] = {0, 0, 0};
    if (!((attr_done[cfg] >> g->device) & 1u)) {
        for (auto& row : tabs[cfg])
            for (auto kf : row) PD_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done[cfg] |= 1ull << g->device;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    tabs[cfg][p.half ? 1 : 0][r]<<<sms * ctas, kThreads32b, smem, g->stream>>>(M, p.d_ctx);
    PD_CUDA(cudaGetLastError());
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
    static const int dbg = [] {
        const char* e = getenv("PD_MARCH_DBG");
        return e ? atoi(e) : 0;
    }();
    M.dbg = dbg;
    const int r = reaction == PD_REACTION_SURFACE_SINK ? 1 : reaction == PD_REACTION_VOLUMETRIC ? 2 : 0;
    static const int ver = [] {
        const char* e = getenv("PD_MARCH32_V");
        return e ? atoi(e) : 43;
    }();
    if (ver == 43 && p.d_ctx) {
        M.sched = march_flagged_schedule(g, p, sched, n);
        march32b_launch(g, p, M, r);
        return;
    }
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
    table[p.half ? 1 : 0][r]<<<sms * kCtas32, kT32, bytes, g->stream>>>(M);
    PD_CUDA(cudaGetLastError());
}

void march32_launch(pd_grid* g, MarchPlan& p, const StepArgs<float>& a, int reaction) {
    march32_launch_sched(g, p, a, reaction, p.d_stream, p.n, p.d_counter + (a.k & 1023));
}

}  // namespace pdb
