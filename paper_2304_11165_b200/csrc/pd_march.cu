// Warp-per-chunk plane-marching FTCS step for 3-D FP64 grids — the bandwidth
// path (BASELINE.json configs C1-C5). Same per-node result, bit for bit, as
// ftcs_step_kernel (pd_ftcs.cu) and the reference (solver.hpp:360-455).
//
// ftcs_march14_kernel (default):
// * Persistent, 4 CTAs x 4 warps per SM. One warp owns one chunk at a time and
//   marches its 8 z-planes; lane (y, xp) owns the x-pair (2xp, 2xp+1) of row y.
// * Every plane (plus the z-halo planes of the z neighbours) is staged by
//   cp.async into the warp's continuous 8-slot ring of shared-memory tiles
//   (rows -1..8 x 8 columns + two x-halo columns; u and D_eff), 5 loads ahead
//   of the plane being computed, across chunk boundaries: no CTA barriers.
//   x halos (8 B) and y halos (64-B rows) come straight from the neighbour
//   chunks' slabs — those chunks are in flight in adjacent warps, so they hit
//   L2 — and z halos are 512-B planes.
// * Cells without a source in the grid (inactive pairs, missing neighbours)
//   copy D_eff from a sentinel chunk (-inf) and never read u, so empty 32-B
//   sectors cost no HBM traffic.
// * Usability without masks: D_eff = fluid ? D : -inf (static per run); a
//   neighbour is usable iff it is fluid (solver.hpp:374,379-381), i.e. iff the
//   face sum d_a + d_b is not -inf.
// * Face fluxes: F(a|b) = ((d_a+d_b)*0.5)*(u_b-u_a) is exactly what both
//   endpoints compute in the reference (dh_p*(p.u-u_c) for a, dh_m*(u_c-m.u)
//   for b). For a substituted face the reference computes
//   ((d_c+d_c)*0.5)*(u_c-u_c) = +-0 when u_c, d_c are finite, and a +-0 term
//   leaves lap = 0.0 + ... bitwise unchanged, so the fast path uses 0. Planes
//   whose nodes and neighbours are all fluid skip the selects and the wall
//   override. Non-finite fast results and Dirichlet-exposed chunks take the
//   exact generic path on operands re-read from the ring.
// * Schedule: chunks are ordered (z-block of kSeg layers, 4x4 tiles of chunk
//   columns, column, z) and claimed one at a time from one atomic counter, so
//   the chunks in flight form one short window of that order and neighbour
//   halos hit L2 (a static interleave was measured to lose that). The claim ->
//   schedule id -> lane masks/descriptor pipeline runs ahead through a
//   per-warp context ring in shared memory.
// * D_eff is stored halved (HALF): (d_a + d_b) * 0.5 == h_a + h_b exactly for
//   normal values, so faces need no 0.5 multiply (plan falls back for tiny D).
// * Uniform chunks (kFlagUnif: all fluid, one D_eff value also on the
//   neighbours' facing layers) load no D_eff and form every face coefficient
//   once (compute14u).
// * PUSH (multi-GPU): boundary chunks also store their new z=0 / z=7 planes
//   into the neighbour GPU's ghost chunks (pd_peer.cu).
// * 3-D FP32 grids run the same design in pd_march32.cu.
//
// Earlier layouts (four nodes per lane "v15/v16", a whole x-row per lane
// "v17") were measured and retired; see DESIGN.md section 4 and commit d37e7fc.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "pd_internal.cuh"
#include "pd_async.cuh"

namespace pdb {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kCtasPerSm = 4;  // march v14 (default): 4 CTAs x 4 warps per SM
constexpr int kSeg = 8;  // measured: 16 and 32 read 0.6 / 2.3 GB more DRAM per C5 step (profiles/r02_ab_schedule.txt)
constexpr unsigned kSentHi = 0xFFF00000u;  // high word of -inf
constexpr int kFlagDirichlet = 2;  // chunk touches a Dirichlet outer face
constexpr int kFlagPushLo = 1 << 16;  // push the new z=0 plane to the lower peer's ghost chunk
constexpr int kFlagPushHi = 1 << 17;  // push the new z=7 plane to the upper peer's ghost chunk
// uniform chunk: its six face neighbours exist, every node is fluid with one
// D_eff bit pattern dv, and so is the facing layer of every neighbour, so each
// face coefficient the reference forms, (d_c + d_n) * 0.5, is (dv + dv) * 0.5:
// the chunk loads no D_eff at all (march v14, compute14u)
constexpr int kFlagUnif = 1 << 18;
// desc flag bits 8..15: plane z is interior-fluid (every node and every face
// neighbour fluid) -> select-free path

__device__ __forceinline__ bool sentinel(double d) {
    return (unsigned)__double2hiint(d) == kSentHi;
}
__device__ __forceinline__ double sent() { return __hiloint2double((int)kSentHi, 0); }


struct MarchArgs {
    StepArgs<double> A;
    const int32_t* __restrict__ sched;
    int64_t n;
    const int32_t* __restrict__ desc;  // 8 ints per chunk: nbr[6], key, flags
    const uint32_t* __restrict__ lm;   // per chunk and lane: active / sink bits
    const double* __restrict__ deff;
    int* counter;                    // chunk-claim counter of this step
    int zero;                        // 0 (opaque to the compiler)
    int64_t n_all;                   // chunks of the grid (D_eff sentinel chunk follows them)
    int dbg;                         // measurement-only halo skip mask (PD_MARCH_DBG)
    // fused halo push (multi-GPU, pd_peer.cu): chunks flagged kFlagPushLo /
    // kFlagPushHi also store their new z=0 / z=7 plane into the lower / upper
    // peer's ghost chunk peer_ord[2c+side] of the peer's u_next column
    double* peer_un[2];
    const int32_t* __restrict__ peer_ord;
    const double* __restrict__ dv;     // per chunk: the uniform D_eff of kFlagUnif chunks
    int pf;                            // v14: L2 prefetch of the next load-side chunk's slabs
};

// Schedule entries carry bit 31 on uniform chunks (flagged_schedule); -1 ends.
__device__ __forceinline__ int sched_id(int e) { return e == -1 ? -1 : (int)((uint32_t)e & 0x7FFFFFFFu); }


struct SlowConsts {
    int64_t size[3];
    double inv_dx2[3];
    double bcv[6];
    double dt, neg_k, src_factor;
    int dirichlet;
    uint32_t huge_hi;
};

// Exact generic node update (solver.hpp:360-441) on already-loaded neighbour
// values nu/nd[axis*2+side]; usability from the D_eff sentinel, outer faces
// from global coordinates.
template <int REACTION>
__device__ __noinline__ double slow_node(const SlowConsts& K, double u_c, double d_c,
                                         const double* nu, const double* nd, int64_t gx,
                                         int64_t gy, int64_t gz, bool sink, double src) {
    const int64_t g[3] = {gx, gy, gz};
    double lap = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
        double u2[2], d2[2];
        for (int side = 0; side < 2; ++side) {
            const int f = ax * 2 + side;
            const int64_t gg = g[ax] + (side ? 1 : -1);
            if (gg < 0 || gg >= K.size[ax]) {
                u2[side] = (K.dirichlet >> f) & 1 ? K.bcv[f] : u_c;
                d2[side] = d_c;
            } else if (sentinel(nd[f])) {
                u2[side] = u_c;
                d2[side] = d_c;
            } else {
                u2[side] = nu[f];
                d2[side] = nd[f];
            }
        }
        const double dh_m = (d_c + d2[0]) * 0.5;
        const double dh_p = (d_c + d2[1]) * 0.5;
        lap += (dh_p * (u2[1] - u_c) - dh_m * (u_c - u2[0])) * K.inv_dx2[ax];
    }
    double rate = 0.0;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        if (sink) rate = K.neg_k * u_c;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        rate = src * K.src_factor;
    }
    return u_c + K.dt * lap + K.dt * rate;
}

// Face flux F(a|b) shared by both endpoints; 0 when either side is not fluid.
// HALF: the ring holds D_eff / 2 (plan.half), so (d_a + d_b) * 0.5 is
// h_a + h_b — the same double, since halving is exact and commutes with
// rounding for normal values (the plan checks every fluid D >= 2^-1021) —
// and the 0.5 multiply disappears.
template <bool HALF>
__device__ __forceinline__ double face(double da, double db, double ua, double ub) {
    const double s = da + db;
    const double f = (HALF ? s : s * 0.5) * (ub - ua);
    return ((unsigned)__double2hiint(s) == kSentHi) ? 0.0 : f;
}
template <bool HALF>
__device__ __forceinline__ double fface(double da, double db, double ua, double ub) {
    return (HALF ? (da + db) : (da + db) * 0.5) * (ub - ua);
}

// One plane tile: u and D_eff of one z-plane of a chunk, rows y = -1..8 of
// the 8 body columns (pitch 8: the lanes' 16-B pair accesses are bank-conflict
// free) and the x- / x+ halo cells of rows 0..7 in two side columns.
struct Tile {
    double u[80], hxu[2][8];
    double d[80], hxd[2][8];
};
constexpr uint32_t kTileBytes = sizeof(Tile);                  // 1536
constexpr uint32_t kDOff = (uint32_t)offsetof(Tile, d);        // u -> D_eff distance (bytes)
constexpr uint32_t kHxOff = (uint32_t)offsetof(Tile, hxu);     // x-halo column (bytes)

// ---- predicated asynchronous copies (LDGSTS), one predicate per pair ----
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Per-lane constants of the tile geometry (byte offsets inside a tile).
struct LaneGeo {
    int y, xp;
    bool xface, yface;
    uint32_t s_c;   // own pair
    uint32_t s_l;   // left neighbour cell (x-halo column for xp = 0)
    uint32_t s_r;   // right neighbour cell (x-halo column for xp = 3)
    uint32_t s_hx;  // x-halo cell this lane fills (x-face lanes)
    uint32_t s_hy;  // y-halo pair this lane fills (y-face lanes)
    uint32_t bp;    // own pair offset inside plane 0 (elements)
};

__device__ __forceinline__ LaneGeo lane_geo(int lane) {
    LaneGeo G;
    G.y = lane >> 2;
    G.xp = lane & 3;
    const int x0 = 2 * G.xp;
    G.xface = G.xp == 0 || G.xp == 3;
    G.yface = G.y == 0 || G.y == 7;
    G.s_c = (uint32_t)(x0 + 8 * (G.y + 1)) * 8u;
    G.s_l = G.xp == 0 ? kHxOff + (uint32_t)G.y * 8u : G.s_c - 8u;
    G.s_r = G.xp == 3 ? kHxOff + (uint32_t)(8 + G.y) * 8u : G.s_c + 16u;
    G.s_hx = kHxOff + (uint32_t)((G.xp == 3 ? 8 : 0) + G.y) * 8u;
    G.s_hy = G.y == 0 ? G.s_c - 64u : G.s_c + 64u;
    G.bp = (uint32_t)(G.y * 8 + x0);
    return G;
}

// |x| >= 2^e_huge or non-finite, from the high word (integer pipe); hi is
// StepArgs::huge_hi (e_huge depends on the grid's slot count and cell volume)
__device__ __forceinline__ bool huge(double x, uint32_t hi) {
    return ((unsigned)__double2hiint(x) & 0x7fffffffu) >= hi;
}

struct Consts {
    double dt, neg_k, src_factor, ix, iy, iz;
};

__device__ __forceinline__ double2 lds2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds1(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
    return v;
}

// Rare-path handling of a node pair whose fast result is huge / non-finite,
// and the Dirichlet-exposed chunks: exact generic update (slow_node) on the
// staged values, then the reference's non-finite / total-mass flags
// (solver.hpp:444, 250-260, 514-515).
template <int REACTION>
__device__ __noinline__ double2 pair_slow(unsigned long long* bad_key, int* flagp, const SlowConsts& K,
                                          int c, int key, int cflags, uint32_t lm, int z,
                                          int xp, int y, const double* nu0, const double* nd0,
                                          const double* nu1, const double* nd1, double uc0, double uc1,
                                          double dc0, double dc1, bool s0, bool s1, double src0,
                                          double src1, double out0, double out1) {
    const bool dirichlet = (cflags & kFlagDirichlet) != 0;
    const int x0 = 2 * xp;
    const int kx = key & 1023, ky = (key >> 10) & 1023, kz = (key >> 20) & 1023;
    const int64_t gx = (int64_t)kx * 8 + x0, gy = (int64_t)ky * 8 + y, gz = (int64_t)kz * 8 + z;
    const bool a0 = (lm >> (2 * z)) & 1u, a1 = (lm >> (2 * z + 1)) & 1u;
    bool h0, h1;
    if (dirichlet) {  // the whole chunk takes the exact generic update
        if (!sentinel(dc0)) out0 = slow_node<REACTION>(K, uc0, dc0, nu0, nd0, gx, gy, gz, s0, src0);
        if (!sentinel(dc1)) out1 = slow_node<REACTION>(K, uc1, dc1, nu1, nd1, gx + 1, gy, gz, s1, src1);
        h0 = a0 && huge(out0, K.huge_hi);
        h1 = a1 && huge(out1, K.huge_hi);
    } else {  // a huge fast result: re-derive the non-finite ones exactly
        h0 = a0 && huge(out0, K.huge_hi);
        h1 = a1 && huge(out1, K.huge_hi);
        if (h0 && !isfinite(out0) && !sentinel(dc0))
            out0 = slow_node<REACTION>(K, uc0, dc0, nu0, nd0, gx, gy, gz, s0, src0);
        if (h1 && !isfinite(out1) && !sentinel(dc1))
            out1 = slow_node<REACTION>(K, uc1, dc1, nu1, nd1, gx + 1, gy, gz, s1, src1);
    }
    if (h0 | h1) {
        const bool bad0 = a0 && !isfinite(out0), bad1 = a1 && !isfinite(out1);
        const int o = z * 64 + y * 8 + x0;
        if (bad0 | bad1) {
            atomicMin(bad_key, ((unsigned long long)c << 10) | (unsigned long long)(o + (bad0 ? 0 : 1)));
            atomicOr(flagp, 1);
        } else {
            atomicOr(flagp, 2);
        }
    }
    return make_double2(out0, out1);
}

// u_next stores: streaming (evict-first) — the values are next read one
// step later, long after they would have left L2.
__device__ __forceinline__ void stg2(double* p, double a, double b) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void stg_pair(double* p, double a, double b, bool a0, bool a1) {
    asm volatile(
        "{\n .reg .pred p, q, r;\n setp.ne.b32 p, %3, 0;\n setp.ne.b32 q, %4, 0;\n"
        " and.pred r, p, q;\n"
        " @r st.global.cs.v2.f64 [%0], {%1, %2};\n"
        " xor.pred p, p, r;\n xor.pred q, q, r;\n"
        " @p st.global.cs.f64 [%0], %1;\n"
        " @q st.global.cs.f64 [%0+8], %2;\n}\n" ::"l"(p),
        "d"(a), "d"(b), "r"((int)a0), "r"((int)a1)
        : "memory");
}

// ---------------------------------------------------------------------------
// v14: the same per-node arithmetic with a rolled plane loop over a
// continuous 8-slot ring (slot = load index & 7, 5 loads ahead), 32-bit
// element offsets against the uniform column bases, and a rare path that
// re-reads its operands from the ring: small code (instruction-cache
// resident) and <= 128 registers, so 16 warps per SM fit (4 CTAs x 4 warps x
// 8 slots x 1.5 KB = 192 KB of ring per SM).
// ---------------------------------------------------------------------------
constexpr int kRing14 = 8;
constexpr int kAhead14 = 5;  // kRing14 - 3 (planes z-1, z, z+1 resident)
constexpr int kCtas14 = 4;
constexpr uint32_t kCtxBytes14 = 176;  // lm[32] | desc[8] | id, pad | uniform D (at 168)
constexpr uint32_t kWarpBytes14 = kRing14 * kTileBytes + 3 * kCtxBytes14;

__device__ __forceinline__ void cp4(uint32_t sa, const void* g, bool pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
        " @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(sa),
        "l"(g), "r"((int)pred));
}

struct LoadCtx14 {
    uint32_t own, zl, zh, xo, yo;  // element offsets of the lane's sources in plane 0
    uint32_t lm;                   // active bits of the lane's pair (0 if no chunk)
    bool zlok, zhok, xok, yok;
    bool dl;                       // load D_eff (false for kFlagUnif chunks)
};

__device__ __forceinline__ LoadCtx14 make_load_ctx14(int c, uint32_t lm, int dv, int dbg, const LaneGeo& G) {
    int nb[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) nb[f] = __shfl_sync(0xffffffffu, dv, 24 + f);
    LoadCtx14 L;
    const bool ok = c >= 0;
    L.dl = !(__shfl_sync(0xffffffffu, dv, 31) & kFlagUnif);
    L.own = ok ? (uint32_t)c * 512u + G.bp : 0u;
    L.lm = ok ? lm : 0u;
    L.zlok = ok && nb[4] >= 0 && !(dbg & 4);
    L.zhok = ok && nb[5] >= 0 && !(dbg & 4);
    L.zl = L.zlok ? (uint32_t)nb[4] * 512u + 448u + G.bp : 0u;
    L.zh = L.zhok ? (uint32_t)nb[5] * 512u + G.bp : 0u;
    const int jx = G.xp == 0 ? nb[0] : nb[1];
    L.xok = ok && G.xface && jx >= 0 && !(dbg & 1);
    L.xo = L.xok ? (uint32_t)jx * 512u + (uint32_t)G.y * 8u + (G.xp == 0 ? 7u : 0u) : 0u;
    const int jy = G.y == 0 ? nb[2] : nb[3];
    L.yok = ok && G.yface && jy >= 0 && !(dbg & 2);
    L.yo = L.yok ? (uint32_t)jy * 512u + (G.y == 0 ? 56u : 0u) + 2u * (uint32_t)G.xp : 0u;
    return L;
}

// Load i (0..9, warp-uniform) of a chunk into the ring slot at st. D_eff
// cells without a source in the grid (inactive pairs, missing neighbours)
// copy the same cells of the sentinel chunk (-inf, at sent_off); their u is
// not loaded (never used: the face terms of a sentinel side are zero).
__device__ __forceinline__ void cp16_ud(uint32_t su, const double* gu, bool pu, uint32_t sd, const double* gd,
                                        bool pd) {
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.b32 p, %4, 0;\n setp.ne.b32 q, %5, 0;\n"
        " @p cp.async.cg.shared.global [%0], [%1], 16;\n"
        " @q cp.async.cg.shared.global [%2], [%3], 16;\n}\n" ::"r"(su),
        "l"(gu), "r"(sd), "l"(gd), "r"((int)pu), "r"((int)pd));
}
__device__ __forceinline__ void cp8_ud(uint32_t su, const double* gu, bool pu, uint32_t sd, const double* gd,
                                       bool pd) {
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.b32 p, %4, 0;\n setp.ne.b32 q, %5, 0;\n"
        " @p cp.async.ca.shared.global [%0], [%1], 8;\n"
        " @q cp.async.ca.shared.global [%2], [%3], 8;\n}\n" ::"r"(su),
        "l"(gu), "r"(sd), "l"(gd), "r"((int)pu), "r"((int)pd));
}
__device__ __forceinline__ void issue14(uint32_t st, const double* __restrict__ u, const double* __restrict__ de,
                                        const LoadCtx14& L, int i, const LaneGeo& G, uint32_t sent_off) {
    if (i == 0 || i == 9) {
        const bool ok = i == 0 ? L.zlok : L.zhok;
        const uint32_t o = i == 0 ? L.zl : L.zh;
        cp16_ud(st + G.s_c, u + o, ok, st + kDOff + G.s_c, de + (ok ? o : sent_off + G.bp), L.dl);
        return;
    }
    const uint32_t p64 = (uint32_t)(i - 1) * 64u;
    const bool ok = ((L.lm >> (2 * (i - 1))) & 3u) != 0u;
    const uint32_t o = L.own + p64;
    cp16_ud(st + G.s_c, u + o, ok, st + kDOff + G.s_c, de + (ok ? o : sent_off + G.bp + p64), L.dl);
    const uint32_t ox = L.xo + p64;
    cp8_ud(st + G.s_hx, u + ox, L.xok, st + kDOff + G.s_hx, de + (L.xok ? ox : sent_off + G.bp + p64),
           G.xface && L.dl);
    const uint32_t oy = L.yo + p64;
    cp16_ud(st + G.s_hy, u + oy, L.yok, st + kDOff + G.s_hy, de + (L.yok ? oy : sent_off + G.bp + p64),
            G.yface && L.dl);
}

struct ChunkCtx14 {
    int c, key, flags;
    uint32_t lm;
    double dv;  // uniform D_eff (kFlagUnif chunks)
};

// Rare path (Dirichlet-exposed chunk, or a huge / non-finite fast result):
// re-reads the pair's operands from the ring and applies the exact generic
// update and the error / mass flags (solver.hpp:360-455, 250-260, 514-515).
template <int REACTION, bool HALF>
__device__ __noinline__ double2 pair_slow14(const MarchArgs& M, const SlowConsts& K, ChunkCtx14 C, int z,
                                            uint32_t tm, uint32_t t0, uint32_t tp, LaneGeo G, double out0,
                                            double out1) {
    const bool un = (C.flags & kFlagUnif) != 0;  // no D_eff in the ring: every d is dv
    const double2 vv = make_double2(C.dv, C.dv);
    const double2 uc = lds2(t0 + G.s_c), dc0 = un ? vv : lds2(t0 + kDOff + G.s_c);
    const double uL = lds1(t0 + G.s_l), dL0 = un ? C.dv : lds1(t0 + kDOff + G.s_l);
    const double uR = lds1(t0 + G.s_r), dR0 = un ? C.dv : lds1(t0 + kDOff + G.s_r);
    const double2 uym = lds2(t0 + G.s_c - 64), dym0 = un ? vv : lds2(t0 + kDOff + G.s_c - 64);
    const double2 uyp = lds2(t0 + G.s_c + 64), dyp0 = un ? vv : lds2(t0 + kDOff + G.s_c + 64);
    const double2 uzm = lds2(tm + G.s_c), dzm0 = un ? vv : lds2(tm + kDOff + G.s_c);
    const double2 uzp = lds2(tp + G.s_c), dzp0 = un ? vv : lds2(tp + kDOff + G.s_c);
    // the ring / dv hold D_eff / 2 under HALF: the generic update needs D (exact doubling)
    auto dd = [](double h) { return HALF ? h + h : h; };
    auto dd2 = [&](double2 h) { return make_double2(dd(h.x), dd(h.y)); };
    const double2 dc = dd2(dc0), dym = dd2(dym0), dyp = dd2(dyp0), dzm = dd2(dzm0), dzp = dd2(dzp0);
    const double dL = dd(dL0), dR = dd(dR0);
    const bool s0 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (16 + 2 * z)) & 1u);
    const bool s1 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (17 + 2 * z)) & 1u);
    double src0 = 0.0, src1 = 0.0;
    if (REACTION == PD_REACTION_VOLUMETRIC) {
        const double* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + G.bp;
        src0 = sp[0];
        src1 = sp[1];
    }
    const double nu0[6] = {uL, uc.y, uym.x, uyp.x, uzm.x, uzp.x};
    const double nd0[6] = {dL, dc.y, dym.x, dyp.x, dzm.x, dzp.x};
    const double nu1[6] = {uc.x, uR, uym.y, uyp.y, uzm.y, uzp.y};
    const double nd1[6] = {dc.x, dR, dym.y, dyp.y, dzm.y, dzp.y};
    return pair_slow<REACTION>(M.A.bad_key, M.A.flags + M.A.k, K, C.c, C.key, C.flags, C.lm, z, G.xp, G.y, nu0,
                               nd0, nu1, nd1, uc.x, uc.y, dc.x, dc.y, s0, s1, src0, src1, out0, out1);
}

// Remote store of a node pair into the peer's ghost chunk (NVLink P2P / same
// device); active nodes only, like the local store.
__device__ __noinline__ void push_pair14(const MarchArgs& M, const ChunkCtx14& C, int z, uint32_t bp, double out0,
                                         double out1, bool a0, bool a1) {
    const int side = z == 0 ? 0 : 1;
    if (!(C.flags & (side ? kFlagPushHi : kFlagPushLo))) return;
    const int32_t o = __ldg(M.peer_ord + 2 * (int64_t)C.c + side);
    double* p = M.peer_un[side] + (int64_t)o * 512 + z * 64 + bp;  // bp even: 16-B aligned pair
    if (a0 && a1) {  // one 16-B remote store (NVLink) for a fully active pair
        *reinterpret_cast<double2*>(p) = make_double2(out0, out1);
    } else {
        if (a0) p[0] = out0;
        if (a1) p[1] = out1;
    }
}

// Uniform chunk (kFlagUnif): every node active and fluid, every face
// coefficient (dv + dv) * 0.5 — the reference's (d_c + d_n) * 0.5 with both
// sides dv — so only u comes from the ring. Same expression order as the
// interior path of compute14.
template <int REACTION, bool PUSH, bool HALF>
__device__ __forceinline__ void compute14u(const MarchArgs& M, const SlowConsts& K, const Consts& Q,
                                           const ChunkCtx14& C, int z, uint32_t tm, uint32_t t0, uint32_t tp,
                                           const LaneGeo& G, double* __restrict__ un, bool& pushed) {
    const uint32_t lz = C.lm >> (2 * z);
    const double2 uc = lds2(t0 + G.s_c);
    const double uL = lds1(t0 + G.s_l), uR = lds1(t0 + G.s_r);
    const double2 uym = lds2(t0 + G.s_c - 64), uyp = lds2(t0 + G.s_c + 64);
    const double2 uzm = lds2(tm + G.s_c), uzp = lds2(tp + G.s_c);
    const double dh = HALF ? C.dv + C.dv : (C.dv + C.dv) * 0.5;
    const double fxl = dh * (uc.x - uL), fxi = dh * (uc.y - uc.x), fxr = dh * (uR - uc.y);
    const double fy0m = dh * (uc.x - uym.x), fy0p = dh * (uyp.x - uc.x);
    const double fz0m = dh * (uc.x - uzm.x), fz0p = dh * (uzp.x - uc.x);
    const double fy1m = dh * (uc.y - uym.y), fy1p = dh * (uyp.y - uc.y);
    const double fz1m = dh * (uc.y - uzm.y), fz1p = dh * (uzp.y - uc.y);
    double lap0 = 0.0;
    lap0 += (fxi - fxl) * Q.ix;
    lap0 += (fy0p - fy0m) * Q.iy;
    lap0 += (fz0p - fz0m) * Q.iz;
    double lap1 = 0.0;
    lap1 += (fxr - fxi) * Q.ix;
    lap1 += (fy1p - fy1m) * Q.iy;
    lap1 += (fz1p - fz1m) * Q.iz;
    double r0 = 0.0, r1 = 0.0;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        r0 = ((lz >> 16) & 1u) ? Q.neg_k * uc.x : 0.0;
        r1 = ((lz >> 17) & 1u) ? Q.neg_k * uc.y : 0.0;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        const double* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + G.bp;
        r0 = sp[0] * Q.src_factor;
        r1 = sp[1] * Q.src_factor;
    }
    double out0 = uc.x + Q.dt * lap0 + Q.dt * r0;
    double out1 = uc.y + Q.dt * lap1 + Q.dt * r1;
    if (huge(out0, M.A.huge_hi) | huge(out1, M.A.huge_hi)) {
        const double2 r = pair_slow14<REACTION, HALF>(M, K, C, z, tm, t0, tp, G, out0, out1);
        out0 = r.x;
        out1 = r.y;
    }
    stg_pair(un + ((uint32_t)C.c * 512u + (uint32_t)z * 64u + G.bp), out0, out1, true, true);
    if (PUSH && (C.flags & (kFlagPushLo | kFlagPushHi)) && (z == 0 || z == 7)) {
        push_pair14(M, C, z, G.bp, out0, out1, true, true);
        pushed = true;
    }
}

template <int REACTION, bool PUSH, bool HALF>
__device__ __forceinline__ void compute14(const MarchArgs& M, const SlowConsts& K, const Consts& Q,
                                          const ChunkCtx14& C, int z, uint32_t tm, uint32_t t0, uint32_t tp,
                                          const LaneGeo& G, double* __restrict__ un, bool& pushed) {
    if (C.flags & kFlagUnif) {  // warp-uniform
        compute14u<REACTION, PUSH, HALF>(M, K, Q, C, z, tm, t0, tp, G, un, pushed);
        return;
    }
    const uint32_t lz = C.lm >> (2 * z);
    const bool a0 = lz & 1u, a1 = (lz >> 1) & 1u;
    const double2 uc = lds2(t0 + G.s_c), dc = lds2(t0 + kDOff + G.s_c);
    const double uL = lds1(t0 + G.s_l), dL = lds1(t0 + kDOff + G.s_l);
    const double uR = lds1(t0 + G.s_r), dR = lds1(t0 + kDOff + G.s_r);
    const double2 uym = lds2(t0 + G.s_c - 64), dym = lds2(t0 + kDOff + G.s_c - 64);
    const double2 uyp = lds2(t0 + G.s_c + 64), dyp = lds2(t0 + kDOff + G.s_c + 64);
    const double2 uzm = lds2(tm + G.s_c), dzm = lds2(tm + kDOff + G.s_c);
    const double2 uzp = lds2(tp + G.s_c), dzp = lds2(tp + kDOff + G.s_c);
    double fxl, fxi, fxr, fy0m, fy0p, fz0m, fz0p, fy1m, fy1p, fz1m, fz1p;
    const bool interior = (C.flags >> (8 + z)) & 1;  // warp-uniform: no walls, no substitution
    if (interior) {
        fxl = fface<HALF>(dL, dc.x, uL, uc.x);
        fxi = fface<HALF>(dc.x, dc.y, uc.x, uc.y);
        fxr = fface<HALF>(dc.y, dR, uc.y, uR);
        fy0m = fface<HALF>(dym.x, dc.x, uym.x, uc.x);
        fy0p = fface<HALF>(dc.x, dyp.x, uc.x, uyp.x);
        fz0m = fface<HALF>(dzm.x, dc.x, uzm.x, uc.x);
        fz0p = fface<HALF>(dc.x, dzp.x, uc.x, uzp.x);
        fy1m = fface<HALF>(dym.y, dc.y, uym.y, uc.y);
        fy1p = fface<HALF>(dc.y, dyp.y, uc.y, uyp.y);
        fz1m = fface<HALF>(dzm.y, dc.y, uzm.y, uc.y);
        fz1p = fface<HALF>(dc.y, dzp.y, uc.y, uzp.y);
    } else {
        fxl = face<HALF>(dL, dc.x, uL, uc.x);
        fxi = face<HALF>(dc.x, dc.y, uc.x, uc.y);
        fxr = face<HALF>(dc.y, dR, uc.y, uR);
        fy0m = face<HALF>(dym.x, dc.x, uym.x, uc.x);
        fy0p = face<HALF>(dc.x, dyp.x, uc.x, uyp.x);
        fz0m = face<HALF>(dzm.x, dc.x, uzm.x, uc.x);
        fz0p = face<HALF>(dc.x, dzp.x, uc.x, uzp.x);
        fy1m = face<HALF>(dym.y, dc.y, uym.y, uc.y);
        fy1p = face<HALF>(dc.y, dyp.y, uc.y, uyp.y);
        fz1m = face<HALF>(dzm.y, dc.y, uzm.y, uc.y);
        fz1p = face<HALF>(dc.y, dzp.y, uc.y, uzp.y);
    }
    double lap0 = 0.0;  // lap starts at T{0} (solver.hpp:420)
    lap0 += (fxi - fxl) * Q.ix;
    lap0 += (fy0p - fy0m) * Q.iy;
    lap0 += (fz0p - fz0m) * Q.iz;
    double lap1 = 0.0;
    lap1 += (fxr - fxi) * Q.ix;
    lap1 += (fy1p - fy1m) * Q.iy;
    lap1 += (fz1p - fz1m) * Q.iz;
    double r0 = 0.0, r1 = 0.0;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        r0 = ((lz >> 16) & 1u) ? Q.neg_k * uc.x : 0.0;
        r1 = ((lz >> 17) & 1u) ? Q.neg_k * uc.y : 0.0;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        const double* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + G.bp;
        r0 = sp[0] * Q.src_factor;
        r1 = sp[1] * Q.src_factor;
    }
    double out0 = uc.x + Q.dt * lap0 + Q.dt * r0;
    double out1 = uc.y + Q.dt * lap1 + Q.dt * r1;
    if (!interior) {  // walls stay frozen (solver.hpp:413-417)
        if (sentinel(dc.x)) out0 = uc.x;
        if (sentinel(dc.y)) out1 = uc.y;
    }
    if ((C.flags & kFlagDirichlet) || ((a0 && huge(out0, M.A.huge_hi)) | (a1 && huge(out1, M.A.huge_hi)))) {
        const double2 r = pair_slow14<REACTION, HALF>(M, K, C, z, tm, t0, tp, G, out0, out1);
        out0 = r.x;
        out1 = r.y;
    }
    stg_pair(un + ((uint32_t)C.c * 512u + (uint32_t)z * 64u + G.bp), out0, out1, a0, a1);
    if (PUSH && (C.flags & (kFlagPushLo | kFlagPushHi)) && (z == 0 || z == 7)) {
        push_pair14(M, C, z, G.bp, out0, out1, a0, a1);
        pushed = true;
    }
}

template <int REACTION, bool PUSH, bool HALF>
__global__ void __launch_bounds__(kThreads, kCtas14) ftcs_march14_kernel(MarchArgs M) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<double>& A = M.A;
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
        K.huge_hi = A.huge_hi;
    }
    __syncthreads();
    Consts Q;
    Q.dt = A.dt;
    Q.neg_k = A.neg_k;
    Q.src_factor = A.src_factor;
    Q.ix = A.inv_dx2[0];
    Q.iy = A.inv_dx2[1];
    Q.iz = A.inv_dx2[2];
    LaneGeo G = lane_geo(lane);
#ifndef PD_M14_NOPIN
    // opaque copies: ptxas cannot rematerialise a shuffle result inside the
    // plane loop, so the lane constants stay in registers
    G.s_c = __shfl_sync(0xffffffffu, G.s_c, lane);
    G.s_l = __shfl_sync(0xffffffffu, G.s_l, lane);
    G.s_r = __shfl_sync(0xffffffffu, G.s_r, lane);
    G.s_hx = __shfl_sync(0xffffffffu, G.s_hx, lane);
    G.s_hy = __shfl_sync(0xffffffffu, G.s_hy, lane);
    G.bp = __shfl_sync(0xffffffffu, G.bp, lane);
#endif
    uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw) + (uint32_t)warp * kWarpBytes14;
#ifndef PD_NOPIN2
    sb = __shfl_sync(0xffffffffu, sb, lane);
    G.xface = __shfl_sync(0xffffffffu, (int)G.xface, lane) != 0;
    G.yface = __shfl_sync(0xffffffffu, (int)G.yface, lane) != 0;
#endif
    const double* __restrict__ u = A.u;
    const double* __restrict__ de = M.deff;
    double* __restrict__ un = A.un;
    const uint32_t sent_off = (uint32_t)M.n_all * 512u;

    // Chunk pipeline, staged through a 3-entry per-warp context ring in shared
    // memory so no register ever waits on a just-issued load: at the advance
    // onto chunk k, entry k%3 holds chunk k's lane masks + descriptor + id,
    // entry (k+1)%3 holds chunk k+1's id, and lane 0 holds the claimed
    // schedule position of chunk k+2. The advance reads entry k%3, issues the
    // cp.async of chunk k+1's masks / descriptor and of chunk k+2's id, and
    // claims the position of chunk k+3 (a plain atomic: the counter address is
    // opaque, ctr + (warp & zero), so ptxas does not warp-aggregate it and
    // shuffle the result right away).
    int* ctr_l = M.counter + ((t >> 5) & M.zero);
    const int n = (int)M.n;
    const uint32_t cb = sb + kRing14 * kTileBytes;  // context ring
    auto cent = [&](int e) -> uint32_t { return cb + (uint32_t)e * kCtxBytes14; };
    int raw = 0;
    auto claim_issue = [&]() {
        if (lane == 0) asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(raw) : "l"(ctr_l) : "memory");
    };
    auto sched_sync = [&]() -> int {
        claim_issue();
        const int p = __shfl_sync(0xffffffffu, raw, 0);
        return p < n ? sched_id(__ldg(&M.sched[p])) : -1;
    };
    auto fetch_ctx = [&](uint32_t e, int c) {  // masks + descriptor + uniform D of chunk c into entry e
        cp4(e + 4u * (uint32_t)lane, M.lm + (int64_t)(c < 0 ? 0 : c) * 32 + lane, c >= 0);
        cp4(e + 128u + 4u * (uint32_t)(lane & 7), M.desc + (int64_t)(c < 0 ? 0 : c) * 8 + (lane & 7),
            c >= 0 && lane < 8);
        cp4(e + 168u + 4u * (uint32_t)(lane & 1),
            reinterpret_cast<const uint32_t*>(M.dv + (c < 0 ? 0 : c)) + (lane & 1), c >= 0 && lane < 2);
    };
    {
        const int id0 = sched_sync();
        if (id0 < 0) return;
        const int id1 = sched_sync();
        if (lane == 0) {
            sts_u32(cent(0) + 160u, (uint32_t)id0);
            sts_u32(cent(1) + 160u, (uint32_t)id1);
        }
        fetch_ctx(cent(0), id0);
        cp_commit();
        cp_wait<0>();
        __syncwarp();
        claim_issue();
    }
    int ek = 0;  // entry of the load-side chunk
    ChunkCtx14 Cld;
    LoadCtx14 Lld;
    auto advance = [&]() {
        const uint32_t e0 = cent(ek);
        const int e1i = ek == 2 ? 0 : ek + 1, e2i = e1i == 2 ? 0 : e1i + 1;
        const uint32_t e1 = cent(e1i), e2 = cent(e2i);
        const int c = sched_id((int)lds_u32(e0 + 160u));
        const uint32_t lm = c >= 0 ? lds_u32(e0 + 4u * (uint32_t)lane) : 0u;
        // descriptor word j lives at lane 24 + j (make_load_ctx14 / ChunkCtx14)
        const int dv = (int)lds_u32(e0 + 128u + 4u * (uint32_t)(lane >= 24 ? lane - 24 : 0));
        Cld = ChunkCtx14{c, __shfl_sync(0xffffffffu, dv, 30), __shfl_sync(0xffffffffu, dv, 31), lm,
                         lds1(e0 + 168u)};
        Lld = make_load_ctx14(c, lm, c >= 0 ? dv : -1, M.dbg, G);
        const int e1raw = (int)lds_u32(e1 + 160u);
        const int c1 = sched_id(e1raw);
        fetch_ctx(e1, c1);
        // DRAM concurrency: also pull chunk c1's slabs towards L2 now (its
        // plane loads start one chunk later); D_eff only for non-uniform chunks
        if (M.pf && lane == 0 && c1 >= 0) {
            prefetch_l2(u + (int64_t)c1 * 512, 4096u);
            if (e1raw >= 0) prefetch_l2(de + (int64_t)c1 * 512, 4096u);
        }
        if (lane == 0) {
            const bool ok = raw < n;
            cp4(e2 + 160u, M.sched + (ok ? raw : 0), ok);
            if (!ok) sts_u32(e2 + 160u, 0xFFFFFFFFu);
        }
        claim_issue();
        ek = e1i;
    };
    advance();
    int p_ld = 0;    // next load index (0..9) of the load-side chunk
    uint32_t Lc = 0;  // loads issued
    auto issue_next = [&]() {
        issue14(sb + (Lc & (kRing14 - 1)) * kTileBytes, u, de, Lld, p_ld, G, sent_off);
        if (++p_ld == 10) {  // the load side moves on to the next chunk
            p_ld = 0;
            advance();
        }
        cp_commit();
        ++Lc;
    };
    ChunkCtx14 Cc = Cld;
    uint32_t base = 0;  // load index of plane -1 of Cc
    bool pushed = false;
#pragma unroll 1
    for (int k = 0; k < 3 + kAhead14; ++k) issue_next();
#pragma unroll 1
    while (Cc.c >= 0) {
#pragma unroll 1
        for (int z = 0; z < 8; ++z) {
            cp_wait<kAhead14>();
            __syncwarp();
            const uint32_t b = base + (uint32_t)z;
            compute14<REACTION, PUSH, HALF>(M, K, Q, Cc, z, sb + (b & 7u) * kTileBytes, sb + ((b + 1u) & 7u) * kTileBytes,
                                      sb + ((b + 2u) & 7u) * kTileBytes, G, un, pushed);
            __syncwarp();
            issue_next();
            if (z == 7) {  // plane 8 of this chunk and plane -1 of the next
                issue_next();
                issue_next();
            }
        }
        base += 10u;
        Cc = Cld;
    }
    cp_wait<0>();
    // the pushed planes are visible system-wide before this kernel completes
    // (the stream's next kernel raises the peer's step counter, pd_peer.cu)
    if (PUSH && pushed) __threadfence_system();
}

// ---------------------------------------------------------------------------
// v20 (PD_MARCH_V=20, measured and kept for A/B): v14's per-node arithmetic and tile layout with a bulk-copy
// load side. One elected lane per warp moves each staged plane with
// cp.async.bulk (TMA bulk copies, UBLKCP): the own u plane and D_eff plane
// (512 B each, contiguous in the column), the y-halo rows of the y
// neighbours (64 B each) and the z-halo planes, completing on one mbarrier
// per ring slot (expect_tx). Only the x-halo cells (8 B at a 64-B stride,
// below the 16-B bulk granule) stay per-lane cp.async, tracked by the same
// mbarrier (cp.async.mbarrier.arrive). This replaces v14's per-lane
// predicated 16-B copies and their address / sentinel selection (~55 of
// v14's ~265 warp instructions per plane). Whole planes are copied, inactive
// slots included: their D_eff is the -inf sentinel in the plan's D_eff
// array and their u is never used, so results are unchanged.
// Measured (profiles/r02_ab_v14_v20.txt): bitwise equal, DRAM unchanged, but
// 1.34x slower: each single-lane cp.async.bulk compiles to an R2UR waterfall
// of ~14 issue slots, so 6 copies per plane cost more than v14's per-lane
// LDGSTS (one warp instruction per 512 B).
// ---------------------------------------------------------------------------
constexpr uint32_t kBarOff20 = kRing14 * kTileBytes + 3 * kCtxBytes14;  // 8 mbarriers (8 B each)
constexpr uint32_t kWarpBytes20 = kBarOff20 + 8u * kRing14;


// Sources of one chunk's loads (element offsets; warp-uniform except the
// x-halo fields).
struct LoadCtx20 {
    uint32_t own, zl, zh, yl, yh;  // own plane 0, z-halo planes, y-halo rows (plane 0)
    uint32_t xo;                   // x-halo cell of this lane (plane 0)
    bool ok, zlok, zhok, ylok, yhok, xok;
    bool dl;                       // load D_eff (false for kFlagUnif chunks)
};

__device__ __forceinline__ LoadCtx20 make_load_ctx20(int c, int dv, int dbg, const LaneGeo& G,
                                                     uint32_t sent_off) {
    int nb[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) nb[f] = __shfl_sync(0xffffffffu, dv, 24 + f);
    LoadCtx20 L;
    L.ok = c >= 0;
    L.dl = L.ok && !(__shfl_sync(0xffffffffu, dv, 31) & kFlagUnif);
    L.own = L.ok ? (uint32_t)c * 512u : 0u;
    L.zlok = L.ok && nb[4] >= 0 && !(dbg & 4);
    L.zhok = L.ok && nb[5] >= 0 && !(dbg & 4);
    // D_eff of a missing neighbour comes from the sentinel chunk (-inf)
    L.zl = L.zlok ? (uint32_t)nb[4] * 512u + 448u : sent_off;
    L.zh = L.zhok ? (uint32_t)nb[5] * 512u : sent_off;
    L.ylok = L.ok && nb[2] >= 0 && !(dbg & 2);
    L.yhok = L.ok && nb[3] >= 0 && !(dbg & 2);
    L.yl = L.ylok ? (uint32_t)nb[2] * 512u + 56u : sent_off;
    L.yh = L.yhok ? (uint32_t)nb[3] * 512u : sent_off;
    const int jx = G.xp == 0 ? nb[0] : nb[1];
    L.xok = L.ok && G.xface && jx >= 0 && !(dbg & 1);
    L.xo = L.xok ? (uint32_t)jx * 512u + (uint32_t)G.y * 8u + (G.xp == 0 ? 7u : 0u) : sent_off + G.bp;
    return L;
}

// Load i (0..9, warp-uniform) of a chunk into the ring slot at st, completing
// on bar: i = 0 / 9 the z-halo planes (plane 7 of the z- neighbour, plane 0
// of the z+ neighbour), i = 1..8 own plane i-1 with its x / y halos.
__device__ __forceinline__ void issue20(uint32_t st, uint32_t bar, const double* __restrict__ u,
                                        const double* __restrict__ de, const LoadCtx20& L, int i,
                                        const LaneGeo& G, int lane) {
    const bool body = i >= 1 && i <= 8;
    const uint32_t p64 = body ? (uint32_t)(i - 1) * 64u : 0u;
    if (body) {  // x-halo cells: per-lane 8-B copies (x-face lanes)
        const uint32_t ox = L.xo + (L.xok ? p64 : 0u);
        cp8_ud(st + G.s_hx, u + ox, L.xok, st + kDOff + G.s_hx, de + ox, G.xface && L.dl);
    }
    cp_mbar_arrive(bar);
    __syncwarp();
    if (lane == 0) {
        // the ring slot's previous contents were read through the generic
        // proxy (all lanes, ordered by the __syncwarp); order those reads
        // before the async-proxy writes below
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bool pu;
        uint32_t src;
        if (body) {
            pu = L.ok;
            src = L.own + p64;
        } else {
            pu = i == 0 ? L.zlok : L.zhok;
            src = i == 0 ? L.zl : L.zh;
        }
        uint32_t bytes = (pu ? 512u : 0u) + (L.dl ? 512u : 0u);
        if (body) bytes += (L.ylok ? 64u : 0u) + (L.yhok ? 64u : 0u) + (L.dl ? 128u : 0u);
        mbar_arrive_tx(bar, bytes);
        if (pu) bulk_g2s(st + 64u, u + src, 512u, bar);
        if (L.dl) bulk_g2s(st + kDOff + 64u, de + src, 512u, bar);
        if (body) {
            const uint32_t yl = L.yl + (L.ylok ? p64 : 0u), yh = L.yh + (L.yhok ? p64 : 0u);
            if (L.ylok) bulk_g2s(st, u + yl, 64u, bar);
            if (L.yhok) bulk_g2s(st + 576u, u + yh, 64u, bar);
            if (L.dl) {
                bulk_g2s(st + kDOff, de + yl, 64u, bar);
                bulk_g2s(st + kDOff + 576u, de + yh, 64u, bar);
            }
        }
    }
}

template <int REACTION, bool PUSH, bool HALF>
__global__ void __launch_bounds__(kThreads, kCtas14) ftcs_march20_kernel(MarchArgs M) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<double>& A = M.A;
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
        K.huge_hi = A.huge_hi;
    }
    __syncthreads();
    Consts Q;
    Q.dt = A.dt;
    Q.neg_k = A.neg_k;
    Q.src_factor = A.src_factor;
    Q.ix = A.inv_dx2[0];
    Q.iy = A.inv_dx2[1];
    Q.iz = A.inv_dx2[2];
    LaneGeo G = lane_geo(lane);
    // opaque copies: ptxas cannot rematerialise a shuffle result inside the
    // plane loop, so the lane constants stay in registers
    G.s_c = __shfl_sync(0xffffffffu, G.s_c, lane);
    G.s_l = __shfl_sync(0xffffffffu, G.s_l, lane);
    G.s_r = __shfl_sync(0xffffffffu, G.s_r, lane);
    G.s_hx = __shfl_sync(0xffffffffu, G.s_hx, lane);
    G.bp = __shfl_sync(0xffffffffu, G.bp, lane);
    uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw) + (uint32_t)warp * kWarpBytes20;
    sb = __shfl_sync(0xffffffffu, sb, lane);
    G.xface = __shfl_sync(0xffffffffu, (int)G.xface, lane) != 0;
    const uint32_t bars = sb + kBarOff20;
    if (lane < kRing14) mbar_init(bars + 8u * (uint32_t)lane, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    const double* __restrict__ u = A.u;
    const double* __restrict__ de = M.deff;
    double* __restrict__ un = A.un;
    const uint32_t sent_off = (uint32_t)M.n_all * 512u;

    // chunk pipeline: as v14 (context ring, claims 3 chunks ahead)
    int* ctr_l = M.counter + ((t >> 5) & M.zero);
    const int n = (int)M.n;
    const uint32_t cb = sb + kRing14 * kTileBytes;  // context ring
    auto cent = [&](int e) -> uint32_t { return cb + (uint32_t)e * kCtxBytes14; };
    int raw = 0;
    auto claim_issue = [&]() {
        if (lane == 0) asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(raw) : "l"(ctr_l) : "memory");
    };
    auto sched_sync = [&]() -> int {
        claim_issue();
        const int p = __shfl_sync(0xffffffffu, raw, 0);
        return p < n ? __ldg(&M.sched[p]) : -1;
    };
    auto fetch_ctx = [&](uint32_t e, int c) {  // masks + descriptor + uniform D of chunk c into entry e
        cp4(e + 4u * (uint32_t)lane, M.lm + (int64_t)(c < 0 ? 0 : c) * 32 + lane, c >= 0);
        cp4(e + 128u + 4u * (uint32_t)(lane & 7), M.desc + (int64_t)(c < 0 ? 0 : c) * 8 + (lane & 7),
            c >= 0 && lane < 8);
        cp4(e + 168u + 4u * (uint32_t)(lane & 1),
            reinterpret_cast<const uint32_t*>(M.dv + (c < 0 ? 0 : c)) + (lane & 1), c >= 0 && lane < 2);
    };
    {
        const int id0 = sched_sync();
        if (id0 < 0) return;
        const int id1 = sched_sync();
        if (lane == 0) {
            sts_u32(cent(0) + 160u, (uint32_t)id0);
            sts_u32(cent(1) + 160u, (uint32_t)id1);
        }
        fetch_ctx(cent(0), id0);
        cp_commit();
        cp_wait<0>();
        __syncwarp();
        claim_issue();
    }
    int ek = 0;  // entry of the load-side chunk
    ChunkCtx14 Cld;
    LoadCtx20 Lld;
    auto advance = [&]() {
        const uint32_t e0 = cent(ek);
        const int e1i = ek == 2 ? 0 : ek + 1, e2i = e1i == 2 ? 0 : e1i + 1;
        const uint32_t e1 = cent(e1i), e2 = cent(e2i);
        const int c = (int)lds_u32(e0 + 160u);
        const uint32_t lm = c >= 0 ? lds_u32(e0 + 4u * (uint32_t)lane) : 0u;
        // descriptor word j lives at lane 24 + j (make_load_ctx20 / ChunkCtx14)
        const int dv = (int)lds_u32(e0 + 128u + 4u * (uint32_t)(lane >= 24 ? lane - 24 : 0));
        Cld = ChunkCtx14{c, __shfl_sync(0xffffffffu, dv, 30), __shfl_sync(0xffffffffu, dv, 31), lm,
                         lds1(e0 + 168u)};
        Lld = make_load_ctx20(c, c >= 0 ? dv : -1, M.dbg, G, sent_off);
        const int c1 = (int)lds_u32(e1 + 160u);
        fetch_ctx(e1, c1);
        if (lane == 0) {
            const bool ok = raw < n;
            cp4(e2 + 160u, M.sched + (ok ? raw : 0), ok);
            if (!ok) sts_u32(e2 + 160u, 0xFFFFFFFFu);
        }
        claim_issue();
        ek = e1i;
    };
    advance();
    int p_ld = 0;     // next load index (0..9) of the load-side chunk
    uint32_t Lc = 0;  // loads issued
    auto issue_next = [&]() {
        const uint32_t slot = Lc & (kRing14 - 1);
        issue20(sb + slot * kTileBytes, bars + 8u * slot, u, de, Lld, p_ld, G, lane);
        if (++p_ld == 10) {  // the load side moves on to the next chunk
            p_ld = 0;
            advance();
        }
        ++Lc;
    };
    auto wait_load = [&](uint32_t l) { mbar_wait(bars + 8u * (l & (kRing14 - 1)), (l >> 3) & 1u); };
    ChunkCtx14 Cc = Cld;
    uint32_t base = 0;  // load index of plane -1 of Cc
    bool pushed = false;
#pragma unroll 1
    for (int k = 0; k < 3 + kAhead14; ++k) issue_next();
#pragma unroll 1
    while (Cc.c >= 0) {
        wait_load(base);
        wait_load(base + 1u);
#pragma unroll 1
        for (int z = 0; z < 8; ++z) {
            const uint32_t b = base + (uint32_t)z;
            wait_load(b + 2u);
            compute14<REACTION, PUSH, HALF>(M, K, Q, Cc, z, sb + (b & 7u) * kTileBytes,
                                            sb + ((b + 1u) & 7u) * kTileBytes, sb + ((b + 2u) & 7u) * kTileBytes,
                                            G, un, pushed);
            __syncwarp();
            issue_next();
            if (z == 7) {  // plane 8 of this chunk and plane -1 of the next
                issue_next();
                issue_next();
            }
        }
        base += 10u;
        Cc = Cld;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    // the pushed planes are visible system-wide before this kernel completes
    // (the stream's next kernel raises the peer's step counter, pd_peer.cu)
    if (PUSH && pushed) __threadfence_system();
}

// ---------------------------------------------------------------------------
// v30: CTA-staged chunk pipeline fed by TMA.
// * A CTA = 4 compute warps + 1 producer warp; 4 CTAs per SM. The CTA works
//   on one chunk at a time per stage; compute warp w owns planes 2w and 2w+1
//   of the chunk, lane (y, xp) the x-pairs (2xp, 2xp+1) of row y: 4 nodes per
//   lane, the two own planes being each other's z neighbours.
// * Three 16.25 KB stages per CTA. One elected producer thread moves a whole
//   chunk per stage with ~15 asynchronous copies completing on the stage's
//   "full" mbarrier: the chunk record (lane masks, descriptor, uniform D;
//   176 B), the own u and D_eff slabs (4 KB bulk copies each), the x-halo
//   columns and y-halo rows of the four lateral neighbours (4-D TMA tensor
//   boxes {2,8,8,1} / {8,1,8,1} over the [chunk][z][y][x] columns) and the
//   two z-halo planes (512-B bulk copies). A v14 plane load needed ~60 warp
//   instructions per 512 B; here one instruction moves up to 4 KB.
// * The compute warps release a stage on its "empty" mbarrier; the producer
//   runs up to three chunks ahead, its claim -> schedule -> descriptor chain
//   software-pipelined two chunks deep.
// * Missing lateral / z neighbours: D_eff comes from the sentinel chunk
//   (-inf), u is not copied (never used, the face term is substituted).
//   Uniform chunks (kFlagUnif) copy no D_eff at all.
// * Per-node arithmetic, walls, reactions, rare path, push: as v14 (same
//   expressions, same order), so results are bitwise identical.
// ---------------------------------------------------------------------------
// configurations (template CFG): stages per CTA, planes per compute warp
// (2: 4 compute warps, 1: 8), CTAs per SM
//   0: 3 stages, 2 planes, 4 CTAs (16 compute warps / SM)
//   1: 4 stages, 1 plane,  3 CTAs (24)
//   2: 3 stages, 1 plane,  3 CTAs (24)
//   3: 5 stages, 1 plane,  2 CTAs (16)
//   4, 5, 6: as 0 with an L2 look-ahead of 2, 4, 6 chunks (0-3: 3)
__host__ __device__ constexpr int nst30(int cfg) { return cfg == 1 ? 4 : cfg == 3 ? 5 : 3; }
__host__ __device__ constexpr int pw30(int cfg) { return cfg == 1 || cfg == 2 || cfg == 3 ? 1 : 2; }
__host__ __device__ constexpr int ctas30(int cfg) { return cfg == 1 || cfg == 2 ? 3 : cfg == 3 ? 2 : 4; }
__host__ __device__ constexpr int look30(int cfg) { return cfg == 4 ? 2 : cfg == 5 ? 4 : cfg == 6 ? 6 : 3; }
__host__ __device__ constexpr int nw30(int cfg) { return 8 / pw30(cfg); }  // compute warps per CTA
__host__ __device__ constexpr int threads30(int cfg) { return 32 * (nw30(cfg) + 1); }  // + one producer warp
// stage layout (bytes): the D_eff half mirrors the u half at +kDHalf30
constexpr uint32_t kOwn30 = 0;      // [z][y][x] own slab (4096)
constexpr uint32_t kYL30 = 4096;    // [z][x]    y- neighbour's row 7 (512)
constexpr uint32_t kYH30 = 4608;    // [z][x]    y+ neighbour's row 0 (512)
constexpr uint32_t kXL30 = 5120;    // [z][y]    x- neighbour's column 7 (512; per-lane copies)
constexpr uint32_t kXH30 = 5632;    // [z][y]    x+ neighbour's column 0 (512; per-lane copies)
constexpr uint32_t kZL30 = 6144;    // [y][x]    z- neighbour's plane 7 (512)
constexpr uint32_t kZH30 = 6656;    // [y][x]    z+ neighbour's plane 0 (512)
constexpr uint32_t kDHalf30 = 7168;
// chunk record (176 B), then at +176 the chunk id and, for the compute
// warps' x-halo prefetch, the next chunk's x- / x+ neighbours, flags and id
constexpr uint32_t kCtx30 = 14336;
constexpr uint32_t kCtxWords30 = 44;
constexpr uint32_t kStage30 = 14336 + 256;
__host__ __device__ constexpr uint32_t bar30(int nst) { return (uint32_t)nst * kStage30; }  // full[nst] then empty[nst]
__host__ __device__ constexpr uint32_t smem30(int nst) { return bar30(nst) + 16u * (uint32_t)nst; }


// Shared-memory byte addresses (u side; D_eff at +kDHalf30) of one plane's
// operands for the lane: own pair, z- / z+ pairs, y- / y+ pairs, x- / x+ cells.
struct Addr30 {
    uint32_t c, zm, zp, ym, yp, l, r;
};

// Rare path: operands re-read from the stage, exact generic update and the
// error / mass flags (solver.hpp:360-455, 250-260, 514-515).
template <int REACTION, bool HALF, uint32_t DH = kDHalf30>
__device__ __noinline__ double2 pair_slow30(const MarchArgs& M, const SlowConsts& K, const ChunkCtx14& C, int z,
                                            int xp, int y, uint32_t bp, Addr30 a, double out0, double out1) {
    const bool un = (C.flags & kFlagUnif) != 0;  // no D_eff in the stage: every d is dv
    const double2 vv = make_double2(C.dv, C.dv);
    const double2 uc = lds2(a.c), dc0 = un ? vv : lds2(a.c + DH);
    const double uL = lds1(a.l), dL0 = un ? C.dv : lds1(a.l + DH);
    const double uR = lds1(a.r), dR0 = un ? C.dv : lds1(a.r + DH);
    const double2 uym = lds2(a.ym), dym0 = un ? vv : lds2(a.ym + DH);
    const double2 uyp = lds2(a.yp), dyp0 = un ? vv : lds2(a.yp + DH);
    const double2 uzm = lds2(a.zm), dzm0 = un ? vv : lds2(a.zm + DH);
    const double2 uzp = lds2(a.zp), dzp0 = un ? vv : lds2(a.zp + DH);
    auto dd = [](double h) { return HALF ? h + h : h; };
    auto dd2 = [&](double2 h) { return make_double2(dd(h.x), dd(h.y)); };
    const double2 dc = dd2(dc0), dym = dd2(dym0), dyp = dd2(dyp0), dzm = dd2(dzm0), dzp = dd2(dzp0);
    const double dL = dd(dL0), dR = dd(dR0);
    const bool s0 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (16 + 2 * z)) & 1u);
    const bool s1 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (17 + 2 * z)) & 1u);
    double src0 = 0.0, src1 = 0.0;
    if (REACTION == PD_REACTION_VOLUMETRIC) {
        const double* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + bp;
        src0 = sp[0];
        src1 = sp[1];
    }
    const double nu0[6] = {uL, uc.y, uym.x, uyp.x, uzm.x, uzp.x};
    const double nd0[6] = {dL, dc.y, dym.x, dyp.x, dzm.x, dzp.x};
    const double nu1[6] = {uc.x, uR, uym.y, uyp.y, uzm.y, uzp.y};
    const double nd1[6] = {dc.x, dR, dym.y, dyp.y, dzm.y, dzp.y};
    return pair_slow<REACTION>(M.A.bad_key, M.A.flags + M.A.k, K, C.c, C.key, C.flags, C.lm, z, xp, y, nu0, nd0,
                               nu1, nd1, uc.x, uc.y, dc.x, dc.y, s0, s1, src0, src1, out0, out1);
}

// One plane of one lane (v14's compute14 / compute14u arithmetic). uc / dc
// (own pair) and the z neighbours are passed in registers (the warp's two
// planes share them); the lateral neighbours are read here.
template <int REACTION, bool PUSH, bool HALF>
__device__ __forceinline__ void compute30(const MarchArgs& M, const SlowConsts& K, const Consts& Q,
                                          const ChunkCtx14& C, int z, int xp, int y, uint32_t bp, const Addr30& a,
                                          double2 uc, double2 dc, double2 uzm, double2 dzm, double2 uzp,
                                          double2 dzp, double* __restrict__ un, bool& pushed) {
    const uint32_t lz = C.lm >> (2 * z);
    const bool unif = (C.flags & kFlagUnif) != 0;  // warp-uniform
    const double uL = lds1(a.l), uR = lds1(a.r);
    const double2 uym = lds2(a.ym), uyp = lds2(a.yp);
    bool a0, a1, interior;
    double fxl, fxi, fxr, fy0m, fy0p, fz0m, fz0p, fy1m, fy1p, fz1m, fz1p;
    if (unif) {
        a0 = a1 = interior = true;
        const double dh = HALF ? C.dv + C.dv : (C.dv + C.dv) * 0.5;
        fxl = dh * (uc.x - uL);
        fxi = dh * (uc.y - uc.x);
        fxr = dh * (uR - uc.y);
        fy0m = dh * (uc.x - uym.x);
        fy0p = dh * (uyp.x - uc.x);
        fz0m = dh * (uc.x - uzm.x);
        fz0p = dh * (uzp.x - uc.x);
        fy1m = dh * (uc.y - uym.y);
        fy1p = dh * (uyp.y - uc.y);
        fz1m = dh * (uc.y - uzm.y);
        fz1p = dh * (uzp.y - uc.y);
    } else {
        a0 = lz & 1u;
        a1 = (lz >> 1) & 1u;
        const double dL = lds1(a.l + kDHalf30), dR = lds1(a.r + kDHalf30);
        const double2 dym = lds2(a.ym + kDHalf30), dyp = lds2(a.yp + kDHalf30);
        interior = (C.flags >> (8 + z)) & 1;  // warp-uniform: no walls, no substitution
        if (interior) {
            fxl = fface<HALF>(dL, dc.x, uL, uc.x);
            fxi = fface<HALF>(dc.x, dc.y, uc.x, uc.y);
            fxr = fface<HALF>(dc.y, dR, uc.y, uR);
            fy0m = fface<HALF>(dym.x, dc.x, uym.x, uc.x);
            fy0p = fface<HALF>(dc.x, dyp.x, uc.x, uyp.x);
            fz0m = fface<HALF>(dzm.x, dc.x, uzm.x, uc.x);
            fz0p = fface<HALF>(dc.x, dzp.x, uc.x, uzp.x);
            fy1m = fface<HALF>(dym.y, dc.y, uym.y, uc.y);
            fy1p = fface<HALF>(dc.y, dyp.y, uc.y, uyp.y);
            fz1m = fface<HALF>(dzm.y, dc.y, uzm.y, uc.y);
            fz1p = fface<HALF>(dc.y, dzp.y, uc.y, uzp.y);
        } else {
            fxl = face<HALF>(dL, dc.x, uL, uc.x);
            fxi = face<HALF>(dc.x, dc.y, uc.x, uc.y);
            fxr = face<HALF>(dc.y, dR, uc.y, uR);
            fy0m = face<HALF>(dym.x, dc.x, uym.x, uc.x);
            fy0p = face<HALF>(dc.x, dyp.x, uc.x, uyp.x);
            fz0m = face<HALF>(dzm.x, dc.x, uzm.x, uc.x);
            fz0p = face<HALF>(dc.x, dzp.x, uc.x, uzp.x);
            fy1m = face<HALF>(dym.y, dc.y, uym.y, uc.y);
            fy1p = face<HALF>(dc.y, dyp.y, uc.y, uyp.y);
            fz1m = face<HALF>(dzm.y, dc.y, uzm.y, uc.y);
            fz1p = face<HALF>(dc.y, dzp.y, uc.y, uzp.y);
        }
    }
    double lap0 = 0.0;  // lap starts at T{0} (solver.hpp:420)
    lap0 += (fxi - fxl) * Q.ix;
    lap0 += (fy0p - fy0m) * Q.iy;
    lap0 += (fz0p - fz0m) * Q.iz;
    double lap1 = 0.0;
    lap1 += (fxr - fxi) * Q.ix;
    lap1 += (fy1p - fy1m) * Q.iy;
    lap1 += (fz1p - fz1m) * Q.iz;
    double r0 = 0.0, r1 = 0.0;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        r0 = ((lz >> 16) & 1u) ? Q.neg_k * uc.x : 0.0;
        r1 = ((lz >> 17) & 1u) ? Q.neg_k * uc.y : 0.0;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        const double* sp = M.A.src + (int64_t)C.c * 512 + z * 64 + bp;
        r0 = sp[0] * Q.src_factor;
        r1 = sp[1] * Q.src_factor;
    }
    double out0 = uc.x + Q.dt * lap0 + Q.dt * r0;
    double out1 = uc.y + Q.dt * lap1 + Q.dt * r1;
    if (!interior) {  // walls stay frozen (solver.hpp:413-417)
        if (sentinel(dc.x)) out0 = uc.x;
        if (sentinel(dc.y)) out1 = uc.y;
    }
    if ((C.flags & kFlagDirichlet) || ((a0 && huge(out0, M.A.huge_hi)) | (a1 && huge(out1, M.A.huge_hi)))) {
        const double2 r = pair_slow30<REACTION, HALF>(M, K, C, z, xp, y, bp, a, out0, out1);
        out0 = r.x;
        out1 = r.y;
    }
    stg_pair(un + ((uint32_t)C.c * 512u + (uint32_t)z * 64u + bp), out0, out1, a0, a1);
    if (PUSH && (C.flags & (kFlagPushLo | kFlagPushHi)) && (z == 0 || z == 7)) {
        push_pair14(M, C, z, bp, out0, out1, a0, a1);
        pushed = true;
    }
}

template <int REACTION, bool PUSH, bool HALF, int CFG>
__global__ void __launch_bounds__(threads30(CFG), ctas30(CFG))
    ftcs_march30_kernel(const __grid_constant__ MarchArgs M, const uint32_t* __restrict__ ctxa,
                        const __grid_constant__ CUtensorMap mux, const __grid_constant__ CUtensorMap muy,
                        const __grid_constant__ CUtensorMap mdx, const __grid_constant__ CUtensorMap mdy) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<double>& A = M.A;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    constexpr int kStages30 = nst30(CFG), kW30 = nw30(CFG), PW = pw30(CFG);
    const uint32_t full0 = sm0 + bar30(kStages30), empty0 = full0 + 8u * kStages30;
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
        K.huge_hi = A.huge_hi;
        for (int s = 0; s < kStages30; ++s) {
            mbar_init(full0 + 8u * s, 1u);
            mbar_init(empty0 + 8u * s, (uint32_t)kW30);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const double* __restrict__ u = A.u;
    const double* __restrict__ de = M.deff;
    const int n = (int)M.n;

    if (warp == kW30) {  // ---------------- producer (one thread) ----------------
        if (lane != 0) return;
        int* ctr = M.counter;
        auto claim = [&]() -> int {
            int r;
            asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(r) : "l"(ctr) : "memory");
            return r;
        };
        // schedule entries carry bit 31 for uniform chunks (no D_eff needed)
        auto id_of = [&](int p) -> int { return p < n ? __ldg(&M.sched[p]) : -1; };
        auto prefetch = [&](const void* g, uint32_t bytes) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(g), "r"(bytes) : "memory");
        };
        auto prefetch_chunk = [&](int e) {  // e: flagged schedule entry (>= 0: none pending)
            if (e == -1) return;
            const int64_t c = (int64_t)((uint32_t)e & 0x7FFFFFFFu);
            prefetch(u + c * 512, 4096u);
            prefetch(ctxa + c * kCtxWords30, 176u);
            if (e >= 0) prefetch(de + c * 512, 4096u);
        };
        auto chunk_of = [](int e) { return e == -1 ? -1 : (int)((uint32_t)e & 0x7FFFFFFFu); };
        const int4* desc4 = reinterpret_cast<const int4*>(M.desc);
        const int sent_c = (int)M.n_all;  // D_eff sentinel chunk
        // Look-ahead (the stages alone hold too few chunks to cover the DRAM
        // latency): the schedule position of chunk k+kLook+1 is claimed, chunk
        // k+kLook's slabs (u, record, and D_eff unless uniform) are prefetched
        // into L2 as soon as its id is known, chunk k+1's descriptor is loaded,
        // chunk k is copied into its stage.
        constexpr int kLook = look30(CFG);
        int q[kLook + 1];  // flagged entries of chunks k .. k+kLook
#pragma unroll
        for (int j = 0; j <= kLook; ++j) {
            q[j] = id_of(claim());
            if (j > 0) prefetch_chunk(q[j]);
        }
        int p_nxt = claim();
        int c_cur = chunk_of(q[0]);
        int4 d0 = make_int4(0, 0, 0, 0), d1 = d0;
        if (c_cur >= 0) {
            d0 = __ldg(desc4 + 2 * (int64_t)c_cur);
            d1 = __ldg(desc4 + 2 * (int64_t)c_cur + 1);
        }
#pragma unroll 1
        for (uint32_t k = 0;; ++k) {
            const uint32_t s = k % kStages30, ph = (k / kStages30) & 1u;
            // descriptor of the next chunk and the look-ahead, before the wait
            const int c_nx = chunk_of(q[1]);
            int4 e0 = make_int4(0, 0, 0, 0), e1 = e0;
            if (c_nx >= 0) {
                e0 = __ldg(desc4 + 2 * (int64_t)c_nx);
                e1 = __ldg(desc4 + 2 * (int64_t)c_nx + 1);
            }
            const int qn = id_of(p_nxt);
            if (c_cur >= 0) p_nxt = claim();
            const uint32_t st = sm0 + s * kStage30, full = full0 + 8u * s;
            if (k >= (uint32_t)kStages30) mbar_wait(empty0 + 8u * s, ph ^ 1u);
            sts_u32(st + kCtx30 + 176u, (uint32_t)c_cur);
            if (c_cur < 0) {  // end marker: the compute warps stop at this stage
                mbar_arrive(full);
                break;
            }
            const int nb2 = d0.z, nb3 = d0.w, nb4 = d1.x, nb5 = d1.y;
            const bool dl = !(d1.w & kFlagUnif);
            uint32_t bytes = 176u + 4096u;
            bytes += (nb2 >= 0 ? 512u : 0u) + (nb3 >= 0 ? 512u : 0u) + (nb4 >= 0 ? 512u : 0u) +
                     (nb5 >= 0 ? 512u : 0u);
            if (dl) bytes += 4096u + 4u * 512u;
            // the next chunk's x neighbours, for the compute warps' x-halo copies
            sts_u32(st + kCtx30 + 180u, (uint32_t)e0.x);
            sts_u32(st + kCtx30 + 184u, (uint32_t)e0.y);
            sts_u32(st + kCtx30 + 188u, (uint32_t)e1.w);
            sts_u32(st + kCtx30 + 192u, (uint32_t)c_nx);
            mbar_arrive_tx(full, bytes);
            const int64_t cb = (int64_t)c_cur * 512;
            bulk_g2s(st + kCtx30, ctxa + (int64_t)c_cur * kCtxWords30, 176u, full);
            bulk_g2s(st + kOwn30, u + cb, 4096u, full);
            if (nb2 >= 0) tma4(st + kYL30, &muy, 0, 7, 0, nb2, full);
            if (nb3 >= 0) tma4(st + kYH30, &muy, 0, 0, 0, nb3, full);
            if (nb4 >= 0) bulk_g2s(st + kZL30, u + (int64_t)nb4 * 512 + 448, 512u, full);
            if (nb5 >= 0) bulk_g2s(st + kZH30, u + (int64_t)nb5 * 512, 512u, full);
            if (dl) {
                const uint32_t sd = st + kDHalf30;
                bulk_g2s(sd + kOwn30, de + cb, 4096u, full);
                tma4(sd + kYL30, &mdy, 0, 7, 0, nb2 >= 0 ? nb2 : sent_c, full);
                tma4(sd + kYH30, &mdy, 0, 0, 0, nb3 >= 0 ? nb3 : sent_c, full);
                bulk_g2s(sd + kZL30, de + (nb4 >= 0 ? (int64_t)nb4 * 512 + 448 : (int64_t)sent_c * 512), 512u, full);
                bulk_g2s(sd + kZH30, de + (nb5 >= 0 ? (int64_t)nb5 * 512 : (int64_t)sent_c * 512), 512u, full);
            }
            prefetch_chunk(qn);
#pragma unroll
            for (int j = 0; j < kLook; ++j) q[j] = q[j + 1];
            q[kLook] = qn;
            c_cur = c_nx;
            d0 = e0;
            d1 = e1;
        }
        return;
    }

    // ---------------- compute warps ----------------
    Consts Q;
    Q.dt = A.dt;
    Q.neg_k = A.neg_k;
    Q.src_factor = A.src_factor;
    Q.ix = A.inv_dx2[0];
    Q.iy = A.inv_dx2[1];
    Q.iz = A.inv_dx2[2];
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp);  // own pair offset in a plane (elements)
    const uint32_t oc = bp * 8u;                     // (bytes)
    // lateral operands: base + z * stride (stage-relative); lanes on a chunk
    // face read the halo buffers
    const uint32_t b_ym = y > 0 ? kOwn30 + oc - 64u : kYL30 + 16u * xp, s_ym = y > 0 ? 512u : 64u;
    const uint32_t b_yp = y < 7 ? kOwn30 + oc + 64u : kYH30 + 16u * xp, s_yp = y < 7 ? 512u : 64u;
    const uint32_t b_l = xp > 0 ? kOwn30 + oc - 8u : kXL30 + 8u * y, s_l = xp > 0 ? 512u : 64u;
    const uint32_t b_r = xp < 3 ? kOwn30 + oc + 16u : kXH30 + 8u * y, s_r = xp < 3 ? 512u : 64u;
    const int z0 = PW == 2 ? 2 * warp : warp, z1 = z0 + 1;
    double* __restrict__ un = A.un;
    bool pushed = false;
    const uint32_t sent_off = (uint32_t)M.n_all * 512u;
    // x-halo cells of this warp's planes, copied per lane (a TMA box would
    // need a 16-B inner dimension: 64 16-B requests per box) into the stage
    // of chunk cn, one chunk ahead: lanes xp = 0 / 3 copy column 7 of the x-
    // neighbour / column 0 of the x+ neighbour (u, and D_eff unless uniform;
    // the sentinel chunk's D_eff for a missing neighbour)
    auto issue_xh = [&](uint32_t stn, int nbl, int nbh, int flags_n) {
        if (xp == 0 || xp == 3) {
            const int j = xp == 0 ? nbl : nbh;
            const uint32_t dst = stn + (xp == 0 ? kXL30 : kXH30) + (uint32_t)(z0 * 8 + y) * 8u;
            const uint32_t src = (uint32_t)j * 512u + (uint32_t)(z0 * 64 + y * 8) + (xp == 0 ? 7u : 0u);
            const bool dl = !(flags_n & kFlagUnif);
#pragma unroll
            for (int q = 0; q < PW; ++q) {
                const uint32_t o = src + 64u * q;
                cp8_ud(dst + 64u * q, u + (j >= 0 ? o : 0u), j >= 0, dst + kDHalf30 + 64u * q,
                       de + (j >= 0 ? o : sent_off), dl);
            }
        }
        cp_commit();
    };
    uint32_t k = 0;
    {
        mbar_wait(full0, 0u);
        const int c = (int)lds_u32(sm0 + kCtx30 + 176u);
        if (c < 0) return;
        issue_xh(sm0, (int)lds_u32(sm0 + kCtx30 + 128u), (int)lds_u32(sm0 + kCtx30 + 132u),
                 (int)lds_u32(sm0 + kCtx30 + 156u));
    }
#pragma unroll 1
    for (;; ++k) {
        const uint32_t s = k % kStages30;
        const uint32_t st = sm0 + s * kStage30;
        const int c = (int)lds_u32(st + kCtx30 + 176u);
        {  // x halos of the next chunk (its stage is free of them: this warp is done with it)
            const int cn = (int)lds_u32(st + kCtx30 + 192u);
            const uint32_t sn = (k + 1) % kStages30;
            if (cn >= 0)
                issue_xh(sm0 + sn * kStage30, (int)lds_u32(st + kCtx30 + 180u), (int)lds_u32(st + kCtx30 + 184u),
                         (int)lds_u32(st + kCtx30 + 188u));
            else
                cp_commit();
        }
        cp_wait<1>();  // this chunk's x halos (this lane's own copies)
        ChunkCtx14 C;
        C.c = c;
        C.lm = lds_u32(st + kCtx30 + 4u * (uint32_t)lane);
        C.key = (int)lds_u32(st + kCtx30 + 128u + 24u);
        C.flags = (int)lds_u32(st + kCtx30 + 128u + 28u);
        C.dv = lds1(st + kCtx30 + 160u);
        const bool unif = (C.flags & kFlagUnif) != 0;
        const double2 vv = make_double2(C.dv, C.dv);
        if constexpr (PW == 2) {
            Addr30 a0, a1;
            a0.c = st + kOwn30 + oc + (uint32_t)z0 * 512u;
            a1.c = a0.c + 512u;
            a0.zm = warp == 0 ? st + kZL30 + oc : a0.c - 512u;
            a0.zp = a1.c;
            a1.zm = a0.c;
            a1.zp = warp == kW30 - 1 ? st + kZH30 + oc : a1.c + 512u;
            a0.ym = st + b_ym + (uint32_t)z0 * s_ym;
            a1.ym = a0.ym + s_ym;
            a0.yp = st + b_yp + (uint32_t)z0 * s_yp;
            a1.yp = a0.yp + s_yp;
            a0.l = st + b_l + (uint32_t)z0 * s_l;
            a1.l = a0.l + s_l;
            a0.r = st + b_r + (uint32_t)z0 * s_r;
            a1.r = a0.r + s_r;
            const double2 uc0 = lds2(a0.c), uc1 = lds2(a1.c), uzm = lds2(a0.zm), uzp = lds2(a1.zp);
            const double2 dc0 = unif ? vv : lds2(a0.c + kDHalf30), dc1 = unif ? vv : lds2(a1.c + kDHalf30);
            const double2 dzm = unif ? vv : lds2(a0.zm + kDHalf30), dzp = unif ? vv : lds2(a1.zp + kDHalf30);
            compute30<REACTION, PUSH, HALF>(M, K, Q, C, z0, xp, y, bp, a0, uc0, dc0, uzm, dzm, uc1, dc1, un,
                                            pushed);
            compute30<REACTION, PUSH, HALF>(M, K, Q, C, z1, xp, y, bp, a1, uc1, dc1, uc0, dc0, uzp, dzp, un,
                                            pushed);
        } else {  // one plane per warp: z = warp
            const int z = z0;
            Addr30 a;
            a.c = st + kOwn30 + oc + (uint32_t)z * 512u;
            a.zm = z == 0 ? st + kZL30 + oc : a.c - 512u;
            a.zp = z == 7 ? st + kZH30 + oc : a.c + 512u;
            a.ym = st + b_ym + (uint32_t)z * s_ym;
            a.yp = st + b_yp + (uint32_t)z * s_yp;
            a.l = st + b_l + (uint32_t)z * s_l;
            a.r = st + b_r + (uint32_t)z * s_r;
            const double2 uc = lds2(a.c), uzm = lds2(a.zm), uzp = lds2(a.zp);
            const double2 dc = unif ? vv : lds2(a.c + kDHalf30);
            const double2 dzm = unif ? vv : lds2(a.zm + kDHalf30), dzp = unif ? vv : lds2(a.zp + kDHalf30);
            compute30<REACTION, PUSH, HALF>(M, K, Q, C, z, xp, y, bp, a, uc, dc, uzm, dzm, uzp, dzp, un, pushed);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * s);
        const uint32_t s1 = (k + 1) % kStages30;
        mbar_wait(full0 + 8u * s1, ((k + 1) / kStages30) & 1u);
        if ((int)lds_u32(sm0 + s1 * kStage30 + kCtx30 + 176u) < 0) break;
    }
    cp_wait<0>();
    // the pushed planes are visible system-wide before this kernel completes
    // (the stream's next kernel raises the peer's step counter, pd_peer.cu)
    if (PUSH && pushed) __threadfence_system();
}

// ---------------------------------------------------------------------------
// v31: v30's CTA-staged chunk pipeline with a lean compute side.
// * The producer is a whole warp: lane 0 claims chunks and issues the bulk /
//   TMA copies (as v30); all 32 lanes copy the x-halo cells (8-B cp.async)
//   and arrive on the stage's "full" mbarrier when those land
//   (cp.async.mbarrier.arrive.noinc), so the compute warps issue no copies.
// * Compute warp w owns planes 2w, 2w+1 of the staged chunk; lane (y, xp)
//   the pairs (2xp, 2xp+1) of row y. Its eleven operand offsets inside a
//   stage are lane constants pinned in registers (no per-chunk address
//   arithmetic beyond stage base + offset).
// * Both planes are computed in one straight-line block (the face between
//   them once), on one of three warp-uniform paths: uniform chunk (no D_eff
//   staged), both planes interior-fluid (select-free faces), generic
//   (sentinel faces, walls). The huge / non-finite test is folded into one
//   max of high words per lane and one warp vote; the exact rare path
//   re-reads everything from the stage.
// * Per-node arithmetic, expression order and stores: as v14 / v30, so the
//   results are bitwise identical.
// ---------------------------------------------------------------------------
// configurations (template CFG): compute groups of 4 warps per CTA (a group
// works on one staged chunk; groups take stages round-robin), stages per CTA,
// CTAs per SM, and how the halos travel (TMA / bulk copies issued by lane 0,
// or per-lane cp.async by the whole producer warp)
//   0: 1 group,  3 stages, 4 CTAs, bulk/TMA halos   (16 compute warps / SM, 12 stages)
//   1: 1 group,  4 stages, 3 CTAs, bulk/TMA halos   (12, 12; 128 registers)
//   2: 1 group,  3 stages, 4 CTAs, per-lane halos
//   3: as 0, the lane's stage offsets re-read from a shared-memory table each
//      chunk instead of held (pinned) in registers
constexpr int kW31 = 4;  // compute warps per group (planes 2w, 2w+1 of the group's chunk)
__host__ __device__ constexpr int grp31(int cfg) { return 1; }
__host__ __device__ constexpr int nst31(int cfg) { return cfg == 1 ? 4 : 3; }
__host__ __device__ constexpr int ctas31(int cfg) { return cfg == 1 ? 3 : 4; }
__host__ __device__ constexpr bool lanehalo31(int cfg) { return cfg == 2; }
__host__ __device__ constexpr bool tab31(int cfg) { return cfg == 3; }
__host__ __device__ constexpr int threads31(int cfg) { return 32 * (kW31 * grp31(cfg) + 1); }  // + the producer warp
// register cap: an SM sub-partition holds 16 K registers for its warps (the
// CTAs' warps spread round-robin over the 4 sub-partitions); multiples of 8
__host__ __device__ constexpr int maxreg31(int cfg) {
    return 16384 / (32 * ((threads31(cfg) / 32 * ctas31(cfg) + 3) / 4)) / 8 * 8;
}
constexpr int kB31 = 4;  // chunks claimed per atomic (producer batch)


// Rare path of one plane pair: everything (chunk record, operands) re-read
// from the stage at st.
template <int REACTION, bool HALF>
__device__ __noinline__ double2 pair_slow31(const MarchArgs& M, const SlowConsts& K, uint32_t st, int lane, int z,
                                            double out0, double out1) {
    ChunkCtx14 C;
    C.c = (int)lds_u32(st + kCtx30 + 176u);
    C.lm = lds_u32(st + kCtx30 + 4u * (uint32_t)lane);
    C.key = (int)lds_u32(st + kCtx30 + 152u);
    C.flags = (int)lds_u32(st + kCtx30 + 156u);
    C.dv = lds1(st + kCtx30 + 160u);
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp), oc = bp * 8u, zz = (uint32_t)z;
    Addr30 a;
    a.c = st + kOwn30 + oc + zz * 512u;
    a.zm = z == 0 ? st + kZL30 + oc : a.c - 512u;
    a.zp = z == 7 ? st + kZH30 + oc : a.c + 512u;
    a.ym = y > 0 ? a.c - 64u : st + kYL30 + zz * 64u + 16u * (uint32_t)xp;
    a.yp = y < 7 ? a.c + 64u : st + kYH30 + zz * 64u + 16u * (uint32_t)xp;
    a.l = xp > 0 ? a.c - 8u : st + kXL30 + zz * 64u + 8u * (uint32_t)y;
    a.r = xp < 3 ? a.c + 16u : st + kXH30 + zz * 64u + 8u * (uint32_t)y;
    return pair_slow30<REACTION, HALF>(M, K, C, z, xp, y, bp, a, out0, out1);
}

// lap and explicit Euler update of one node, the reference's order
// (solver.hpp:420-441): lap = 0 + dx term + dy term + dz term;
// u + dt * lap + dt * r
template <int REACTION>
__device__ __forceinline__ double node31(const Consts& Q, double uc, double fxm, double fxp, double fym, double fyp,
                                         double fzm, double fzp, bool sink, double src) {
    double lap = 0.0;
    lap += (fxp - fxm) * Q.ix;
    lap += (fyp - fym) * Q.iy;
    lap += (fzp - fzm) * Q.iz;
    // no reaction: dt * 0 is +0 (dt is validated positive and finite,
    // solver.hpp:305), so the reference's u + dt*lap + dt*r is u + dt*lap + 0
    if (REACTION == PD_REACTION_NONE) return uc + Q.dt * lap + 0.0;
    double r = 0.0;
    if (REACTION == PD_REACTION_SURFACE_SINK) r = sink ? Q.neg_k * uc : 0.0;
    else if (REACTION == PD_REACTION_VOLUMETRIC) r = src * Q.src_factor;
    return uc + Q.dt * lap + Q.dt * r;
}

template <int REACTION, bool PUSH, bool HALF, int CFG>
__global__ void __maxnreg__(maxreg31(CFG))
    ftcs_march31_kernel(const __grid_constant__ MarchArgs M, const uint32_t* __restrict__ ctxa,
                        const __grid_constant__ CUtensorMap muy, const __grid_constant__ CUtensorMap mdy) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    constexpr int kSt = nst31(CFG), kG = grp31(CFG);
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<double>& A = M.A;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = sm0 + bar30(kSt), empty0 = full0 + 8u * kSt;
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
        K.huge_hi = A.huge_hi;
        for (int s = 0; s < kSt; ++s) {
            mbar_init(full0 + 8u * s, 33u);  // lane 0's expect_tx arrive + 32 x-halo arrivals
            mbar_init(empty0 + 8u * s, (uint32_t)kW31);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const double* __restrict__ u = A.u;
    const double* __restrict__ de = M.deff;
    const int n = (int)M.n;

    if (warp == kW31 * kG) {  // ---------------- producer warp ----------------
        // Chunks are claimed kB31 schedule positions per atomic; lane j < kB31
        // holds chunk j of a batch (flagged schedule entry, descriptor). The
        // chain claim -> entries -> descriptors runs one batch per stage: the
        // claim of batch b+3, the entries of b+2, the descriptors and the L2
        // prefetch of b+1 are issued while batch b is copied, so no
        // long-latency result is consumed in the batch it was requested in.
        int* ctr = M.counter;
        const int4* desc4 = reinterpret_cast<const int4*>(M.desc);
        const int sent_c = (int)M.n_all;  // D_eff sentinel chunk
        const uint32_t sent_off = (uint32_t)M.n_all * 512u;
        auto claim = [&]() -> int {  // lane 0 holds the result
            int r = 0;
            if (lane == 0)
                asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(ctr), "r"(kB31) : "memory");
            return r;
        };
        auto entries = [&](int p0) -> int {  // lane j < kB31: entry of position p0 + j
            const int p = __shfl_sync(0xffffffffu, p0, 0) + lane;
            return lane < kB31 && p < n ? __ldg(&M.sched[p]) : -1;
        };
        auto chunk_of = [](int e) { return e == -1 ? -1 : (int)((uint32_t)e & 0x7FFFFFFFu); };
        auto descs = [&](int e, int4& d0, int4& d1) {
            const int c = chunk_of(e);
            if (lane < kB31 && c >= 0) {
                d0 = __ldg(desc4 + 2 * (int64_t)c);
                d1 = __ldg(desc4 + 2 * (int64_t)c + 1);
            }
        };
        auto prefetch = [&](int e) {  // the batch's slabs into L2 (u, record, and D_eff unless uniform)
            const int64_t c = (int64_t)chunk_of(e);
            if (lane < kB31 && c >= 0) {
                prefetch_l2(u + c * 512, 4096u);
                prefetch_l2(ctxa + c * kCtxWords30, 176u);
                if (e >= 0) prefetch_l2(de + c * 512, 4096u);
            }
        };
        int e_c = entries(claim());
        int e_n = entries(claim());
        int p_nn = claim();
        int4 d0c = make_int4(0, 0, 0, 0), d1c = d0c;
        descs(e_c, d0c, d1c);
        prefetch(e_c);
        const uint32_t xo0 = (uint32_t)lane * 8u;  // this lane's x-halo cells: (z, y) = lane + 32 j
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
            for (int j = 0; j < kB31; ++j, ++k) {
                const int c_cur = chunk_of(__shfl_sync(0xffffffffu, e_c, j));
                const uint32_t st = sm0 + s * kStage30, full = full0 + 8u * s;
                if (k >= (uint32_t)kSt) mbar_wait(empty0 + 8u * s, ph ^ 1u);
                if (c_cur < 0) {  // end markers: one per group, in its next stage
#pragma unroll 1
                    for (int m = 0; m < kG; ++m) {
                        if (m > 0) {
                            if (++s == (uint32_t)kSt) {
                                s = 0;
                                ph ^= 1u;
                            }
                            if (k + m >= (uint32_t)kSt) mbar_wait(empty0 + 8u * s, ph ^ 1u);
                        }
                        const uint32_t stm = sm0 + s * kStage30, fm = full0 + 8u * s;
                        if (lane == 0) {
                            sts_u32(stm + kCtx30 + 176u, 0xFFFFFFFFu);
                            mbar_arrive(fm);
                        }
                        cp_mbar_arrive_noinc(fm);
                    }
                    done = true;
                    break;
                }
                const int nb0 = __shfl_sync(0xffffffffu, d0c.x, j), nb1 = __shfl_sync(0xffffffffu, d0c.y, j);
                const int nb2 = __shfl_sync(0xffffffffu, d0c.z, j), nb3 = __shfl_sync(0xffffffffu, d0c.w, j);
                const int nb4 = __shfl_sync(0xffffffffu, d1c.x, j), nb5 = __shfl_sync(0xffffffffu, d1c.y, j);
                const bool dl = !(__shfl_sync(0xffffffffu, d1c.w, j) & kFlagUnif);
                if (M.dbg & 48) {  // measurement only: no copies (16) / own slabs only (32)
                    if (lane == 0) {
                        sts_u32(st + kCtx30 + 176u, (uint32_t)c_cur);
                        if (M.dbg & 16) {
                            mbar_arrive(full);
                        } else {
                            mbar_arrive_tx(full, dl ? 8192u : 4096u);
                            bulk_g2s(st + kOwn30, u + (int64_t)c_cur * 512, 4096u, full);
                            if (dl) bulk_g2s(st + kDHalf30 + kOwn30, de + (int64_t)c_cur * 512, 4096u, full);
                        }
                    }
                    cp_mbar_arrive_noinc(full);
                    if (++s == (uint32_t)kSt) {
                        s = 0;
                        ph ^= 1u;
                    }
                    continue;
                }
                if (!lanehalo31(CFG) && lane == 0) {
                    sts_u32(st + kCtx30 + 176u, (uint32_t)c_cur);
                    uint32_t bytes = 176u + 4096u;
                    bytes += (nb2 >= 0 ? 512u : 0u) + (nb3 >= 0 ? 512u : 0u) + (nb4 >= 0 ? 512u : 0u) +
                             (nb5 >= 0 ? 512u : 0u);
                    if (dl) bytes += 4096u + 4u * 512u;
                    mbar_arrive_tx(full, bytes);
                    const int64_t cb = (int64_t)c_cur * 512;
                    bulk_g2s(st + kCtx30, ctxa + (int64_t)c_cur * kCtxWords30, 176u, full);
                    bulk_g2s(st + kOwn30, u + cb, 4096u, full);
                    if (nb2 >= 0) tma4(st + kYL30, &muy, 0, 7, 0, nb2, full);
                    if (nb3 >= 0) tma4(st + kYH30, &muy, 0, 0, 0, nb3, full);
                    if (nb4 >= 0) bulk_g2s(st + kZL30, u + (int64_t)nb4 * 512 + 448, 512u, full);
                    if (nb5 >= 0) bulk_g2s(st + kZH30, u + (int64_t)nb5 * 512, 512u, full);
                    if (dl) {
                        const uint32_t sd = st + kDHalf30;
                        bulk_g2s(sd + kOwn30, de + cb, 4096u, full);
                        tma4(sd + kYL30, &mdy, 0, 7, 0, nb2 >= 0 ? nb2 : sent_c, full);
                        tma4(sd + kYH30, &mdy, 0, 0, 0, nb3 >= 0 ? nb3 : sent_c, full);
                        bulk_g2s(sd + kZL30, de + (nb4 >= 0 ? (int64_t)nb4 * 512 + 448 : (int64_t)sent_c * 512),
                                 512u, full);
                        bulk_g2s(sd + kZH30, de + (nb5 >= 0 ? (int64_t)nb5 * 512 : (int64_t)sent_c * 512), 512u,
                                 full);
                    }
                }
                if (lanehalo31(CFG)) {
                    // lane 0: the two own slabs (4 KB bulk copies); every lane:
                    // its 16-B pieces of the chunk record and of the y / z halos
                    if (lane == 0) {
                        sts_u32(st + kCtx30 + 176u, (uint32_t)c_cur);
                        mbar_arrive_tx(full, dl ? 8192u : 4096u);
                        const int64_t cb = (int64_t)c_cur * 512;
                        bulk_g2s(st + kOwn30, u + cb, 4096u, full);
                        if (dl) bulk_g2s(st + kDHalf30 + kOwn30, de + cb, 4096u, full);
                    }
                    if (lane < 11) cp16(st + kCtx30 + 16u * (uint32_t)lane, ctxa + (int64_t)c_cur * kCtxWords30 + 4 * lane, true);
                    const uint32_t l16 = 16u * (uint32_t)lane, l2 = 2u * (uint32_t)lane;
                    // z halos: plane 7 of the z- neighbour, plane 0 of the z+ neighbour (16 B per lane)
                    const uint32_t zl = (uint32_t)nb4 * 512u + 448u + l2, zh = (uint32_t)nb5 * 512u + l2;
                    cp16(st + kZL30 + l16, u + (nb4 >= 0 ? zl : 0u), nb4 >= 0);
                    cp16(st + kZH30 + l16, u + (nb5 >= 0 ? zh : 0u), nb5 >= 0);
                    cp16(st + kDHalf30 + kZL30 + l16, de + (nb4 >= 0 ? zl : sent_off + l2), dl);
                    cp16(st + kDHalf30 + kZH30 + l16, de + (nb5 >= 0 ? zh : sent_off + l2), dl);
                    // y halos: row 7 of the y- neighbour, row 0 of the y+ neighbour, as [z][x];
                    // 32 16-B pieces per side: lane -> plane lane >> 2, x pair lane & 3
                    const uint32_t yo = (uint32_t)(lane >> 2) * 64u + 2u * (uint32_t)(lane & 3);
                    const uint32_t yl = (uint32_t)nb2 * 512u + 56u + yo, yh = (uint32_t)nb3 * 512u + yo;
                    cp16(st + kYL30 + l16, u + (nb2 >= 0 ? yl : 0u), nb2 >= 0);
                    cp16(st + kYH30 + l16, u + (nb3 >= 0 ? yh : 0u), nb3 >= 0);
                    cp16(st + kDHalf30 + kYL30 + l16, de + (nb2 >= 0 ? yl : sent_off + yo), dl);
                    cp16(st + kDHalf30 + kYH30 + l16, de + (nb3 >= 0 ? yh : sent_off + yo), dl);
                }
                {  // x halos: column 7 of the x- neighbour, column 0 of the x+ neighbour
                    // (u only where the neighbour exists; D_eff from the sentinel chunk otherwise)
                    const uint32_t gl = (uint32_t)nb0 * 512u + (uint32_t)lane * 8u + 7u;
                    const uint32_t gh = (uint32_t)nb1 * 512u + (uint32_t)lane * 8u;
                    const uint32_t gs = sent_off + (uint32_t)lane * 8u;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {  // cells (z, y) = lane + 32 jj of each side
                        const uint32_t dL = st + kXL30 + xo0 + (uint32_t)jj * 256u;
                        const uint32_t dH = st + kXH30 + xo0 + (uint32_t)jj * 256u;
                        const uint32_t oL = gl + (uint32_t)jj * 256u, oH = gh + (uint32_t)jj * 256u;
                        cp8(dL, u + (nb0 >= 0 ? oL : 0u), nb0 >= 0);
                        cp8(dH, u + (nb1 >= 0 ? oH : 0u), nb1 >= 0);
                        cp8(dL + kDHalf30, de + (nb0 >= 0 ? oL : gs + (uint32_t)jj * 256u), dl);
                        cp8(dH + kDHalf30, de + (nb1 >= 0 ? oH : gs + (uint32_t)jj * 256u), dl);
                    }
                    cp_mbar_arrive_noinc(full);
                }
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
    Consts Q;
    Q.dt = A.dt;
    Q.neg_k = A.neg_k;
    Q.src_factor = A.src_factor;
    Q.ix = A.inv_dx2[0];
    Q.iy = A.inv_dx2[1];
    Q.iz = A.inv_dx2[2];
    const int y = lane >> 2, xp = lane & 3;
    const int grp = warp / kW31, wq = warp % kW31;  // group, plane pair
    const uint32_t z0 = 2u * (uint32_t)wq;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp);  // own pair offset in a plane (elements)
    const uint32_t oc = bp * 8u;
    // operand offsets inside a stage (u side; D_eff at +kDHalf30): pinned in
    // registers, or (tab31) a per-warp table in shared memory re-read each
    // chunk (3 LDS.128 + 1 LDS issued before the stage wait)
    const uint32_t s_ym = y > 0 ? 512u : 64u, s_yp = y < 7 ? 512u : 64u;
    const uint32_t s_l = xp > 0 ? 512u : 64u, s_r = xp < 3 ? 512u : 64u;
    const uint32_t b_ym = y > 0 ? kOwn30 + oc - 64u + z0 * 512u : kYL30 + 16u * (uint32_t)xp + z0 * 64u;
    const uint32_t b_yp = y < 7 ? kOwn30 + oc + 64u + z0 * 512u : kYH30 + 16u * (uint32_t)xp + z0 * 64u;
    const uint32_t b_l = xp > 0 ? kOwn30 + oc - 8u + z0 * 512u : kXL30 + 8u * (uint32_t)y + z0 * 64u;
    const uint32_t b_r = xp < 3 ? kOwn30 + oc + 16u + z0 * 512u : kXH30 + 8u * (uint32_t)y + z0 * 64u;
    const uint32_t v_c = kOwn30 + oc + z0 * 512u;
    const uint32_t v_zm = wq == 0 ? kZL30 + oc : kOwn30 + oc + z0 * 512u - 512u;
    const uint32_t v_zp = wq == kW31 - 1 ? kZH30 + oc : kOwn30 + oc + z0 * 512u + 1024u;
    const uint32_t v_lm = kCtx30 + 4u * (uint32_t)lane, v_g = z0 * 64u + bp;
    uint32_t tab = 0, p_c = 0, p_zm = 0, p_zp = 0, p_ym0 = 0, p_ym1 = 0, p_yp0 = 0, p_yp1 = 0, p_l0 = 0, p_l1 = 0,
             p_r0 = 0, p_r1 = 0, p_lm = 0, p_g = 0;
    if (tab31(CFG)) {
        tab = pin(sm0 + smem30(kSt) + (uint32_t)warp * 2048u + 16u * (uint32_t)lane, lane);
        sts4(tab, v_c, v_zm, v_zp, b_ym);
        sts4(tab + 512u, b_ym + s_ym, b_yp, b_yp + s_yp, b_l);
        sts4(tab + 1024u, b_l + s_l, b_r, b_r + s_r, v_lm);
        sts4(tab + 1536u, v_g, 0u, 0u, 0u);
    } else {
        p_c = pin(v_c, lane), p_zm = pin(v_zm, lane), p_zp = pin(v_zp, lane);
        p_ym0 = pin(b_ym, lane), p_ym1 = pin(b_ym + s_ym, lane), p_yp0 = pin(b_yp, lane);
        p_yp1 = pin(b_yp + s_yp, lane), p_l0 = pin(b_l, lane), p_l1 = pin(b_l + s_l, lane);
        p_r0 = pin(b_r, lane), p_r1 = pin(b_r + s_r, lane), p_lm = pin(v_lm, lane), p_g = pin(v_g, lane);
    }
    const uint32_t zsh = 2u * z0;  // lm bit of plane z0
    double* __restrict__ un = A.un;
    const uint32_t huge_hi = A.huge_hi;
    bool pushed = false;
    uint32_t s = (uint32_t)grp, ph = 0;  // this group's chunks: k = grp, grp + kG, ...
#pragma unroll 1
    for (;;) {
        uint32_t o_c = p_c, o_zm = p_zm, o_zp = p_zp, o_ym0 = p_ym0, o_ym1 = p_ym1, o_yp0 = p_yp0, o_yp1 = p_yp1;
        uint32_t o_l0 = p_l0, o_l1 = p_l1, o_r0 = p_r0, o_r1 = p_r1, o_lm = p_lm, g_off = p_g;
        if (tab31(CFG)) {
            const uint4 t0 = lds4(tab), t1 = lds4(tab + 512u), t2 = lds4(tab + 1024u);
            g_off = lds_u32(tab + 1536u);
            o_c = t0.x, o_zm = t0.y, o_zp = t0.z, o_ym0 = t0.w, o_ym1 = t1.x, o_yp0 = t1.y;
            o_yp1 = t1.z, o_l0 = t1.w, o_l1 = t2.x, o_r0 = t2.y, o_r1 = t2.z, o_lm = t2.w;
        }
        mbar_wait(full0 + 8u * s, ph);
        const uint32_t st = sm0 + s * kStage30;
        const int c = (int)lds_u32(st + kCtx30 + 176u);
        if (c < 0) break;
        const uint32_t lm = lds_u32(st + o_lm);
        const int flags = (int)lds_u32(st + kCtx30 + 156u);
        const uint32_t ab = (lm >> zsh) & 0xFu;  // active bits: plane z0 (x0, x1), plane z1 (x0, x1)
        const uint32_t sk = (lm >> (16u + zsh)) & 0xFu;
        double src[4] = {0.0, 0.0, 0.0, 0.0};
        if (REACTION == PD_REACTION_VOLUMETRIC) {
            const double* sp = A.src + (int64_t)c * 512 + g_off;
            src[0] = sp[0];
            src[1] = sp[1];
            src[2] = sp[64];
            src[3] = sp[65];
        }
        // u operands (both planes)
        const double2 uc0 = lds2(st + o_c), uc1 = lds2(st + o_c + 512u);
        const double2 uzm = lds2(st + o_zm), uzp = lds2(st + o_zp);
        const double uL0 = lds1(st + o_l0), uR0 = lds1(st + o_r0), uL1 = lds1(st + o_l1), uR1 = lds1(st + o_r1);
        const double2 uym0 = lds2(st + o_ym0), uyp0 = lds2(st + o_yp0);
        const double2 uym1 = lds2(st + o_ym1), uyp1 = lds2(st + o_yp1);
        double o00, o01, o10, o11;  // plane z0 (x0, x1), plane z1 (x0, x1)
        const uint32_t ib = ((uint32_t)flags >> (8u + z0)) & 3u;
        if (flags & kFlagUnif) {
            const double dv = lds1(st + kCtx30 + 160u);
            const double dh = HALF ? dv + dv : (dv + dv) * 0.5;
            const double fzx = dh * (uc1.x - uc0.x), fzy = dh * (uc1.y - uc0.y);  // face z0 | z1
            const double f0i = dh * (uc0.y - uc0.x), f1i = dh * (uc1.y - uc1.x);
            o00 = node31<REACTION>(Q, uc0.x, dh * (uc0.x - uL0), f0i, dh * (uc0.x - uym0.x), dh * (uyp0.x - uc0.x),
                                   dh * (uc0.x - uzm.x), fzx, sk & 1u, src[0]);
            o01 = node31<REACTION>(Q, uc0.y, f0i, dh * (uR0 - uc0.y), dh * (uc0.y - uym0.y), dh * (uyp0.y - uc0.y),
                                   dh * (uc0.y - uzm.y), fzy, sk & 2u, src[1]);
            o10 = node31<REACTION>(Q, uc1.x, dh * (uc1.x - uL1), f1i, dh * (uc1.x - uym1.x), dh * (uyp1.x - uc1.x),
                                   fzx, dh * (uzp.x - uc1.x), sk & 4u, src[2]);
            o11 = node31<REACTION>(Q, uc1.y, f1i, dh * (uR1 - uc1.y), dh * (uc1.y - uym1.y), dh * (uyp1.y - uc1.y),
                                   fzy, dh * (uzp.y - uc1.y), sk & 8u, src[3]);
        } else {
            const uint32_t dh_ = kDHalf30;
            const double2 dc0 = lds2(st + o_c + dh_), dc1 = lds2(st + o_c + 512u + dh_);
            const double2 dzm = lds2(st + o_zm + dh_), dzp = lds2(st + o_zp + dh_);
            const double dL0 = lds1(st + o_l0 + dh_), dR0 = lds1(st + o_r0 + dh_);
            const double dL1 = lds1(st + o_l1 + dh_), dR1 = lds1(st + o_r1 + dh_);
            const double2 dym0 = lds2(st + o_ym0 + dh_), dyp0 = lds2(st + o_yp0 + dh_);
            const double2 dym1 = lds2(st + o_ym1 + dh_), dyp1 = lds2(st + o_yp1 + dh_);
            if (ib == 3u) {  // both planes interior-fluid: no sentinel faces, no walls
                const double fzx = fface<HALF>(dc0.x, dc1.x, uc0.x, uc1.x), fzy = fface<HALF>(dc0.y, dc1.y, uc0.y, uc1.y);
                const double f0i = fface<HALF>(dc0.x, dc0.y, uc0.x, uc0.y), f1i = fface<HALF>(dc1.x, dc1.y, uc1.x, uc1.y);
                o00 = node31<REACTION>(Q, uc0.x, fface<HALF>(dL0, dc0.x, uL0, uc0.x), f0i,
                                       fface<HALF>(dym0.x, dc0.x, uym0.x, uc0.x), fface<HALF>(dc0.x, dyp0.x, uc0.x, uyp0.x),
                                       fface<HALF>(dzm.x, dc0.x, uzm.x, uc0.x), fzx, sk & 1u, src[0]);
                o01 = node31<REACTION>(Q, uc0.y, f0i, fface<HALF>(dc0.y, dR0, uc0.y, uR0),
                                       fface<HALF>(dym0.y, dc0.y, uym0.y, uc0.y), fface<HALF>(dc0.y, dyp0.y, uc0.y, uyp0.y),
                                       fface<HALF>(dzm.y, dc0.y, uzm.y, uc0.y), fzy, sk & 2u, src[1]);
                o10 = node31<REACTION>(Q, uc1.x, fface<HALF>(dL1, dc1.x, uL1, uc1.x), f1i,
                                       fface<HALF>(dym1.x, dc1.x, uym1.x, uc1.x), fface<HALF>(dc1.x, dyp1.x, uc1.x, uyp1.x),
                                       fzx, fface<HALF>(dc1.x, dzp.x, uc1.x, uzp.x), sk & 4u, src[2]);
                o11 = node31<REACTION>(Q, uc1.y, f1i, fface<HALF>(dc1.y, dR1, uc1.y, uR1),
                                       fface<HALF>(dym1.y, dc1.y, uym1.y, uc1.y), fface<HALF>(dc1.y, dyp1.y, uc1.y, uyp1.y),
                                       fzy, fface<HALF>(dc1.y, dzp.y, uc1.y, uzp.y), sk & 8u, src[3]);
            } else {  // generic: faces with a sentinel side contribute 0; walls stay frozen
                const double fzx = face<HALF>(dc0.x, dc1.x, uc0.x, uc1.x), fzy = face<HALF>(dc0.y, dc1.y, uc0.y, uc1.y);
                const double f0i = face<HALF>(dc0.x, dc0.y, uc0.x, uc0.y), f1i = face<HALF>(dc1.x, dc1.y, uc1.x, uc1.y);
                o00 = node31<REACTION>(Q, uc0.x, face<HALF>(dL0, dc0.x, uL0, uc0.x), f0i,
                                       face<HALF>(dym0.x, dc0.x, uym0.x, uc0.x), face<HALF>(dc0.x, dyp0.x, uc0.x, uyp0.x),
                                       face<HALF>(dzm.x, dc0.x, uzm.x, uc0.x), fzx, sk & 1u, src[0]);
                o01 = node31<REACTION>(Q, uc0.y, f0i, face<HALF>(dc0.y, dR0, uc0.y, uR0),
                                       face<HALF>(dym0.y, dc0.y, uym0.y, uc0.y), face<HALF>(dc0.y, dyp0.y, uc0.y, uyp0.y),
                                       face<HALF>(dzm.y, dc0.y, uzm.y, uc0.y), fzy, sk & 2u, src[1]);
                o10 = node31<REACTION>(Q, uc1.x, face<HALF>(dL1, dc1.x, uL1, uc1.x), f1i,
                                       face<HALF>(dym1.x, dc1.x, uym1.x, uc1.x), face<HALF>(dc1.x, dyp1.x, uc1.x, uyp1.x),
                                       fzx, face<HALF>(dc1.x, dzp.x, uc1.x, uzp.x), sk & 4u, src[2]);
                o11 = node31<REACTION>(Q, uc1.y, f1i, face<HALF>(dc1.y, dR1, uc1.y, uR1),
                                       face<HALF>(dym1.y, dc1.y, uym1.y, uc1.y), face<HALF>(dc1.y, dyp1.y, uc1.y, uyp1.y),
                                       fzy, face<HALF>(dc1.y, dzp.y, uc1.y, uzp.y), sk & 8u, src[3]);
                if (sentinel(dc0.x)) o00 = uc0.x;  // walls (solver.hpp:413-417)
                if (sentinel(dc0.y)) o01 = uc0.y;
                if (sentinel(dc1.x)) o10 = uc1.x;
                if (sentinel(dc1.y)) o11 = uc1.y;
            }
        }
        // rare path: Dirichlet-exposed chunk, or a huge / non-finite result
        // (inactive slots keep u there: a huge one only costs the re-check)
        const uint32_t hm = max(max((uint32_t)__double2hiint(o00) & 0x7fffffffu, (uint32_t)__double2hiint(o01) & 0x7fffffffu),
                                max((uint32_t)__double2hiint(o10) & 0x7fffffffu, (uint32_t)__double2hiint(o11) & 0x7fffffffu));
        const bool slow = (flags & kFlagDirichlet) || hm >= huge_hi;
        if (__any_sync(0xffffffffu, slow)) {
            if (slow) {
                const double2 r0 = pair_slow31<REACTION, HALF>(M, K, st, lane, (int)z0, o00, o01);
                const double2 r1 = pair_slow31<REACTION, HALF>(M, K, st, lane, (int)z0 + 1, o10, o11);
                o00 = r0.x;
                o01 = r0.y;
                o10 = r1.x;
                o11 = r1.y;
            }
        }
        double* gp = un + ((uint32_t)c * 512u + g_off);
        stg_pair(gp, o00, o01, ab & 1u, ab & 2u);
        stg_pair(gp + 64, o10, o11, ab & 4u, ab & 8u);
        if (PUSH && (flags & (kFlagPushLo | kFlagPushHi)) && (z0 == 0 || z0 == 6)) {
            ChunkCtx14 C;
            C.c = c;
            C.key = (int)lds_u32(st + kCtx30 + 152u);
            C.flags = flags;
            C.lm = lm;
            C.dv = 0.0;
            if (z0 == 0) push_pair14(M, C, 0, bp, o00, o01, ab & 1u, ab & 2u);
            else push_pair14(M, C, 7, bp, o10, o11, ab & 4u, ab & 8u);
            pushed = true;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * s);
        s += (uint32_t)kG;
        if (s >= (uint32_t)kSt) {
            s -= (uint32_t)kSt;
            ph ^= 1u;
        }
    }
    // the pushed planes are visible system-wide before this kernel completes
    // (the stream's next kernel raises the peer's step counter, pd_peer.cu)
    if (PUSH && pushed) __threadfence_system();
}

// ---------------------------------------------------------------------------
// v41: v31's pipeline with a padded stage layout (v40, commit history) and x
// neighbours by shuffle.
// * A stage half (u; D_eff at +kHalf41) holds 10 planes z = -1..8 at a 640-B
//   pitch, rows y = -1..8 of 64 B: own node (x, y, z) at (z+1)*640 +
//   (y+1)*64 + 8x, the y halos as rows -1 / 8 of each plane, the z halos as
//   planes -1 / 8; then the x- halo column block [z][y] (512 B) and, 64 B
//   further (other banks), the x+ block.
// * A lane's z / y neighbours are its own address -+640 / -+64 (no per-lane
//   halo offsets: v31 pinned eleven stage offsets per lane and spilled); its
//   x neighbours are its row neighbours' pair halves (shfl up / down), lanes
//   on the chunk's x faces take the halo cell, read by one conflict-free 8-B
//   load per plane (v40 read x neighbours with 8-B loads: rows 64 B apart put
//   four rows on the same banks, 3x replays).
// * The producer warp moves the chunk with per-lane 16-B / 8-B cp.async into
//   that layout (a bulk or TMA copy cannot scatter rows to a 640-B pitch);
//   the 176-B chunk record is one bulk copy. Completion: lane 0's expect_tx
//   + 32 cp.async arrivals (cp.async.mbarrier.arrive.noinc).
// * Arithmetic, paths, rare path and stores: as v31 (bitwise identical).
// ---------------------------------------------------------------------------
constexpr uint32_t kPP41 = 640;                 // plane pitch
constexpr uint32_t kXL41 = 10 * kPP41, kXH41 = kXL41 + 576;  // x-halo blocks [z][y]
constexpr uint32_t kHalf41 = kXH41 + 512;       // D_eff half (7488)
constexpr uint32_t kCtx41 = 2 * kHalf41;        // chunk record, then the chunk id at +176
constexpr uint32_t kStage41 = kCtx41 + 256;     // 15232
constexpr int kSt41 = 3, kCtas41 = 4;
constexpr int kThreads41 = 32 * (kW31 + 1);
constexpr uint32_t smem41() { return kSt41 * kStage41 + 16u * kSt41; }

template <int REACTION, bool HALF>
__device__ __noinline__ double2 pair_slow41(const MarchArgs& M, const SlowConsts& K, uint32_t st, int lane, int z,
                                            double out0, double out1) {
    ChunkCtx14 C;
    C.c = (int)lds_u32(st + kCtx41 + 176u);
    C.lm = lds_u32(st + kCtx41 + 4u * (uint32_t)lane);
    C.key = (int)lds_u32(st + kCtx41 + 152u);
    C.flags = (int)lds_u32(st + kCtx41 + 156u);
    C.dv = lds1(st + kCtx41 + 160u);
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp), pz = st + (uint32_t)(z + 1) * kPP41;
    Addr30 a;
    a.c = pz + (uint32_t)(y + 1) * 64u + 16u * (uint32_t)xp;
    a.zm = a.c - kPP41;
    a.zp = a.c + kPP41;
    a.ym = a.c - 64u;
    a.yp = a.c + 64u;
    a.l = xp > 0 ? a.c - 8u : st + kXL41 + (uint32_t)z * 64u + 8u * (uint32_t)y;
    a.r = xp < 3 ? a.c + 16u : st + kXH41 + (uint32_t)z * 64u + 8u * (uint32_t)y;
    return pair_slow30<REACTION, HALF, kHalf41>(M, K, C, z, xp, y, bp, a, out0, out1);
}

template <int REACTION, bool PUSH, bool HALF>
__global__ void __launch_bounds__(kThreads41, kCtas41)
    ftcs_march41_kernel(const __grid_constant__ MarchArgs M, const uint32_t* __restrict__ ctxa) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<double>& A = M.A;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = sm0 + kSt41 * kStage41, empty0 = full0 + 8u * kSt41;
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
        K.huge_hi = A.huge_hi;
        for (int s = 0; s < kSt41; ++s) {
            mbar_init(full0 + 8u * s, 33u);  // lane 0's expect_tx arrive + 32 cp.async arrivals
            mbar_init(empty0 + 8u * s, (uint32_t)kW31);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const double* __restrict__ u = A.u;
    const double* __restrict__ de = M.deff;
    const int n = (int)M.n;

    if (warp == kW31) {  // ---------------- producer warp ----------------
        // batch pipeline as v31: claim of batch b+3, entries of b+2,
        // descriptors and L2 prefetch of b+1 issued while batch b is copied
        int* ctr = M.counter;
        const int4* desc4 = reinterpret_cast<const int4*>(M.desc);
        const uint32_t sent_off = (uint32_t)M.n_all * 512u;  // D_eff sentinel chunk (elements)
        auto claim = [&]() -> int {
            int r = 0;
            if (lane == 0)
                asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(ctr), "r"(kB31) : "memory");
            return r;
        };
        auto entries = [&](int p0) -> int {
            const int p = __shfl_sync(0xffffffffu, p0, 0) + lane;
            return lane < kB31 && p < n ? __ldg(&M.sched[p]) : -1;
        };
        auto chunk_of = [](int e) { return e == -1 ? -1 : (int)((uint32_t)e & 0x7FFFFFFFu); };
        auto descs = [&](int e, int4& d0, int4& d1) {
            const int c = chunk_of(e);
            if (lane < kB31 && c >= 0) {
                d0 = __ldg(desc4 + 2 * (int64_t)c);
                d1 = __ldg(desc4 + 2 * (int64_t)c + 1);
            }
        };
        auto prefetch = [&](int e) {
            const int64_t c = (int64_t)chunk_of(e);
            if (lane < kB31 && c >= 0) {
                prefetch_l2(u + c * 512, 4096u);
                prefetch_l2(ctxa + c * kCtxWords30, 176u);
                if (e >= 0) prefetch_l2(de + c * 512, 4096u);
            }
        };
        int e_c = entries(claim());
        int e_n = entries(claim());
        int p_nn = claim();
        int4 d0c = make_int4(0, 0, 0, 0), d1c = d0c;
        descs(e_c, d0c, d1c);
        prefetch(e_c);
        // per-lane destinations (stage-relative) and source element offsets
        const uint32_t L = (uint32_t)lane;
        const uint32_t d_own = kPP41 + 64u + 16u * L;                        // + 640 i: row pair L of plane i
        const uint32_t d_ylo = kPP41 * ((L >> 2) + 1u) + 16u * (L & 3u);      // row -1 of plane L/4
        const uint32_t s_ylo = 64u * (L >> 2) + 2u * (L & 3u);                // of the y- / y+ neighbour
        const uint32_t d_x0 = 8u * L;                                         // x cell (z, y) = L
        const uint32_t d_x1 = d_x0 + 256u;                                    //              = L + 32
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
            for (int j = 0; j < kB31; ++j, ++k) {
                const int c_cur = chunk_of(__shfl_sync(0xffffffffu, e_c, j));
                const uint32_t st = sm0 + s * kStage41, full = full0 + 8u * s;
                if (k >= (uint32_t)kSt41) mbar_wait(empty0 + 8u * s, ph ^ 1u);
                if (c_cur < 0) {  // end marker: the compute warps stop at this stage
                    if (lane == 0) {
                        sts_u32(st + kCtx41 + 176u, 0xFFFFFFFFu);
                        mbar_arrive(full);
                    }
                    cp_mbar_arrive_noinc(full);
                    done = true;
                    break;
                }
                const int nb0 = __shfl_sync(0xffffffffu, d0c.x, j), nb1 = __shfl_sync(0xffffffffu, d0c.y, j);
                const int nb2 = __shfl_sync(0xffffffffu, d0c.z, j), nb3 = __shfl_sync(0xffffffffu, d0c.w, j);
                const int nb4 = __shfl_sync(0xffffffffu, d1c.x, j), nb5 = __shfl_sync(0xffffffffu, d1c.y, j);
                const bool dl = !(__shfl_sync(0xffffffffu, d1c.w, j) & kFlagUnif);
                if (lane == 0) {
                    sts_u32(st + kCtx41 + 176u, (uint32_t)c_cur);
                    mbar_arrive_tx(full, 176u);
                    bulk_g2s(st + kCtx41, ctxa + (int64_t)c_cur * kCtxWords30, 176u, full);
                }
                // own slabs: plane i, rows 2 (L/8).. as 16-B pieces (8 per lane)
                const uint32_t so = (uint32_t)c_cur * 512u + 2u * L;
                const double* gu = u + so;
                const double* gd = de + so;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cp16(st + d_own + (uint32_t)i * kPP41, gu + 64 * i, true);
                    cp16(st + kHalf41 + d_own + (uint32_t)i * kPP41, gd + 64 * i, dl);
                }
                // z halos: plane 7 of the z- neighbour -> plane -1, plane 0 of the z+ neighbour -> plane 8
                {
                    const uint32_t zl = (uint32_t)nb4 * 512u + 448u + 2u * L, zh = (uint32_t)nb5 * 512u + 2u * L;
                    cp16(st + 64u + 16u * L, u + (nb4 >= 0 ? zl : 0u), nb4 >= 0);
                    cp16(st + 9u * kPP41 + 64u + 16u * L, u + (nb5 >= 0 ? zh : 0u), nb5 >= 0);
                    cp16(st + kHalf41 + 64u + 16u * L, de + (nb4 >= 0 ? zl : sent_off + 2u * L), dl);
                    cp16(st + kHalf41 + 9u * kPP41 + 64u + 16u * L, de + (nb5 >= 0 ? zh : sent_off + 2u * L), dl);
                }
                // y halos: row 7 of the y- neighbour -> row -1, row 0 of the y+ neighbour -> row 8
                {
                    const uint32_t yl = (uint32_t)nb2 * 512u + 56u + s_ylo, yh = (uint32_t)nb3 * 512u + s_ylo;
                    cp16(st + d_ylo, u + (nb2 >= 0 ? yl : 0u), nb2 >= 0);
                    cp16(st + d_ylo + 576u, u + (nb3 >= 0 ? yh : 0u), nb3 >= 0);
                    cp16(st + kHalf41 + d_ylo, de + (nb2 >= 0 ? yl : sent_off + s_ylo), dl);
                    cp16(st + kHalf41 + d_ylo + 576u, de + (nb3 >= 0 ? yh : sent_off + s_ylo), dl);
                }
                // x halos: column 7 of the x- neighbour, column 0 of the x+ neighbour, cells (z, y) = L, L + 32
                {
                    const uint32_t xl = (uint32_t)nb0 * 512u + 8u * L + 7u, xh = (uint32_t)nb1 * 512u + 8u * L;
                    const uint32_t xs = sent_off + 8u * L;
                    cp8(st + d_x0 + kXL41, u + (nb0 >= 0 ? xl : 0u), nb0 >= 0);
                    cp8(st + d_x1 + kXL41, u + (nb0 >= 0 ? xl + 256u : 0u), nb0 >= 0);
                    cp8(st + d_x0 + kXH41, u + (nb1 >= 0 ? xh : 0u), nb1 >= 0);
                    cp8(st + d_x1 + kXH41, u + (nb1 >= 0 ? xh + 256u : 0u), nb1 >= 0);
                    cp8(st + kHalf41 + d_x0 + kXL41, de + (nb0 >= 0 ? xl : xs), dl);
                    cp8(st + kHalf41 + d_x1 + kXL41, de + (nb0 >= 0 ? xl + 256u : xs + 256u), dl);
                    cp8(st + kHalf41 + d_x0 + kXH41, de + (nb1 >= 0 ? xh : xs), dl);
                    cp8(st + kHalf41 + d_x1 + kXH41, de + (nb1 >= 0 ? xh + 256u : xs + 256u), dl);
                }
                cp_mbar_arrive_noinc(full);
                if (++s == (uint32_t)kSt41) {
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
    Consts Q;
    Q.dt = A.dt;
    Q.neg_k = A.neg_k;
    Q.src_factor = A.src_factor;
    Q.ix = A.inv_dx2[0];
    Q.iy = A.inv_dx2[1];
    Q.iz = A.inv_dx2[2];
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t z0 = 2u * (uint32_t)warp;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp);
    const uint32_t pz0 = (z0 + 1u) * kPP41;
    const uint32_t v_c = pz0 + (uint32_t)(y + 1) * 64u + 16u * (uint32_t)xp;
    const uint32_t o_c = pin(v_c, lane);
    // x-halo cell of plane z0 (x+ block for xp = 3; x- block otherwise: the
    // interior lanes' copy of their row's x- cell is a broadcast, unused)
    const uint32_t o_x = pin((xp == 3 ? kXH41 : kXL41) + z0 * 64u + 8u * (uint32_t)y, lane);
    const bool xlo = xp == 0, xhi = xp == 3;
    const uint32_t zsh = 2u * z0;
    double* __restrict__ un = A.un;
    const uint32_t huge_hi = A.huge_hi;
    bool pushed = false;
    uint32_t s = 0, ph = 0;
#pragma unroll 1
    for (;;) {
        mbar_wait(full0 + 8u * s, ph);
        const uint32_t st = sm0 + s * kStage41;
        const int c = (int)lds_u32(st + kCtx41 + 176u);
        if (c < 0) break;
        const uint32_t lm = lds_u32(st + kCtx41 + 4u * (uint32_t)lane);
        const int flags = (int)lds_u32(st + kCtx41 + 156u);
        const uint32_t ab = (lm >> zsh) & 0xFu;
        const uint32_t sk = (lm >> (16u + zsh)) & 0xFu;
        const uint32_t g_off = z0 * 64u + bp;
        double src[4] = {0.0, 0.0, 0.0, 0.0};
        if (REACTION == PD_REACTION_VOLUMETRIC) {
            const double* sp = A.src + (int64_t)c * 512 + g_off;
            src[0] = sp[0];
            src[1] = sp[1];
            src[2] = sp[64];
            src[3] = sp[65];
        }
        const uint32_t a = st + o_c, ax = st + o_x;
        const double2 uc0 = lds2(a), uc1 = lds2(a + kPP41);
        const double2 uzm = lds2(a - kPP41), uzp = lds2(a + 2u * kPP41);
        const double uh0 = lds1(ax), uh1 = lds1(ax + 64u);
        // every lane shuffles (full mask), then the face lanes take the halo cell
        const double su0 = __shfl_up_sync(0xffffffffu, uc0.y, 1), sd0 = __shfl_down_sync(0xffffffffu, uc0.x, 1);
        const double su1 = __shfl_up_sync(0xffffffffu, uc1.y, 1), sd1 = __shfl_down_sync(0xffffffffu, uc1.x, 1);
        const double uL0 = xlo ? uh0 : su0, uR0 = xhi ? uh0 : sd0;
        const double uL1 = xlo ? uh1 : su1, uR1 = xhi ? uh1 : sd1;
        const double2 uym0 = lds2(a - 64u), uyp0 = lds2(a + 64u);
        const double2 uym1 = lds2(a + kPP41 - 64u), uyp1 = lds2(a + kPP41 + 64u);
        double o00, o01, o10, o11;
        const uint32_t ib = ((uint32_t)flags >> (8u + z0)) & 3u;
        if (flags & kFlagUnif) {
            const double dv = lds1(st + kCtx41 + 160u);
            const double dh = HALF ? dv + dv : (dv + dv) * 0.5;
            const double fzx = dh * (uc1.x - uc0.x), fzy = dh * (uc1.y - uc0.y);
            const double f0i = dh * (uc0.y - uc0.x), f1i = dh * (uc1.y - uc1.x);
            o00 = node31<REACTION>(Q, uc0.x, dh * (uc0.x - uL0), f0i, dh * (uc0.x - uym0.x), dh * (uyp0.x - uc0.x),
                                   dh * (uc0.x - uzm.x), fzx, sk & 1u, src[0]);
            o01 = node31<REACTION>(Q, uc0.y, f0i, dh * (uR0 - uc0.y), dh * (uc0.y - uym0.y), dh * (uyp0.y - uc0.y),
                                   dh * (uc0.y - uzm.y), fzy, sk & 2u, src[1]);
            o10 = node31<REACTION>(Q, uc1.x, dh * (uc1.x - uL1), f1i, dh * (uc1.x - uym1.x), dh * (uyp1.x - uc1.x),
                                   fzx, dh * (uzp.x - uc1.x), sk & 4u, src[2]);
            o11 = node31<REACTION>(Q, uc1.y, f1i, dh * (uR1 - uc1.y), dh * (uc1.y - uym1.y), dh * (uyp1.y - uc1.y),
                                   fzy, dh * (uzp.y - uc1.y), sk & 8u, src[3]);
        } else {
            const uint32_t b = a + kHalf41, bx = ax + kHalf41;
            const double2 dc0 = lds2(b), dc1 = lds2(b + kPP41);
            const double2 dzm = lds2(b - kPP41), dzp = lds2(b + 2u * kPP41);
            const double dh0 = lds1(bx), dh1 = lds1(bx + 64u);
            const double tu0 = __shfl_up_sync(0xffffffffu, dc0.y, 1), td0 = __shfl_down_sync(0xffffffffu, dc0.x, 1);
            const double tu1 = __shfl_up_sync(0xffffffffu, dc1.y, 1), td1 = __shfl_down_sync(0xffffffffu, dc1.x, 1);
            const double dL0 = xlo ? dh0 : tu0, dR0 = xhi ? dh0 : td0;
            const double dL1 = xlo ? dh1 : tu1, dR1 = xhi ? dh1 : td1;
            const double2 dym0 = lds2(b - 64u), dyp0 = lds2(b + 64u);
            const double2 dym1 = lds2(b + kPP41 - 64u), dyp1 = lds2(b + kPP41 + 64u);
            if (ib == 3u) {
                const double fzx = fface<HALF>(dc0.x, dc1.x, uc0.x, uc1.x), fzy = fface<HALF>(dc0.y, dc1.y, uc0.y, uc1.y);
                const double f0i = fface<HALF>(dc0.x, dc0.y, uc0.x, uc0.y), f1i = fface<HALF>(dc1.x, dc1.y, uc1.x, uc1.y);
                o00 = node31<REACTION>(Q, uc0.x, fface<HALF>(dL0, dc0.x, uL0, uc0.x), f0i,
                                       fface<HALF>(dym0.x, dc0.x, uym0.x, uc0.x), fface<HALF>(dc0.x, dyp0.x, uc0.x, uyp0.x),
                                       fface<HALF>(dzm.x, dc0.x, uzm.x, uc0.x), fzx, sk & 1u, src[0]);
                o01 = node31<REACTION>(Q, uc0.y, f0i, fface<HALF>(dc0.y, dR0, uc0.y, uR0),
                                       fface<HALF>(dym0.y, dc0.y, uym0.y, uc0.y), fface<HALF>(dc0.y, dyp0.y, uc0.y, uyp0.y),
                                       fface<HALF>(dzm.y, dc0.y, uzm.y, uc0.y), fzy, sk & 2u, src[1]);
                o10 = node31<REACTION>(Q, uc1.x, fface<HALF>(dL1, dc1.x, uL1, uc1.x), f1i,
                                       fface<HALF>(dym1.x, dc1.x, uym1.x, uc1.x), fface<HALF>(dc1.x, dyp1.x, uc1.x, uyp1.x),
                                       fzx, fface<HALF>(dc1.x, dzp.x, uc1.x, uzp.x), sk & 4u, src[2]);
                o11 = node31<REACTION>(Q, uc1.y, f1i, fface<HALF>(dc1.y, dR1, uc1.y, uR1),
                                       fface<HALF>(dym1.y, dc1.y, uym1.y, uc1.y), fface<HALF>(dc1.y, dyp1.y, uc1.y, uyp1.y),
                                       fzy, fface<HALF>(dc1.y, dzp.y, uc1.y, uzp.y), sk & 8u, src[3]);
            } else {
                const double fzx = face<HALF>(dc0.x, dc1.x, uc0.x, uc1.x), fzy = face<HALF>(dc0.y, dc1.y, uc0.y, uc1.y);
                const double f0i = face<HALF>(dc0.x, dc0.y, uc0.x, uc0.y), f1i = face<HALF>(dc1.x, dc1.y, uc1.x, uc1.y);
                o00 = node31<REACTION>(Q, uc0.x, face<HALF>(dL0, dc0.x, uL0, uc0.x), f0i,
                                       face<HALF>(dym0.x, dc0.x, uym0.x, uc0.x), face<HALF>(dc0.x, dyp0.x, uc0.x, uyp0.x),
                                       face<HALF>(dzm.x, dc0.x, uzm.x, uc0.x), fzx, sk & 1u, src[0]);
                o01 = node31<REACTION>(Q, uc0.y, f0i, face<HALF>(dc0.y, dR0, uc0.y, uR0),
                                       face<HALF>(dym0.y, dc0.y, uym0.y, uc0.y), face<HALF>(dc0.y, dyp0.y, uc0.y, uyp0.y),
                                       face<HALF>(dzm.y, dc0.y, uzm.y, uc0.y), fzy, sk & 2u, src[1]);
                o10 = node31<REACTION>(Q, uc1.x, face<HALF>(dL1, dc1.x, uL1, uc1.x), f1i,
                                       face<HALF>(dym1.x, dc1.x, uym1.x, uc1.x), face<HALF>(dc1.x, dyp1.x, uc1.x, uyp1.x),
                                       fzx, face<HALF>(dc1.x, dzp.x, uc1.x, uzp.x), sk & 4u, src[2]);
                o11 = node31<REACTION>(Q, uc1.y, f1i, face<HALF>(dc1.y, dR1, uc1.y, uR1),
                                       face<HALF>(dym1.y, dc1.y, uym1.y, uc1.y), face<HALF>(dc1.y, dyp1.y, uc1.y, uyp1.y),
                                       fzy, face<HALF>(dc1.y, dzp.y, uc1.y, uzp.y), sk & 8u, src[3]);
                if (sentinel(dc0.x)) o00 = uc0.x;
                if (sentinel(dc0.y)) o01 = uc0.y;
                if (sentinel(dc1.x)) o10 = uc1.x;
                if (sentinel(dc1.y)) o11 = uc1.y;
            }
        }
        const uint32_t hm = max(max((uint32_t)__double2hiint(o00) & 0x7fffffffu, (uint32_t)__double2hiint(o01) & 0x7fffffffu),
                                max((uint32_t)__double2hiint(o10) & 0x7fffffffu, (uint32_t)__double2hiint(o11) & 0x7fffffffu));
        const bool slow = (flags & kFlagDirichlet) || hm >= huge_hi;
        if (__any_sync(0xffffffffu, slow)) {
            if (slow) {
                const double2 r0 = pair_slow41<REACTION, HALF>(M, K, st, lane, (int)z0, o00, o01);
                const double2 r1 = pair_slow41<REACTION, HALF>(M, K, st, lane, (int)z0 + 1, o10, o11);
                o00 = r0.x;
                o01 = r0.y;
                o10 = r1.x;
                o11 = r1.y;
            }
        }
        double* gp = un + ((uint32_t)c * 512u + g_off);
        stg_pair(gp, o00, o01, ab & 1u, ab & 2u);
        stg_pair(gp + 64, o10, o11, ab & 4u, ab & 8u);
        if (PUSH && (flags & (kFlagPushLo | kFlagPushHi)) && (z0 == 0 || z0 == 6)) {
            ChunkCtx14 C;
            C.c = c;
            C.key = (int)lds_u32(st + kCtx41 + 152u);
            C.flags = flags;
            C.lm = lm;
            C.dv = 0.0;
            if (z0 == 0) push_pair14(M, C, 0, bp, o00, o01, ab & 1u, ab & 2u);
            else push_pair14(M, C, 7, bp, o10, o11, ab & 4u, ab & 8u);
            pushed = true;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * s);
        if (++s == (uint32_t)kSt41) {
            s = 0;
            ph ^= 1u;
        }
    }
    if (PUSH && pushed) __threadfence_system();
}

// ---------------------------------------------------------------------------
// v43: v41 with the x halos on the TMA engine. In v41 the producer's 8-B
// x-halo gathers (64 rows of a neighbour's column per side) cost ~94
// shared-memory wavefronts per chunk (15 per instruction against 2 ideal).
// A TMA box {2,8,8,1} moves columns 6-7 of the x- neighbour / 0-1 of the x+
// neighbour into an [z][y][pair] block (1 KB per side) without the LSU;
// lanes on the x faces read x = 7 / x = 0 of their row's pair
// (conflict-free: the x- and x+ blocks use alternate 8-B halves of a bank
// pair). Everything else as v41.
// ---------------------------------------------------------------------------
constexpr uint32_t kPP43 = 640;                 // plane pitch
constexpr uint32_t kXL43 = 10 * kPP43, kXH43 = kXL43 + 1024;  // x-halo blocks [z][y][pair] (TMA, 128-B aligned)
constexpr uint32_t kHalf43 = kXH43 + 1024;      // D_eff half (8448)
constexpr uint32_t kCtx43 = 2 * kHalf43;        // chunk record, then the chunk id at +176
constexpr uint32_t kStage43 = kCtx43 + 256;     // 17152
constexpr int kSt43 = 3, kCtas43 = 4;
constexpr int kThreads43 = 32 * (kW31 + 1);
constexpr uint32_t smem43() { return kSt43 * kStage43 + 16u * kSt43; }

template <int REACTION, bool HALF>
__device__ __noinline__ double2 pair_slow43(const MarchArgs& M, const SlowConsts& K, uint32_t st, int lane, int z,
                                            double out0, double out1) {
    ChunkCtx14 C;
    C.c = (int)lds_u32(st + kCtx43 + 176u);
    C.lm = lds_u32(st + kCtx43 + 4u * (uint32_t)lane);
    C.key = (int)lds_u32(st + kCtx43 + 152u);
    C.flags = (int)lds_u32(st + kCtx43 + 156u);
    C.dv = lds1(st + kCtx43 + 160u);
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp), pz = st + (uint32_t)(z + 1) * kPP43;
    Addr30 a;
    a.c = pz + (uint32_t)(y + 1) * 64u + 16u * (uint32_t)xp;
    a.zm = a.c - kPP43;
    a.zp = a.c + kPP43;
    a.ym = a.c - 64u;
    a.yp = a.c + 64u;
    a.l = xp > 0 ? a.c - 8u : st + kXL43 + ((uint32_t)z * 8u + (uint32_t)y) * 16u + 8u;
    a.r = xp < 3 ? a.c + 16u : st + kXH43 + ((uint32_t)z * 8u + (uint32_t)y) * 16u;
    return pair_slow30<REACTION, HALF, kHalf43>(M, K, C, z, xp, y, bp, a, out0, out1);
}

// u + dt * lap of one node (solver.hpp:420-441 without the reaction term,
// which ftcs_march43_kernel adds per warp)
__device__ __forceinline__ double node31x(const Consts& Q, double uc, double fxm, double fxp, double fym, double fyp,
                                          double fzm, double fzp) {
    double lap = 0.0;
    lap += (fxp - fxm) * Q.ix;
    lap += (fyp - fym) * Q.iy;
    lap += (fzp - fzm) * Q.iz;
    return uc + Q.dt * lap;
}

template <int REACTION, bool PUSH, bool HALF>
__global__ void __launch_bounds__(kThreads43, kCtas43)
    ftcs_march43_kernel(const __grid_constant__ MarchArgs M, const uint32_t* __restrict__ ctxa,
                        const __grid_constant__ CUtensorMap mux, const __grid_constant__ CUtensorMap mdx) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const StepArgs<double>& A = M.A;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = sm0 + kSt43 * kStage43, empty0 = full0 + 8u * kSt43;
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
        K.huge_hi = A.huge_hi;
        for (int s = 0; s < kSt43; ++s) {
            mbar_init(full0 + 8u * s, 33u);  // lane 0's expect_tx arrive + 32 cp.async arrivals
            mbar_init(empty0 + 8u * s, (uint32_t)kW31);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const double* __restrict__ u = A.u;
    const double* __restrict__ de = M.deff;
    const int n = (int)M.n;

    if (warp == kW31) {  // ---------------- producer warp ----------------
        // batch pipeline as v31: claim of batch b+3, entries of b+2,
        // descriptors and L2 prefetch of b+1 issued while batch b is copied
        int* ctr = M.counter;
        const int4* desc4 = reinterpret_cast<const int4*>(M.desc);
        const uint32_t sent_off = (uint32_t)M.n_all * 512u;  // D_eff sentinel chunk (elements)
        auto claim = [&]() -> int {
            int r = 0;
            if (lane == 0)
                asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(ctr), "r"(kB31) : "memory");
            return r;
        };
        auto entries = [&](int p0) -> int {
            const int p = __shfl_sync(0xffffffffu, p0, 0) + lane;
            return lane < kB31 && p < n ? __ldg(&M.sched[p]) : -1;
        };
        auto chunk_of = [](int e) { return e == -1 ? -1 : (int)((uint32_t)e & 0x7FFFFFFFu); };
        auto descs = [&](int e, int4& d0, int4& d1) {
            const int c = chunk_of(e);
            if (lane < kB31 && c >= 0) {
                d0 = __ldg(desc4 + 2 * (int64_t)c);
                d1 = __ldg(desc4 + 2 * (int64_t)c + 1);
            }
        };
        // M.pf: bit 0 L2 prefetch of the next batch's u slabs and records,
        // bit 1 of its D_eff slabs, bit 2 skip the own-slab copies of pairs
        // with no active node (their D_eff is written as the sentinel)
        const int pf = M.pf;
        auto prefetch = [&](int e) {
            const int64_t c = (int64_t)chunk_of(e);
            if (lane < kB31 && c >= 0) {
                if (pf & 1) {
                    prefetch_l2(u + c * 512, 4096u);
                    prefetch_l2(ctxa + c * kCtxWords30, 176u);
                }
                if ((pf & 2) && e >= 0) prefetch_l2(de + c * 512, 4096u);
            }
        };
        // this lane's active-pair word (chunk record lm[lane]) of chunk j of a batch
        auto lm_of = [&](int e, int j) -> uint32_t {
            const int c = chunk_of(__shfl_sync(0xffffffffu, e, j));
            return (pf & 4) && c >= 0 ? __ldg(ctxa + (int64_t)c * kCtxWords30 + lane) : 0xFFFFu;
        };
        int e_c = entries(claim());
        int e_n = entries(claim());
        int p_nn = claim();
        int4 d0c = make_int4(0, 0, 0, 0), d1c = d0c;
        descs(e_c, d0c, d1c);
        prefetch(e_c);
        static_assert(kB31 == 4, "v43 rotates four per-chunk lane-mask words per batch");
        uint32_t lc0 = lm_of(e_c, 0), lc1 = lm_of(e_c, 1), lc2 = lm_of(e_c, 2), lc3 = lm_of(e_c, 3);
        // per-lane destinations (stage-relative) and source element offsets
        const uint32_t L = (uint32_t)lane;
        const uint32_t d_own = kPP43 + 64u + 16u * L;                        // + 640 i: row pair L of plane i
        const uint32_t d_ylo = kPP43 * ((L >> 2) + 1u) + 16u * (L & 3u);      // row -1 of plane L/4
        const uint32_t s_ylo = 64u * (L >> 2) + 2u * (L & 3u);                // of the y- / y+ neighbour
        uint32_t s = 0, ph = 0, k = 0;
#pragma unroll 1
        for (;;) {
            int4 d0n = make_int4(0, 0, 0, 0), d1n = d0n;
            descs(e_n, d0n, d1n);
            prefetch(e_n);
            const uint32_t ln0 = lm_of(e_n, 0), ln1 = lm_of(e_n, 1), ln2 = lm_of(e_n, 2), ln3 = lm_of(e_n, 3);
            const int e_nn = entries(p_nn);
            p_nn = claim();
            bool done = false;
#pragma unroll 1
            for (int j = 0; j < kB31; ++j, ++k) {
                const int c_cur = chunk_of(__shfl_sync(0xffffffffu, e_c, j));
                const uint32_t st = sm0 + s * kStage43, full = full0 + 8u * s;
                if (k >= (uint32_t)kSt43) mbar_wait(empty0 + 8u * s, ph ^ 1u);
                if (c_cur < 0) {  // end marker: the compute warps stop at this stage
                    if (lane == 0) {
                        sts_u32(st + kCtx43 + 176u, 0xFFFFFFFFu);
                        mbar_arrive(full);
                    }
                    cp_mbar_arrive_noinc(full);
                    done = true;
                    break;
                }
                const int nb0 = __shfl_sync(0xffffffffu, d0c.x, j), nb1 = __shfl_sync(0xffffffffu, d0c.y, j);
                const int nb2 = __shfl_sync(0xffffffffu, d0c.z, j), nb3 = __shfl_sync(0xffffffffu, d0c.w, j);
                const int nb4 = __shfl_sync(0xffffffffu, d1c.x, j), nb5 = __shfl_sync(0xffffffffu, d1c.y, j);
                const bool dl = !(__shfl_sync(0xffffffffu, d1c.w, j) & kFlagUnif);
                if (lane == 0) {
                    sts_u32(st + kCtx43 + 176u, (uint32_t)c_cur);
                    mbar_arrive_tx(full, 176u + (nb0 >= 0 ? 1024u : 0u) + (nb1 >= 0 ? 1024u : 0u) + (dl ? 2048u : 0u));
                    bulk_g2s(st + kCtx43, ctxa + (int64_t)c_cur * kCtxWords30, 176u, full);
                    if (nb0 >= 0) tma4(st + kXL43, &mux, 6, 0, 0, nb0, full);
                    if (nb1 >= 0) tma4(st + kXH43, &mux, 0, 0, 0, nb1, full);
                    if (dl) {
                        const int sent_c = (int)M.n_all;
                        tma4(st + kHalf43 + kXL43, &mdx, 6, 0, 0, nb0 >= 0 ? nb0 : sent_c, full);
                        tma4(st + kHalf43 + kXH43, &mdx, 0, 0, 0, nb1 >= 0 ? nb1 : sent_c, full);
                    }
                }
                // own slabs: plane i, rows 2 (L/8).. as 16-B pieces (8 per lane)
                const uint32_t so = (uint32_t)c_cur * 512u + 2u * L;
                const double* gu = u + so;
                const double* gd = de + so;
                const uint32_t lmj = lc0;  // this lane's pair bits (2 per plane)
                lc0 = lc1;
                lc1 = lc2;
                lc2 = lc3;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool act = (lmj >> (2 * i)) & 3u;
                    cp16(st + d_own + (uint32_t)i * kPP43, gu + 64 * i, act);
                    cp16(st + kHalf43 + d_own + (uint32_t)i * kPP43, gd + 64 * i, dl && act);
                    if (dl && !act) {  // no active node: D_eff = sentinel, u never used
                        const uint32_t sh = kSentHi;
                        sts4(st + kHalf43 + d_own + (uint32_t)i * kPP43, 0u, sh, 0u, sh);
                    }
                }
                // z halos: plane 7 of the z- neighbour -> plane -1, plane 0 of the z+ neighbour -> plane 8
                {
                    const uint32_t zl = (uint32_t)nb4 * 512u + 448u + 2u * L, zh = (uint32_t)nb5 * 512u + 2u * L;
                    cp16(st + 64u + 16u * L, u + (nb4 >= 0 ? zl : 0u), nb4 >= 0);
                    cp16(st + 9u * kPP43 + 64u + 16u * L, u + (nb5 >= 0 ? zh : 0u), nb5 >= 0);
                    cp16(st + kHalf43 + 64u + 16u * L, de + (nb4 >= 0 ? zl : sent_off + 2u * L), dl);
                    cp16(st + kHalf43 + 9u * kPP43 + 64u + 16u * L, de + (nb5 >= 0 ? zh : sent_off + 2u * L), dl);
                }
                // y halos: row 7 of the y- neighbour -> row -1, row 0 of the y+ neighbour -> row 8
                {
                    const uint32_t yl = (uint32_t)nb2 * 512u + 56u + s_ylo, yh = (uint32_t)nb3 * 512u + s_ylo;
                    cp16(st + d_ylo, u + (nb2 >= 0 ? yl : 0u), nb2 >= 0);
                    cp16(st + d_ylo + 576u, u + (nb3 >= 0 ? yh : 0u), nb3 >= 0);
                    cp16(st + kHalf43 + d_ylo, de + (nb2 >= 0 ? yl : sent_off + s_ylo), dl);
                    cp16(st + kHalf43 + d_ylo + 576u, de + (nb3 >= 0 ? yh : sent_off + s_ylo), dl);
                }
                cp_mbar_arrive_noinc(full);
                if (++s == (uint32_t)kSt43) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (done) break;
            e_c = e_n;
            d0c = d0n;
            d1c = d1n;
            e_n = e_nn;
            lc0 = ln0;
            lc1 = ln1;
            lc2 = ln2;
            lc3 = ln3;
        }
        return;
    }

    // ---------------- compute warps ----------------
    if (M.dbg & 8) {  // measurement only (PD_MARCH_DBG=8): release every stage unread (the copy pipeline alone)
        uint32_t s = 0, ph = 0;
        for (;;) {
            mbar_wait(full0 + 8u * s, ph);
            if ((int)lds_u32(sm0 + s * kStage43 + kCtx43 + 176u) < 0) break;
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8u * s);
            if (++s == (uint32_t)kSt43) {
                s = 0;
                ph ^= 1u;
            }
        }
        return;
    }
    Consts Q;
    Q.dt = A.dt;
    Q.neg_k = A.neg_k;
    Q.src_factor = A.src_factor;
    Q.ix = A.inv_dx2[0];
    Q.iy = A.inv_dx2[1];
    Q.iz = A.inv_dx2[2];
    const int y = lane >> 2, xp = lane & 3;
    const uint32_t z0 = 2u * (uint32_t)warp;
    const uint32_t bp = (uint32_t)(y * 8 + 2 * xp);
    const uint32_t pz0 = (z0 + 1u) * kPP43;
    const uint32_t v_c = pz0 + (uint32_t)(y + 1) * 64u + 16u * (uint32_t)xp;
    const uint32_t o_c = pin(v_c, lane);
    // x-halo cell of plane z0 (x+ block for xp = 3; x- block otherwise: the
    // interior lanes' copy of their row's x- cell is a broadcast, unused)
    const uint32_t o_x = pin(xp == 3 ? kXH43 + (z0 * 8u + (uint32_t)y) * 16u : kXL43 + (z0 * 8u + (uint32_t)y) * 16u + 8u, lane);
    const bool xlo = xp == 0, xhi = xp == 3;
    const uint32_t zsh = 2u * z0;
    double* __restrict__ un = A.un;
    const uint32_t huge_hi = A.huge_hi;
    bool pushed = false;
    uint32_t s = 0, ph = 0;
#pragma unroll 1
    for (;;) {
        mbar_wait(full0 + 8u * s, ph);
        const uint32_t st = sm0 + s * kStage43;
        const int c = (int)lds_u32(st + kCtx43 + 176u);
        if (c < 0) break;
        const uint32_t lm = lds_u32(st + kCtx43 + 4u * (uint32_t)lane);
        const int flags = (int)lds_u32(st + kCtx43 + 156u);
        const uint32_t ab = (lm >> zsh) & 0xFu;
        const uint32_t sk = (lm >> (16u + zsh)) & 0xFu;
        const uint32_t g_off = z0 * 64u + bp;
        double src[4] = {0.0, 0.0, 0.0, 0.0};
        if (REACTION == PD_REACTION_VOLUMETRIC) {
            const double* sp = A.src + (int64_t)c * 512 + g_off;
            src[0] = sp[0];
            src[1] = sp[1];
            src[2] = sp[64];
            src[3] = sp[65];
        }
        const uint32_t a = st + o_c, ax = st + o_x;
        const double2 uc0 = lds2(a), uc1 = lds2(a + kPP43);
        const double2 uzm = lds2(a - kPP43), uzp = lds2(a + 2u * kPP43);
        const double uh0 = lds1(ax), uh1 = lds1(ax + 128u);
        // every lane shuffles (full mask), then the face lanes take the halo cell
        const double su0 = __shfl_up_sync(0xffffffffu, uc0.y, 1), sd0 = __shfl_down_sync(0xffffffffu, uc0.x, 1);
        const double su1 = __shfl_up_sync(0xffffffffu, uc1.y, 1), sd1 = __shfl_down_sync(0xffffffffu, uc1.x, 1);
        const double uL0 = xlo ? uh0 : su0, uR0 = xhi ? uh0 : sd0;
        const double uL1 = xlo ? uh1 : su1, uR1 = xhi ? uh1 : sd1;
        const double2 uym0 = lds2(a - 64u), uyp0 = lds2(a + 64u);
        const double2 uym1 = lds2(a + kPP43 - 64u), uyp1 = lds2(a + kPP43 + 64u);
        double o00, o01, o10, o11;  // u + dt * lap first, the reaction term below
        bool w00 = false, w01 = false, w10 = false, w11 = false;
        const uint32_t ib = ((uint32_t)flags >> (8u + z0)) & 3u;
        if (flags & kFlagUnif) {
            const double dv = lds1(st + kCtx43 + 160u);
            const double dh = HALF ? dv + dv : (dv + dv) * 0.5;
            const double fzx = dh * (uc1.x - uc0.x), fzy = dh * (uc1.y - uc0.y);
            const double f0i = dh * (uc0.y - uc0.x), f1i = dh * (uc1.y - uc1.x);
            o00 = node31x(Q, uc0.x, dh * (uc0.x - uL0), f0i, dh * (uc0.x - uym0.x), dh * (uyp0.x - uc0.x),
                                   dh * (uc0.x - uzm.x), fzx);
            o01 = node31x(Q, uc0.y, f0i, dh * (uR0 - uc0.y), dh * (uc0.y - uym0.y), dh * (uyp0.y - uc0.y),
                                   dh * (uc0.y - uzm.y), fzy);
            o10 = node31x(Q, uc1.x, dh * (uc1.x - uL1), f1i, dh * (uc1.x - uym1.x), dh * (uyp1.x - uc1.x),
                                   fzx, dh * (uzp.x - uc1.x));
            o11 = node31x(Q, uc1.y, f1i, dh * (uR1 - uc1.y), dh * (uc1.y - uym1.y), dh * (uyp1.y - uc1.y),
                                   fzy, dh * (uzp.y - uc1.y));
        } else {
            const uint32_t b = a + kHalf43, bx = ax + kHalf43;
            const double2 dc0 = lds2(b), dc1 = lds2(b + kPP43);
            const double2 dzm = lds2(b - kPP43), dzp = lds2(b + 2u * kPP43);
            const double dh0 = lds1(bx), dh1 = lds1(bx + 128u);
            const double tu0 = __shfl_up_sync(0xffffffffu, dc0.y, 1), td0 = __shfl_down_sync(0xffffffffu, dc0.x, 1);
            const double tu1 = __shfl_up_sync(0xffffffffu, dc1.y, 1), td1 = __shfl_down_sync(0xffffffffu, dc1.x, 1);
            const double dL0 = xlo ? dh0 : tu0, dR0 = xhi ? dh0 : td0;
            const double dL1 = xlo ? dh1 : tu1, dR1 = xhi ? dh1 : td1;
            const double2 dym0 = lds2(b - 64u), dyp0 = lds2(b + 64u);
            const double2 dym1 = lds2(b + kPP43 - 64u), dyp1 = lds2(b + kPP43 + 64u);
            if (ib == 3u) {
                const double fzx = fface<HALF>(dc0.x, dc1.x, uc0.x, uc1.x), fzy = fface<HALF>(dc0.y, dc1.y, uc0.y, uc1.y);
                const double f0i = fface<HALF>(dc0.x, dc0.y, uc0.x, uc0.y), f1i = fface<HALF>(dc1.x, dc1.y, uc1.x, uc1.y);
                o00 = node31x(Q, uc0.x, fface<HALF>(dL0, dc0.x, uL0, uc0.x), f0i,
                                       fface<HALF>(dym0.x, dc0.x, uym0.x, uc0.x), fface<HALF>(dc0.x, dyp0.x, uc0.x, uyp0.x),
                                       fface<HALF>(dzm.x, dc0.x, uzm.x, uc0.x), fzx);
                o01 = node31x(Q, uc0.y, f0i, fface<HALF>(dc0.y, dR0, uc0.y, uR0),
                                       fface<HALF>(dym0.y, dc0.y, uym0.y, uc0.y), fface<HALF>(dc0.y, dyp0.y, uc0.y, uyp0.y),
                                       fface<HALF>(dzm.y, dc0.y, uzm.y, uc0.y), fzy);
                o10 = node31x(Q, uc1.x, fface<HALF>(dL1, dc1.x, uL1, uc1.x), f1i,
                                       fface<HALF>(dym1.x, dc1.x, uym1.x, uc1.x), fface<HALF>(dc1.x, dyp1.x, uc1.x, uyp1.x),
                                       fzx, fface<HALF>(dc1.x, dzp.x, uc1.x, uzp.x));
                o11 = node31x(Q, uc1.y, f1i, fface<HALF>(dc1.y, dR1, uc1.y, uR1),
                                       fface<HALF>(dym1.y, dc1.y, uym1.y, uc1.y), fface<HALF>(dc1.y, dyp1.y, uc1.y, uyp1.y),
                                       fzy, fface<HALF>(dc1.y, dzp.y, uc1.y, uzp.y));
            } else {
                const double fzx = face<HALF>(dc0.x, dc1.x, uc0.x, uc1.x), fzy = face<HALF>(dc0.y, dc1.y, uc0.y, uc1.y);
                const double f0i = face<HALF>(dc0.x, dc0.y, uc0.x, uc0.y), f1i = face<HALF>(dc1.x, dc1.y, uc1.x, uc1.y);
                o00 = node31x(Q, uc0.x, face<HALF>(dL0, dc0.x, uL0, uc0.x), f0i,
                                       face<HALF>(dym0.x, dc0.x, uym0.x, uc0.x), face<HALF>(dc0.x, dyp0.x, uc0.x, uyp0.x),
                                       face<HALF>(dzm.x, dc0.x, uzm.x, uc0.x), fzx);
                o01 = node31x(Q, uc0.y, f0i, face<HALF>(dc0.y, dR0, uc0.y, uR0),
                                       face<HALF>(dym0.y, dc0.y, uym0.y, uc0.y), face<HALF>(dc0.y, dyp0.y, uc0.y, uyp0.y),
                                       face<HALF>(dzm.y, dc0.y, uzm.y, uc0.y), fzy);
                o10 = node31x(Q, uc1.x, face<HALF>(dL1, dc1.x, uL1, uc1.x), f1i,
                                       face<HALF>(dym1.x, dc1.x, uym1.x, uc1.x), face<HALF>(dc1.x, dyp1.x, uc1.x, uyp1.x),
                                       fzx, face<HALF>(dc1.x, dzp.x, uc1.x, uzp.x));
                o11 = node31x(Q, uc1.y, f1i, face<HALF>(dc1.y, dR1, uc1.y, uR1),
                                       face<HALF>(dym1.y, dc1.y, uym1.y, uc1.y), face<HALF>(dc1.y, dyp1.y, uc1.y, uyp1.y),
                                       fzy, face<HALF>(dc1.y, dzp.y, uc1.y, uzp.y));
                w00 = sentinel(dc0.x);  // walls (solver.hpp:413-417), applied after the reaction term
                w01 = sentinel(dc0.y);
                w10 = sentinel(dc1.x);
                w11 = sentinel(dc1.y);
            }
        }
        // + dt * r (solver.hpp:437-441): r = 0 on nodes without a reaction, and
        // dt * 0 = +0 (dt validated positive and finite), so warps without a
        // sink node add +0 and skip the two products
        if (REACTION == PD_REACTION_SURFACE_SINK && __any_sync(0xffffffffu, sk != 0u)) {
            o00 = o00 + Q.dt * ((sk & 1u) ? Q.neg_k * uc0.x : 0.0);
            o01 = o01 + Q.dt * ((sk & 2u) ? Q.neg_k * uc0.y : 0.0);
            o10 = o10 + Q.dt * ((sk & 4u) ? Q.neg_k * uc1.x : 0.0);
            o11 = o11 + Q.dt * ((sk & 8u) ? Q.neg_k * uc1.y : 0.0);
        } else if (REACTION == PD_REACTION_VOLUMETRIC) {
            o00 = o00 + Q.dt * (src[0] * Q.src_factor);
            o01 = o01 + Q.dt * (src[1] * Q.src_factor);
            o10 = o10 + Q.dt * (src[2] * Q.src_factor);
            o11 = o11 + Q.dt * (src[3] * Q.src_factor);
        } else {
            o00 = o00 + 0.0;
            o01 = o01 + 0.0;
            o10 = o10 + 0.0;
            o11 = o11 + 0.0;
        }
        if (w00) o00 = uc0.x;
        if (w01) o01 = uc0.y;
        if (w10) o10 = uc1.x;
        if (w11) o11 = uc1.y;
        const uint32_t hm = max(max((uint32_t)__double2hiint(o00) & 0x7fffffffu, (uint32_t)__double2hiint(o01) & 0x7fffffffu),
                                max((uint32_t)__double2hiint(o10) & 0x7fffffffu, (uint32_t)__double2hiint(o11) & 0x7fffffffu));
        const bool slow = (flags & kFlagDirichlet) || hm >= huge_hi;
        if (__any_sync(0xffffffffu, slow)) {
            if (slow) {
                const double2 r0 = pair_slow43<REACTION, HALF>(M, K, st, lane, (int)z0, o00, o01);
                const double2 r1 = pair_slow43<REACTION, HALF>(M, K, st, lane, (int)z0 + 1, o10, o11);
                o00 = r0.x;
                o01 = r0.y;
                o10 = r1.x;
                o11 = r1.y;
            }
        }
        double* gp = un + ((uint32_t)c * 512u + g_off);
        if ((flags & kFlagUnif) || ib == 3u) {  // every node of both planes active: plain 16-B stores
            stg2(gp, o00, o01);
            stg2(gp + 64, o10, o11);
        } else {
            stg_pair(gp, o00, o01, ab & 1u, ab & 2u);
            stg_pair(gp + 64, o10, o11, ab & 4u, ab & 8u);
        }
        if (PUSH && (flags & (kFlagPushLo | kFlagPushHi)) && (z0 == 0 || z0 == 6)) {
            ChunkCtx14 C;
            C.c = c;
            C.key = (int)lds_u32(st + kCtx43 + 152u);
            C.flags = flags;
            C.lm = lm;
            C.dv = 0.0;
            if (z0 == 0) push_pair14(M, C, 0, bp, o00, o01, ab & 1u, ab & 2u);
            else push_pair14(M, C, 7, bp, o10, o11, ab & 4u, ab & 8u);
            pushed = true;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * s);
        if (++s == (uint32_t)kSt43) {
            s = 0;
            ph ^= 1u;
        }
    }
    if (PUSH && pushed) __threadfence_system();
}

__global__ void sentinel_fill_kernel(double* p) { p[threadIdx.x] = sent(); }

// desc flags of the fused halo push: bit set iff the chunk has a peer ghost
__global__ void push_flags_kernel(int32_t* __restrict__ desc, const int32_t* __restrict__ ord, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int f = desc[i * 8 + 7] & ~(kFlagPushLo | kFlagPushHi);
    if (ord[2 * i] >= 0) f |= kFlagPushLo;
    if (ord[2 * i + 1] >= 0) f |= kFlagPushHi;
    desc[i * 8 + 7] = f;
}

// v30 chunk records: lm[32] | desc[8] | dv (2 words) | 2 pad words, one
// 176-B bulk copy per chunk
__global__ void pack_ctx_kernel(const uint32_t* __restrict__ lm, const int32_t* __restrict__ desc,
                                const uint32_t* __restrict__ dv, int dvw, int64_t n, uint32_t* __restrict__ ctx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * 44) return;
    const int64_t c = i / 44;
    const int w = (int)(i - c * 44);
    uint32_t v = 0;
    if (w < 32) v = lm[c * 32 + w];
    else if (w < 40) v = (uint32_t)desc[c * 8 + (w - 32)];
    else if (w < 40 + dvw) v = dv[c * dvw + (w - 40)];  // uniform D_eff: FP64 2 words, FP32 1
    ctx[i] = v;
}

void march_pack_ctx(pd_grid* g, MarchPlan& p) {
    const int64_t n = g->n_chunks;
    if (!p.d_ctx) PD_CUDA(pd_malloc(&p.d_ctx, sizeof(uint32_t) * 44 * (size_t)n));
    pack_ctx_kernel<<<(unsigned)((n * 44 + 255) / 256), 256, 0, g->stream>>>(
        p.d_lm, p.d_desc, static_cast<const uint32_t*>(p.d_dv), g->tbytes / 4, n, p.d_ctx);
    PD_CUDA(cudaGetLastError());
}

void march_push_flags(pd_grid* g, MarchPlan& p, const int32_t* d_ord) {
    if (!p.ready || g->n_chunks == 0) return;
    push_flags_kernel<<<(unsigned)((g->n_chunks + 255) / 256), 256, 0, g->stream>>>(p.d_desc, d_ord, g->n_chunks);
    PD_CUDA(cudaGetLastError());
    if (p.d_ctx) march_pack_ctx(g, p);
}

__global__ void desc_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ keys,
                            const uint64_t* __restrict__ flu, int64_t n, int64_t s0, int64_t s1,
                            int64_t s2, int dirichlet, int32_t* __restrict__ desc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k[3] = {keys[i * 3], keys[i * 3 + 1], keys[i * 3 + 2]};
    const int64_t s[3] = {s0, s1, s2};
    bool exposed = false;
    for (int a = 0; a < 3; ++a) {
        const bool lo = k[a] == 0;
        const bool hi = (int64_t)k[a] * 8 + 8 >= s[a];
        exposed = exposed || (lo && ((dirichlet >> (2 * a)) & 1)) || (hi && ((dirichlet >> (2 * a + 1)) & 1));
    }
    int nb[6];
    for (int f = 0; f < 6; ++f) nb[f] = nbr[i * 6 + f];
    uint64_t F[8];
    for (int z = 0; z < 8; ++z) F[z] = flu[i * 8 + z];
    int flags = exposed ? kFlagDirichlet : 0;
    // interior-fluid planes: the plane and every face neighbour of its nodes fluid
    const uint64_t ALL = ~0ull;
    const uint64_t zlo = nb[4] >= 0 ? flu[(int64_t)nb[4] * 8 + 7] : 0ull;
    const uint64_t zhi = nb[5] >= 0 ? flu[(int64_t)nb[5] * 8 + 0] : 0ull;
    for (int z = 0; z < 8 && !exposed; ++z) {
        bool ok = F[z] == ALL;
        ok = ok && (z > 0 ? F[z - 1] == ALL : zlo == ALL);
        ok = ok && (z < 7 ? F[z + 1] == ALL : zhi == ALL);
        ok = ok && nb[0] >= 0 && (flu[(int64_t)nb[0] * 8 + z] & 0x8080808080808080ull) == 0x8080808080808080ull;
        ok = ok && nb[1] >= 0 && (flu[(int64_t)nb[1] * 8 + z] & 0x0101010101010101ull) == 0x0101010101010101ull;
        ok = ok && nb[2] >= 0 && (flu[(int64_t)nb[2] * 8 + z] >> 56) == 0xFFull;
        ok = ok && nb[3] >= 0 && (flu[(int64_t)nb[3] * 8 + z] & 0xFFull) == 0xFFull;
        if (ok) flags |= 1 << (8 + z);
    }
    for (int f = 0; f < 6; ++f) desc[i * 8 + f] = nb[f];
    desc[i * 8 + 6] = k[0] | (k[1] << 10) | (k[2] << 20);
    desc[i * 8 + 7] = flags;
}

// Per chunk and lane (y = lane>>2, pair x0 = 2*(lane&3)): bit 2z+n = node n of
// the lane's pair in plane z is active, bit 16+2z+n = it is a sink node.
__global__ void lanemask_kernel(const uint64_t* __restrict__ act, const uint64_t* __restrict__ snk,
                                int64_t n, uint32_t* __restrict__ lm) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * 32) return;
    const int64_t c = t >> 5;
    const int lane = (int)(t & 31);
    const int bp = (lane >> 2) * 8 + 2 * (lane & 3);
    uint32_t v = 0;
    for (int z = 0; z < 8; ++z) {
        v |= (uint32_t)((act[c * 8 + z] >> bp) & 3ull) << (2 * z);
        v |= (uint32_t)((snk[c * 8 + z] >> bp) & 3ull) << (16 + 2 * z);
    }
    lm[t] = v;
}

// D_eff = fluid ? D : -inf over every slot; counts fluid nodes whose D is not
// finite (then the fast path is disabled: its sentinel logic assumes finite D).
// Uniform chunks (kFlagUnif): per chunk the common D_eff bit pattern of its
// 512 slots (all fluid), else the marker ~0 (a NaN, never a valid D_eff). B
// is the scalar's bit type (uint64 for FP64, uint32 for FP32 grids).
template <class B>
__global__ void unif_dv_kernel(const B* __restrict__ deff, int64_t n, B* __restrict__ dv, B sent_bits) {
    const int64_t c = blockIdx.x;
    const int lane = threadIdx.x;
    if (c >= n) return;
    const B* d = deff + c * 512;
    const B v0 = d[0];
    bool same = v0 != sent_bits;
    for (int i = lane; i < 512; i += 32) same = same && d[i] == v0;
    same = __all_sync(0xffffffffu, same);
    if (lane == 0) dv[c] = same ? v0 : (B)~(B)0;
}

// A chunk is uniform when its own slots share one D_eff value dv (all fluid)
// and the facing layer of each of its six neighbours (the only cells its
// faces read) holds dv too: one warp per chunk.
template <class B>
__global__ void unif_flag_kernel(int32_t* __restrict__ desc, const B* __restrict__ d, const B* __restrict__ dv,
                                 int64_t n) {
    const int64_t c = blockIdx.x;
    const int lane = threadIdx.x;
    if (c >= n) return;
    const B v = dv[c];
    if (v == (B)~(B)0) return;
    bool ok = true;
    for (int f = 0; f < 6; ++f) {
        const int j = desc[c * 8 + f];
        if (j < 0) {
            ok = false;
            break;
        }
        for (int k = lane; k < 64; k += 32) {  // facing layer of neighbour j
            const int a = k & 7, b = k >> 3;
            int off;
            switch (f) {
                case 0: off = (b << 6) | (a << 3) | 7; break;  // x- neighbour: its x = 7 column
                case 1: off = (b << 6) | (a << 3); break;      // x+ : x = 0
                case 2: off = (b << 6) | (7 << 3) | a; break;  // y- : y = 7 row
                case 3: off = (b << 6) | a; break;             // y+ : y = 0
                case 4: off = (7 << 6) | (b << 3) | a; break;  // z- : z = 7 plane
                default: off = (b << 3) | a; break;            // z+ : z = 0
            }
            ok = ok && d[(int64_t)j * 512 + off] == v;
        }
        ok = __all_sync(0xffffffffu, ok);
        if (!ok) break;
    }
    if (lane == 0 && ok) desc[c * 8 + 7] |= kFlagUnif;
}

template <class B>
void mark_uniform(pd_grid* g, MarchPlan* plan, B sent_bits) {
    const int64_t n_all = g->n_chunks;
    B* dv = nullptr;
    PD_CUDA(pd_malloc(&dv, sizeof(B) * (size_t)n_all));
    plan->d_dv = dv;
    const B* deff = static_cast<const B*>(plan->d_deff);
    unif_dv_kernel<B><<<(unsigned)n_all, 32, 0, g->stream>>>(deff, n_all, dv, sent_bits);
    unif_flag_kernel<B><<<(unsigned)n_all, 32, 0, g->stream>>>(plan->d_desc, deff, dv, n_all);
    PD_CUDA(cudaGetLastError());
}

// D_eff = fluid ? D * (half ? 0.5 : 1) : -inf. bad[0] counts fluid nodes with
// a non-finite D (march disabled), bad[1] those with |D| < 2^-1021, where
// halving would not be exact (the plan keeps D unhalved then).
__global__ void deff_kernel(const double* __restrict__ dcol, const uint64_t* __restrict__ fluid,
                            int64_t n_slots, double* __restrict__ deff, unsigned long long* bad, int half) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_slots) return;
    const bool fl = (fluid[i >> 6] >> (i & 63)) & 1ull;
    const double v = dcol[i];
    deff[i] = fl ? (half ? v * 0.5 : v) : sent();
    if (fl && !isfinite(v)) atomicAdd(bad, 1ull);
    // halving is exact and commutes with the face sum only away from the
    // extremes: below 2^-1021 it would round, and at >= 2^1022 the reference's
    // d_a + d_b can overflow where h_a + h_b does not -- keep D unhalved then
    if (fl && (fabs(v) < 0x1p-1021 || fabs(v) >= 0x1p1022)) atomicAdd(bad + 1, 1ull);
}

void march_free(MarchPlan* p) {
    for (auto& sp : p->subs) {
        pd_free(sp.d_stream);
        pd_free(sp.d_counter);
    }
    pd_free(p->d_stream);
    pd_free(p->d_desc);
    pd_free(p->d_dv);
    pd_free(p->d_deff);
    pd_free(p->d_counter);
    pd_free(p->d_lm);
    pd_free(p->d_ctx);
    for (auto& f : p->flagged) pd_free(f.second);
    *p = MarchPlan{};
}

// Device schedule of the chunk ordinals [begin, end): (z-block of kSeg
// layers, 4x4 column tiles, column, z), so the chunks in flight form one
// short window and neighbour halos hit L2.
__global__ void sched_key_kernel(const int32_t* __restrict__ keys, int64_t begin, int64_t n,
                                 unsigned long long* __restrict__ sk, int32_t* __restrict__ ord, int seg, int tx,
                                 int ty) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t* k = keys + (begin + i) * 3;
    const unsigned long long x = (unsigned)k[0], y = (unsigned)k[1], z = (unsigned)k[2];
    // (z-block of seg layers, 2^tx x 2^ty column tile, column, z); keys < 1024
    // per axis, 10 bits per field
    sk[i] = ((z / (unsigned)seg) << 50) | ((y >> ty) << 40) | ((x >> tx) << 30) | (y << 20) | (x << 10) | z;
    ord[i] = (int32_t)(begin + i);
}

int32_t* march_schedule(pd_grid* g, int64_t begin, int64_t end) {
    // device radix sort of per-chunk schedule keys (the host sort cost ~20 ms
    // at 10^5 chunks)
    const int64_t n = end - begin;
    int32_t* d = nullptr;
    PD_CUDA(pd_malloc(&d, sizeof(int32_t) * (size_t)std::max<int64_t>(1, n)));
    if (n == 0) return d;
    unsigned long long *k_in = nullptr, *k_out = nullptr;
    int32_t* o_in = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    try {
        PD_CUDA(pd_malloc(&k_in, sizeof(unsigned long long) * (size_t)n));
        PD_CUDA(pd_malloc(&k_out, sizeof(unsigned long long) * (size_t)n));
        PD_CUDA(pd_malloc(&o_in, sizeof(int32_t) * (size_t)n));
        // PD_SCHED="seg,tx,ty" (A/B only): z-block depth and log2 column-tile sides
        static const int3 sc = [] {
            int3 v = make_int3(kSeg, 2, 2);
            if (const char* e = getenv("PD_SCHED")) {
                if (sscanf(e, "%d,%d,%d", &v.x, &v.y, &v.z) != 3 || v.x < 1 || v.y < 0 || v.y > 9 || v.z < 0 || v.z > 9)
                    v = make_int3(kSeg, 2, 2);
            }
            return v;
        }();
        sched_key_kernel<<<(unsigned)((n + 255) / 256), 256, 0, g->stream>>>(g->d_keys, begin, n, k_in, o_in, sc.x,
                                                                               sc.y, sc.z);
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, o_in, d, (int)n, 0, 60, g->stream));
        PD_CUDA(pd_malloc(&tmp, tb));
        PD_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, o_in, d, (int)n, 0, 60, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    } catch (...) {
        pd_free(k_in);
        pd_free(k_out);
        pd_free(o_in);
        pd_free(tmp);
        pd_free(d);
        throw;
    }
    pd_free(k_in);
    pd_free(k_out);
    pd_free(o_in);
    pd_free(tmp);
    return d;
}

void march_build(pd_grid* g, const int32_t* d_nbr, const uint64_t* d_fluid, const uint64_t* d_sink,
                 const void* d_dcol, int dirichlet, int64_t begin, int64_t end, MarchPlan* plan) {
    march_free(plan);
    if (g->dims != 3) return;
    if (g->cc[0] > 1024 || g->cc[1] > 1024 || g->cc[2] > 1024) return;  // key packing limit
    const int64_t n_all = g->n_chunks;
    if (n_all == 0 || end <= begin) return;
    if (n_all * 512 >= (int64_t)0xFFFFFFFF) return;  // 32-bit slot offsets (>16 GB per column)
    PD_CUDA(pd_malloc(&plan->d_desc, sizeof(int32_t) * 8 * (size_t)n_all));
    desc_kernel<<<(unsigned)((n_all + 255) / 256), 256, 0, g->stream>>>(
        d_nbr, g->d_keys, d_fluid, n_all, g->size[0], g->size[1], g->size[2], dirichlet, plan->d_desc);
    PD_CUDA(cudaGetLastError());
    PD_CUDA(pd_malloc(&plan->d_lm, sizeof(uint32_t) * 32 * (size_t)n_all));
    lanemask_kernel<<<(unsigned)((n_all * 32 + 255) / 256), 256, 0, g->stream>>>(g->d_masks, d_sink,
                                                                                n_all, plan->d_lm);
    PD_CUDA(cudaGetLastError());
    const int64_t slots = n_all * 512;
    PD_CUDA(pd_malloc(&plan->d_counter, sizeof(int) * 1024));
    if (g->tbytes == 4) {
        if (!march32_deff(g, d_dcol, d_fluid, &plan->d_deff, &plan->half)) {
            march_free(plan);  // non-finite D on a fluid node: keep the exact tile kernel
            return;
        }
        mark_uniform<unsigned>(g, plan, 0xFF800000u);
        march_pack_ctx(g, *plan);
    } else {
        // one extra chunk of sentinels after the last one: the source of every
        // D_eff cell a plane load does not read from the grid (inactive pairs,
        // missing neighbours), so the loads need no shared-memory sentinel stores
        double* deff = nullptr;
        PD_CUDA(pd_malloc(&deff, sizeof(double) * (size_t)(slots + 512)));
        plan->d_deff = deff;
        sentinel_fill_kernel<<<1, 512, 0, g->stream>>>(deff + slots);
        unsigned long long* d_bad = nullptr;
        PD_CUDA(pd_malloc(&d_bad, 2 * sizeof(unsigned long long)));
        PD_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(unsigned long long), g->stream));
        static const int half_env = [] {
            const char* e = getenv("PD_MARCH_HALF");
            return e ? atoi(e) : 1;
        }();
        deff_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, g->stream>>>((const double*)d_dcol, d_fluid, slots,
                                                                            deff, d_bad, half_env);
        PD_CUDA(cudaGetLastError());
        unsigned long long bad[2] = {0, 0};
        PD_CUDA(cudaMemcpyAsync(bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        if (bad[0]) {  // non-finite D on a fluid node: keep the exact tile kernel
            pd_free(d_bad);
            march_free(plan);
            return;
        }
        plan->half = half_env && !bad[1];
        if (half_env && bad[1]) {  // tiny D somewhere: store D unhalved
            PD_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(unsigned long long), g->stream));
            deff_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, g->stream>>>((const double*)d_dcol, d_fluid,
                                                                                slots, deff, d_bad, 0);
            PD_CUDA(cudaGetLastError());
        }
        pd_free(d_bad);
        mark_uniform<unsigned long long>(g, plan, 0xFFF0000000000000ull);
        march_pack_ctx(g, *plan);
    }
    const int64_t n = end - begin;
    plan->d_stream = march_schedule(g, begin, end);
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    plan->grid = sms * kCtasPerSm;
    plan->n = n;
    plan->ready = true;
}

int march_counters_per_step() { return 1; }

void march_launch(pd_grid* g, MarchPlan& p, const StepArgs<double>& a, int reaction, const PeerLaunch* pl) {
    march_launch_sched(g, p, a, reaction, p.d_stream, p.n, p.d_counter + (a.k & 1023), pl);
}

// Sub-range schedule of the plan (built once per distinct [begin, end)).
MarchPlan::Sub& march_sub(pd_grid* g, MarchPlan& p, int64_t begin, int64_t end) {
    for (auto& sp : p.subs)
        if (sp.begin == begin && sp.end == end) return sp;
    MarchPlan::Sub sp;
    sp.begin = begin;
    sp.end = end;
    sp.n = end - begin;
    sp.d_stream = march_schedule(g, begin, end);
    PD_CUDA(pd_malloc(&sp.d_counter, sizeof(int)));
    p.subs.push_back(sp);
    return p.subs.back();
}

// ---- v30 host side: TMA tensor maps over the [chunk][z][y][x] columns ----
namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    if (!fn) fail(PD_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old for TMA)");
    return fn;
}

// 4-D FP64 view of a column: dims (x 8, y 8, z 8, chunk n), box `box`
CUtensorMap column_map(const double* base, int64_t n_chunks, const cuuint32_t box[4]) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {8, 8, 8, (cuuint64_t)n_chunks};
    const cuuint64_t strides[3] = {64, 512, 4096};  // bytes, dims 1..3
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(PD_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}
}  // namespace

__global__ void flag_sched_kernel(const int32_t* __restrict__ sched, const int32_t* __restrict__ desc, int64_t n,
                                  int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t c = sched[i];
    out[i] = (desc[(int64_t)c * 8 + 7] & kFlagUnif) ? (int32_t)((uint32_t)c | 0x80000000u) : c;
}

const int32_t* flagged_schedule(pd_grid* g, MarchPlan& p, const int32_t* sched, int64_t n) {
    for (auto& f : p.flagged)
        if (f.first == sched) return f.second;
    int32_t* d = nullptr;
    PD_CUDA(pd_malloc(&d, sizeof(int32_t) * (size_t)std::max<int64_t>(1, n)));
    if (n > 0) {
        flag_sched_kernel<<<(unsigned)((n + 255) / 256), 256, 0, g->stream>>>(sched, p.d_desc, n, d);
        PD_CUDA(cudaGetLastError());
    }
    p.flagged.emplace_back(sched, d);
    return d;
}

const int32_t* march_flagged_schedule(pd_grid* g, MarchPlan& p, const int32_t* sched, int64_t n) {
    return flagged_schedule(g, p, sched, n);
}

void march30_launch(pd_grid* g, MarchPlan& p, MarchArgs M, int r, bool push) {
    if (!p.d_ctx) fail(PD_E_INPUT, "march v30 needs the packed chunk records (3-D FP64 plan)");
    M.sched = flagged_schedule(g, p, M.sched, M.n);
    static const cuuint32_t bx[4] = {2, 8, 8, 1}, by[4] = {8, 1, 8, 1};
    const CUtensorMap mux = column_map(M.A.u, g->n_chunks, bx), muy = column_map(M.A.u, g->n_chunks, by);
    const CUtensorMap mdx = column_map(M.deff, g->n_chunks + 1, bx), mdy = column_map(M.deff, g->n_chunks + 1, by);
    using K30 = void (*)(const MarchArgs, const uint32_t*, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                         const CUtensorMap);
#define PD_M_TABLE(N)                                                                                         \
    {{{ftcs_march30_kernel<0, false, false, N>, ftcs_march30_kernel<1, false, false, N>,                       \
       ftcs_march30_kernel<2, false, false, N>},                                                               \
      {ftcs_march30_kernel<0, true, false, N>, ftcs_march30_kernel<1, true, false, N>,                         \
       ftcs_march30_kernel<2, true, false, N>}},                                                               \
     {{ftcs_march30_kernel<0, false, true, N>, ftcs_march30_kernel<1, false, true, N>,                         \
       ftcs_march30_kernel<2, false, true, N>},                                                                \
      {ftcs_march30_kernel<0, true, true, N>, ftcs_march30_kernel<1, true, true, N>,                           \
       ftcs_march30_kernel<2, true, true, N>}}}
    static const K30 tabs[7][2][2][3] = {PD_M_TABLE(0), PD_M_TABLE(1), PD_M_TABLE(2), PD_M_TABLE(3),
                                         PD_M_TABLE(4), PD_M_TABLE(5), PD_M_TABLE(6)};
#undef PD_M_TABLE
    static const int cfg = [] {
        const char* e = getenv("PD_M30_CFG");
        const int v = e ? atoi(e) : 5;
        return v >= 0 && v <= 6 ? v : 5;
    }();
    const K30(*tab)[2][3] = tabs[cfg];
    const uint32_t smem = smem30(nst30(cfg));
    const int ctas = ctas30(cfg);
    static uint64_t attr_done = 0;
    const int dev = g->device;
    if (dev < 0 || dev >= 64) fail(PD_E_INPUT, "device index out of range");
    if (!((attr_done >> dev) & 1u)) {
        for (int h = 0; h < 2; ++h)
            for (int q = 0; q < 2; ++q)
                for (int rr = 0; rr < 3; ++rr)
                    PD_CUDA(cudaFuncSetAttribute(tab[h][q][rr], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done |= 1ull << dev;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    tab[p.half ? 1 : 0][push ? 1 : 0][r]<<<sms * ctas, threads30(cfg), smem, g->stream>>>(M, p.d_ctx, mux, muy, mdx,
                                                                                          mdy);
    PD_CUDA(cudaGetLastError());
}

void march31_launch(pd_grid* g, MarchPlan& p, MarchArgs M, int r, bool push) {
    if (!p.d_ctx) fail(PD_E_INPUT, "march v31 needs the packed chunk records (3-D FP64 plan)");
    M.sched = flagged_schedule(g, p, M.sched, M.n);
    static const cuuint32_t by[4] = {8, 1, 8, 1};
    const CUtensorMap muy = column_map(M.A.u, g->n_chunks, by);
    const CUtensorMap mdy = column_map(M.deff, g->n_chunks + 1, by);
    using K31 = void (*)(const MarchArgs, const uint32_t*, const CUtensorMap, const CUtensorMap);
#define PD_M_TABLE(N)                                                                                         \
    {{{ftcs_march31_kernel<0, false, false, N>, ftcs_march31_kernel<1, false, false, N>,                       \
       ftcs_march31_kernel<2, false, false, N>},                                                               \
      {ftcs_march31_kernel<0, true, false, N>, ftcs_march31_kernel<1, true, false, N>,                         \
       ftcs_march31_kernel<2, true, false, N>}},                                                               \
     {{ftcs_march31_kernel<0, false, true, N>, ftcs_march31_kernel<1, false, true, N>,                         \
       ftcs_march31_kernel<2, false, true, N>},                                                                \
      {ftcs_march31_kernel<0, true, true, N>, ftcs_march31_kernel<1, true, true, N>,                           \
       ftcs_march31_kernel<2, true, true, N>}}}
    static const K31 tabs[4][2][2][3] = {PD_M_TABLE(0), PD_M_TABLE(1), PD_M_TABLE(2), PD_M_TABLE(3)};
#undef PD_M_TABLE
    static const int cfg = [] {
        const char* e = getenv("PD_M31_CFG");
        const int v = e ? atoi(e) : 0;
        return v >= 0 && v <= 3 ? v : 0;
    }();
    const K31(*tab)[2][3] = tabs[cfg];
    const uint32_t smem = smem30(nst31(cfg)) + (tab31(cfg) ? 2048u * (uint32_t)(kW31 * grp31(cfg)) : 0u);  // + offset tables
    static uint64_t attr_done[4] = {0, 0, 0, 0};
    const int dev = g->device;
    if (dev < 0 || dev >= 64) fail(PD_E_INPUT, "device index out of range");
    if (!((attr_done[cfg] >> dev) & 1u)) {
        for (int h = 0; h < 2; ++h)
            for (int q = 0; q < 2; ++q)
                for (int rr = 0; rr < 3; ++rr)
                    PD_CUDA(cudaFuncSetAttribute(tab[h][q][rr], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done[cfg] |= 1ull << dev;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (M.dbg & 64) {  // measurement only: resident CTAs per SM of this configuration
        static bool said = false;
        int occ = 0;
        PD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tab[p.half ? 1 : 0][push ? 1 : 0][r],
                                                              threads31(cfg), smem));
        if (!said) fprintf(stderr, "march31 cfg %d: %d threads, %u B smem, %d CTAs/SM resident (launching %d)\n", cfg,
                           threads31(cfg), smem, occ, ctas31(cfg));
        said = true;
    }
    tab[p.half ? 1 : 0][push ? 1 : 0][r]<<<sms * ctas31(cfg), threads31(cfg), smem, g->stream>>>(M, p.d_ctx, muy, mdy);
    PD_CUDA(cudaGetLastError());
}

void march41_launch(pd_grid* g, MarchPlan& p, MarchArgs M, int r, bool push) {
    if (!p.d_ctx) fail(PD_E_INPUT, "march v41 needs the packed chunk records (3-D FP64 plan)");
    M.sched = flagged_schedule(g, p, M.sched, M.n);
    using K41 = void (*)(const MarchArgs, const uint32_t*);
    static const K41 tab[2][2][3] = {
        {{ftcs_march41_kernel<0, false, false>, ftcs_march41_kernel<1, false, false>, ftcs_march41_kernel<2, false, false>},
         {ftcs_march41_kernel<0, true, false>, ftcs_march41_kernel<1, true, false>, ftcs_march41_kernel<2, true, false>}},
        {{ftcs_march41_kernel<0, false, true>, ftcs_march41_kernel<1, false, true>, ftcs_march41_kernel<2, false, true>},
         {ftcs_march41_kernel<0, true, true>, ftcs_march41_kernel<1, true, true>, ftcs_march41_kernel<2, true, true>}}};
    const uint32_t smem = smem41();
    static uint64_t attr_done = 0;
    const int dev = g->device;
    if (dev < 0 || dev >= 64) fail(PD_E_INPUT, "device index out of range");
    if (!((attr_done >> dev) & 1u)) {
        for (int h = 0; h < 2; ++h)
            for (int q = 0; q < 2; ++q)
                for (int rr = 0; rr < 3; ++rr)
                    PD_CUDA(cudaFuncSetAttribute(tab[h][q][rr], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done |= 1ull << dev;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    tab[p.half ? 1 : 0][push ? 1 : 0][r]<<<sms * kCtas41, kThreads41, smem, g->stream>>>(M, p.d_ctx);
    PD_CUDA(cudaGetLastError());
}

void march43_launch(pd_grid* g, MarchPlan& p, MarchArgs M, int r, bool push) {
    static const int pf = [] {
        const char* e = getenv("PD_M43_PF");
        return e ? atoi(e) : 5;
    }();
    M.pf = pf;
    if (!p.d_ctx) fail(PD_E_INPUT, "march v43 needs the packed chunk records (3-D FP64 plan)");
    M.sched = flagged_schedule(g, p, M.sched, M.n);
    static const cuuint32_t bx[4] = {2, 8, 8, 1};
    const CUtensorMap mux = column_map(M.A.u, g->n_chunks, bx), mdx = column_map(M.deff, g->n_chunks + 1, bx);
    using K43 = void (*)(const MarchArgs, const uint32_t*, const CUtensorMap, const CUtensorMap);
    static const K43 tab[2][2][3] = {
        {{ftcs_march43_kernel<0, false, false>, ftcs_march43_kernel<1, false, false>, ftcs_march43_kernel<2, false, false>},
         {ftcs_march43_kernel<0, true, false>, ftcs_march43_kernel<1, true, false>, ftcs_march43_kernel<2, true, false>}},
        {{ftcs_march43_kernel<0, false, true>, ftcs_march43_kernel<1, false, true>, ftcs_march43_kernel<2, false, true>},
         {ftcs_march43_kernel<0, true, true>, ftcs_march43_kernel<1, true, true>, ftcs_march43_kernel<2, true, true>}}};
    const uint32_t smem = smem43();
    static uint64_t attr_done = 0;
    const int dev = g->device;
    if (dev < 0 || dev >= 64) fail(PD_E_INPUT, "device index out of range");
    if (!((attr_done >> dev) & 1u)) {
        for (int h = 0; h < 2; ++h)
            for (int q = 0; q < 2; ++q)
                for (int rr = 0; rr < 3; ++rr)
                    PD_CUDA(cudaFuncSetAttribute(tab[h][q][rr], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done |= 1ull << dev;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    tab[p.half ? 1 : 0][push ? 1 : 0][r]<<<sms * kCtas43, kThreads43, smem, g->stream>>>(M, p.d_ctx, mux, mdx);
    PD_CUDA(cudaGetLastError());
}

void march_launch_sched(pd_grid* g, MarchPlan& p, const StepArgs<double>& a, int reaction, const int32_t* sched,
                        int64_t n, int* counter, const PeerLaunch* pl) {
    MarchArgs M;
    M.peer_un[0] = pl ? pl->un[0] : nullptr;
    M.peer_un[1] = pl ? pl->un[1] : nullptr;
    M.peer_ord = pl ? pl->ord : nullptr;
    M.A = a;
    M.sched = sched;
    M.n = n;
    M.desc = p.d_desc;
    M.lm = p.d_lm;
    M.deff = static_cast<const double*>(p.d_deff);
    M.dv = static_cast<const double*>(p.d_dv);
    M.counter = counter;
    static const int dbg = [] {
        const char* e = getenv("PD_MARCH_DBG");
        return e ? atoi(e) : 0;
    }();
    M.dbg = dbg;
    M.zero = 0;
    M.n_all = g->n_chunks;
    static const int ver = [] {
        const char* e = getenv("PD_MARCH_V");
        return e ? atoi(e) : 43;
    }();
    using KernT = void (*)(MarchArgs);
    const int r = reaction == PD_REACTION_SURFACE_SINK ? 1 : reaction == PD_REACTION_VOLUMETRIC ? 2 : 0;
#define PD_M_TABLE(K)                                                                            \
    {{{K<0, false, false>, K<1, false, false>, K<2, false, false>},                              \
      {K<0, true, false>, K<1, true, false>, K<2, true, false>}},                                \
     {{K<0, false, true>, K<1, false, true>, K<2, false, true>},                                 \
      {K<0, true, true>, K<1, true, true>, K<2, true, true>}}}
    static const KernT t14[2][2][3] = PD_M_TABLE(ftcs_march14_kernel);  // [half][push][reaction]
    static const KernT t20[2][2][3] = PD_M_TABLE(ftcs_march20_kernel);
#undef PD_M_TABLE
    if (ver == 30) {
        march30_launch(g, p, M, r, pl != nullptr);
        return;
    }
    if (ver == 31) {
        march31_launch(g, p, M, r, pl != nullptr);
        return;
    }
    if (ver == 41) {
        march41_launch(g, p, M, r, pl != nullptr);
        return;
    }
    if (ver == 43) {
        march43_launch(g, p, M, r, pl != nullptr);
        return;
    }
    static const int pf = [] {
        const char* e = getenv("PD_M14_PF");
        return e ? atoi(e) : 1;
    }();
    M.pf = pf;
    if (ver == 14) M.sched = flagged_schedule(g, p, M.sched, M.n);
    const bool v20 = ver != 14;
    const size_t bytes = (size_t)(v20 ? kWarpBytes20 : kWarpBytes14) * kWarps;
    // the dynamic shared-memory opt-in is per device: set it once per device
    static uint64_t attr_done[2] = {0, 0};
    const int dev = g->device;
    if (dev < 0 || dev >= 64) fail(PD_E_INPUT, "device index out of range");
    if (!((attr_done[v20] >> dev) & 1u)) {
        for (auto& half : (v20 ? t20 : t14))
            for (auto& row : half)
                for (auto k : row)
                    PD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        attr_done[v20] |= 1ull << dev;
    }
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    (v20 ? t20 : t14)[p.half ? 1 : 0][pl ? 1 : 0][r]<<<sms * kCtas14, kThreads, bytes, g->stream>>>(M);
    PD_CUDA(cudaGetLastError());
}

}  // namespace pdb
