// Warp-per-chunk, register-marching FTCS step for 3-D FP64 grids — the
// bandwidth path (BASELINE.json configs C1-C5).
//
// Same per-node result, bit for bit, as ftcs_step_kernel (pd_ftcs.cu) and the
// reference (solver.hpp:360-455). Design (measured alternatives — a staged
// 10^3 smem tile with CTA barriers, and a TMA/cp.async producer warp feeding
// mbarrier-synchronised consumer warps — were latency- or producer-bound, see
// DESIGN.md):
//
// * One warp owns one chunk at a time and marches its 8 z-planes; lane
//   (y, xp) holds the x-adjacent node pair (2xp, 2xp+1) of row y in every
//   plane. u and D of the planes z-1, z, z+1 live in registers (the z
//   stencil), x and y neighbours come from warp shuffles, and only the
//   chunk-face lanes read halo values from memory. No shared memory, no
//   barriers; loads for plane z+2 are in flight while plane z is computed, and
//   20 warps per SM keep enough bytes in flight to cover HBM latency.
// * Pairs without an active node are never loaded (predicated 16-B loads), so
//   empty 32-B sectors cost no HBM traffic.
// * Contiguous halos. x faces are 8-B strided in a chunk slab, so every step
//   also writes the x=0 / x=7 planes of u_next into a side array (64 doubles
//   per face, contiguous) and the stepper keeps the same for D_eff; y halos
//   are 64-B rows and z halos 512-B planes of the neighbour chunks.
// * Schedule. Chunks are ordered (z-block of kSeg layers, 4x4 tiles of chunk
//   columns, column, z) and claimed kBatch at a time from one atomic counter,
//   so the chunks in flight always form one short window of that order: the
//   z halos were streamed by the same warp a moment ago and the x/y halos by
//   the warps next to it in the window (L2 hits). (Cutting the order into
//   several independently claimed parts spreads y neighbours hundreds of
//   microseconds apart and was measured to miss L2.)
// * Usability without masks. D_eff = fluid ? D : -inf (static per run); a
//   neighbour is usable iff it is fluid (solver.hpp:374,379-381), i.e. iff the
//   face sum d_a + d_b is not -inf.
// * Face fluxes. F(a|b) = ((d_a+d_b)*0.5)*(u_b-u_a) is exactly the value both
//   endpoints compute in the reference (dh_p*(p.u-u_c) for a, dh_m*(u_c-m.u)
//   for b). For a substituted face the reference computes
//   ((d_c+d_c)*0.5)*(u_c-u_c) = +-0 when u_c, d_c are finite, and a +-0 term
//   leaves lap = 0.0 + ... bitwise unchanged, so the fast path uses 0. Planes
//   whose nodes and neighbours are all fluid skip the selects entirely. Nodes
//   whose fast result is non-finite, and chunks that touch a Dirichlet outer
//   face, take the exact generic path on the same register values.
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kCtasPerSm = 4;  // default occupancy (PD_MARCH_OCC=3 selects 3)
constexpr int kBatch = 1;  // one chunk per claim: neighbours in the schedule run close in time
constexpr int kParts = 1;
constexpr int kSeg = 16;
constexpr unsigned kSentHi = 0xFFF00000u;  // high word of -inf
constexpr int kFlagDirichlet = 2;  // chunk touches a Dirichlet outer face
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
    const double* __restrict__ xfu;  // x-face planes of u       [c][side][64]
    const double* __restrict__ xfd;  // x-face planes of D_eff   [c][side][64]
    double* __restrict__ xfun;       // x-face planes of u_next (written)
    int* counter;                    // kParts counters of this step
    int dbg;                         // measurement-only halo skip mask (PD_MARCH_DBG)
};


struct SlowConsts {
    int64_t size[3];
    double inv_dx2[3];
    double bcv[6];
    double dt, neg_k, src_factor;
    int dirichlet;
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
__device__ __forceinline__ double face(double da, double db, double ua, double ub) {
    const double s = da + db;
    const double f = (s * 0.5) * (ub - ua);
    return ((unsigned)__double2hiint(s) == kSentHi) ? 0.0 : f;
}
__device__ __forceinline__ double fface(double da, double db, double ua, double ub) {
    return ((da + db) * 0.5) * (ub - ua);
}

struct ChunkCtx {  // what the compute side needs of a chunk
    int c, key, flags;
    uint32_t lm;
};

// Per-warp ring of plane tiles in shared memory. A tile holds u and D_eff of
// one z-plane of a chunk: rows y = -1..8 of the 8 body columns (pitch 8, so
// the lanes' 16-B pair accesses are bank-conflict free) and the x- / x+ halo
// cells of rows 0..7 in two side columns.
constexpr int kRing = 8;   // power of two: slot = load index & 7
constexpr int kAhead = 5;  // kRing - 3 (planes z-1, z, z+1 resident)
struct Tile {
    double u[80], hxu[2][8];
    double d[80], hxd[2][8];
};
__device__ __forceinline__ int tix(int x, int y) { return x + 8 * (y + 1); }

__device__ __forceinline__ void cp16_if(void* smem, const void* gmem, bool pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
        " @p cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(smem)),
        "l"(gmem), "r"((int)pred));
}
__device__ __forceinline__ void cp8_if(void* smem, const void* gmem, bool pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
        " @p cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(smem)),
        "l"(gmem), "r"((int)pred));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Lane-specific source offsets (elements, 32-bit: u holds < 2^32 slots, see
// march_build) of one chunk, computed once per chunk on the load side.
constexpr uint32_t kNone = 0xFFFFFFFFu;
struct LoadCtx {
    int c;
    uint32_t lm;
    uint32_t own;   // the lane's pair in plane 0
    uint32_t zlo;   // pair in the z- neighbour's plane 7
    uint32_t zhi;   // pair in the z+ neighbour's plane 0
    uint32_t xoff;  // x-halo cell of plane 0 in the side planes (face lanes)
    uint32_t yoff;  // y-halo pair of plane 0 (face lanes)
};

template <int XD>
__device__ __forceinline__ LoadCtx make_load_ctx(int c, uint32_t lm, int dv, const MarchArgs& M, int y,
                                                 int xp, int x0) {
    int nb[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) nb[f] = __shfl_sync(0xffffffffu, dv, 24 + f);
    LoadCtx L;
    L.c = c;
    L.lm = lm;
    const uint32_t bp = (uint32_t)(y * 8 + x0);
    L.own = (uint32_t)(c < 0 ? 0 : c) * 512u + bp;
    const bool zk = !(M.dbg & 4);
    L.zlo = (zk && nb[4] >= 0) ? (uint32_t)nb[4] * 512u + 448u + bp : kNone;
    L.zhi = (zk && nb[5] >= 0) ? (uint32_t)nb[5] * 512u + bp : kNone;
    const int jx = (M.dbg & 1) ? -1 : (xp == 0 ? nb[0] : nb[1]);
    if (XD)  // x halo straight from the neighbour's slab (x = 7 / x = 0 column)
        L.xoff = ((xp == 0 || xp == 3) && jx >= 0) ? (uint32_t)jx * 512u + (uint32_t)y * 8u + (xp == 0 ? 7u : 0u)
                                                   : kNone;
    else
        L.xoff = ((xp == 0 || xp == 3) && jx >= 0) ? ((uint32_t)jx * 2u + (xp == 0 ? 1u : 0u)) * 64u + (uint32_t)y
                                                   : kNone;
    const int jy = (M.dbg & 2) ? -1 : (y == 0 ? nb[2] : nb[3]);
    L.yoff = ((y == 0 || y == 7) && jy >= 0) ? (uint32_t)jy * 512u + (y == 0 ? 56u : 0u) + (uint32_t)x0 : kNone;
    return L;
}

// Issues the lane's share of plane p (-1..8) into tile T: predicated 16-B
// copies of its node pair (pairs with no active node are never read; their
// D_eff cells get the sentinel) and, for chunk-face lanes, the x / y halo
// cells. p = -1 / 8 are the z halo planes of the z neighbours.
template <int XD>
__device__ __forceinline__ void issue_plane(Tile& T, const MarchArgs& M, const LoadCtx& L, int p,
                                            int y, int xp, int t0) {
    const double sv = sent();
    const bool body = (unsigned)p <= 7u;
    const uint32_t o = body ? L.own + (uint32_t)p * 64u : (p < 0 ? L.zlo : L.zhi);
    const bool ok = L.c >= 0 && (body ? ((L.lm >> (2 * p)) & 3u) != 0 : o != kNone);
    const uint32_t oo = ok ? o : 0u;
    cp16_if(&T.u[t0], M.A.u + oo, ok);
    cp16_if(&T.d[t0], M.deff + oo, ok);
    if (!ok) *reinterpret_cast<double2*>(&T.d[t0]) = make_double2(sv, sv);
    if (!body) return;  // warp-uniform
    const bool xl = xp == 0 || xp == 3, yl = y == 0 || y == 7;
    const int side = xp == 0 ? 0 : 1;
    const bool xok = L.c >= 0 && L.xoff != kNone;
    const uint32_t ox = xok ? L.xoff + (uint32_t)p * (XD ? 64u : 8u) : 0u;
    cp8_if(&T.hxu[side][y], (XD ? M.A.u : M.xfu) + ox, xok);
    cp8_if(&T.hxd[side][y], (XD ? M.deff : M.xfd) + ox, xok);
    if (xl && !xok) T.hxd[side][y] = sv;
    const bool yok = L.c >= 0 && L.yoff != kNone;
    const int ty = y == 0 ? t0 - 8 : t0 + 8;
    const uint32_t oy = yok ? L.yoff + (uint32_t)p * 64u : 0u;
    cp16_if(&T.u[ty], M.A.u + oy, yok);
    cp16_if(&T.d[ty], M.deff + oy, yok);
    if (yl && !yok) *reinterpret_cast<double2*>(&T.d[ty]) = make_double2(sv, sv);
}

// |x| >= 2^990 or non-finite, from the high word (integer pipe)
__device__ __forceinline__ bool huge(double x) {
    return ((unsigned)__double2hiint(x) & 0x7fffffffu) >= 0x7DD00000u;
}

template <int REACTION, int XD>
__device__ __forceinline__ void compute_plane(const MarchArgs& M, const SlowConsts& K,
                                              const ChunkCtx& C, int z, const Tile& Tm,
                                              const Tile& T0, const Tile& Tp, int y, int xp, int x0,
                                              int t0, int lofs, int rofs) {
    const bool a0 = (C.lm >> (2 * z)) & 1u, a1 = (C.lm >> (2 * z + 1)) & 1u;
    if (!(a0 | a1)) return;
    const double2 uc = *reinterpret_cast<const double2*>(&T0.u[t0]);
    const double2 dc = *reinterpret_cast<const double2*>(&T0.d[t0]);
    constexpr int kD = (int)(offsetof(Tile, d) / sizeof(double));  // u -> d distance
    const double uL = T0.u[lofs], dL = T0.u[lofs + kD];
    const double uR = T0.u[rofs], dR = T0.u[rofs + kD];
    const double2 uym = *reinterpret_cast<const double2*>(&T0.u[t0 - 8]);
    const double2 dym = *reinterpret_cast<const double2*>(&T0.d[t0 - 8]);
    const double2 uyp = *reinterpret_cast<const double2*>(&T0.u[t0 + 8]);
    const double2 dyp = *reinterpret_cast<const double2*>(&T0.d[t0 + 8]);
    const double2 uzm = *reinterpret_cast<const double2*>(&Tm.u[t0]);
    const double2 dzm = *reinterpret_cast<const double2*>(&Tm.d[t0]);
    const double2 uzp = *reinterpret_cast<const double2*>(&Tp.u[t0]);
    const double2 dzp = *reinterpret_cast<const double2*>(&Tp.d[t0]);
    const StepArgs<double>& A = M.A;
    const int o = z * 64 + y * 8 + x0;
    const int c = C.c;
    const bool s0 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (16 + 2 * z)) & 1u);
    const bool s1 = REACTION == PD_REACTION_SURFACE_SINK && ((C.lm >> (17 + 2 * z)) & 1u);
    double src0 = 0.0, src1 = 0.0;
    if (REACTION == PD_REACTION_VOLUMETRIC) {
        src0 = A.src[(int64_t)c * 512 + o];
        src1 = A.src[(int64_t)c * 512 + o + 1];
    }
    const double ix = K.inv_dx2[0], iy = K.inv_dx2[1], iz = K.inv_dx2[2];
    const bool dirichlet = (C.flags & kFlagDirichlet) != 0;  // warp-uniform
    double out0, out1;
    if (!dirichlet) {
        double fxl, fxi, fxr, fy0m, fy0p, fz0m, fz0p, fy1m, fy1p, fz1m, fz1p;
        if ((C.flags >> (8 + z)) & 1) {
            // interior-fluid plane (warp-uniform): no substitution anywhere
            fxl = fface(dL, dc.x, uL, uc.x);
            fxi = fface(dc.x, dc.y, uc.x, uc.y);
            fxr = fface(dc.y, dR, uc.y, uR);
            fy0m = fface(dym.x, dc.x, uym.x, uc.x);
            fy0p = fface(dc.x, dyp.x, uc.x, uyp.x);
            fz0m = fface(dzm.x, dc.x, uzm.x, uc.x);
            fz0p = fface(dc.x, dzp.x, uc.x, uzp.x);
            fy1m = fface(dym.y, dc.y, uym.y, uc.y);
            fy1p = fface(dc.y, dyp.y, uc.y, uyp.y);
            fz1m = fface(dzm.y, dc.y, uzm.y, uc.y);
            fz1p = fface(dc.y, dzp.y, uc.y, uzp.y);
        } else {
            fxl = face(dL, dc.x, uL, uc.x);
            fxi = face(dc.x, dc.y, uc.x, uc.y);
            fxr = face(dc.y, dR, uc.y, uR);
            fy0m = face(dym.x, dc.x, uym.x, uc.x);
            fy0p = face(dc.x, dyp.x, uc.x, uyp.x);
            fz0m = face(dzm.x, dc.x, uzm.x, uc.x);
            fz0p = face(dc.x, dzp.x, uc.x, uzp.x);
            fy1m = face(dym.y, dc.y, uym.y, uc.y);
            fy1p = face(dc.y, dyp.y, uc.y, uyp.y);
            fz1m = face(dzm.y, dc.y, uzm.y, uc.y);
            fz1p = face(dc.y, dzp.y, uc.y, uzp.y);
        }
        double lap0 = 0.0;  // lap starts at T{0} (solver.hpp:420)
        lap0 += (fxi - fxl) * ix;
        lap0 += (fy0p - fy0m) * iy;
        lap0 += (fz0p - fz0m) * iz;
        double lap1 = 0.0;
        lap1 += (fxr - fxi) * ix;
        lap1 += (fy1p - fy1m) * iy;
        lap1 += (fz1p - fz1m) * iz;
        double r0 = 0.0, r1 = 0.0;
        if (REACTION == PD_REACTION_SURFACE_SINK) {
            if (s0) r0 = K.neg_k * uc.x;
            if (s1) r1 = K.neg_k * uc.y;
        } else if (REACTION == PD_REACTION_VOLUMETRIC) {
            r0 = src0 * K.src_factor;
            r1 = src1 * K.src_factor;
        }
        out0 = uc.x + K.dt * lap0 + K.dt * r0;
        out1 = uc.y + K.dt * lap1 + K.dt * r1;
    } else {
        const int kx = C.key & 1023, ky = (C.key >> 10) & 1023, kz = (C.key >> 20) & 1023;
        const int64_t gx = (int64_t)kx * 8 + x0, gy = (int64_t)ky * 8 + y, gz = (int64_t)kz * 8 + z;
        const double nu0[6] = {uL, uc.y, uym.x, uyp.x, uzm.x, uzp.x};
        const double nd0[6] = {dL, dc.y, dym.x, dyp.x, dzm.x, dzp.x};
        out0 = slow_node<REACTION>(K, uc.x, dc.x, nu0, nd0, gx, gy, gz, s0, src0);
        const double nu1[6] = {uc.x, uR, uym.y, uyp.y, uzm.y, uzp.y};
        const double nd1[6] = {dc.x, dR, dym.y, dyp.y, dzm.y, dzp.y};
        out1 = slow_node<REACTION>(K, uc.y, dc.y, nu1, nd1, gx + 1, gy, gz, s1, src1);
    }
    // walls (active, not fluid) stay frozen (solver.hpp:413-417)
    if (sentinel(dc.x)) out0 = uc.x;
    if (sentinel(dc.y)) out1 = uc.y;
    const bool h0 = a0 && huge(out0), h1 = a1 && huge(out1);
    if (h0 | h1) {
        // rare: a non-finite fast-path result is re-derived exactly (the
        // +-0 substitution shortcut needs finite operands), then the
        // reference's non-finite / total-mass checks are flagged
        // (solver.hpp:444, 250-260, 514-515)
        const int kx = C.key & 1023, ky = (C.key >> 10) & 1023, kz = (C.key >> 20) & 1023;
        const int64_t gx = (int64_t)kx * 8 + x0, gy = (int64_t)ky * 8 + y, gz = (int64_t)kz * 8 + z;
        if (h0 && !isfinite(out0) && !sentinel(dc.x) && !dirichlet) {
            const double nu[6] = {uL, uc.y, uym.x, uyp.x, uzm.x, uzp.x};
            const double nd[6] = {dL, dc.y, dym.x, dyp.x, dzm.x, dzp.x};
            out0 = slow_node<REACTION>(K, uc.x, dc.x, nu, nd, gx, gy, gz, s0, src0);
        }
        if (h1 && !isfinite(out1) && !sentinel(dc.y) && !dirichlet) {
            const double nu[6] = {uc.x, uR, uym.y, uyp.y, uzm.y, uzp.y};
            const double nd[6] = {dc.x, dR, dym.y, dyp.y, dzm.y, dzp.y};
            out1 = slow_node<REACTION>(K, uc.y, dc.y, nu, nd, gx + 1, gy, gz, s1, src1);
        }
        const bool bad0 = a0 && !isfinite(out0), bad1 = a1 && !isfinite(out1);
        if (bad0 | bad1) {
            atomicMin(A.bad_key, ((unsigned long long)c << 10) | (unsigned long long)(o + (bad0 ? 0 : 1)));
            atomicOr(&A.flags[A.k], 1);
        } else {
            atomicOr(&A.flags[A.k], 2);
        }
    }
    double* dst = A.un + (int64_t)c * 512 + o;
    if (a0 && a1) {
        *reinterpret_cast<double2*>(dst) = make_double2(out0, out1);
    } else {
        if (a0) dst[0] = out0;
        if (a1) dst[1] = out1;
    }
    // x-face side planes of u_next for the next step's x halos
    if (XD) return;
    if (xp == 0 && a0) M.xfun[((int64_t)c * 2 + 0) * 64 + z * 8 + y] = out0;
    if (xp == 3 && a1) M.xfun[((int64_t)c * 2 + 1) * 64 + z * 8 + y] = out1;
}

__device__ __forceinline__ void load_ctx(const MarchArgs& M, int c, int lane, uint32_t& lm, int& dv) {
    lm = 0u;
    dv = -1;
    if (c < 0) return;
    lm = __ldg(&M.lm[(int64_t)c * 32 + lane]);
    if (lane >= 24) dv = __ldg(&M.desc[(int64_t)c * 8 + lane - 24]);
}

__device__ __forceinline__ ChunkCtx make_ctx(int c, uint32_t lm, int dv) {
    ChunkCtx C;
    C.c = c;
    C.lm = lm;
    C.key = __shfl_sync(0xffffffffu, dv, 30);
    C.flags = __shfl_sync(0xffffffffu, dv, 31);
    return C;
}

// One warp streams a sequence of chunks. Its plane loads (10 per chunk:
// z-halo below, the 8 body planes, z-halo above) form one continuous
// sequence through a kRing-slot tile ring, kAhead loads ahead of the plane
// being computed, across chunk boundaries.
template <int REACTION, int OCC, int XD>
__global__ void __launch_bounds__(kThreads, OCC) ftcs_march_kernel(MarchArgs M) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int y = lane >> 2, xp = lane & 3, x0 = 2 * xp;
    Tile* ring = reinterpret_cast<Tile*>(smem_raw) + warp * kRing;
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
    }
    __syncthreads();
    const int lofs = xp == 0 ? (int)(offsetof(Tile, hxu) / sizeof(double)) + y : tix(x0, y) - 1;
    const int rofs = xp == 3 ? (int)(offsetof(Tile, hxu) / sizeof(double)) + 8 + y : tix(x0, y) + 2;

    // ---- chunk stream: kBatch-chunk claims from one counter ----
    int* ctr = M.counter;
    auto claim = [&]() -> int {
        int v = 0;
        if (lane == 0) v = atomicAdd(ctr, kBatch);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    int b_cur = claim(), b_nxt = claim();
    int bi = 0;  // position of the next chunk to fetch inside b_cur
    const int n = (int)M.n;
    auto next_id = [&]() -> int {
        if (bi == kBatch) {
            b_cur = b_nxt;
            b_nxt = claim();
            bi = 0;
        }
        const int p = b_cur + bi++;
        return p < n ? __ldg(&M.sched[p]) : -1;
    };

    // loading side: chunk whose planes are being issued, and the next one
    int c_ld = next_id();
    if (c_ld < 0) return;
    uint32_t lm0, lm1;
    int dv0, dv1;
    load_ctx(M, c_ld, lane, lm0, dv0);
    ChunkCtx Cld = make_ctx(c_ld, lm0, dv0);
    const int t0 = tix(x0, y);
    LoadCtx Lld = make_load_ctx<XD>(c_ld, lm0, dv0, M, y, xp, x0);
    int c_nx = next_id();
    load_ctx(M, c_nx, lane, lm1, dv1);
    int p_ld = -1;  // next plane of Cld to issue (-1..8)
    int L = 0;      // loads issued
    auto issue_next = [&]() {
        if (Lld.c >= 0) issue_plane<XD>(ring[L & (kRing - 1)], M, Lld, p_ld, y, xp, t0);
        cp_commit();
        ++L;
        if (++p_ld == 9) {  // advance the load side to the next chunk
            p_ld = -1;
            Cld = make_ctx(c_nx, lm1, dv1);
            Lld = make_load_ctx<XD>(c_nx, lm1, dv1, M, y, xp, x0);
            c_nx = Cld.c >= 0 ? next_id() : -1;
            load_ctx(M, c_nx, lane, lm1, dv1);
        }
    };
    // compute side: follows the load side, which is never more than one
    // chunk ahead (kAhead + 3 < 10 loads)
    ChunkCtx Cc = Cld;
    int base = 0;  // load index of plane -1 of Cc
    // prologue: planes -1, 0, 1 needed for z = 0, plus kAhead more
    for (int k = 0; k < 3 + kAhead; ++k) issue_next();
    while (Cc.c >= 0) {
#pragma unroll 1
        for (int z = 0; z < 8; ++z) {
            // loads up to index base+z+2 complete; exactly kAhead newer groups
            // are in flight at this point of every iteration
            cp_wait<kAhead>();
            __syncwarp();
            compute_plane<REACTION, XD>(M, K, Cc, z, ring[(base + z) & (kRing - 1)],
                                    ring[(base + z + 1) & (kRing - 1)],
                                    ring[(base + z + 2) & (kRing - 1)], y, xp, x0, t0, lofs, rofs);
            __syncwarp();
            issue_next();
            if (z == 7) {  // planes 8 of this chunk and -1 of the next
                issue_next();
                issue_next();
            }
        }
        base += 10;
        Cc = Cld;
    }
    cp_wait<0>();
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
__global__ void deff_kernel(const double* __restrict__ dcol, const uint64_t* __restrict__ fluid,
                            int64_t n_slots, double* __restrict__ deff, unsigned long long* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_slots) return;
    const bool fl = (fluid[i >> 6] >> (i & 63)) & 1ull;
    const double v = dcol[i];
    deff[i] = fl ? v : sent();
    if (fl && !isfinite(v)) atomicAdd(bad, 1ull);
}

// x=0 / x=7 planes of a column into the side array [c][side][z*8+y].
__global__ void xface_kernel(const double* __restrict__ col, int64_t n, double* __restrict__ xf) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * 128) return;
    const int64_t c = t >> 7;
    const int side = (int)((t >> 6) & 1), p = (int)(t & 63);
    const int z = p >> 3, y = p & 7;
    xf[t] = col[c * 512 + z * 64 + y * 8 + (side ? 7 : 0)];
}

void march_free(MarchPlan* p) {
    cudaFree(p->d_stream);
    cudaFree(p->d_desc);
    cudaFree(p->d_deff);
    cudaFree(p->d_xfd);
    cudaFree(p->d_xf[0]);
    cudaFree(p->d_xf[1]);
    cudaFree(p->d_counter);
    cudaFree(p->d_lm);
    *p = MarchPlan{};
}

void march_extract_xfaces(pd_grid* g, MarchPlan& p, const void* col) {
    const int64_t n = g->n_chunks;
    if (n == 0 || !p.ready) return;
    xface_kernel<<<(unsigned)((n * 128 + 255) / 256), 256, 0, g->stream>>>((const double*)col, n,
                                                                          p.d_xf[p.cur]);
    PD_CUDA(cudaGetLastError());
}

void march_build(pd_grid* g, const int32_t* d_nbr, const uint64_t* d_fluid, const uint64_t* d_sink,
                 const void* d_dcol, int dirichlet, int64_t begin, int64_t end, MarchPlan* plan) {
    march_free(plan);
    if (g->dims != 3 || g->tbytes != 8) return;
    if (g->cc[0] > 1024 || g->cc[1] > 1024 || g->cc[2] > 1024) return;  // key packing limit
    const int64_t n_all = g->n_chunks;
    if (n_all == 0 || end <= begin) return;
    if (n_all * 512 >= (int64_t)0xFFFFFFFF) return;  // 32-bit slot offsets (>16 GB per column)
    PD_CUDA(cudaMalloc(&plan->d_desc, sizeof(int32_t) * 8 * (size_t)n_all));
    desc_kernel<<<(unsigned)((n_all + 255) / 256), 256, 0, g->stream>>>(
        d_nbr, g->d_keys, d_fluid, n_all, g->size[0], g->size[1], g->size[2], dirichlet, plan->d_desc);
    PD_CUDA(cudaGetLastError());
    PD_CUDA(cudaMalloc(&plan->d_lm, sizeof(uint32_t) * 32 * (size_t)n_all));
    lanemask_kernel<<<(unsigned)((n_all * 32 + 255) / 256), 256, 0, g->stream>>>(g->d_masks, d_sink,
                                                                                n_all, plan->d_lm);
    PD_CUDA(cudaGetLastError());
    const int64_t slots = n_all * 512;
    PD_CUDA(cudaMalloc(&plan->d_deff, sizeof(double) * (size_t)slots));
    PD_CUDA(cudaMalloc(&plan->d_xfd, sizeof(double) * 128 * (size_t)n_all));
    PD_CUDA(cudaMalloc(&plan->d_xf[0], sizeof(double) * 128 * (size_t)n_all));
    PD_CUDA(cudaMalloc(&plan->d_xf[1], sizeof(double) * 128 * (size_t)n_all));
    PD_CUDA(cudaMalloc(&plan->d_counter, sizeof(int) * 1024 * kParts));
    unsigned long long* d_bad = nullptr;
    PD_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
    PD_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), g->stream));
    deff_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, g->stream>>>(
        (const double*)d_dcol, d_fluid, slots, plan->d_deff, d_bad);
    PD_CUDA(cudaGetLastError());
    xface_kernel<<<(unsigned)((n_all * 128 + 255) / 256), 256, 0, g->stream>>>(plan->d_deff, n_all,
                                                                              plan->d_xfd);
    PD_CUDA(cudaGetLastError());
    unsigned long long bad = 0;
    PD_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, g->stream));
    // schedule of the owned range: (zblock, y, x, z)
    const int64_t n = end - begin;
    std::vector<int32_t> keys((size_t)n * 3);
    PD_CUDA(cudaMemcpyAsync(keys.data(), g->d_keys + begin * 3, sizeof(int32_t) * 3 * (size_t)n,
                            cudaMemcpyDeviceToHost, g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    cudaFree(d_bad);
    if (bad) {  // non-finite D on a fluid node: keep the exact tile kernel
        march_free(plan);
        return;
    }
    std::vector<int32_t> order((size_t)n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        const int32_t* ka = &keys[(size_t)a * 3];
        const int32_t* kb = &keys[(size_t)b * 3];
        // z-block, then 4x4 column tiles, then columns inside the tile, then z
        const int za = ka[2] / kSeg, zb = kb[2] / kSeg;
        if (za != zb) return za < zb;
        if (ka[1] / 4 != kb[1] / 4) return ka[1] / 4 < kb[1] / 4;
        if (ka[0] / 4 != kb[0] / 4) return ka[0] / 4 < kb[0] / 4;
        if (ka[1] != kb[1]) return ka[1] < kb[1];
        if (ka[0] != kb[0]) return ka[0] < kb[0];
        return ka[2] < kb[2];
    });
    for (auto& o : order) o = (int32_t)(o + begin);
    PD_CUDA(cudaMalloc(&plan->d_stream, sizeof(int32_t) * order.size()));
    PD_CUDA(cudaMemcpyAsync(plan->d_stream, order.data(), sizeof(int32_t) * order.size(),
                            cudaMemcpyHostToDevice, g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    int sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    static const int occ = [] {
        const char* e = getenv("PD_MARCH_OCC");
        return (e && atoi(e) == 3) ? 3 : kCtasPerSm;
    }();
    plan->grid = sms * occ;
    plan->n = n;
    plan->ready = true;
    plan->cur = 0;
}

int march_counters_per_step() { return kParts; }

void march_launch(pd_grid* g, MarchPlan& p, const StepArgs<double>& a, int reaction) {
    MarchArgs M;
    M.A = a;
    M.sched = p.d_stream;
    M.n = p.n;
    M.desc = p.d_desc;
    M.lm = p.d_lm;
    M.deff = p.d_deff;
    M.xfu = p.d_xf[p.cur];
    M.xfd = p.d_xfd;
    M.xfun = p.d_xf[1 - p.cur];
    M.counter = p.d_counter + (int64_t)(a.k & 1023) * kParts;
    static const int dbg = [] {
        const char* e = getenv("PD_MARCH_DBG");
        return e ? atoi(e) : 0;
    }();
    M.dbg = dbg;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const bool occ3 = p.grid == sms * 3;
    const size_t bytes = sizeof(Tile) * kRing * kWarps;
    static const int xd = [] {
        const char* e = getenv("PD_MARCH_XSIDE");
        return (e && atoi(e) == 1) ? 0 : 1;
    }();
    using KernT = void (*)(MarchArgs);
    static const KernT table[2][2][3] = {
        {{ftcs_march_kernel<0, kCtasPerSm, 0>, ftcs_march_kernel<1, kCtasPerSm, 0>, ftcs_march_kernel<2, kCtasPerSm, 0>},
         {ftcs_march_kernel<0, 3, 0>, ftcs_march_kernel<1, 3, 0>, ftcs_march_kernel<2, 3, 0>}},
        {{ftcs_march_kernel<0, kCtasPerSm, 1>, ftcs_march_kernel<1, kCtasPerSm, 1>, ftcs_march_kernel<2, kCtasPerSm, 1>},
         {ftcs_march_kernel<0, 3, 1>, ftcs_march_kernel<1, 3, 1>, ftcs_march_kernel<2, 3, 1>}}};
    static bool attr_set = false;
    if (!attr_set) {
        for (auto& a : table)
            for (auto& b : a)
                for (auto k : b) PD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        attr_set = true;
    }
    const int r = reaction == PD_REACTION_SURFACE_SINK ? 1 : reaction == PD_REACTION_VOLUMETRIC ? 2 : 0;
    table[xd][occ3 ? 1 : 0][r]<<<p.grid, kThreads, bytes, g->stream>>>(M);
    PD_CUDA(cudaGetLastError());
    p.cur = 1 - p.cur;
}

}  // namespace pdb
