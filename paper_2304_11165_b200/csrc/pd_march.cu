// Warp-specialized, mbarrier-pipelined FTCS step for 3-D FP64 grids — the
// bandwidth path (BASELINE.json configs C1-C5).
//
// Same per-node result, bit for bit, as ftcs_step_kernel (pd_ftcs.cu) and the
// reference (solver.hpp:360-455); what changes is how bytes and instructions
// are spent.
//
// * Schedule. Chunks are ordered (z-block of kSeg layers, y, x, z): runs of a
//   chunk column inside a z-block are contiguous and neighbouring columns
//   follow each other. Persistent CTAs (2 per SM) grab kBatch consecutive
//   chunks of that order with an atomic counter, so the chunks in flight are
//   always a contiguous window of the schedule and the face halos a CTA reads
//   were just streamed by its neighbours (L2 hits).
// * Producer warp. One warp per CTA streams chunk after chunk into a
//   kStages-deep shared-memory ring with cp.async (16-B copies; body pairs
//   with no active / fluid node are never read from HBM) and signals each
//   stage through an mbarrier (cp.async.mbarrier.arrive). Descriptors and
//   masks are prefetched one chunk ahead, chunk ids one batch ahead, so the
//   producer never waits on its own loads.
// * Contiguous halos. x faces are 8-B strided in a chunk slab, so every step
//   also writes the x=0 / x=7 planes of u_next into a side array (64 doubles
//   per face, contiguous) and the stepper keeps the same for D_eff; y and z
//   face layers are read directly (64-B rows / 512-B planes).
// * Consumer warps (8). Warp w computes z-plane w, two x-adjacent nodes per
//   thread, from shared memory only.
// * Usability without masks. D_eff = fluid ? D : -inf (static per run). A
//   neighbour is usable iff it is fluid (solver.hpp:374,379-381), i.e. iff the
//   face sum d_a + d_b is not -inf.
// * Face fluxes. F(a|b) = ((d_a+d_b)*0.5)*(u_b-u_a) is exactly the value both
//   endpoints compute in the reference (dh_p*(p.u-u_c) for a, dh_m*(u_c-m.u)
//   for b). For a substituted face the reference computes
//   ((d_c+d_c)*0.5)*(u_c-u_c) = +-0 when u_c, d_c are finite, and a +-0 term
//   leaves lap = 0.0 + ... bitwise unchanged, so the fast path uses 0. Nodes
//   whose fast result is non-finite, and chunks that touch a Dirichlet outer
//   face, take the exact generic path on the same loaded values.
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {

constexpr int kConsumerWarps = 8;
constexpr int kMarchThreads = 32 * (kConsumerWarps + 1);
constexpr int kStages = 6;
constexpr int kSeg = 16;
constexpr int kBatch = 32;
constexpr int kCtasPerSm = 2;
constexpr unsigned kSentHi = 0xFFF00000u;  // high word of -inf
constexpr int kFlagDirichlet = 2;  // chunk touches a Dirichlet outer face
constexpr int kFlagBulk = 4;       // dense chunk: stream body slabs with TMA bulk copies
// bits 8..15: plane z is interior-fluid (all nodes and all their face
// neighbours fluid) -> select-free consumer path

// One pipeline stage. The u region and the D_eff region have identical
// layouts, kDOff doubles apart, so every D load is the matching u address plus
// an immediate.
constexpr int kRegion = 896;  // body 512 + x faces 128 + y faces 128 + z faces 128
constexpr int kHX = 512, kHY = 640, kHZ = 768;
constexpr int kDOff = kRegion;
struct __align__(16) MarchStage {
    double v[2 * kRegion];  // [0, 896): u, [896, 1792): D_eff
    uint64_t act[8], snk[8];
    int4 meta;  // chunk ordinal (-1 = end), packed key, flags
    int4 pad;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
// TMA bulk copy global -> shared, completion reported to an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ bool sentinel(double d) {
    return (unsigned)__double2hiint(d) == kSentHi;
}
__device__ __forceinline__ double sent() { return __hiloint2double((int)kSentHi, 0); }

struct MarchArgs {
    StepArgs<double> A;
    const int32_t* __restrict__ sched;
    int64_t n;
    const int32_t* __restrict__ desc;  // 8 ints per chunk
    const uint16_t* __restrict__ pm;   // per chunk, per lane: pair has active / fluid node
    const double* __restrict__ deff;
    const double* __restrict__ xfu;  // x-face planes of u       [c][side][64]
    const double* __restrict__ xfd;  // x-face planes of D_eff   [c][side][64]
    double* __restrict__ xfun;       // x-face planes of u_next (written)
    int* counter;                    // per-step batch counter
};

// Per-lane prefetch of one chunk's descriptor: lanes 0-7 active words,
// 16-23 sink words, 24-31 the 8 descriptor ints; plus the lane's pair mask.
struct LaneDesc {
    uint64_t v;
    unsigned pm;
};
__device__ __forceinline__ LaneDesc load_lane_desc(const MarchArgs& M, int c, int lane) {
    LaneDesc d{0ull, 0u};
    if (c < 0) return d;
    d.pm = __ldg(&M.pm[(int64_t)c * 32 + lane]);
    if (lane < 8)
        d.v = __ldg(&M.A.active[(int64_t)c * 8 + lane]);
    else if (lane >= 16 && lane < 24)
        d.v = M.A.reaction == PD_REACTION_SURFACE_SINK ? __ldg(&M.A.sink[(int64_t)c * 8 + lane - 16])
                                                        : 0ull;
    else if (lane >= 24)
        d.v = (uint64_t)(uint32_t)__ldg(&M.desc[(int64_t)c * 8 + lane - 24]);
    return d;
}

__device__ __forceinline__ void produce(MarchStage& S, uint64_t* full, const MarchArgs& M, int c,
                                        const LaneDesc& L, int lane) {
    const double* U = M.A.u;
    const double* Dd = M.deff;
    const double sv = sent();
    double* V = S.v;
    if (c >= 0) {
        const int64_t cb = (int64_t)c * 512;
        int nb[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) nb[f] = (int)__shfl_sync(0xffffffffu, (unsigned)L.v, 24 + f);
        const int key = (int)__shfl_sync(0xffffffffu, (unsigned)L.v, 30);
        const int flg = (int)__shfl_sync(0xffffffffu, (unsigned)L.v, 31);
        const bool bulk = flg & kFlagBulk;
        if (lane == 0) {
            // stage memory was last touched through the generic proxy
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            // bytes of every bulk copy of this stage, registered before issue
            unsigned bytes = bulk ? 8192u : 0u;
#pragma unroll
            for (int f = 0; f < 6; ++f)
                if ((f < 2 || f >= 4) && nb[f] >= 0) bytes += 1024u;
            if (bytes) mbar_expect_tx(full, bytes);
            if (bulk) {
                bulk_g2s(&V[0], U + cb, 4096u, full);
                bulk_g2s(&V[kDOff], Dd + cb, 4096u, full);
            }
            // x faces from the contiguous side arrays: x- halo = neighbour's
            // x=7 plane (side 1), x+ halo = neighbour's x=0 plane (side 0)
#pragma unroll
            for (int f = 0; f < 2; ++f)
                if (nb[f] >= 0) {
                    const int64_t src = ((int64_t)nb[f] * 2 + (1 - f)) * 64;
                    bulk_g2s(&V[kHX + f * 64], M.xfu + src, 512u, full);
                    bulk_g2s(&V[kDOff + kHX + f * 64], M.xfd + src, 512u, full);
                }
            // z faces: plane z=7 (z- halo) / z=0 (z+ halo)
#pragma unroll
            for (int f = 0; f < 2; ++f)
                if (nb[4 + f] >= 0) {
                    const int64_t src = (int64_t)nb[4 + f] * 512 + (f == 0 ? 448 : 0);
                    bulk_g2s(&V[kHZ + f * 64], U + src, 512u, full);
                    bulk_g2s(&V[kDOff + kHZ + f * 64], Dd + src, 512u, full);
                }
        }
        if (!bulk) {
            // sparse chunk: 16-B copies of pairs holding an active (u) /
            // fluid (D) node only, so empty sectors are never read
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int off = r * 64 + 2 * lane;
                if ((L.pm >> (2 * r)) & 1u) cp16(&V[off], U + cb + off);
                if ((L.pm >> (2 * r + 1)) & 1u)
                    cp16(&V[kDOff + off], Dd + cb + off);
                else
                    *reinterpret_cast<double2*>(&V[kDOff + off]) = make_double2(sv, sv);
            }
        }
#pragma unroll
        for (int f = 0; f < 6; ++f)
            if ((f < 2 || f >= 4) && nb[f] < 0) {
                const int base = f < 2 ? kHX + f * 64 : kHZ + (f - 4) * 64;
                *reinterpret_cast<double2*>(&V[kDOff + base + 2 * lane]) = make_double2(sv, sv);
            }
        // y faces: row y=7 (y- halo) / y=0 (y+ halo) of every plane, index z*8+x
        {
            const int z = lane >> 2, k = 2 * (lane & 3);
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const int j = nb[2 + f];
                const int dst = kHY + f * 64 + z * 8 + k;
                if (j >= 0) {
                    const int64_t src = (int64_t)j * 512 + z * 64 + (f == 0 ? 56 : 0) + k;
                    cp16(&V[dst], U + src);
                    cp16(&V[kDOff + dst], Dd + src);
                } else {
                    *reinterpret_cast<double2*>(&V[kDOff + dst]) = make_double2(sv, sv);
                }
            }
        }
        if (lane < 8) S.act[lane] = L.v;
        if (lane >= 16 && lane < 24) S.snk[lane - 16] = L.v;
        if (lane == 0) S.meta = make_int4(c, key, flg, 0);
    } else if (lane == 0) {
        S.meta = make_int4(-1, 0, 0, 0);
    }
    cp_async_arrive_noinc(full);  // completes when this lane's copies land
    mbar_arrive(full);            // orders this lane's plain smem stores
}

// Face flux F(a|b) shared by both endpoints; 0 when either side is not fluid.
__device__ __forceinline__ double face(double da, double db, double ua, double ub) {
    const double s = da + db;
    const double f = (s * 0.5) * (ub - ua);
    return ((unsigned)__double2hiint(s) == kSentHi) ? 0.0 : f;
}

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

// Loop-invariant per-thread element offsets inside a stage region.
struct Offs {
    int c, l, r, ym, yp, zm, zp;
};

template <int REACTION>
__device__ __forceinline__ void consume(const MarchStage& S, const MarchArgs& M,
                                        const SlowConsts& K, const Offs& O, int z, int lane) {
    const StepArgs<double>& A = M.A;
    const int y = lane >> 2, xp = lane & 3, x0 = 2 * xp;
    const int bp = y * 8 + x0;
    const uint64_t actw = S.act[z];
    const bool a0 = (actw >> bp) & 1ull, a1 = (actw >> (bp + 1)) & 1ull;
    if (!(a0 | a1)) return;
    const double* V = S.v;
    const int4 meta = S.meta;
    const int c = meta.x;
    const double2 uc = *reinterpret_cast<const double2*>(&V[O.c]);
    const double2 dc = *reinterpret_cast<const double2*>(&V[O.c + kDOff]);
    const double uL = V[O.l], dL = V[O.l + kDOff];
    const double uR = V[O.r], dR = V[O.r + kDOff];
    const double2 uym = *reinterpret_cast<const double2*>(&V[O.ym]);
    const double2 dym = *reinterpret_cast<const double2*>(&V[O.ym + kDOff]);
    const double2 uyp = *reinterpret_cast<const double2*>(&V[O.yp]);
    const double2 dyp = *reinterpret_cast<const double2*>(&V[O.yp + kDOff]);
    const double2 uzm = *reinterpret_cast<const double2*>(&V[O.zm]);
    const double2 dzm = *reinterpret_cast<const double2*>(&V[O.zm + kDOff]);
    const double2 uzp = *reinterpret_cast<const double2*>(&V[O.zp]);
    const double2 dzp = *reinterpret_cast<const double2*>(&V[O.zp + kDOff]);
    const bool s0 = REACTION == PD_REACTION_SURFACE_SINK && ((S.snk[z] >> bp) & 1ull);
    const bool s1 = REACTION == PD_REACTION_SURFACE_SINK && ((S.snk[z] >> (bp + 1)) & 1ull);
    const int o = O.c;  // body offset of node 0 == in-chunk offset
    double src0 = 0.0, src1 = 0.0;
    if (REACTION == PD_REACTION_VOLUMETRIC) {
        src0 = A.src[(int64_t)c * 512 + o];
        src1 = A.src[(int64_t)c * 512 + o + 1];
    }
    double out0 = 0.0, out1 = 0.0;
    bool slow0 = (meta.z & kFlagDirichlet) != 0, slow1 = slow0;
    if ((meta.z >> (8 + z)) & 1) {
        // interior-fluid plane: every node and every neighbour is fluid, so
        // no face needs the substitution select (warp-uniform branch)
        auto fface = [](double da, double db, double ua, double ub) {
            return ((da + db) * 0.5) * (ub - ua);
        };
        const double fxl = fface(dL, dc.x, uL, uc.x);
        const double fxi = fface(dc.x, dc.y, uc.x, uc.y);
        const double fxr = fface(dc.y, dR, uc.y, uR);
        const double ix = K.inv_dx2[0], iy = K.inv_dx2[1], iz = K.inv_dx2[2];
        double lap0 = 0.0;
        lap0 += (fxi - fxl) * ix;
        lap0 += (fface(dc.x, dyp.x, uc.x, uyp.x) - fface(dym.x, dc.x, uym.x, uc.x)) * iy;
        lap0 += (fface(dc.x, dzp.x, uc.x, uzp.x) - fface(dzm.x, dc.x, uzm.x, uc.x)) * iz;
        double lap1 = 0.0;
        lap1 += (fxr - fxi) * ix;
        lap1 += (fface(dc.y, dyp.y, uc.y, uyp.y) - fface(dym.y, dc.y, uym.y, uc.y)) * iy;
        lap1 += (fface(dc.y, dzp.y, uc.y, uzp.y) - fface(dzm.y, dc.y, uzm.y, uc.y)) * iz;
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
        slow0 = !isfinite(out0);
        slow1 = !isfinite(out1);
    } else if (!slow0) {
        const double fxl = face(dL, dc.x, uL, uc.x);
        const double fxi = face(dc.x, dc.y, uc.x, uc.y);
        const double fxr = face(dc.y, dR, uc.y, uR);
        const double ix = K.inv_dx2[0], iy = K.inv_dx2[1], iz = K.inv_dx2[2];
        double lap0 = 0.0;  // lap starts at T{0} (solver.hpp:420)
        lap0 += (fxi - fxl) * ix;
        lap0 += (face(dc.x, dyp.x, uc.x, uyp.x) - face(dym.x, dc.x, uym.x, uc.x)) * iy;
        lap0 += (face(dc.x, dzp.x, uc.x, uzp.x) - face(dzm.x, dc.x, uzm.x, uc.x)) * iz;
        double lap1 = 0.0;
        lap1 += (fxr - fxi) * ix;
        lap1 += (face(dc.y, dyp.y, uc.y, uyp.y) - face(dym.y, dc.y, uym.y, uc.y)) * iy;
        lap1 += (face(dc.y, dzp.y, uc.y, uzp.y) - face(dzm.y, dc.y, uzm.y, uc.y)) * iz;
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
        slow0 = !isfinite(out0);
        slow1 = !isfinite(out1);
    }
    if (slow0 | slow1) {
        const int kx = meta.y & 1023, ky = (meta.y >> 10) & 1023, kz = (meta.y >> 20) & 1023;
        const int64_t gx = (int64_t)kx * 8 + x0, gy = (int64_t)ky * 8 + y, gz = (int64_t)kz * 8 + z;
        if (slow0) {
            const double nu[6] = {uL, uc.y, uym.x, uyp.x, uzm.x, uzp.x};
            const double nd[6] = {dL, dc.y, dym.x, dyp.x, dzm.x, dzp.x};
            out0 = slow_node<REACTION>(K, uc.x, dc.x, nu, nd, gx, gy, gz, s0, src0);
        }
        if (slow1) {
            const double nu[6] = {uc.x, uR, uym.y, uyp.y, uzm.y, uzp.y};
            const double nd[6] = {dc.x, dR, dym.y, dyp.y, dzm.y, dzp.y};
            out1 = slow_node<REACTION>(K, uc.y, dc.y, nu, nd, gx + 1, gy, gz, s1, src1);
        }
    }
    // walls (active, not fluid) stay frozen (solver.hpp:413-417)
    if (sentinel(dc.x)) out0 = uc.x;
    if (sentinel(dc.y)) out1 = uc.y;
    double* dst = A.un + (int64_t)c * 512 + o;
    if (a0 && a1)
        *reinterpret_cast<double2*>(dst) = make_double2(out0, out1);
    else if (a0)
        dst[0] = out0;
    else
        dst[1] = out1;
    // x-face side planes of u_next for the next step's x halos
    if (xp == 0 && a0) M.xfun[((int64_t)c * 2 + 0) * 64 + z * 8 + y] = out0;
    if (xp == 3 && a1) M.xfun[((int64_t)c * 2 + 1) * 64 + z * 8 + y] = out1;
    // non-finite / huge detection (solver.hpp:444, 250-260, 514-515)
    const bool bad0 = a0 && !isfinite(out0), bad1 = a1 && !isfinite(out1);
    if (bad0 | bad1) {
        atomicMin(A.bad_key, ((unsigned long long)c << 10) | (unsigned long long)(o + (bad0 ? 0 : 1)));
        atomicOr(&A.flags[A.k], 1);
    } else if ((a0 && !(fabs(out0) < 0x1p990)) || (a1 && !(fabs(out1) < 0x1p990))) {
        atomicOr(&A.flags[A.k], 2);
    }
}

template <int REACTION>
__global__ void __launch_bounds__(kMarchThreads, kCtasPerSm) ftcs_march_kernel(MarchArgs M) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MarchStage* st = reinterpret_cast<MarchStage*>(smem_raw);
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const StepArgs<double>& A = M.A;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    if (t == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 64);               // 32 async + 32 plain arrivals
            mbar_init(&empty[s], kConsumerWarps);  // one per consumer warp
        }
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

    if (warp == kConsumerWarps) {
        // ---- producer: ids per batch in lane registers, descriptors kAhead
        // chunks ahead, the batch after next claimed while this one streams ----
        constexpr int kAhead = 4;
        int b_cur = 0, b_nxt = 0, b_far = 0;
        if (lane == 0) {
            b_cur = atomicAdd(M.counter, kBatch);
            b_nxt = atomicAdd(M.counter, kBatch);
        }
        b_cur = __shfl_sync(0xffffffffu, b_cur, 0);
        b_nxt = __shfl_sync(0xffffffffu, b_nxt, 0);
        auto ld_id = [&](int b) -> int {
            const int64_t p = (int64_t)b + lane;
            return p < M.n ? __ldg(&M.sched[p]) : -1;
        };
        int id_cur = ld_id(b_cur), id_nxt = ld_id(b_nxt), id_far = -1;
        int pos = 0;  // position of the chunk being produced inside batch b_cur
        auto id_ahead = [&](int k) -> int {  // chunk id k positions after pos
            const int p = pos + k;
            return p < kBatch ? __shfl_sync(0xffffffffu, id_cur, p)
                              : __shfl_sync(0xffffffffu, id_nxt, p - kBatch);
        };
        int cid[kAhead];
        LaneDesc ring[kAhead];
#pragma unroll
        for (int k = 0; k < kAhead; ++k) {
            cid[k] = id_ahead(k);
            ring[k] = load_lane_desc(M, cid[k], lane);
        }
        bool done = false;
        for (int q0 = 0; !done; q0 += kStages) {
#pragma unroll
            for (int s = 0; s < kStages; ++s) {
                if (q0 > 0) mbar_wait(&empty[s], ((q0 / kStages) - 1) & 1);
                const int c = cid[0];
                produce(st[s], &full[s], M, c, ring[0], lane);
                if (c < 0) {
                    done = true;
                    break;
                }
                // advance the prefetch window by one chunk
                const int c_new = cid[kAhead - 1] < 0 ? -1 : id_ahead(kAhead);
#pragma unroll
                for (int k = 0; k + 1 < kAhead; ++k) {
                    cid[k] = cid[k + 1];
                    ring[k] = ring[k + 1];
                }
                cid[kAhead - 1] = c_new;
                ring[kAhead - 1] = load_lane_desc(M, c_new, lane);
                ++pos;
                if (pos == 1 && lane == 0) b_far = atomicAdd(M.counter, kBatch);
                if (pos == kBatch / 2) id_far = ld_id(__shfl_sync(0xffffffffu, b_far, 0));
                if (pos == kBatch) {
                    pos = 0;
                    id_cur = id_nxt;
                    id_nxt = id_far;
                }
            }
        }
    } else {
        // ---- consumers: warp w = z-plane w ----
        const int z = warp, y = lane >> 2, xp = lane & 3, x0 = 2 * xp;
        const int o = z * 64 + y * 8 + x0;
        Offs O;
        O.c = o;
        O.l = xp == 0 ? kHX + z * 8 + y : o - 1;
        O.r = xp == 3 ? kHX + 64 + z * 8 + y : o + 2;
        O.ym = y == 0 ? kHY + z * 8 + x0 : o - 8;
        O.yp = y == 7 ? kHY + 64 + z * 8 + x0 : o + 8;
        O.zm = z == 0 ? kHZ + y * 8 + x0 : o - 64;
        O.zp = z == 7 ? kHZ + 64 + y * 8 + x0 : o + 64;
        for (int q0 = 0;; q0 += kStages) {
#pragma unroll
            for (int s = 0; s < kStages; ++s) {
                mbar_wait(&full[s], (q0 / kStages) & 1);
                if (st[s].meta.x < 0) return;
                consume<REACTION>(st[s], M, K, O, z, lane);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
    }
}

__global__ void desc_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ keys,
                            const uint64_t* __restrict__ act, const uint64_t* __restrict__ flu,
                            int64_t n, int64_t s0, int64_t s1, int64_t s2, int dirichlet,
                            int32_t* __restrict__ desc) {
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
    // dense chunks stream their body with bulk copies
    int pairs = 0;
    uint64_t F[8];
    for (int z = 0; z < 8; ++z) {
        const uint64_t w = act[i * 8 + z];
        pairs += __popcll((w | (w >> 1)) & 0x5555555555555555ull);
        F[z] = flu[i * 8 + z];
    }
    int flags = (exposed ? kFlagDirichlet : 0) | (pairs >= 128 ? kFlagBulk : 0);
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

// Per chunk and producer lane: bit 2r = the lane's pair in plane r has an
// active node, bit 2r+1 = it has a fluid node.
__global__ void pairmask_kernel(const uint64_t* __restrict__ act, const uint64_t* __restrict__ flu,
                                int64_t n, uint16_t* __restrict__ pm) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * 32) return;
    const int64_t c = t >> 5;
    const int lane = (int)(t & 31);
    unsigned v = 0;
    for (int r = 0; r < 8; ++r) {
        if ((act[c * 8 + r] >> (2 * lane)) & 3ull) v |= 1u << (2 * r);
        if ((flu[c * 8 + r] >> (2 * lane)) & 3ull) v |= 1u << (2 * r + 1);
    }
    pm[t] = (uint16_t)v;
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
    cudaFree(p->d_pm);
    *p = MarchPlan{};
}

void march_extract_xfaces(pd_grid* g, MarchPlan& p, const void* col) {
    const int64_t n = g->n_chunks;
    if (n == 0 || !p.ready) return;
    xface_kernel<<<(unsigned)((n * 128 + 255) / 256), 256, 0, g->stream>>>((const double*)col, n,
                                                                          p.d_xf[p.cur]);
    PD_CUDA(cudaGetLastError());
}

void march_build(pd_grid* g, const int32_t* d_nbr, const uint64_t* d_fluid, const void* d_dcol,
                 int dirichlet, int64_t begin, int64_t end, MarchPlan* plan) {
    march_free(plan);
    if (g->dims != 3 || g->tbytes != 8) return;
    if (g->cc[0] > 1024 || g->cc[1] > 1024 || g->cc[2] > 1024) return;  // key packing limit
    const int64_t n_all = g->n_chunks;
    if (n_all == 0 || end <= begin) return;
    PD_CUDA(cudaMalloc(&plan->d_desc, sizeof(int32_t) * 8 * (size_t)n_all));
    desc_kernel<<<(unsigned)((n_all + 255) / 256), 256, 0, g->stream>>>(
        d_nbr, g->d_keys, g->d_masks, d_fluid, n_all, g->size[0], g->size[1], g->size[2], dirichlet,
        plan->d_desc);
    PD_CUDA(cudaGetLastError());
    const int64_t slots = n_all * 512;
    PD_CUDA(cudaMalloc(&plan->d_deff, sizeof(double) * (size_t)slots));
    PD_CUDA(cudaMalloc(&plan->d_xfd, sizeof(double) * 128 * (size_t)n_all));
    PD_CUDA(cudaMalloc(&plan->d_xf[0], sizeof(double) * 128 * (size_t)n_all));
    PD_CUDA(cudaMalloc(&plan->d_xf[1], sizeof(double) * 128 * (size_t)n_all));
    PD_CUDA(cudaMalloc(&plan->d_counter, sizeof(int) * 1024));
    PD_CUDA(cudaMalloc(&plan->d_pm, sizeof(uint16_t) * 32 * (size_t)n_all));
    pairmask_kernel<<<(unsigned)((n_all * 32 + 255) / 256), 256, 0, g->stream>>>(g->d_masks, d_fluid,
                                                                                n_all, plan->d_pm);
    PD_CUDA(cudaGetLastError());
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
        const int za = ka[2] / kSeg, zb = kb[2] / kSeg;
        if (za != zb) return za < zb;
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
    plan->grid = sms * kCtasPerSm;
    plan->n = n;
    plan->ready = true;
    plan->cur = 0;
    static bool attr_set = false;
    if (!attr_set) {
        const int bytes = (int)(sizeof(MarchStage) * kStages);
        PD_CUDA(cudaFuncSetAttribute(ftcs_march_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        PD_CUDA(cudaFuncSetAttribute(ftcs_march_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        PD_CUDA(cudaFuncSetAttribute(ftcs_march_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        attr_set = true;
    }
}

void march_launch(pd_grid* g, MarchPlan& p, const StepArgs<double>& a, int reaction) {
    const size_t bytes = sizeof(MarchStage) * kStages;
    MarchArgs M;
    M.A = a;
    M.sched = p.d_stream;
    M.n = p.n;
    M.desc = p.d_desc;
    M.pm = p.d_pm;
    M.deff = p.d_deff;
    M.xfu = p.d_xf[p.cur];
    M.xfd = p.d_xfd;
    M.xfun = p.d_xf[1 - p.cur];
    M.counter = p.d_counter + (a.k & 1023);
    if (reaction == PD_REACTION_SURFACE_SINK)
        ftcs_march_kernel<1><<<p.grid, kMarchThreads, bytes, g->stream>>>(M);
    else if (reaction == PD_REACTION_VOLUMETRIC)
        ftcs_march_kernel<2><<<p.grid, kMarchThreads, bytes, g->stream>>>(M);
    else
        ftcs_march_kernel<0><<<p.grid, kMarchThreads, bytes, g->stream>>>(M);
    PD_CUDA(cudaGetLastError());
    p.cur = 1 - p.cur;
}

}  // namespace pdb
