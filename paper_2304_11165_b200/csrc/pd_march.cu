// Column-ordered, cp.async-pipelined FTCS step for 3-D FP64 grids — the
// bandwidth path (BASELINE.json configs C1-C5).
//
// Same per-node result, bit for bit, as ftcs_step_kernel (pd_ftcs.cu) and the
// reference (solver.hpp:360-455); what changes is how bytes and instructions
// are spent:
//
// * Schedule. Chunks are ordered (z-block of kSeg layers, y, x, z): runs of a
//   chunk column inside a z-block are contiguous, neighbouring columns follow
//   each other. Each CTA takes kBatch consecutive chunks of that order; the
//   hardware dispatches CTAs in order as SM slots free up, so the set of chunks
//   in flight is always a contiguous window of the schedule and every x/y/z
//   face halo a CTA reads was just streamed by its neighbours (L2 hit).
// * Staging. A kStages-deep cp.async ring stages each chunk's u / D into a
//   padded 10^3 tile (body + the six one-node face layers of the neighbour
//   chunks). Body pairs without an active (u) or fluid (D) node are never read
//   from HBM.
// * Usability without masks. The stepper keeps D_eff = fluid ? D : -inf
//   (static per run). A neighbour is usable iff it is fluid
//   (solver.hpp:374,379-381), i.e. iff the face sum d_a + d_b is not -inf, so
//   the substitution rule costs one integer compare per face.
// * Face fluxes. F(a|b) = ((d_a+d_b)*0.5)*(u_b-u_a) is exactly the value both
//   endpoints compute in the reference (dh_p*(p.u-u_c) for a, dh_m*(u_c-m.u)
//   for b), so it is computed once per face. For a substituted face the
//   reference computes ((d_c+d_c)*0.5)*(u_c-u_c) = +-0 when u_c, d_c are
//   finite, and any +-0 term leaves lap = 0.0 + ... bitwise unchanged, so the
//   fast path uses 0. Nodes whose fast result is non-finite, and chunks that
//   touch a Dirichlet outer face, take the exact generic path.
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {

constexpr int kMarchThreads = 256;
constexpr int kStages = 4;
constexpr int kSeg = 16;
constexpr int kBatch = 32;
constexpr int kTile = 1002;  // 1 pad + 10^3 + 1
constexpr unsigned kSentHi = 0xFFF00000u;  // high word of -inf
constexpr int kFlagInterior = 1, kFlagDirichlet = 2;

struct MarchStage {
    double u[kTile];
    double d[kTile];
    uint64_t act[8], snk[8];
};

__device__ __forceinline__ int tix(int x, int y, int z) {
    return 2 + x + 10 * (y + 1) + 100 * (z + 1);
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ bool sentinel(double d) {
    return (unsigned)__double2hiint(d) == kSentHi;
}

struct Desc {
    int4 a, b;  // a = nbr 0..3, b = {nbr4, nbr5, key packed 10:10:10, flags}
    uint64_t act, flu, snk;
};

__device__ __forceinline__ Desc load_desc(const StepArgs<double>& A, const int4* __restrict__ desc,
                                          int c, int z) {
    Desc d;
    d.a = __ldg(&desc[2 * (int64_t)c]);
    d.b = __ldg(&desc[2 * (int64_t)c + 1]);
    d.act = __ldg(&A.active[(int64_t)c * 8 + z]);
    d.flu = __ldg(&A.fluid[(int64_t)c * 8 + z]);
    d.snk = A.reaction == PD_REACTION_SURFACE_SINK ? __ldg(&A.sink[(int64_t)c * 8 + z]) : 0ull;
    return d;
}

// Stage one chunk: u and D_eff (sentinel -inf on non-fluid nodes) of the body
// and of the six neighbour face layers; absent neighbours get the sentinel.
__device__ __forceinline__ void issue(MarchStage& S, int4& meta, const StepArgs<double>& A,
                                      const double* __restrict__ deff, int c, const Desc& D,
                                      int t, int dbg) {
    const int z = t >> 5, y = (t >> 2) & 7, xp = t & 3, x0 = 2 * xp, lane = t & 31;
    const int o = z * 64 + y * 8 + x0;
    const int bp = y * 8 + x0;
    const int T = tix(x0, y, z);
    const double* U = A.u;
    const int64_t cb = (int64_t)c * 512;
    const double sent = __hiloint2double((int)kSentHi, 0);
    if ((D.act >> bp) & 3ull) cp16(&S.u[T], U + cb + o);
    if ((D.flu >> bp) & 3ull)
        cp16(&S.d[T], deff + cb + o);
    else
        *reinterpret_cast<double2*>(&S.d[T]) = make_double2(sent, sent);
    if (xp == 0) {
        const int j = (dbg & 1) ? -1 : D.a.x;
        if (j >= 0) {
            const int64_t src = (int64_t)j * 512 + z * 64 + y * 8 + 7;
            cp8(&S.u[T - 1], U + src);
            cp8(&S.d[T - 1], deff + src);
        } else {
            S.d[T - 1] = sent;
        }
    }
    if (xp == 3) {
        const int j = (dbg & 1) ? -1 : D.a.y;
        if (j >= 0) {
            const int64_t src = (int64_t)j * 512 + z * 64 + y * 8;
            cp8(&S.u[T + 2], U + src);
            cp8(&S.d[T + 2], deff + src);
        } else {
            S.d[T + 2] = sent;
        }
    }
    if (y == 0) {
        const int j = (dbg & 2) ? -1 : D.a.z;
        if (j >= 0) {
            const int64_t src = (int64_t)j * 512 + z * 64 + 56 + x0;
            cp16(&S.u[T - 10], U + src);
            cp16(&S.d[T - 10], deff + src);
        } else {
            *reinterpret_cast<double2*>(&S.d[T - 10]) = make_double2(sent, sent);
        }
    }
    if (y == 7) {
        const int j = (dbg & 2) ? -1 : D.a.w;
        if (j >= 0) {
            const int64_t src = (int64_t)j * 512 + z * 64 + x0;
            cp16(&S.u[T + 10], U + src);
            cp16(&S.d[T + 10], deff + src);
        } else {
            *reinterpret_cast<double2*>(&S.d[T + 10]) = make_double2(sent, sent);
        }
    }
    if (z == 0) {
        const int j = (dbg & 4) ? -1 : D.b.x;
        if (j >= 0) {
            const int64_t src = (int64_t)j * 512 + 448 + y * 8 + x0;
            cp16(&S.u[T - 100], U + src);
            cp16(&S.d[T - 100], deff + src);
        } else {
            *reinterpret_cast<double2*>(&S.d[T - 100]) = make_double2(sent, sent);
        }
    }
    if (z == 7) {
        const int j = (dbg & 4) ? -1 : D.b.y;
        if (j >= 0) {
            const int64_t src = (int64_t)j * 512 + y * 8 + x0;
            cp16(&S.u[T + 100], U + src);
            cp16(&S.d[T + 100], deff + src);
        } else {
            *reinterpret_cast<double2*>(&S.d[T + 100]) = make_double2(sent, sent);
        }
    }
    if (lane == 0) {
        S.act[z] = D.act;
        S.snk[z] = D.snk;
    }
    if (t == 0) meta = make_int4(c, D.b.z, D.b.w, 0);
}

// Face flux F(a|b) shared by both endpoints; 0 when either side is not fluid.
__device__ __forceinline__ double face(double da, double db, double ua, double ub) {
    const double s = da + db;
    const double f = (s * 0.5) * (ub - ua);
    return ((unsigned)__double2hiint(s) == kSentHi) ? 0.0 : f;
}

// Exact generic node update (solver.hpp:360-441 with the tile as the data
// source): used for Dirichlet-exposed chunks and to re-derive any non-finite
// fast-path result so post-error state matches the reference bit for bit.
// Per-launch constants of the generic path, copied to shared memory once so
// the out-of-line slow path does not force the kernel arguments onto the stack.
struct SlowConsts {
    int64_t size[3];
    double inv_dx2[3];
    double bcv[6];
    double dt, neg_k, src_factor;
    int dirichlet;
};

template <int REACTION>
__device__ __noinline__ double slow_node(const MarchStage& S, const SlowConsts& A, int T, int x,
                                         int y, int z, int kx, int ky, int kz, bool sink,
                                         double src) {
    const double u_c = S.u[T], d_c = S.d[T];
    const int64_t g[3] = {(int64_t)kx * 8 + x, (int64_t)ky * 8 + y, (int64_t)kz * 8 + z};
    const int stride[3] = {1, 10, 100};
    double lap = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        double nu[2], nd[2];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const int Tn = T + (side ? stride[ax] : -stride[ax]);
            const int64_t gg = g[ax] + (side ? 1 : -1);
            if (gg < 0 || gg >= A.size[ax]) {
                const int f = ax * 2 + side;
                nu[side] = (A.dirichlet >> f) & 1 ? A.bcv[f] : u_c;
                nd[side] = d_c;
            } else if (sentinel(S.d[Tn])) {
                nu[side] = u_c;
                nd[side] = d_c;
            } else {
                nu[side] = S.u[Tn];
                nd[side] = S.d[Tn];
            }
        }
        const double dh_m = (d_c + nd[0]) * 0.5;
        const double dh_p = (d_c + nd[1]) * 0.5;
        lap += (dh_p * (nu[1] - u_c) - dh_m * (u_c - nu[0])) * A.inv_dx2[ax];
    }
    double rate = 0.0;
    if (REACTION == PD_REACTION_SURFACE_SINK) {
        if (sink) rate = A.neg_k * u_c;
    } else if (REACTION == PD_REACTION_VOLUMETRIC) {
        rate = src * A.src_factor;
    }
    return u_c + A.dt * lap + A.dt * rate;
}

template <int REACTION>
__device__ __forceinline__ void compute(const MarchStage& S, const int4 meta,
                                        const StepArgs<double>& A, const SlowConsts& K, int t) {
    const int z = t >> 5, y = (t >> 2) & 7, xp = t & 3, x0 = 2 * xp;
    const int o = z * 64 + y * 8 + x0;
    const int bp = y * 8 + x0;
    const uint64_t actw = S.act[z];
    const bool a0 = (actw >> bp) & 1ull, a1 = (actw >> (bp + 1)) & 1ull;
    if (!(a0 | a1)) return;
    const int c = meta.x;
    const int T = tix(x0, y, z);
    const double2 uc = *reinterpret_cast<const double2*>(&S.u[T]);
    const double2 dc = *reinterpret_cast<const double2*>(&S.d[T]);
    const bool s0 = REACTION == PD_REACTION_SURFACE_SINK && ((S.snk[z] >> bp) & 1ull);
    const bool s1 = REACTION == PD_REACTION_SURFACE_SINK && ((S.snk[z] >> (bp + 1)) & 1ull);
    double src0 = 0.0, src1 = 0.0;
    if (REACTION == PD_REACTION_VOLUMETRIC) {
        src0 = A.src[(int64_t)c * 512 + o];
        src1 = A.src[(int64_t)c * 512 + o + 1];
    }
    double out0, out1;
    if (meta.z & kFlagDirichlet) {
        const int kx = meta.y & 1023, ky = (meta.y >> 10) & 1023, kz = (meta.y >> 20) & 1023;
        out0 = sentinel(dc.x) ? uc.x : slow_node<REACTION>(S, K, T, x0, y, z, kx, ky, kz, s0, src0);
        out1 = sentinel(dc.y) ? uc.y : slow_node<REACTION>(S, K, T + 1, x0 + 1, y, z, kx, ky, kz, s1, src1);
    } else {
        const double uL = S.u[T - 1], dL = S.d[T - 1];
        const double uR = S.u[T + 2], dR = S.d[T + 2];
        const double2 uym = *reinterpret_cast<const double2*>(&S.u[T - 10]);
        const double2 dym = *reinterpret_cast<const double2*>(&S.d[T - 10]);
        const double2 uyp = *reinterpret_cast<const double2*>(&S.u[T + 10]);
        const double2 dyp = *reinterpret_cast<const double2*>(&S.d[T + 10]);
        const double2 uzm = *reinterpret_cast<const double2*>(&S.u[T - 100]);
        const double2 dzm = *reinterpret_cast<const double2*>(&S.d[T - 100]);
        const double2 uzp = *reinterpret_cast<const double2*>(&S.u[T + 100]);
        const double2 dzp = *reinterpret_cast<const double2*>(&S.d[T + 100]);
        const double fxl = face(dL, dc.x, uL, uc.x);
        const double fxi = face(dc.x, dc.y, uc.x, uc.y);
        const double fxr = face(dc.y, dR, uc.y, uR);
        const double ix = A.inv_dx2[0], iy = A.inv_dx2[1], iz = A.inv_dx2[2];
        // node 0 (lap starts at T{0}, solver.hpp:420)
        double lap0 = 0.0;
        lap0 += (fxi - fxl) * ix;
        lap0 += (face(dc.x, dyp.x, uc.x, uyp.x) - face(dym.x, dc.x, uym.x, uc.x)) * iy;
        lap0 += (face(dc.x, dzp.x, uc.x, uzp.x) - face(dzm.x, dc.x, uzm.x, uc.x)) * iz;
        double lap1 = 0.0;
        lap1 += (fxr - fxi) * ix;
        lap1 += (face(dc.y, dyp.y, uc.y, uyp.y) - face(dym.y, dc.y, uym.y, uc.y)) * iy;
        lap1 += (face(dc.y, dzp.y, uc.y, uzp.y) - face(dzm.y, dc.y, uzm.y, uc.y)) * iz;
        double r0 = 0.0, r1 = 0.0;
        if (REACTION == PD_REACTION_SURFACE_SINK) {
            if (s0) r0 = A.neg_k * uc.x;
            if (s1) r1 = A.neg_k * uc.y;
        } else if (REACTION == PD_REACTION_VOLUMETRIC) {
            r0 = src0 * A.src_factor;
            r1 = src1 * A.src_factor;
        }
        out0 = uc.x + A.dt * lap0 + A.dt * r0;
        out1 = uc.y + A.dt * lap1 + A.dt * r1;
        // walls (active, not fluid) stay frozen (solver.hpp:413-417)
        if (sentinel(dc.x)) out0 = uc.x;
        if (sentinel(dc.y)) out1 = uc.y;
        if (!isfinite(out0) && !sentinel(dc.x)) {
            const int kx = meta.y & 1023, ky = (meta.y >> 10) & 1023, kz = (meta.y >> 20) & 1023;
            out0 = slow_node<REACTION>(S, K, T, x0, y, z, kx, ky, kz, s0, src0);
        }
        if (!isfinite(out1) && !sentinel(dc.y)) {
            const int kx = meta.y & 1023, ky = (meta.y >> 10) & 1023, kz = (meta.y >> 20) & 1023;
            out1 = slow_node<REACTION>(S, K, T + 1, x0 + 1, y, z, kx, ky, kz, s1, src1);
        }
    }
    double* dst = A.un + (int64_t)c * 512 + o;
    if (a0 && a1)
        *reinterpret_cast<double2*>(dst) = make_double2(out0, out1);
    else if (a0)
        dst[0] = out0;
    else
        dst[1] = out1;
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
__global__ void __launch_bounds__(kMarchThreads, 3)
    ftcs_march_kernel(StepArgs<double> A, const int32_t* __restrict__ sched, int64_t n,
                      const int4* __restrict__ desc, const double* __restrict__ deff, int dbg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MarchStage* st = reinterpret_cast<MarchStage*>(smem_raw);
    __shared__ int4 meta[kStages];
    __shared__ SlowConsts K;
    const int t = threadIdx.x;
    const int z = t >> 5;
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
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    const int64_t q0 = (int64_t)blockIdx.x * kBatch;
    const int cnt = (int)min((int64_t)kBatch, n - q0);
    const int32_t* ids = sched + q0;

    int c_issue = ids[0];
    Desc d_issue = load_desc(A, desc, c_issue, z);
    int c_next = cnt > 1 ? ids[1] : 0;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        Desc d_next = d_issue;
        int c_after = 0;
        if (s + 1 < cnt) d_next = load_desc(A, desc, c_next, z);
        if (s + 2 < cnt) c_after = ids[s + 2];
        if (s < cnt) issue(st[s], meta[s], A, deff, c_issue, d_issue, t, dbg);
        cp_commit();
        c_issue = c_next;
        d_issue = d_next;
        c_next = c_after;
    }
    for (int k = 0; k < cnt; ++k) {
        const int qi = k + kStages - 1;
        Desc d_next = d_issue;
        int c_after = 0;
        if (qi + 1 < cnt) d_next = load_desc(A, desc, c_next, z);
        if (qi + 2 < cnt) c_after = ids[qi + 2];
        if (qi < cnt) issue(st[qi % kStages], meta[qi % kStages], A, deff, c_issue, d_issue, t, dbg);
        cp_commit();
        c_issue = c_next;
        d_issue = d_next;
        c_next = c_after;
        cp_wait<kStages - 1>();
        __syncthreads();
        compute<REACTION>(st[k % kStages], meta[k % kStages], A, K, t);
        __syncthreads();
    }
}

__global__ void desc_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ keys,
                            int64_t n, int64_t s0, int64_t s1, int64_t s2, int dirichlet,
                            int4* __restrict__ desc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k[3] = {keys[i * 3], keys[i * 3 + 1], keys[i * 3 + 2]};
    const int64_t s[3] = {s0, s1, s2};
    bool interior = true, exposed = false;
    for (int a = 0; a < 3; ++a) {
        const bool lo = k[a] == 0;
        const bool hi = (int64_t)k[a] * 8 + 8 >= s[a];
        interior = interior && !lo && !hi;
        exposed = exposed || (lo && ((dirichlet >> (2 * a)) & 1)) || (hi && ((dirichlet >> (2 * a + 1)) & 1));
    }
    desc[2 * i] = make_int4(nbr[i * 6 + 0], nbr[i * 6 + 1], nbr[i * 6 + 2], nbr[i * 6 + 3]);
    desc[2 * i + 1] = make_int4(nbr[i * 6 + 4], nbr[i * 6 + 5], k[0] | (k[1] << 10) | (k[2] << 20),
                                (interior ? kFlagInterior : 0) | (exposed ? kFlagDirichlet : 0));
}

// D_eff = fluid ? D : -inf over every slot; counts fluid nodes whose D is not
// finite (then the fast path is disabled: its sentinel logic assumes finite D).
__global__ void deff_kernel(const double* __restrict__ dcol, const uint64_t* __restrict__ fluid,
                            int64_t n_slots, double* __restrict__ deff, unsigned long long* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_slots) return;
    const bool fl = (fluid[i >> 6] >> (i & 63)) & 1ull;
    const double v = dcol[i];
    deff[i] = fl ? v : __hiloint2double((int)kSentHi, 0);
    if (fl && !isfinite(v)) atomicAdd(bad, 1ull);
}

void march_free(MarchPlan* p) {
    cudaFree(p->d_stream);
    cudaFree(p->d_stream_off);
    cudaFree(p->d_desc);
    cudaFree(p->d_deff);
    *p = MarchPlan{};
}

void march_build(pd_grid* g, const int32_t* d_nbr, const uint64_t* d_fluid, const void* d_dcol,
                 int dirichlet, int64_t begin, int64_t end, MarchPlan* plan) {
    march_free(plan);
    if (g->dims != 3 || g->tbytes != 8) return;
    if (g->cc[0] > 1024 || g->cc[1] > 1024 || g->cc[2] > 1024) return;  // key packing limit
    const int64_t n_all = g->n_chunks;
    if (n_all == 0) return;
    PD_CUDA(cudaMalloc(&plan->d_desc, sizeof(int4) * 2 * (size_t)n_all));
    desc_kernel<<<(unsigned)((n_all + 255) / 256), 256, 0, g->stream>>>(
        d_nbr, g->d_keys, n_all, g->size[0], g->size[1], g->size[2], dirichlet, plan->d_desc);
    PD_CUDA(cudaGetLastError());
    const int64_t slots = n_all * 512;
    PD_CUDA(cudaMalloc(&plan->d_deff, sizeof(double) * (size_t)slots));
    unsigned long long* d_bad = nullptr;
    PD_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
    PD_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), g->stream));
    deff_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, g->stream>>>(
        (const double*)d_dcol, d_fluid, slots, plan->d_deff, d_bad);
    PD_CUDA(cudaGetLastError());
    unsigned long long bad = 0;
    PD_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, g->stream));
    // schedule of the owned range: (zblock, y, x, z)
    const int64_t n = end - begin;
    std::vector<int32_t> keys((size_t)std::max<int64_t>(1, n) * 3);
    if (n > 0)
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
    PD_CUDA(cudaMalloc(&plan->d_stream, sizeof(int32_t) * std::max<size_t>(1, order.size())));
    if (!order.empty())
        PD_CUDA(cudaMemcpyAsync(plan->d_stream, order.data(), sizeof(int32_t) * order.size(),
                                cudaMemcpyHostToDevice, g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    plan->grid = (int)((n + kBatch - 1) / kBatch);
    plan->n = n;
    plan->ready = n > 0;
    static bool attr_set = false;
    if (!attr_set) {
        const int bytes = (int)(sizeof(MarchStage) * kStages);
        PD_CUDA(cudaFuncSetAttribute(ftcs_march_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        PD_CUDA(cudaFuncSetAttribute(ftcs_march_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        PD_CUDA(cudaFuncSetAttribute(ftcs_march_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        attr_set = true;
    }
}

void march_launch(pd_grid* g, const MarchPlan& p, const StepArgs<double>& a, int reaction) {
    const size_t bytes = sizeof(MarchStage) * kStages;
    // PD_MARCH_DBG: measurement-only switch that skips halo classes
    // (1 x, 2 y, 4 z); results are then wrong. Never set in tests/bench.
    static const int dbg = [] {
        const char* e = getenv("PD_MARCH_DBG");
        return e ? atoi(e) : 0;
    }();
    if (reaction == PD_REACTION_SURFACE_SINK)
        ftcs_march_kernel<1><<<p.grid, kMarchThreads, bytes, g->stream>>>(a, p.d_stream, p.n, p.d_desc, p.d_deff, dbg);
    else if (reaction == PD_REACTION_VOLUMETRIC)
        ftcs_march_kernel<2><<<p.grid, kMarchThreads, bytes, g->stream>>>(a, p.d_stream, p.n, p.d_desc, p.d_deff, dbg);
    else
        ftcs_march_kernel<0><<<p.grid, kMarchThreads, bytes, g->stream>>>(a, p.d_stream, p.n, p.d_desc, p.d_deff, dbg);
    PD_CUDA(cudaGetLastError());
}

}  // namespace pdb
