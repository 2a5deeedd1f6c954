// Column-marching, cp.async-pipelined FTCS step for 3-D FP64 grids — the
// bandwidth path (BASELINE.json configs C1-C5).
//
// Same per-node arithmetic as ftcs_step_kernel (pd_ftcs.cu) and the reference
// (solver.hpp:360-455); what changes is how bytes move:
//   * Persistent CTAs (256 threads, 3 per SM) each own a static stream of
//     chunks. Streams are built once per stepper from "segments": runs of up
//     to kSeg chunks of one chunk column (x,y) that are consecutive in z,
//     scheduled z-block-major (zblock, y, x) and dealt round-robin to CTAs, so
//     at any instant the machine sweeps one z-block slab: the x/y face halos a
//     CTA reads were just read (or are being read) by its neighbours' CTAs and
//     hit L2, and the z halos are the planes of the chunks the same CTA read
//     one iteration earlier / is about to read.
//   * A kStages-deep cp.async ring stages body u/D (16-B copies, zero-filled
//     without a global read for pairs with no active / fluid node, so sectors
//     without active nodes cost no HBM traffic) and the six one-node face
//     halos of each chunk; descriptors (neighbour ordinals, masks) are
//     prefetched one stage ahead in registers, so no load waits on another.
//   * Warp w computes z-plane w of the chunk, two x-adjacent nodes per
//     thread; u_next is written with 16-B stores (8-B for half-active pairs).
#include <algorithm>
#include <numeric>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {

constexpr int kMarchThreads = 256;
constexpr int kStages = 4;
constexpr int kSeg = 16;
constexpr int kMarchCtasPerSm = 3;

struct MarchStage {
    double u[512], d[512];
    double hu[6][64], hd[6][64];  // face halos: x: z*8+y, y: z*8+x, z: y*8+x
    uint64_t act[8], flu[8], snk[8];
    uint64_t fl[6][8];  // neighbour fluid words (x/y faces per plane; z faces word 0)
};

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp8(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
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

__device__ __forceinline__ int nb_of(const Desc& d, int f) {
    return f == 0 ? d.a.x : f == 1 ? d.a.y : f == 2 ? d.a.z : f == 3 ? d.a.w : f == 4 ? d.b.x : d.b.y;
}

__device__ __forceinline__ void issue(MarchStage& S, int4& meta, const StepArgs<double>& A,
                                      int c, const Desc& D, int t) {
    const int z = t >> 5, y = (t >> 2) & 7, xp = t & 3, x0 = 2 * xp, lane = t & 31;
    const int o = z * 64 + y * 8 + x0;
    const int bp = y * 8 + x0;
    const double* U = A.u;
    const double* Dd = A.d;
    const int64_t cb = (int64_t)c * 512;
    cp16(&S.u[o], U + cb + o, ((D.act >> bp) & 3ull) != 0);
    cp16(&S.d[o], Dd + cb + o, ((D.flu >> bp) & 3ull) != 0);
    if (xp == 0) {
        const int j = D.a.x;
        const int64_t src = j >= 0 ? (int64_t)j * 512 + z * 64 + y * 8 + 7 : 0;
        cp8(&S.hu[0][z * 8 + y], U + src, j >= 0);
        cp8(&S.hd[0][z * 8 + y], Dd + src, j >= 0);
    }
    if (xp == 3) {
        const int j = D.a.y;
        const int64_t src = j >= 0 ? (int64_t)j * 512 + z * 64 + y * 8 : 0;
        cp8(&S.hu[1][z * 8 + y], U + src, j >= 0);
        cp8(&S.hd[1][z * 8 + y], Dd + src, j >= 0);
    }
    if (y == 0) {
        const int j = D.a.z;
        const int64_t src = j >= 0 ? (int64_t)j * 512 + z * 64 + 56 + x0 : 0;
        cp16(&S.hu[2][z * 8 + x0], U + src, j >= 0);
        cp16(&S.hd[2][z * 8 + x0], Dd + src, j >= 0);
    }
    if (y == 7) {
        const int j = D.a.w;
        const int64_t src = j >= 0 ? (int64_t)j * 512 + z * 64 + x0 : 0;
        cp16(&S.hu[3][z * 8 + x0], U + src, j >= 0);
        cp16(&S.hd[3][z * 8 + x0], Dd + src, j >= 0);
    }
    if (z == 0) {
        const int j = D.b.x;
        const int64_t src = j >= 0 ? (int64_t)j * 512 + 448 + y * 8 + x0 : 0;
        cp16(&S.hu[4][y * 8 + x0], U + src, j >= 0);
        cp16(&S.hd[4][y * 8 + x0], Dd + src, j >= 0);
    }
    if (z == 7) {
        const int j = D.b.y;
        const int64_t src = j >= 0 ? (int64_t)j * 512 + y * 8 + x0 : 0;
        cp16(&S.hu[5][y * 8 + x0], U + src, j >= 0);
        cp16(&S.hd[5][y * 8 + x0], Dd + src, j >= 0);
    }
    if (lane == 0) {
        S.act[z] = D.act;
        S.flu[z] = D.flu;
        S.snk[z] = D.snk;
    } else if (lane <= 4) {
        const int j = nb_of(D, lane - 1);
        cp8(&S.fl[lane - 1][z], A.fluid + (j >= 0 ? (int64_t)j * 8 + z : 0), j >= 0);
    } else if (lane == 5 && (z == 0 || z == 7)) {
        const int f = z == 0 ? 4 : 5;
        const int j = nb_of(D, f);
        cp8(&S.fl[f][0], A.fluid + (j >= 0 ? (int64_t)j * 8 + (z == 0 ? 7 : 0) : 0), j >= 0);
    }
    if (t == 0) meta = make_int4(c, D.b.z, D.b.w, 0);
}

// One neighbour value pair with the reference's substitution rule
// (solver.hpp:363-382): usable neighbour -> (u_nb, d_nb); Dirichlet outer
// face -> (value, d_c); anything else -> (u_c, d_c).
struct Nb {
    double u, d;
};

template <int REACTION>
__device__ __forceinline__ double update_node(const StepArgs<double>& A, const Nb (&nb)[6],
                                              double u_c, double d_c, bool sink,
                                              double src) {
    double lap = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const Nb m = nb[2 * ax], p = nb[2 * ax + 1];
        const double dh_m = (d_c + m.d) * 0.5;
        const double dh_p = (d_c + p.d) * 0.5;
        lap += (dh_p * (p.u - u_c) - dh_m * (u_c - m.u)) * A.inv_dx2[ax];
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
                                        const StepArgs<double>& A, int t) {
    const int z = t >> 5, y = (t >> 2) & 7, xp = t & 3, x0 = 2 * xp;
    const int o = z * 64 + y * 8 + x0;
    const int bp = y * 8 + x0;
    const uint64_t actw = S.act[z], fluw = S.flu[z];
    const bool a0 = (actw >> bp) & 1ull, a1 = (actw >> (bp + 1)) & 1ull;
    if (!(a0 | a1)) return;
    const bool f0 = (fluw >> bp) & 1ull, f1 = (fluw >> (bp + 1)) & 1ull;
    const int c = meta.x;
    const bool interior = meta.z & 1;
    const int kx = meta.y & 1023, ky = (meta.y >> 10) & 1023, kz = (meta.y >> 20) & 1023;
    const double u0 = S.u[o], u1 = S.u[o + 1];
    const double d0 = S.d[o], d1 = S.d[o + 1];
    const uint64_t fl_zm = z > 0 ? S.flu[z - 1] : 0ull, fl_zp = z < 7 ? S.flu[z + 1] : 0ull;
    double out[2];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
        const double u_c = n ? u1 : u0;
        const double d_c = n ? d1 : d0;
        const bool fl = n ? f1 : f0;
        const int x = x0 + n, oo = o + n, b = bp + n;
        if (!fl) {
            out[n] = u_c;  // solid-side node: frozen (solver.hpp:413-417)
            continue;
        }
        Nb nb[6];
        bool ok[6];
        // x-
        if (x == 0) {
            nb[0] = {S.hu[0][z * 8 + y], S.hd[0][z * 8 + y]};
            ok[0] = (S.fl[0][z] >> (y * 8 + 7)) & 1ull;
        } else if (n == 1) {
            nb[0] = {u0, d0};
            ok[0] = f0;
        } else {
            nb[0] = {S.u[oo - 1], S.d[oo - 1]};
            ok[0] = (fluw >> (b - 1)) & 1ull;
        }
        // x+
        if (x == 7) {
            nb[1] = {S.hu[1][z * 8 + y], S.hd[1][z * 8 + y]};
            ok[1] = (S.fl[1][z] >> (y * 8)) & 1ull;
        } else if (n == 0) {
            nb[1] = {u1, d1};
            ok[1] = f1;
        } else {
            nb[1] = {S.u[oo + 1], S.d[oo + 1]};
            ok[1] = (fluw >> (b + 1)) & 1ull;
        }
        // y-
        if (y == 0) {
            nb[2] = {S.hu[2][z * 8 + x], S.hd[2][z * 8 + x]};
            ok[2] = (S.fl[2][z] >> (56 + x)) & 1ull;
        } else {
            nb[2] = {S.u[oo - 8], S.d[oo - 8]};
            ok[2] = (fluw >> (b - 8)) & 1ull;
        }
        // y+
        if (y == 7) {
            nb[3] = {S.hu[3][z * 8 + x], S.hd[3][z * 8 + x]};
            ok[3] = (S.fl[3][z] >> x) & 1ull;
        } else {
            nb[3] = {S.u[oo + 8], S.d[oo + 8]};
            ok[3] = (fluw >> (b + 8)) & 1ull;
        }
        // z-
        if (z == 0) {
            nb[4] = {S.hu[4][y * 8 + x], S.hd[4][y * 8 + x]};
            ok[4] = (S.fl[4][0] >> (y * 8 + x)) & 1ull;
        } else {
            nb[4] = {S.u[oo - 64], S.d[oo - 64]};
            ok[4] = (fl_zm >> b) & 1ull;
        }
        // z+
        if (z == 7) {
            nb[5] = {S.hu[5][y * 8 + x], S.hd[5][y * 8 + x]};
            ok[5] = (S.fl[5][0] >> (y * 8 + x)) & 1ull;
        } else {
            nb[5] = {S.u[oo + 64], S.d[oo + 64]};
            ok[5] = (fl_zp >> b) & 1ull;
        }
#pragma unroll
        for (int f = 0; f < 6; ++f)
            if (!ok[f]) nb[f] = {u_c, d_c};
        if (!interior) {
            // outer box faces (solver.hpp:363-369) take precedence
            const int64_t g[3] = {(int64_t)kx * 8 + x, (int64_t)ky * 8 + y, (int64_t)kz * 8 + z};
#pragma unroll
            for (int f = 0; f < 6; ++f) {
                const int ax = f >> 1;
                const int64_t gg = g[ax] + ((f & 1) ? 1 : -1);
                if (gg < 0 || gg >= A.size[ax])
                    nb[f] = (A.dirichlet >> f) & 1 ? Nb{A.bcv[f], d_c} : Nb{u_c, d_c};
            }
        }
        const bool sk = REACTION == PD_REACTION_SURFACE_SINK && ((S.snk[z] >> b) & 1ull);
        const double src = REACTION == PD_REACTION_VOLUMETRIC ? A.src[(int64_t)c * 512 + oo] : 0.0;
        out[n] = update_node<REACTION>(A, nb, u_c, d_c, sk, src);
    }
    double* dst = A.un + (int64_t)c * 512 + o;
    if (a0 && a1)
        *reinterpret_cast<double2*>(dst) = make_double2(out[0], out[1]);
    else if (a0)
        dst[0] = out[0];
    else
        dst[1] = out[1];
    // non-finite / huge detection (solver.hpp:444, 250-260, 514-515)
#pragma unroll
    for (int n = 0; n < 2; ++n) {
        if (!(n ? a1 : a0)) continue;
        const double v = out[n];
        if (!isfinite(v)) {
            atomicMin(A.bad_key, ((unsigned long long)c << 10) | (unsigned long long)(o + n));
            atomicOr(&A.flags[A.k], 1);
        } else if (!(fabs(v) < 0x1p990)) {
            atomicOr(&A.flags[A.k], 2);
        }
    }
}

template <int REACTION>
__global__ void __launch_bounds__(kMarchThreads, kMarchCtasPerSm)
    ftcs_march_kernel(StepArgs<double> A, const int32_t* __restrict__ stream,
                      const int32_t* __restrict__ stream_off, const int4* __restrict__ desc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MarchStage* st = reinterpret_cast<MarchStage*>(smem_raw);
    __shared__ int4 meta[kStages];
    const int t = threadIdx.x;
    const int z = t >> 5;
    if (A.k > 0) {
        const int prev = A.flags[A.k - 1];
        if (prev) {
            if (t == 0 && blockIdx.x == 0) A.flags[A.k] = prev;
            return;
        }
    }
    const int q0 = stream_off[blockIdx.x];
    const int n = stream_off[blockIdx.x + 1] - q0;
    if (n <= 0) return;

    // software pipeline: chunk ids 2 ahead, descriptors 1 ahead of issue
    int c_issue = stream[q0];
    Desc d_issue = load_desc(A, desc, c_issue, z);
    int c_next = n > 1 ? stream[q0 + 1] : -1;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        Desc d_next;
        int c_after = -1;
        if (s + 1 < n) d_next = load_desc(A, desc, c_next, z);
        if (s + 2 < n) c_after = stream[q0 + s + 2];
        if (s < n) issue(st[s], meta[s], A, c_issue, d_issue, t);
        cp_commit();
        c_issue = c_next;
        d_issue = d_next;
        c_next = c_after;
    }
    for (int k = 0; k < n; ++k) {
        const int qi = k + kStages - 1;
        Desc d_next;
        int c_after = -1;
        if (qi + 1 < n) d_next = load_desc(A, desc, c_next, z);
        if (qi + 2 < n) c_after = stream[q0 + qi + 2];
        if (qi < n) issue(st[qi % kStages], meta[qi % kStages], A, c_issue, d_issue, t);
        cp_commit();
        c_issue = c_next;
        d_issue = d_next;
        c_next = c_after;
        cp_wait<kStages - 1>();
        __syncthreads();
        compute<REACTION>(st[k % kStages], meta[k % kStages], A, t);
        __syncthreads();
    }
}

__global__ void desc_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ keys,
                            int64_t n, int64_t s0, int64_t s1, int64_t s2, int4* __restrict__ desc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int kx = keys[i * 3], ky = keys[i * 3 + 1], kz = keys[i * 3 + 2];
    // interior: every node's 6 neighbours are inside the box
    const bool interior = kx >= 1 && ky >= 1 && kz >= 1 && (int64_t)kx * 8 + 8 < s0 &&
                          (int64_t)ky * 8 + 8 < s1 && (int64_t)kz * 8 + 8 < s2;
    desc[2 * i] = make_int4(nbr[i * 6 + 0], nbr[i * 6 + 1], nbr[i * 6 + 2], nbr[i * 6 + 3]);
    desc[2 * i + 1] = make_int4(nbr[i * 6 + 4], nbr[i * 6 + 5], kx | (ky << 10) | (kz << 20),
                                interior ? 1 : 0);
}

void march_free(MarchPlan* p) {
    cudaFree(p->d_stream);
    cudaFree(p->d_stream_off);
    cudaFree(p->d_desc);
    *p = MarchPlan{};
}

void march_build(pd_grid* g, const int32_t* d_nbr, int64_t begin, int64_t end, MarchPlan* plan) {
    march_free(plan);
    if (g->dims != 3 || g->tbytes != 8) return;
    if (g->cc[0] > 1024 || g->cc[1] > 1024 || g->cc[2] > 1024) return;  // key packing limit
    const int64_t n_all = g->n_chunks;
    // descriptors for every chunk (ghost chunks are referenced by ordinal only)
    PD_CUDA(cudaMalloc(&plan->d_desc, sizeof(int4) * 2 * (size_t)std::max<int64_t>(1, n_all)));
    if (n_all > 0) {
        desc_kernel<<<(unsigned)((n_all + 255) / 256), 256, 0, g->stream>>>(
            d_nbr, g->d_keys, n_all, g->size[0], g->size[1], g->size[2], plan->d_desc);
        PD_CUDA(cudaGetLastError());
    }
    // segments of the owned range
    const int64_t n = end - begin;
    std::vector<int32_t> keys((size_t)std::max<int64_t>(1, n) * 3), nb((size_t)std::max<int64_t>(1, n) * 6);
    if (n > 0) {
        PD_CUDA(cudaMemcpyAsync(keys.data(), g->d_keys + begin * 3, sizeof(int32_t) * 3 * (size_t)n,
                                cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaMemcpyAsync(nb.data(), d_nbr + begin * 6, sizeof(int32_t) * 6 * (size_t)n,
                                cudaMemcpyDeviceToHost, g->stream));
    }
    PD_CUDA(cudaStreamSynchronize(g->stream));
    auto in_range = [&](int32_t j) { return j >= begin && j < end; };
    std::vector<int64_t> starts;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t below = nb[(size_t)i * 6 + 4];
        if (!in_range(below) || keys[(size_t)i * 3 + 2] % kSeg == 0) starts.push_back(i);
    }
    std::sort(starts.begin(), starts.end(), [&](int64_t a, int64_t b) {
        const int32_t* ka = &keys[(size_t)a * 3];
        const int32_t* kb = &keys[(size_t)b * 3];
        const int za = ka[2] / kSeg, zb = kb[2] / kSeg;
        if (za != zb) return za < zb;
        if (ka[1] != kb[1]) return ka[1] < kb[1];
        return ka[0] < kb[0];
    });
    int dev_sms = 148;
    PD_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, g->device));
    const int grid = std::max(1, dev_sms * kMarchCtasPerSm);
    std::vector<std::vector<int32_t>> streams((size_t)grid);
    for (size_t s = 0; s < starts.size(); ++s) {
        auto& out = streams[s % (size_t)grid];
        int64_t i = starts[s];
        while (true) {
            out.push_back((int32_t)(begin + i));
            const int32_t up = nb[(size_t)i * 6 + 5];
            if (!in_range(up)) break;
            const int64_t ni = up - begin;
            if (keys[(size_t)ni * 3 + 2] % kSeg == 0) break;
            i = ni;
        }
    }
    std::vector<int32_t> flat, off((size_t)grid + 1, 0);
    flat.reserve((size_t)std::max<int64_t>(1, n));
    for (int b = 0; b < grid; ++b) {
        off[(size_t)b] = (int32_t)flat.size();
        flat.insert(flat.end(), streams[(size_t)b].begin(), streams[(size_t)b].end());
    }
    off[(size_t)grid] = (int32_t)flat.size();
    if ((int64_t)flat.size() != n) fail(PD_E_CUDA, "march plan lost chunks");
    PD_CUDA(cudaMalloc(&plan->d_stream, sizeof(int32_t) * std::max<size_t>(1, flat.size())));
    PD_CUDA(cudaMalloc(&plan->d_stream_off, sizeof(int32_t) * off.size()));
    if (!flat.empty())
        PD_CUDA(cudaMemcpyAsync(plan->d_stream, flat.data(), sizeof(int32_t) * flat.size(),
                                cudaMemcpyHostToDevice, g->stream));
    PD_CUDA(cudaMemcpyAsync(plan->d_stream_off, off.data(), sizeof(int32_t) * off.size(),
                            cudaMemcpyHostToDevice, g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    plan->grid = grid;
    plan->n = n;
    plan->ready = true;
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
    if (reaction == PD_REACTION_SURFACE_SINK)
        ftcs_march_kernel<1><<<p.grid, kMarchThreads, bytes, g->stream>>>(a, p.d_stream, p.d_stream_off, p.d_desc);
    else if (reaction == PD_REACTION_VOLUMETRIC)
        ftcs_march_kernel<2><<<p.grid, kMarchThreads, bytes, g->stream>>>(a, p.d_stream, p.d_stream_off, p.d_desc);
    else
        ftcs_march_kernel<0><<<p.grid, kMarchThreads, bytes, g->stream>>>(a, p.d_stream, p.d_stream_off, p.d_desc);
    PD_CUDA(cudaGetLastError());
}

}  // namespace pdb
