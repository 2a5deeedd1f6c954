// Fused FTCS reaction-diffusion step on the device sparse block grid
// (north_star subsystem 3). Restates FtcsStepper (solver.hpp:183-467) for
// sm_100a:
//   - one CTA per chunk: the chunk's u/D and its 2*Dims one-node face layers
//     from the neighbour chunks are staged in shared memory as a 10^Dims tile
//     with a per-cell face status, so every gather (solver.hpp:360-383) is a
//     shared-memory read;
//   - only active nodes are loaded and written (predicated), so 32-B sectors
//     without an active node cost no HBM traffic and inactive slots keep their
//     contents exactly as in the reference;
//   - phi is never read per step: the static wall / sink predicates
//     (solver.hpp:210-212,413,436) are precomputed once per stepper into
//     per-chunk bitmasks;
//   - arithmetic mirrors the reference expression tree with FMA contraction
//     disabled (--fmad=false; reference builds with -ffp-contract=off,
//     CMakeLists.txt:14), so results are bit-identical;
//   - diagnostics (mass / min / max, solver.hpp:444-454,264-278) are produced
//     only on record steps; every step still detects non-finite values with
//     the reference's lowest-ordinal/first-offset rule (solver.hpp:250-260).
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <initializer_list>
#include <limits>

#include <cstring>

#include "pd_internal.cuh"
#include <cstring>

namespace pdb {



__device__ __forceinline__ double min_left(double l, double r) { return (r < l) ? r : l; }
__device__ __forceinline__ double max_left(double l, double r) { return (l < r) ? r : l; }

// |x| >= 2^990 (or non-finite): a non-record step whose values are this large
// could overflow the total mass, which the reference checks every step
// (solver.hpp:514-515); such steps fall back to an exact mass evaluation.
__device__ __forceinline__ bool is_huge(double x, double thr) { return !(fabs(x) < thr); }

template <class T, int D, bool DIAG>
__global__ void __launch_bounds__(Geo<D>::V) ftcs_step_kernel(StepArgs<T> a) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W, FA = Geo<D>::FA, NH = Geo<D>::NH;
    constexpr int TV = Geo<D>::TV;
    __shared__ T su[TV];
    __shared__ T sd[TV];
    __shared__ uint8_t st[TV];  // 0 substitute centre, 1 neighbour, 2 Dirichlet halo

    const int64_t i = a.ord0 + blockIdx.x;
    const int off = threadIdx.x;
    if (a.k > 0) {
        const int prev = a.flags[a.k - 1];
        if (prev) {  // an earlier step of the batch failed: stay a no-op
            if (off == 0) a.flags[a.k] = prev;
            return;
        }
    }
    int c[3];
    c[0] = off & 7;
    c[1] = (off >> 3) & 7;
    c[2] = D == 3 ? (off >> 6) : 0;
    int64_t base[3];
#pragma unroll
    for (int ax = 0; ax < D; ++ax) base[ax] = (int64_t)a.keys[i * D + ax] << 3;

    const uint64_t aw = a.active[i * W + (off >> 6)];
    const uint64_t fw = a.fluid[i * W + (off >> 6)];
    const bool act = (aw >> (off & 63)) & 1u;
    const bool flu = (fw >> (off & 63)) & 1u;
    T u_c = T(0), d_c = T(0);
    if (act) u_c = a.u[i * V + off];
    if (flu) d_c = a.d[i * V + off];

    const int t = (c[0] + 1) + 10 * (c[1] + 1) + (D == 3 ? 100 * (c[2] + 1) : 0);
    {
        uint8_t s = flu ? 1 : 0;
        T tu = u_c;
        if (!act) {
            // in-chunk node beyond the box edge (size not a multiple of 8):
            // acts as the outer face (solver.hpp:363-369)
#pragma unroll
            for (int ax = 0; ax < D; ++ax)
                if (base[ax] + c[ax] >= a.size[ax]) {
                    if (a.dirichlet & (1 << (ax * 2 + 1))) {
                        s = 2;
                        tu = a.bcv[ax * 2 + 1];
                    }
                    break;
                }
        }
        su[t] = tu;
        sd[t] = d_c;
        st[t] = s;
    }
    // halo face layers from the 2*Dims neighbour chunks (build_neighbor_table,
    // solver.hpp:333-351; cross-chunk branch of gather, solver.hpp:377-382)
    for (int h = off; h < NH; h += V) {
        const int f = h / FA;
        const int p = h % FA;
        const int ax = f >> 1, side = f & 1;
        int q[3] = {0, 0, 0};
        {
            int r = p, b = 0;
#pragma unroll
            for (int bx = 0; bx < D; ++bx) {
                if (bx == ax) continue;
                q[bx] = (b == 0) ? (r & 7) : (r >> 3);
                ++b;
            }
        }
        q[ax] = side ? 8 : -1;
        const int th = (q[0] + 1) + 10 * (q[1] + 1) + (D == 3 ? 100 * (q[2] + 1) : 0);
        const int64_t g = base[ax] + q[ax];
        uint8_t s = 0;
        T tu = T(0), td = T(0);
        if (g < 0 || g >= a.size[ax]) {
            if (a.dirichlet & (1 << f)) {
                s = 2;
                tu = a.bcv[f];
            }
        } else {
            const int32_t j = a.nbr[i * 2 * D + f];
            if (j >= 0) {
                q[ax] = side ? 0 : 7;
                const int o2 = q[0] | (q[1] << 3) | (D == 3 ? (q[2] << 6) : 0);
                if ((a.fluid[(int64_t)j * W + (o2 >> 6)] >> (o2 & 63)) & 1u) {
                    s = 1;
                    tu = a.u[(int64_t)j * V + o2];
                    td = a.d[(int64_t)j * V + o2];
                }
            }
        }
        su[th] = tu;
        sd[th] = td;
        st[th] = s;
    }
    __syncthreads();

    T un = u_c;
    if (flu) {
        T lap = T(0);
#pragma unroll
        for (int ax = 0; ax < D; ++ax) {
            const int ts = ax == 0 ? 1 : (ax == 1 ? 10 : 100);
            const int tm = t - ts, tp = t + ts;
            const uint8_t sm = st[tm], sp = st[tp];
            const T mu = sm ? su[tm] : u_c;
            const T md = sm == 1 ? sd[tm] : d_c;
            const T pu = sp ? su[tp] : u_c;
            const T pdd = sp == 1 ? sd[tp] : d_c;
            const T dh_m = (d_c + md) * T(0.5);
            const T dh_p = (d_c + pdd) * T(0.5);
            lap += (dh_p * (pu - u_c) - dh_m * (u_c - mu)) * a.inv_dx2[ax];
        }
        T rate = T(0);
        if (a.reaction == PD_REACTION_SURFACE_SINK) {
            if ((a.sink[i * W + (off >> 6)] >> (off & 63)) & 1u) rate = a.neg_k * u_c;
        } else if (a.reaction == PD_REACTION_VOLUMETRIC) {
            rate = a.src[i * V + off] * a.src_factor;
        }
        un = u_c + a.dt * lap + a.dt * rate;
    }
    if (act) a.un[i * V + off] = un;

    const double v = (double)un;
    const bool bad = act && !isfinite(v);
    if (bad) {
        atomicMin(a.bad_key, ((unsigned long long)i << 10) | (unsigned long long)off);
        atomicOr(&a.flags[a.k], 1);
    }
    if constexpr (!DIAG) {
        if (act && !bad && is_huge(v, a.huge_abs)) atomicOr(&a.flags[a.k], 2);
    } else {
        // per-chunk partials (solver.hpp:444-454)
        __syncthreads();  // tile no longer needed: reuse su as scratch
        double* sv = reinterpret_cast<double*>(su);
        __shared__ double smn[V], smx[V];
        __shared__ uint64_t am[W];
        if (off < W) am[off] = a.active[i * W + off];
        if constexpr (sizeof(T) == 8) {
            sv[off] = v;
        }
        const bool ok = act && !isnan(v);
        smn[off] = ok ? v : INFINITY;
        smx[off] = ok ? v : -INFINITY;
        __syncthreads();
        for (int s = 1; s < V; s <<= 1) {
            if ((off & (2 * s - 1)) == 0) {
                smn[off] = min_left(smn[off], smn[off + s]);
                smx[off] = max_left(smx[off], smx[off + s]);
            }
            __syncthreads();
        }
        if constexpr (sizeof(T) != 8) {
            // float tile is too small for V doubles: reuse smx after the tree
            const double m0 = smn[0], x0 = smx[0];
            __syncthreads();
            smx[off] = v;
            __syncthreads();
            if (off == 0) {
                double acc = 0.0;
                for (int w = 0; w < W; ++w) {
                    uint64_t bits = am[w];
                    while (bits) {
                        const int b = __ffsll((long long)bits) - 1;
                        acc += smx[w * 64 + b];
                        bits &= bits - 1;
                    }
                }
                a.p_mass[i] = acc;
                a.p_mn[i] = m0;
                a.p_mx[i] = x0;
            }
        } else {
            if (off == 0) {
                double acc = 0.0;
                for (int w = 0; w < W; ++w) {
                    uint64_t bits = am[w];
                    while (bits) {
                        const int b = __ffsll((long long)bits) - 1;
                        acc += sv[w * 64 + b];
                        bits &= bits - 1;
                    }
                }
                a.p_mass[i] = acc;
                a.p_mn[i] = smn[0];
                a.p_mx[i] = smx[0];
            }
        }
    }
}

// Static per-stepper predicates from phi (never re-read per step):
//   fluid = active && !(phi <= wall)          (solver.hpp:374,381,413)
//   sink  = fluid && |double(phi)| <= w*hmin  (solver.hpp:436)
template <class T, int D>
__global__ void __launch_bounds__(Geo<D>::V)
    predicate_kernel(const T* __restrict__ phi, const uint64_t* __restrict__ active, T wall,
                     double sink_band, uint64_t* __restrict__ fluid, uint64_t* __restrict__ sink) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t i = blockIdx.x;
    const int off = threadIdx.x;
    const bool act = (active[i * W + (off >> 6)] >> (off & 63)) & 1u;
    bool fl = false, sk = false;
    if (act) {
        const T p = phi[i * V + off];
        fl = !(p <= wall);
        sk = fl && fabs((double)p) <= sink_band;
    }
    const unsigned bf = __ballot_sync(0xffffffffu, fl);
    const unsigned bs = __ballot_sync(0xffffffffu, sk);
    if ((off & 31) == 0) {
        const int w = off >> 6, hi = (off >> 5) & 1;
        reinterpret_cast<unsigned*>(fluid)[(i * W + w) * 2 + hi] = bf;
        reinterpret_cast<unsigned*>(sink)[(i * W + w) * 2 + hi] = bs;
    }
}

template <int D>
__global__ void neighbor_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ table,
                                int64_t n, int64_t cc0, int64_t cc1, int64_t cc2,
                                int32_t* __restrict__ nbr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t cc[3] = {cc0, cc1, cc2};
    for (int ax = 0; ax < D; ++ax)
        for (int s = 0; s < 2; ++s) {
            int64_t k[3] = {0, 0, 0};
            for (int b = 0; b < D; ++b) k[b] = keys[i * D + b];
            k[ax] += s == 0 ? -1 : 1;
            int32_t o = -1;
            if (k[ax] >= 0 && k[ax] < cc[ax]) {
                int64_t lin = k[D - 1];
                for (int b = D - 2; b >= 0; --b) lin = lin * cc[b] + k[b];
                o = table[lin];
            }
            nbr[i * 2 * D + ax * 2 + s] = o;
        }
}

}  // namespace pdb

using namespace pdb;

struct pd_stepper {
    pd_grid* g = nullptr;
    pd_sim_config cfg{};
    int prop_phi = -1, prop_u = -1, prop_d = -1, prop_next = -1, prop_src = -1;
    uint64_t* d_fluid = nullptr;
    uint64_t* d_sink = nullptr;
    int32_t* d_nbr = nullptr;
    int* d_flags = nullptr;
    unsigned long long* d_bad = nullptr;
    double* d_rows = nullptr;  // 3 per row of the batch
    int64_t batch_cap = 0;
    double inv_dx2[3] = {0, 0, 0};
    double hmin = 0.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_ms = 0.0;
    int64_t launches = 0;
    int64_t begin = 0, end = 0;  // owned ordinal range
    pdb::MarchPlan plan;         // 3-D FP64 column-march fast path
    bool use_march = true;
    // region-mass observer (run_frap, analysis.hpp:211-219): box sum of u at
    // every recorded step
    bool has_region = false;
    int64_t rlo[3] = {0, 0, 0}, rhi[3] = {0, 0, 0};
    double* d_region = nullptr;  // one per row of the batch
    std::vector<double> region_out;
    // steady-state observer (pd_observe.cu): max |u_new - u_old| per record
    bool has_conv = false;
    unsigned long long* d_conv = nullptr;  // one per row of the batch (bit patterns)
    std::vector<double> conv_out;
    pdb::PeerState peer;  // fused multi-GPU halo push (pd_peer.cu)
    int e_huge = 990;     // huge_exponent(): set at creation
    uint64_t ver_phi = 0, ver_d = 0;  // prop versions the static state was built from
    // run_simulation's per-step non-finite-mass check (solver.hpp:514-515);
    // off for pd_stepper_step, which is FtcsStepper::step (returns the row)
    bool check_mass = true;
};

namespace {

constexpr int64_t kBatch = 512;

// Below this many chunks per launch the one-CTA-per-chunk tile kernel is
// faster than the persistent march kernel (its pipeline fill / drain and
// per-warp claims dominate): measured crossover between 4 k and 14 k chunks
// (128^3 / 192^3 free boxes); PD_MARCH_MIN_CHUNKS overrides.
int64_t march_min_chunks() {
    static const int64_t v = [] {
        const char* e = getenv("PD_MARCH_MIN_CHUNKS");
        return e ? (int64_t)atoll(e) : (int64_t)6144;
    }();
    return v;
}

void march_build_for(pd_stepper* s, int64_t begin, int64_t end) {
    pd_grid* g = s->g;
    int dir = 0;
    for (int f = 0; f < 2 * g->dims; ++f)
        if (s->cfg.bc_type[f] == PD_BC_DIRICHLET) dir |= 1 << f;
    const void* dcol = g->cols[(size_t)g->column_of[(size_t)s->prop_d]];
    march_build(g, s->d_nbr, s->d_fluid, s->d_sink, dcol, dir, begin, end, &s->plan);
}

// Static per-run state derived from phi (fluid / sink bitmasks) and the
// neighbour table (solver.hpp:206-215, 333-351).
void build_predicates(pd_stepper* s) {
    pd_grid* g = s->g;
    if (g->n_chunks > 0) {
        const void* phi = g->cols[(size_t)g->column_of[(size_t)s->prop_phi]];
        const double sink_band = s->cfg.band_half_width * s->hmin;  // solver.hpp:212
        const unsigned nb = (unsigned)g->n_chunks;
        if (g->tbytes == 8) {
            // wall = T(b_low) + T(eps)   (solver.hpp:210-211)
            const double wall = (double)s->cfg.b_low + (double)s->cfg.boundary_epsilon;
            if (g->dims == 3)
                predicate_kernel<double, 3><<<nb, 512, 0, g->stream>>>(
                    (const double*)phi, g->d_masks, wall, sink_band, s->d_fluid, s->d_sink);
            else
                predicate_kernel<double, 2><<<nb, 64, 0, g->stream>>>(
                    (const double*)phi, g->d_masks, wall, sink_band, s->d_fluid, s->d_sink);
        } else {
            const float wall = (float)s->cfg.b_low + (float)s->cfg.boundary_epsilon;
            if (g->dims == 3)
                predicate_kernel<float, 3><<<nb, 512, 0, g->stream>>>(
                    (const float*)phi, g->d_masks, wall, sink_band, s->d_fluid, s->d_sink);
            else
                predicate_kernel<float, 2><<<nb, 64, 0, g->stream>>>(
                    (const float*)phi, g->d_masks, wall, sink_band, s->d_fluid, s->d_sink);
        }
        PD_CUDA(cudaGetLastError());
        const int blocks = (int)((g->n_chunks + 255) / 256);
        if (g->dims == 3)
            neighbor_kernel<3><<<blocks, 256, 0, g->stream>>>(
                g->d_keys, g->d_table, g->n_chunks, g->cc[0], g->cc[1], g->cc[2], s->d_nbr);
        else
            neighbor_kernel<2><<<blocks, 256, 0, g->stream>>>(
                g->d_keys, g->d_table, g->n_chunks, g->cc[0], g->cc[1], 1, s->d_nbr);
        PD_CUDA(cudaGetLastError());
    }
    s->ver_phi = prop_version(g, s->prop_phi);
    s->ver_d = prop_version(g, s->prop_d);
}

// phi or D was written since the stepper derived its static state (the
// reference reads both on every step, solver.hpp:407-441): rebuild the
// predicates and the march plan over the owned range.
void refresh_if_stale(pd_stepper* s) {
    pd_grid* g = s->g;
    if (prop_version(g, s->prop_phi) == s->ver_phi && prop_version(g, s->prop_d) == s->ver_d) return;
    build_predicates(s);
    if (s->use_march) {
        march_build_for(s, s->begin, s->end);
        s->peer.flags_dirty = s->peer.on;
    }
    PD_CUDA(cudaStreamSynchronize(g->stream));
}

void validate(const pd_grid* g, const pd_sim_config* c, int prop_src,
              std::initializer_list<int> solver_props) {
    // solver.hpp:304-331, messages verbatim
    if (!(c->dt > 0.0) || !std::isfinite(c->dt))
        fail(PD_E_INPUT, "time step must be positive and finite");
    if (c->n_steps < 1) fail(PD_E_INPUT, "step count must be at least 1");
    if (c->record_every < 1) fail(PD_E_INPUT, "record_every must be at least 1");
    if (!(c->b_low < c->b_up)) fail(PD_E_INPUT, "phase band is empty (b_low must be < b_up)");
    if (c->boundary_epsilon < 0.0 || !std::isfinite(c->boundary_epsilon))
        fail(PD_E_INPUT, "boundary_epsilon must be finite and >= 0");
    if (c->reaction_kind == PD_REACTION_SURFACE_SINK) {
        if (c->rate < 0.0) fail(PD_E_INPUT, "surface sink rate must be >= 0");
        if (!(c->band_half_width > 0.0))
            fail(PD_E_INPUT, "surface sink band half-width must be > 0");
    }
    for (int p : solver_props)
        if (p < 0 || p >= (int)g->column_of.size())
            fail(PD_E_INPUT,
                 "grid lacks a solver channel; build simulation grids with channels "
                 "{phi, u, D, u_next}");
    if (c->reaction_kind == PD_REACTION_VOLUMETRIC &&
        (prop_src < 0 || prop_src >= (int)g->column_of.size()))
        fail(PD_E_PROPERTY, "unknown property (volumetric source channel)");
}

template <class T>
void fill_args(const pd_stepper* s, StepArgs<T>& a, const void* u, void* un, double factor) {
    const pd_grid* g = s->g;
    const pd_sim_config& c = s->cfg;
    a.u = (const T*)u;
    a.un = (T*)un;
    a.d = (const T*)g->cols[(size_t)g->column_of[(size_t)s->prop_d]];
    a.src = s->prop_src >= 0 ? (const T*)g->cols[(size_t)g->column_of[(size_t)s->prop_src]]
                             : nullptr;
    a.active = g->d_masks;
    a.fluid = s->d_fluid;
    a.sink = s->d_sink;
    a.nbr = s->d_nbr;
    a.keys = g->d_keys;
    for (int ax = 0; ax < 3; ++ax) a.size[ax] = g->size[ax];
    // inv_dx2[a] = T(1) / T(h_a * h_a)   (solver.hpp:202-205)
    for (int ax = 0; ax < 3; ++ax)
        a.inv_dx2[ax] = ax < g->dims ? T(1) / static_cast<T>(g->spacing[ax] * g->spacing[ax]) : T(0);
    a.dt = static_cast<T>(c.dt);                 // solver.hpp:206
    a.neg_k = -static_cast<T>(c.rate);           // solver.hpp:437
    a.src_factor = static_cast<T>(factor);       // solver.hpp:231-234
    a.dirichlet = 0;
    for (int f = 0; f < 6; ++f) {
        a.bcv[f] = static_cast<T>(c.bc_value[f]);  // solver.hpp:367
        if (f < 2 * g->dims && c.bc_type[f] == PD_BC_DIRICHLET) a.dirichlet |= 1 << f;
    }
    a.reaction = c.reaction_kind;
    a.p_mass = g->red.part[0];
    a.p_mn = g->red.part[1];
    a.p_mx = g->red.part[2];
    a.bad_key = s->d_bad;
    a.flags = s->d_flags;
    a.huge_abs = std::ldexp(1.0, s->e_huge);
    a.huge_hi = s->e_huge < -1022 ? 0u : (uint32_t)(s->e_huge + 1023) << 20;
}

// Exponent below which no value can make the step's total mass non-finite
// (the reference checks pairwise_sum(partials) * cell_volume every step,
// solver.hpp:264-267, 514-515): n_slots values of magnitude < 2^e sum, in
// any order, to < n_slots * 2^e <= 2^1022, and times cell_volume stays finite
// while n_slots * 2^e * max(1, cell_volume) <= 2^1022.
int huge_exponent(const pd_grid* g) {
    const double n_slots = std::max(1.0, (double)g->n_chunks * (g->dims == 3 ? 512.0 : 64.0));
    double cv = 1.0;
    for (int ax = 0; ax < g->dims; ++ax) cv *= g->spacing[ax];
    const int ln = (int)std::ceil(std::log2(n_slots));
    const int lc = cv > 1.0 ? (int)std::ceil(std::log2(cv)) : 0;
    return std::max(-1100, 1022 - ln - lc);
}

// One step of the owned range with the fused halo push: wait for the
// neighbours' previous step, march (boundary planes stored into their ghost
// chunks as they are computed), raise their counters.
void launch_peer_step(pd_stepper* s, const StepArgs<double>& a) {
    pd_grid* g = s->g;
    if (!s->plan.ready) fail(PD_E_INPUT, "the fused peer halo push needs the march path (3-D FP64 grid)");
    if (s->peer.flags_dirty) {
        march_push_flags(g, s->plan, s->peer.d_ord);
        s->peer.flags_dirty = false;
    }
    PeerLaunch pl;
    const int cn = g->column_of[(size_t)s->prop_next];
    for (int side = 0; side < 2; ++side)
        pl.un[side] = s->peer.side[side] ? static_cast<double*>(s->peer.cols[side][cn]) : nullptr;
    pl.ord = s->peer.d_ord;
    peer_wait(g->stream, s->peer);
    march_launch(g, s->plan, a, s->cfg.reaction_kind, &pl);
    peer_signal(g->stream, s->peer);
    s->peer.epoch++;
}

void launch_step(pd_stepper* s, const void* u, void* un, double factor, bool diag, int k) {
    pd_grid* g = s->g;
    if (s->end <= s->begin) return;
    const unsigned nb = (unsigned)(s->end - s->begin);
    if (g->tbytes == 8) {
        StepArgs<double> a;
        fill_args<double>(s, a, u, un, factor);
        a.k = k;
        a.ord0 = s->begin;
        if (s->peer.on) {
            launch_peer_step(s, a);
            if (diag) launch_chunk_stats(g, un, g->d_masks);
        } else if (s->use_march && s->plan.ready && s->end - s->begin >= march_min_chunks()) {
            march_launch(g, s->plan, a, s->cfg.reaction_kind);
            // record step: per-chunk sequential mass / min / max of the new u
            // in the reference's order (solver.hpp:264-278), a second pass
            // (8 B/node) instead of the slower generic diagnostics kernel
            if (diag) launch_chunk_stats(g, un, g->d_masks);
        } else if (g->dims == 3) {
            if (diag) ftcs_step_kernel<double, 3, true><<<nb, 512, 0, g->stream>>>(a);
            else ftcs_step_kernel<double, 3, false><<<nb, 512, 0, g->stream>>>(a);
        } else {
            if (diag) ftcs_step_kernel<double, 2, true><<<nb, 64, 0, g->stream>>>(a);
            else ftcs_step_kernel<double, 2, false><<<nb, 64, 0, g->stream>>>(a);
        }
    } else {
        StepArgs<float> a;
        fill_args<float>(s, a, u, un, factor);
        a.k = k;
        a.ord0 = s->begin;
        if (s->use_march && s->plan.ready && s->end - s->begin >= march_min_chunks()) {
            march32_launch(g, s->plan, a, s->cfg.reaction_kind);
            if (diag) launch_chunk_stats(g, un, g->d_masks);
        } else if (g->dims == 3) {
            if (diag) ftcs_step_kernel<float, 3, true><<<nb, 512, 0, g->stream>>>(a);
            else ftcs_step_kernel<float, 3, false><<<nb, 512, 0, g->stream>>>(a);
        } else {
            if (diag) ftcs_step_kernel<float, 2, true><<<nb, 64, 0, g->stream>>>(a);
            else ftcs_step_kernel<float, 2, false><<<nb, 64, 0, g->stream>>>(a);
        }
    }
    PD_CUDA(cudaGetLastError());
    s->launches++;
}

std::string node_message(const pd_grid* g, int64_t step_number, unsigned long long key) {
    const int64_t ordinal = (int64_t)(key >> 10);
    const int off = (int)(key & 1023u);
    std::vector<int32_t> k((size_t)g->dims);
    PD_CUDA(cudaMemcpy(k.data(), g->d_keys + ordinal * g->dims, sizeof(int32_t) * (size_t)g->dims,
                       cudaMemcpyDeviceToHost));
    // solver.hpp:253-258 (node_index, sparse_block_grid.hpp:244-250)
    std::string m = "non-finite value at step " + std::to_string(step_number) + ", node (";
    for (int a = 0; a < g->dims; ++a) {
        const int64_t idx = ((int64_t)k[(size_t)a] << 3) | ((off >> (3 * a)) & 7);
        m += (a ? "," : "") + std::to_string(idx);
    }
    return m + ")";
}

}  // namespace

extern "C" {

int pd_stepper_create(pd_grid* g, const pd_sim_config* cfg, int prop_phi, int prop_u, int prop_d,
                      int prop_next, pd_stepper** out) {
    return guarded([&] {
        *out = nullptr;
        const int prop_src = cfg->reaction_kind == PD_REACTION_VOLUMETRIC ? cfg->source_prop : -1;
        validate(g, cfg, prop_src, {prop_phi, prop_u, prop_d, prop_next});
        DeviceGuard dg(g->device);
        auto* s = new pd_stepper();
        try {
            s->g = g;
            ++g->refs;
            s->cfg = *cfg;
            s->prop_phi = prop_phi;
            s->prop_u = prop_u;
            s->prop_d = prop_d;
            s->prop_next = prop_next;
            s->prop_src = prop_src;
            s->begin = 0;
            s->end = g->n_chunks;
            s->hmin = g->spacing[0];
            for (int a = 1; a < g->dims; ++a) s->hmin = std::min(s->hmin, g->spacing[a]);
            const int64_t n = std::max<int64_t>(1, g->n_chunks);
            PD_CUDA(pd_malloc(&s->d_fluid, sizeof(uint64_t) * (size_t)(n * g->W)));
            PD_CUDA(pd_malloc(&s->d_sink, sizeof(uint64_t) * (size_t)(n * g->W)));
            PD_CUDA(pd_malloc(&s->d_nbr, sizeof(int32_t) * (size_t)(n * 2 * g->dims)));
            PD_CUDA(pd_malloc(&s->d_flags, sizeof(int) * (size_t)kBatch));
            PD_CUDA(pd_malloc(&s->d_bad, sizeof(unsigned long long)));
            PD_CUDA(pd_malloc(&s->d_rows, sizeof(double) * 3 * (size_t)kBatch));
            PD_CUDA(pd_malloc(&s->d_region, sizeof(double) * (size_t)kBatch));
            PD_CUDA(pd_malloc(&s->d_conv, sizeof(unsigned long long) * (size_t)kBatch));
            PD_CUDA(cudaMemsetAsync(s->d_flags, 0, sizeof(int) * (size_t)kBatch, g->stream));
            PD_CUDA(cudaMemsetAsync(s->d_bad, 0xff, sizeof(unsigned long long), g->stream));
            PD_CUDA(cudaEventCreate(&s->ev0));
            PD_CUDA(cudaEventCreate(&s->ev1));
            build_predicates(s);
            ensure_scratch(g);
            // 4 bits of margin: a sharded domain's global mass sums up to 16
            // ranks' slots (shard.py)
            s->e_huge = huge_exponent(g) - 4;
            const char* nm = getenv("PD_NO_MARCH");
            s->use_march = !(nm && nm[0] == '1');
            // the FP32 march kernel has no huge-value check: float values
            // (< 2^128) must not be able to overflow the double total mass
            if (g->tbytes == 4 && s->e_huge < 129) s->use_march = false;
            if (s->use_march) march_build_for(s, 0, g->n_chunks);
            PD_CUDA(cudaStreamSynchronize(g->stream));
        } catch (...) {
            pd_stepper_destroy(s);
            throw;
        }
        *out = s;
    });
}

int pd_stepper_destroy(pd_stepper* s) {
    if (!s) return PD_OK;
    {
        DeviceGuard dg(s->g->device);
        cudaStreamSynchronize(s->g->stream);
        pd_free(s->d_fluid);
        pd_free(s->d_sink);
        pd_free(s->d_nbr);
        pd_free(s->d_flags);
        pd_free(s->d_bad);
        pd_free(s->d_rows);
        pd_free(s->d_region);
        pd_free(s->d_conv);
        pd_free(s->peer.d_ord);
        pd_free(s->peer.d_err);
        if (s->peer.d_sync) cudaFree(s->peer.d_sync);
        march_free(&s->plan);
        if (s->ev0) cudaEventDestroy(s->ev0);
        if (s->ev1) cudaEventDestroy(s->ev1);
    }
    grid_release(s->g);
    delete s;
    return PD_OK;
}

int pd_stepper_set_range(pd_stepper* s, int64_t begin, int64_t end) {
    return guarded([&] {
        if (begin < 0 || end > s->g->n_chunks || begin > end)
            fail(PD_E_INPUT, "stepper ordinal range outside the grid");
        s->begin = begin;
        s->end = end;
        if (s->use_march && s->g->dims == 3) {
            DeviceGuard dg(s->g->device);
            march_build_for(s, begin, end);
        }
    });
}

int pd_stepper_stability_bound(pd_stepper* s, double* out) {
    return guarded([&] {
        double dmax = 0.0;
        const int rc = pd_grid_max_active(s->g, s->prop_d, &dmax);
        if (rc != PD_OK) fail(rc, pd_last_error());
        if (!(dmax > 0.0)) {
            *out = std::numeric_limits<double>::infinity();
            return;
        }
        // stability_dt (solver.hpp:111-120)
        double inv_sum = 0.0;
        for (int a = 0; a < s->g->dims; ++a) {
            const double h = s->g->spacing[a];
            inv_sum += 1.0 / (h * h);
        }
        *out = 1.0 / (2.0 * dmax) / inv_sum;
    });
}

int pd_stepper_snapshot_diag(pd_stepper* s, pd_diag* out) {
    return guarded([&] {
        pd_grid* g = s->g;
        DeviceGuard dg(g->device);
        const void* u = g->cols[(size_t)g->column_of[(size_t)s->prop_u]];
        launch_chunk_stats(g, u, g->d_masks);
        launch_pairwise_finalize(g, g->d_row, nullptr);
        double row[3];
        PD_CUDA(cudaMemcpyAsync(row, g->d_row, sizeof row, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        out->step = 0;
        out->time = 0.0;
        out->total_mass = row[0];
        out->min_u = row[1];
        out->max_u = row[2];
    });
}

int pd_stepper_run(pd_stepper* s, int64_t step0, int64_t n_steps, int64_t final_step,
                   const double* factors, pd_diag* rows, int64_t* n_rows) {
    return guarded([&] {
        *n_rows = 0;
        if (n_steps <= 0) return;
        pd_grid* g = s->g;
        DeviceGuard dg(g->device);
        refresh_if_stale(s);
        const pd_sim_config& c = s->cfg;
        const int64_t rec = c.record_every;
        double total_ms = 0.0;
        int64_t j = 0;
        std::vector<int> hflags((size_t)kBatch);
        std::vector<double> hrows((size_t)kBatch * 3);
        std::vector<int64_t> row_step((size_t)kBatch);
        std::vector<double> hregion((size_t)kBatch);
        std::vector<unsigned long long> hconv((size_t)kBatch);
        s->region_out.clear();
        s->conv_out.clear();
        while (j < n_steps) {
            const int64_t nb = std::min<int64_t>(kBatch, n_steps - j);
            PD_CUDA(cudaMemsetAsync(s->d_flags, 0, sizeof(int) * (size_t)nb, g->stream));
            PD_CUDA(cudaMemsetAsync(s->d_bad, 0xff, sizeof(unsigned long long), g->stream));
            if (s->plan.ready)
                PD_CUDA(cudaMemsetAsync(s->plan.d_counter, 0,
                                        sizeof(int) * (size_t)(nb * march_counters_per_step()), g->stream));
            int64_t nr = 0;
            if (s->has_conv)
                PD_CUDA(cudaMemsetAsync(s->d_conv, 0, sizeof(unsigned long long) * (size_t)nb, g->stream));
            PD_CUDA(cudaEventRecord(s->ev0, g->stream));
            for (int64_t k = 0; k < nb; ++k) {
                const int64_t st = step0 + j + k;  // global step index being taken
                const bool record = ((st + 1) % rec == 0) || (st + 1 == final_step);
                const int cu = g->column_of[(size_t)s->prop_u];
                const int cn = g->column_of[(size_t)s->prop_next];
                const double f = factors ? factors[j + k] : 1.0;
                launch_step(s, g->cols[(size_t)cu], g->cols[(size_t)cn], f, record, (int)k);
                if (record) {
                    launch_pairwise_finalize(g, s->d_rows + 3 * nr, s->d_flags + k, s->begin,
                                             s->end - s->begin);
                    if (s->has_region) launch_box_sum(g, g->cols[(size_t)cn], s->rlo, s->rhi, s->d_region + nr);
                    if (s->has_conv) launch_absdiff_max(g, g->cols[(size_t)cn], g->cols[(size_t)cu], s->d_conv + nr);
                    row_step[(size_t)nr] = st + 1;
                    ++nr;
                }
                // swap_channels("u", "u_next")  (solver.hpp:262)
                std::swap(g->column_of[(size_t)s->prop_u], g->column_of[(size_t)s->prop_next]);
            }
            PD_CUDA(cudaEventRecord(s->ev1, g->stream));
            PD_CUDA(cudaMemcpyAsync(hflags.data(), s->d_flags, sizeof(int) * (size_t)nb,
                                    cudaMemcpyDeviceToHost, g->stream));
            if (nr > 0)
                PD_CUDA(cudaMemcpyAsync(hrows.data(), s->d_rows, sizeof(double) * 3 * (size_t)nr,
                                        cudaMemcpyDeviceToHost, g->stream));
            if (nr > 0 && s->has_region)
                PD_CUDA(cudaMemcpyAsync(hregion.data(), s->d_region, sizeof(double) * (size_t)nr,
                                        cudaMemcpyDeviceToHost, g->stream));
            if (nr > 0 && s->has_conv)
                PD_CUDA(cudaMemcpyAsync(hconv.data(), s->d_conv, sizeof(unsigned long long) * (size_t)nr,
                                        cudaMemcpyDeviceToHost, g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            float ms = 0.f;
            PD_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
            total_ms += ms;

            int64_t fail_k = -1;
            const int fail_mask = s->check_mass ? ~0 : 1;  // step(): only non-finite nodes throw
            for (int64_t k = 0; k < nb; ++k)
                if (hflags[(size_t)k] & fail_mask) {
                    fail_k = k;
                    break;
                }
            // rows of steps before the failing one are valid
            for (int64_t r = 0; r < nr; ++r) {
                const int64_t step_no = row_step[(size_t)r];
                if (fail_k >= 0 && step_no > step0 + j + fail_k) break;
                pd_diag& d = rows[(*n_rows)++];
                d.step = step_no;
                d.time = static_cast<double>(step_no) * c.dt;  // solver.hpp:266
                d.total_mass = hrows[(size_t)r * 3];
                d.min_u = hrows[(size_t)r * 3 + 1];
                d.max_u = hrows[(size_t)r * 3 + 2];
                if (s->has_region) s->region_out.push_back(hregion[(size_t)r]);
                if (s->has_conv) {
                    double v;
                    std::memcpy(&v, &hconv[(size_t)r], sizeof v);
                    s->conv_out.push_back(v);
                }
            }
            if (fail_k < 0) {
                j += nb;
                continue;
            }
            const int code = hflags[(size_t)fail_k];
            const int64_t st = step0 + j + fail_k;
            // undo the swaps of the steps that did not complete: the failing
            // step itself is undone only for a non-finite node (the reference
            // throws before its swap, solver.hpp:250-262)
            int64_t undo = nb - fail_k - ((code & 1) ? 0 : 1);
            if (undo % 2)
                std::swap(g->column_of[(size_t)s->prop_u], g->column_of[(size_t)s->prop_next]);
            if (code & 1) {
                unsigned long long key = 0;
                PD_CUDA(cudaMemcpy(&key, s->d_bad, sizeof key, cudaMemcpyDeviceToHost));
                s->last_ms = total_ms;
                fail(PD_E_NUMERIC, node_message(g, st + 1, key));
            }
            if (code & 4) {  // recorded step with a non-finite total mass
                s->last_ms = total_ms;
                fail(PD_E_NUMERIC, "non-finite total mass at step " + std::to_string(st + 1));
            }
            // code 2: huge values on a non-recorded step: evaluate that step's
            // total mass exactly (same per-chunk order as step()).
            const void* u_now = g->cols[(size_t)g->column_of[(size_t)s->prop_u]];
            launch_chunk_stats(g, u_now, g->d_masks);
            launch_pairwise_finalize(g, g->d_row, nullptr);
            double row[3];
            PD_CUDA(cudaMemcpyAsync(row, g->d_row, sizeof row, cudaMemcpyDeviceToHost, g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            if (!std::isfinite(row[0])) {
                s->last_ms = total_ms;
                fail(PD_E_NUMERIC, "non-finite total mass at step " + std::to_string(st + 1));
            }
            j += fail_k + 1;
        }
        s->last_ms = total_ms;
    });
}

int pd_stepper_step(pd_stepper* s, int64_t step_index, double factor, pd_diag* row) {
    s->check_mass = false;
    int64_t n = 0;
    const int rc = pd_stepper_run(s, step_index, 1, step_index + 1, &factor, row, &n);
    s->check_mass = true;
    return rc;
}

int pd_stepper_enqueue(pd_stepper* s, int64_t step_index, int64_t begin, int64_t end, double factor) {
    return guarded([&] {
        pd_grid* g = s->g;
        if (begin < s->begin || end > s->end || begin > end)
            fail(PD_E_INPUT, "enqueue range outside the stepper's owned range");
        if (end == begin) return;
        DeviceGuard dg(g->device);
        refresh_if_stale(s);
        (void)step_index;  // steps are stream-ordered; errors accumulate in flags[0]
        const void* u = g->cols[(size_t)g->column_of[(size_t)s->prop_u]];
        void* un = g->cols[(size_t)g->column_of[(size_t)s->prop_next]];
        const unsigned nb = (unsigned)(end - begin);
        if (s->peer.on) {
            if (begin != s->begin || end != s->end)
                fail(PD_E_INPUT, "with the fused peer exchange a step covers the whole owned range");
            StepArgs<double> a;
            fill_args<double>(s, a, u, un, factor);
            a.k = 0;
            a.ord0 = begin;
            PD_CUDA(cudaMemsetAsync(s->plan.d_counter, 0, sizeof(int), g->stream));
            launch_peer_step(s, a);
            PD_CUDA(cudaGetLastError());
            s->launches++;
            return;
        }
        if (g->tbytes == 8) {
            StepArgs<double> a;
            fill_args<double>(s, a, u, un, factor);
            a.k = 0;
            a.ord0 = begin;
            if (s->use_march && s->plan.ready && end - begin >= march_min_chunks()) {
                auto& sp = march_sub(g, s->plan, begin, end);
                PD_CUDA(cudaMemsetAsync(sp.d_counter, 0, sizeof(int), g->stream));
                march_launch_sched(g, s->plan, a, s->cfg.reaction_kind, sp.d_stream, sp.n, sp.d_counter);
            } else if (g->dims == 3) {
                ftcs_step_kernel<double, 3, false><<<nb, 512, 0, g->stream>>>(a);
            } else {
                ftcs_step_kernel<double, 2, false><<<nb, 64, 0, g->stream>>>(a);
            }
        } else {
            StepArgs<float> a;
            fill_args<float>(s, a, u, un, factor);
            a.k = 0;
            a.ord0 = begin;
            if (s->use_march && s->plan.ready && end - begin >= march_min_chunks()) {
                auto& sp = march_sub(g, s->plan, begin, end);
                PD_CUDA(cudaMemsetAsync(sp.d_counter, 0, sizeof(int), g->stream));
                march32_launch_sched(g, s->plan, a, s->cfg.reaction_kind, sp.d_stream, sp.n, sp.d_counter);
            } else if (g->dims == 3)
                ftcs_step_kernel<float, 3, false><<<nb, 512, 0, g->stream>>>(a);
            else
                ftcs_step_kernel<float, 2, false><<<nb, 64, 0, g->stream>>>(a);
        }
        PD_CUDA(cudaGetLastError());
        s->launches++;
    });
}

int pd_stepper_sync_words(pd_stepper* s, void** ptr) {
    return guarded([&] {
        DeviceGuard dg(s->g->device);
        if (!s->peer.d_sync) {  // cudaMalloc: exportable through CUDA IPC
            PD_CUDA(cudaMalloc(&s->peer.d_sync, 64));
            PD_CUDA(cudaMemset(s->peer.d_sync, 0, 64));
        }
        *ptr = s->peer.d_sync;
    });
}

int pd_stepper_sync_ipc_handle(pd_stepper* s, void* out) {
    return guarded([&] {
        void* p = nullptr;
        int rc = pd_stepper_sync_words(s, &p);
        if (rc != PD_OK) fail(rc, pd_last_error());
        DeviceGuard dg(s->g->device);
        cudaIpcMemHandle_t h;
        PD_CUDA(cudaIpcGetMemHandle(&h, p));
        std::memcpy(out, &h, sizeof h);
    });
}

int pd_stepper_set_peer(pd_stepper* s, int side, void* const* peer_cols, int n_cols, void* peer_sync,
                        const int32_t* src_ords, const int32_t* dst_ords, int64_t n) {
    return guarded([&] {
        pd_grid* g = s->g;
        if (side != 0 && side != 1) fail(PD_E_INPUT, "side must be 0 (lower) or 1 (upper)");
        if (n_cols != (int)g->cols.size() || n_cols > 16) fail(PD_E_INPUT, "one peer column per grid property");
        if (g->dims != 3 || g->tbytes != 8 || !s->plan.ready)
            fail(PD_E_INPUT, "the fused peer halo push needs the march path (3-D FP64 grid)");
        DeviceGuard dg(g->device);
        void* own = nullptr;
        int rc = pd_stepper_sync_words(s, &own);
        if (rc != PD_OK) fail(rc, pd_last_error());
        if (!s->peer.d_ord) {
            PD_CUDA(pd_malloc(&s->peer.d_ord, sizeof(int32_t) * 2 * (size_t)std::max<int64_t>(1, g->n_chunks)));
            PD_CUDA(cudaMemsetAsync(s->peer.d_ord, 0xff, sizeof(int32_t) * 2 * (size_t)std::max<int64_t>(1, g->n_chunks),
                                    g->stream));
            // [0] timeout flag, [2..3] total wait ns, [4..5] waits (pd_peer.cu)
            PD_CUDA(pd_malloc(&s->peer.d_err, 32));
            PD_CUDA(cudaMemsetAsync(s->peer.d_err, 0, 32, g->stream));
        }
        std::vector<int32_t> ord((size_t)g->n_chunks * 2);
        PD_CUDA(cudaMemcpyAsync(ord.data(), s->peer.d_ord, sizeof(int32_t) * ord.size(), cudaMemcpyDeviceToHost,
                                g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        for (int64_t c = 0; c < g->n_chunks; ++c) ord[(size_t)(2 * c + side)] = -1;
        for (int64_t i = 0; i < n; ++i) {
            if (src_ords[i] < s->begin || src_ords[i] >= s->end)
                fail(PD_E_INPUT, "push source chunk outside the stepper's owned range");
            ord[(size_t)(2 * src_ords[i] + side)] = dst_ords[i];
        }
        PD_CUDA(cudaMemcpyAsync(s->peer.d_ord, ord.data(), sizeof(int32_t) * ord.size(), cudaMemcpyHostToDevice,
                                g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        for (int c = 0; c < n_cols; ++c) s->peer.cols[side][c] = peer_cols[c];
        s->peer.sync[side] = static_cast<unsigned*>(peer_sync);
        s->peer.side[side] = peer_sync != nullptr;
        s->peer.on = s->peer.side[0] || s->peer.side[1];
        s->peer.flags_dirty = true;
    });
}

int pd_stepper_peer_reset(pd_stepper* s) {
    return guarded([&] {
        DeviceGuard dg(s->g->device);
        if (s->peer.d_sync) PD_CUDA(cudaMemset(s->peer.d_sync, 0, 64));
        if (s->peer.d_err) PD_CUDA(cudaMemset(s->peer.d_err, 0, 32));
        s->peer.epoch = 0;
        PD_CUDA(cudaDeviceSynchronize());
    });
}

int pd_stepper_peer_stats(pd_stepper* s, uint64_t* wait_ns, int64_t* waits) {
    return guarded([&] {
        unsigned long long h[2] = {0, 0};
        if (s->peer.d_err) {
            DeviceGuard dg(s->g->device);
            PD_CUDA(cudaStreamSynchronize(s->g->stream));
            PD_CUDA(cudaMemcpy(h, reinterpret_cast<unsigned long long*>(s->peer.d_err) + 1, sizeof h,
                               cudaMemcpyDeviceToHost));
        }
        if (wait_ns) *wait_ns = h[0];
        if (waits) *waits = (int64_t)h[1];
    });
}

int pd_stepper_swap(pd_stepper* s) {
    std::swap(s->g->column_of[(size_t)s->prop_u], s->g->column_of[(size_t)s->prop_next]);
    return PD_OK;
}

int pd_stepper_status(pd_stepper* s, int64_t step_number) {
    return guarded([&] {
        pd_grid* g = s->g;
        DeviceGuard dg(g->device);
        int f = 0;
        PD_CUDA(cudaMemcpyAsync(&f, s->d_flags, sizeof f, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        if (s->peer.d_err) {
            int e = 0;
            PD_CUDA(cudaMemcpy(&e, s->peer.d_err, sizeof e, cudaMemcpyDeviceToHost));
            if (e) fail(PD_E_CUDA, "peer halo exchange: a neighbour's step counter did not advance within 30 s");
        }
        if (!(f & 1)) {
            PD_CUDA(cudaMemsetAsync(s->d_flags, 0, sizeof(int), g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            return;
        }
        unsigned long long key = 0;
        PD_CUDA(cudaMemcpy(&key, s->d_bad, sizeof key, cudaMemcpyDeviceToHost));
        PD_CUDA(cudaMemsetAsync(s->d_flags, 0, sizeof(int), g->stream));
        PD_CUDA(cudaMemsetAsync(s->d_bad, 0xff, sizeof(unsigned long long), g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        fail(PD_E_NUMERIC, node_message(g, step_number, key));
    });
}

int pd_stepper_partials(pd_stepper* s, double* dev_mass, double* dev_min, double* dev_max) {
    return guarded([&] {
        pd_grid* g = s->g;
        DeviceGuard dg(g->device);
        const void* u = g->cols[(size_t)g->column_of[(size_t)s->prop_u]];
        launch_chunk_stats(g, u, g->d_masks);
        const int64_t n = s->end - s->begin;
        if (n > 0) {
            double* dst[3] = {dev_mass, dev_min, dev_max};
            for (int k = 0; k < 3; ++k)
                PD_CUDA(cudaMemcpyAsync(dst[k], g->red.part[k] + s->begin, sizeof(double) * (size_t)n,
                                        cudaMemcpyDeviceToDevice, g->stream));
        }
    });
}

int pd_reduce_partials(pd_grid* g, const double* dev_mass, const double* dev_min, const double* dev_max, int64_t n,
                       double* row) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const int64_t cap = std::max<int64_t>(1, (n + 1023) / 1024);
        double* scratch = nullptr;
        PD_CUDA(pd_malloc(&scratch, sizeof(double) * (size_t)(6 * cap + 3)));
        const cudaError_t e0 = [&] {
            launch_pairwise_arrays(g, dev_mass, dev_min, dev_max, n, scratch + 6 * cap, scratch);
            return cudaMemcpyAsync(row, scratch + 6 * cap, 3 * sizeof(double), cudaMemcpyDeviceToHost, g->stream);
        }();
        const cudaError_t e1 = cudaStreamSynchronize(g->stream);
        pd_free(scratch);
        PD_CUDA(e0);
        PD_CUDA(e1);
    });
}

int pd_stepper_set_region(pd_stepper* s, const int64_t* lo, const int64_t* hi) {
    return guarded([&] {
        if (!lo || !hi) {
            s->has_region = false;
            return;
        }
        check_box(s->g, lo, hi);
        for (int a = 0; a < 3; ++a) {
            s->rlo[a] = a < s->g->dims ? lo[a] : 0;
            s->rhi[a] = a < s->g->dims ? hi[a] : 1;
        }
        s->has_region = true;
    });
}

int pd_stepper_region_sums(const pd_stepper* s, double* out, int64_t cap, int64_t* n) {
    *n = (int64_t)s->region_out.size();
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n); ++i) out[i] = s->region_out[(size_t)i];
    return PD_OK;
}

int pd_stepper_set_convergence(pd_stepper* s, int on) {
    s->has_conv = on != 0;
    return PD_OK;
}

int pd_stepper_convergence(const pd_stepper* s, double* out, int64_t cap, int64_t* n) {
    *n = (int64_t)s->conv_out.size();
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n); ++i) out[i] = s->conv_out[(size_t)i];
    return PD_OK;
}

int pd_stepper_plane_flux(pd_stepper* s, int axis, int64_t layer, double* face_sum, double* flux,
                          int64_t* faces) {
    return guarded([&] {
        pd_grid* g = s->g;
        if (axis < 0 || axis >= g->dims) fail(PD_E_INPUT, "flux axis out of range");
        if (layer < 0 || layer + 1 >= g->size[axis]) fail(PD_E_INPUT, "flux plane outside the box interior");
        DeviceGuard dg(g->device);
        refresh_if_stale(s);
        const void* u = g->cols[(size_t)g->column_of[(size_t)s->prop_u]];
        const void* d = g->cols[(size_t)g->column_of[(size_t)s->prop_d]];
        int64_t nf = 0;
        const double sum = plane_face_sum(g, u, d, s->d_fluid, s->d_nbr, axis, layer, &nf);
        // Fick's law across the faces: F = -sum dh (u_{L+1} - u_L) / h_axis * A_face
        double area = 1.0;
        for (int a = 0; a < g->dims; ++a)
            if (a != axis) area *= g->spacing[a];
        if (face_sum) *face_sum = sum;
        if (flux) *flux = -sum / g->spacing[axis] * area;
        if (faces) *faces = nf;
    });
}

int pd_stepper_last_ms(const pd_stepper* s, double* ms) {
    *ms = s->last_ms;
    return PD_OK;
}

int pd_stepper_launch_count(const pd_stepper* s, int64_t* launches) {
    *launches = s->launches;
    return PD_OK;
}

}  // extern "C"
