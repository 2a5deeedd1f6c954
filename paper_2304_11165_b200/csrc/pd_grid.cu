// Device sparse block grid store (north_star subsystem 1) and its exact
// chunk-ordered reductions.
//
// Layout in HBM (chunk-ordinal-major SoA, the reference's per-chunk
// property-major payload turned inside out so each property is one
// contiguous array; sparse_block_grid.hpp:40-56,180-187):
//   keys    int32 [n_chunks][Dims]          ascending chunk linear index
//   masks   uint64[n_chunks][V/64]          allocation bitmask
//   table   int32 [prod(ceil(size/8))]      linear index -> ordinal, -1 absent
//   column  T     [n_chunks][V]             one array per physical column
#include <cub/device/device_scan.cuh>

#include <cmath>
#include <cstring>
#include <limits>

#include "pd_internal.cuh"
#include "pd_libm_exp.h"

namespace pdb {

namespace {
thread_local std::string t_err;
}
void set_error(const std::string& msg) { t_err = msg; }

int device_of(const pd_grid* g) { return g->device; }

// ---------------------------------------------------------------------------
// chunk table
// ---------------------------------------------------------------------------

template <int D>
__global__ void build_table_kernel(const int32_t* __restrict__ keys, int64_t n,
                                   int64_t cc0, int64_t cc1, int32_t* __restrict__ table) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t lin = keys[i * D + D - 1];
    if (D == 3) lin = lin * cc1 + keys[i * D + 1];
    lin = lin * cc0 + keys[i * D + 0];
    table[lin] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// per-chunk statistics: sequential active-offset sum (solver.hpp:165-168) and
// the std::min / std::max folds (solver.hpp:290-297) as left-preference trees
// (the fold keeps the earliest of equal values; NaN never enters the fold)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double min_left(double l, double r) { return (r < l) ? r : l; }
__device__ __forceinline__ double max_left(double l, double r) { return (l < r) ? r : l; }

// One thread per chunk: the reference's sequential per-chunk mass over the
// active offsets in ascending order, and the std::min / std::max folds in the
// same order (the first of equal values is kept; NaN never enters the fold).
// A thread walks its own slab; consecutive offsets share L1 lines.
template <class T, int D>
__global__ void __launch_bounds__(128)
    chunk_stats_kernel(const T* __restrict__ x, const uint64_t* __restrict__ masks, int64_t n,
                       double* __restrict__ mass, double* __restrict__ mn, double* __restrict__ mx) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const T* xs = x + i * V;
    double acc = 0.0, lo = INFINITY, hi = -INFINITY;
    for (int w = 0; w < W; ++w) {
        uint64_t bits = __ldg(&masks[i * W + w]);
        while (bits) {
            const int b = __ffsll((long long)bits) - 1;
            bits &= bits - 1;
            const double v = (double)__ldg(&xs[w * 64 + b]);
            acc += v;
            if (!isnan(v)) {
                lo = min_left(lo, v);
                hi = max_left(hi, v);
            }
        }
    }
    mass[i] = acc;
    mn[i] = lo;
    mx[i] = hi;
}

// pairwise_sum (parallel.hpp:68-84): element j of level L covers leaves
// [j*2^L, min((j+1)*2^L, n)), so aligned blocks of 1024 leaves reduce
// independently and their results are the leaves of the next pass.
constexpr int kPairBlock = 1024;

__global__ void __launch_bounds__(kPairBlock)
    pairwise_pass_kernel(const double* __restrict__ m, const double* __restrict__ a,
                         const double* __restrict__ b, int64_t n, double* __restrict__ om,
                         double* __restrict__ oa, double* __restrict__ ob,
                         double* __restrict__ row, double cell_volume, int* flags) {
    __shared__ double s[kPairBlock], smn[kPairBlock], smx[kPairBlock];
    const int tid = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * kPairBlock;
    const int cnt = (int)((n - base) < kPairBlock ? (n - base) : kPairBlock);
    s[tid] = tid < cnt ? m[base + tid] : 0.0;
    smn[tid] = tid < cnt ? a[base + tid] : INFINITY;
    smx[tid] = tid < cnt ? b[base + tid] : -INFINITY;
    __syncthreads();
    for (int st = 1; st < kPairBlock; st <<= 1) {
        if ((tid & (2 * st - 1)) == 0 && tid + st < cnt) {
            s[tid] = s[tid] + s[tid + st];
            smn[tid] = min_left(smn[tid], smn[tid + st]);
            smx[tid] = max_left(smx[tid], smx[tid + st]);
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (row) {
            const double total = s[0] * cell_volume;
            row[0] = total;
            row[1] = smn[0];
            row[2] = smx[0];
            if (flags && !isfinite(total)) atomicOr(flags, 4);
        } else {
            om[blockIdx.x] = s[0];
            oa[blockIdx.x] = smn[0];
            ob[blockIdx.x] = smx[0];
        }
    }
}

__global__ void empty_row_kernel(double* row) {
    row[0] = 0.0;
    row[1] = INFINITY;
    row[2] = -INFINITY;
}

template <class T, int D>
__global__ void __launch_bounds__(Geo<D>::V)
    chunk_max_kernel(const T* __restrict__ x, const uint64_t* __restrict__ masks,
                     double* __restrict__ mass, double* __restrict__ mn,
                     double* __restrict__ mx) {
    // max_diffusivity: same fold as smx above; mass/mn are filled with the
    // identities so the pairwise finalize can be reused unchanged.
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    __shared__ double smx[V];
    const int64_t i = blockIdx.x;
    const int off = threadIdx.x;
    const bool act = (masks[i * W + (off >> 6)] >> (off & 63)) & 1u;
    const double v = act ? (double)x[i * V + off] : -INFINITY;
    smx[off] = (act && !isnan(v)) ? v : -INFINITY;
    __syncthreads();
    for (int s = 1; s < V; s <<= 1) {
        if ((off & (2 * s - 1)) == 0) smx[off] = max_left(smx[off], smx[off + s]);
        __syncthreads();
    }
    if (off == 0) {
        mass[i] = 0.0;
        mn[i] = INFINITY;
        mx[i] = smx[0];
    }
}

template <class T, int D>
__global__ void __launch_bounds__(Geo<D>::V)
    fill_hash_kernel(T* __restrict__ x, const uint64_t* __restrict__ masks,
                     const int32_t* __restrict__ keys, int64_t s0, int64_t s1, uint64_t seed) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t i = blockIdx.x;
    const int off = threadIdx.x;
    if (!((masks[i * W + (off >> 6)] >> (off & 63)) & 1u)) return;
    const int64_t gx = ((int64_t)keys[i * D] << 3) | (off & 7);
    const int64_t gy = ((int64_t)keys[i * D + 1] << 3) | ((off >> 3) & 7);
    int64_t flat = gy * s0 + gx;
    if (D == 3) {
        const int64_t gz = ((int64_t)keys[i * D + 2] << 3) | ((off >> 6) & 7);
        flat = (gz * s1 + gy) * s0 + gx;
    }
    // hash_unit_value (config.hpp:558-564)
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * ((uint64_t)flat + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    x[i * V + off] = (T)((double)(z >> 11) * 0x1.0p-53);
}

template <class T, int D>
__global__ void __launch_bounds__(Geo<D>::V)
    fill_const_kernel(T* __restrict__ x, const uint64_t* __restrict__ masks, double value) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t i = blockIdx.x;
    const int off = threadIdx.x;
    if ((masks[i * W + (off >> 6)] >> (off & 63)) & 1u) x[i * V + off] = (T)value;
}

// smooth_diffusion_coefficient (geometry.hpp:182-187) on active nodes
// (populate_diffusion_channel, geometry.hpp:191-206), with the reference's
// libm exp restated bit for bit (pd_libm_exp.h): D is the reference's bits.
template <class T, int D>
__global__ void __launch_bounds__(Geo<D>::V)
    populate_d_kernel(const T* __restrict__ phi, T* __restrict__ d,
                      const uint64_t* __restrict__ masks, double dmin, double dmax, double g1,
                      double g2) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t i = blockIdx.x;
    const int off = threadIdx.x;
    if (!((masks[i * W + (off >> 6)] >> (off & 63)) & 1u)) return;
    const double p = (double)phi[i * V + off];
    d[i * V + off] = (T)pd_smooth_diffusion(p, dmin, dmax, g1, g2);
}

// ---------------------------------------------------------------------------
// sphere-pack geometry build (build_sparse_grid on field_from(pack.fluid_sdf),
// geometry.hpp:148-176, synthetic.hpp:32-40)
// ---------------------------------------------------------------------------

constexpr int kMaxCand = 1024;

struct PackArgs {
    int64_t size[3];
    double spacing[3], origin[3];
    int64_t cc[3];
    int64_t rlo[3], rext[3];  // chunk-key region [rlo, rlo+rext)
    const double* centers;
    const double* radii;
    int64_t n_spheres;
};

// Candidate spheres of one chunk: every sphere whose lower bound over the
// chunk's node box can reach the chunk's best upper bound. min() is exact, so
// any candidate superset of the per-node argmin reproduces fluid_sdf bitwise.
__device__ int gather_candidates(const PackArgs& p, const int64_t k[3], int* cand,
                                 int* n_cand, double* s_ub) {
    const int tid = threadIdx.x;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        const int64_t i0 = k[a] * 8;
        const int64_t i1 = (k[a] * 8 + 7) < (p.size[a] - 1) ? (k[a] * 8 + 7) : (p.size[a] - 1);
        lo[a] = p.origin[a] + (double)i0 * p.spacing[a];
        hi[a] = p.origin[a] + (double)i1 * p.spacing[a];
    }
    // pass 1: best upper bound (max distance to the box) over spheres
    double ub = INFINITY;
    for (int64_t s = tid; s < p.n_spheres; s += blockDim.x) {
        double far2 = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double c = p.centers[s * 3 + a];
            const double f = fmax(fabs(c - lo[a]), fabs(c - hi[a]));
            far2 += f * f;
        }
        ub = fmin(ub, sqrt(far2) - p.radii[s]);
    }
    for (int o = 16; o; o >>= 1) ub = fmin(ub, __shfl_xor_sync(0xffffffffu, ub, o));
    if ((tid & 31) == 0) s_ub[tid >> 5] = ub;
    __syncthreads();
    if (tid == 0) {
        double u = INFINITY;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) u = fmin(u, s_ub[w]);
        s_ub[0] = u;
        *n_cand = 0;
    }
    __syncthreads();
    ub = s_ub[0];
    const double slack = 1e-9 * (1.0 + fabs(ub));
    for (int64_t s = tid; s < p.n_spheres; s += blockDim.x) {
        double near2 = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double c = p.centers[s * 3 + a];
            const double q = fmin(fmax(c, lo[a]), hi[a]);
            near2 += (c - q) * (c - q);
        }
        if (sqrt(near2) - p.radii[s] <= ub + slack) {
            const int slot = atomicAdd(n_cand, 1);
            if (slot < kMaxCand) cand[slot] = (int)s;
        }
    }
    __syncthreads();
    return *n_cand;
}

// fluid_sdf at node (gx, gy, gz): min over spheres of |x - c| - r, the
// squared distance accumulated axis by axis from 0.0 (synthetic.hpp:35-37).
__device__ __forceinline__ double sdf_at(const PackArgs& p, int64_t gx, int64_t gy, int64_t gz,
                                         const int* cand, int n_cand) {
    const double x0 = p.origin[0] + (double)gx * p.spacing[0];
    const double x1 = p.origin[1] + (double)gy * p.spacing[1];
    const double x2 = p.origin[2] + (double)gz * p.spacing[2];
    double best = INFINITY;
    const bool all = n_cand > kMaxCand;
    const int64_t n = all ? p.n_spheres : n_cand;
    for (int64_t q = 0; q < n; ++q) {
        const int64_t s = all ? q : cand[q];
        const double d0 = x0 - p.centers[s * 3 + 0];
        const double d1 = x1 - p.centers[s * 3 + 1];
        const double d2 = x2 - p.centers[s * 3 + 2];
        double r2 = 0.0;
        r2 += d0 * d0;
        r2 += d1 * d1;
        r2 += d2 * d2;
        const double v = sqrt(r2) - p.radii[s];
        best = (v < best) ? v : best;
    }
    return best;
}

template <class T>
__global__ void __launch_bounds__(512)
    pack_mask_kernel(PackArgs p, T lo_t, T hi_t, uint64_t* __restrict__ slot_masks,
                     int32_t* __restrict__ slot_flag) {
    __shared__ int cand[kMaxCand];
    __shared__ int n_cand;
    __shared__ double s_ub[16];
    const int64_t slot = blockIdx.x;
    int64_t k[3];
    k[0] = p.rlo[0] + slot % p.rext[0];
    k[1] = p.rlo[1] + (slot / p.rext[0]) % p.rext[1];
    k[2] = p.rlo[2] + slot / (p.rext[0] * p.rext[1]);
    const int nc = gather_candidates(p, k, cand, &n_cand, s_ub);
    const int off = threadIdx.x;
    const int64_t gx = k[0] * 8 + (off & 7), gy = k[1] * 8 + ((off >> 3) & 7),
                  gz = k[2] * 8 + (off >> 6);
    bool act = false;
    if (gx < p.size[0] && gy < p.size[1] && gz < p.size[2]) {
        const T phi = (T)sdf_at(p, gx, gy, gz, cand, nc);
        act = phi > lo_t && phi < hi_t;
    }
    const unsigned b = __ballot_sync(0xffffffffu, act);
    __shared__ unsigned words[16];
    if ((off & 31) == 0) words[off >> 5] = b;
    __syncthreads();
    if (off < 8) {
        const uint64_t w = (uint64_t)words[2 * off] | ((uint64_t)words[2 * off + 1] << 32);
        slot_masks[slot * 8 + off] = w;
    }
    if (off == 0) {
        int any = 0;
        for (int w = 0; w < 16; ++w) any |= words[w] != 0;
        slot_flag[slot] = any;
    }
}

template <class T>
__global__ void __launch_bounds__(512)
    pack_fill_kernel(PackArgs p, const uint64_t* __restrict__ slot_masks,
                     const int32_t* __restrict__ slot_flag, const int32_t* __restrict__ ordinal,
                     int32_t* __restrict__ keys, uint64_t* __restrict__ masks,
                     int32_t* __restrict__ table, T* __restrict__ phi_col) {
    __shared__ int cand[kMaxCand];
    __shared__ int n_cand;
    __shared__ double s_ub[16];
    const int64_t slot = blockIdx.x;
    if (!slot_flag[slot]) return;
    const int64_t i = ordinal[slot];
    int64_t k[3];
    k[0] = p.rlo[0] + slot % p.rext[0];
    k[1] = p.rlo[1] + (slot / p.rext[0]) % p.rext[1];
    k[2] = p.rlo[2] + slot / (p.rext[0] * p.rext[1]);
    const int nc = gather_candidates(p, k, cand, &n_cand, s_ub);
    const int off = threadIdx.x;
    if (off < 3) keys[i * 3 + off] = (int32_t)k[off];
    if (off < 8) masks[i * 8 + off] = slot_masks[slot * 8 + off];
    if (off == 0) table[(k[2] * p.cc[1] + k[1]) * p.cc[0] + k[0]] = (int32_t)i;
    const bool act = (slot_masks[slot * 8 + (off >> 6)] >> (off & 63)) & 1u;
    T v = 0;
    if (act) {
        const int64_t gx = k[0] * 8 + (off & 7), gy = k[1] * 8 + ((off >> 3) & 7),
                      gz = k[2] * 8 + (off >> 6);
        v = (T)sdf_at(p, gx, gy, gz, cand, nc);
    }
    phi_col[i * 512 + off] = v;
}

__global__ void popcount_kernel(const uint64_t* __restrict__ masks, int64_t n_words,
                                unsigned long long* out) {
    unsigned long long c = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_words;
         w += (int64_t)gridDim.x * blockDim.x)
        c += __popcll(masks[w]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// one-node face plane of a chunk: side 0 -> coordinate 0, side 1 -> 7
template <class T, int D>
__global__ void face_pack_kernel(const T* __restrict__ col, const int32_t* __restrict__ ords,
                                 int64_t n, int face, T* __restrict__ out, bool unpack,
                                 const T* __restrict__ in, T* __restrict__ dst) {
    constexpr int V = Geo<D>::V, FA = Geo<D>::FA;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * FA) return;
    const int64_t c = t / FA;
    const int p = (int)(t % FA);
    const int ax = face >> 1, side = face & 1;
    int q[3] = {0, 0, 0};
    int b = 0;
    for (int bx = 0; bx < D; ++bx) {
        if (bx == ax) continue;
        q[bx] = b == 0 ? (p & 7) : (p >> 3);
        ++b;
    }
    q[ax] = side ? 7 : 0;
    const int off = q[0] | (q[1] << 3) | (D == 3 ? (q[2] << 6) : 0);
    const int64_t j = ords[c];
    if (unpack)
        dst[j * V + off] = in[t];
    else
        out[t] = col[j * V + off];
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------

template <class F>
void dispatch(const pd_grid* g, F&& f) {
    if (g->tbytes == 8 && g->dims == 3)
        f((double*)nullptr, std::integral_constant<int, 3>{});
    else if (g->tbytes == 8)
        f((double*)nullptr, std::integral_constant<int, 2>{});
    else if (g->dims == 3)
        f((float*)nullptr, std::integral_constant<int, 3>{});
    else
        f((float*)nullptr, std::integral_constant<int, 2>{});
}

void ensure_scratch(pd_grid* g) {
    const int64_t need = g->n_chunks > 0 ? g->n_chunks : 1;
    if (g->red.cap >= need) return;
    for (int k = 0; k < 3; ++k) {
        if (g->red.part[k]) pd_free(g->red.part[k]);
        if (g->red.tmp_a[k]) pd_free(g->red.tmp_a[k]);
        if (g->red.tmp_b[k]) pd_free(g->red.tmp_b[k]);
        const int64_t nb = (need + kPairBlock - 1) / kPairBlock;
        PD_CUDA(pd_malloc(&g->red.part[k], sizeof(double) * need));
        PD_CUDA(pd_malloc(&g->red.tmp_a[k], sizeof(double) * nb));
        PD_CUDA(pd_malloc(&g->red.tmp_b[k], sizeof(double) * nb));
    }
    g->red.cap = need;
}

void launch_chunk_stats(pd_grid* g, const void* col, const uint64_t* masks) {
    ensure_scratch(g);
    if (g->n_chunks == 0) return;
    dispatch(g, [&](auto tp, auto dc) {
        using T = std::remove_pointer_t<decltype(tp)>;
        constexpr int D = decltype(dc)::value;
        chunk_stats_kernel<T, D><<<(unsigned)((g->n_chunks + 127) / 128), 128, 0, g->stream>>>(
            (const T*)col, masks, g->n_chunks, g->red.part[0], g->red.part[1], g->red.part[2]);
    });
    PD_CUDA(cudaGetLastError());
}

void launch_chunk_max(pd_grid* g, const void* col) {
    ensure_scratch(g);
    if (g->n_chunks == 0) return;
    dispatch(g, [&](auto tp, auto dc) {
        using T = std::remove_pointer_t<decltype(tp)>;
        constexpr int D = decltype(dc)::value;
        chunk_max_kernel<T, D><<<(unsigned)g->n_chunks, Geo<D>::V, 0, g->stream>>>(
            (const T*)col, g->d_masks, g->red.part[0], g->red.part[1], g->red.part[2]);
    });
    PD_CUDA(cudaGetLastError());
}

void launch_pairwise_finalize(pd_grid* g, double* dst, int* flags, int64_t begin, int64_t count) {
    ensure_scratch(g);
    if (count < 0) count = g->n_chunks - begin;
    if (count <= 0) {
        empty_row_kernel<<<1, 1, 0, g->stream>>>(dst);
        PD_CUDA(cudaGetLastError());
        return;
    }
    const double* in[3] = {g->red.part[0] + begin, g->red.part[1] + begin, g->red.part[2] + begin};
    int64_t n = count;
    bool use_a = true;
    while (true) {
        const int64_t nb = (n + kPairBlock - 1) / kPairBlock;
        double** out = use_a ? g->red.tmp_a : g->red.tmp_b;
        pairwise_pass_kernel<<<(unsigned)nb, kPairBlock, 0, g->stream>>>(
            in[0], in[1], in[2], n, out[0], out[1], out[2], nb == 1 ? dst : nullptr,
            g->cell_volume, flags);
        PD_CUDA(cudaGetLastError());
        if (nb == 1) break;
        for (int k = 0; k < 3; ++k) in[k] = out[k];
        n = nb;
        use_a = !use_a;
    }
}

void launch_pairwise_arrays(pd_grid* g, const double* m, const double* a, const double* b, int64_t n,
                            double* dst, double* scratch) {
    // scratch: 6 * ceil(n / kPairBlock) doubles (two ping-pong triples)
    if (n <= 0) {
        empty_row_kernel<<<1, 1, 0, g->stream>>>(dst);
        PD_CUDA(cudaGetLastError());
        return;
    }
    const int64_t cap = (n + kPairBlock - 1) / kPairBlock;
    double* ta[3] = {scratch, scratch + cap, scratch + 2 * cap};
    double* tb[3] = {scratch + 3 * cap, scratch + 4 * cap, scratch + 5 * cap};
    const double* in[3] = {m, a, b};
    bool use_a = true;
    while (true) {
        const int64_t nb = (n + kPairBlock - 1) / kPairBlock;
        double** out = use_a ? ta : tb;
        pairwise_pass_kernel<<<(unsigned)nb, kPairBlock, 0, g->stream>>>(
            in[0], in[1], in[2], n, out[0], out[1], out[2], nb == 1 ? dst : nullptr, g->cell_volume, nullptr);
        PD_CUDA(cudaGetLastError());
        if (nb == 1) break;
        for (int k = 0; k < 3; ++k) in[k] = out[k];
        n = nb;
        use_a = !use_a;
    }
}

void check_prop(const pd_grid* g, int prop) {
    if (prop < 0 || prop >= (int)g->column_of.size())
        fail(PD_E_PROPERTY, "unknown property index " + std::to_string(prop));
}

void* col_ptr(pd_grid* g, int prop) {
    check_prop(g, prop);
    return g->cols[(size_t)g->column_of[(size_t)prop]];
}

size_t slab_bytes(const pd_grid* g) {
    return (size_t)g->n_chunks * (size_t)g->V * (size_t)g->tbytes;
}

void alloc_columns(pd_grid* g, int n_props) {
    g->cols.assign((size_t)n_props, nullptr);
    g->column_of.resize((size_t)n_props);
    for (int p = 0; p < n_props; ++p) {
        g->column_of[(size_t)p] = p;
        if (g->n_chunks > 0) {
            PD_CUDA(pd_malloc(&g->cols[(size_t)p], slab_bytes(g)));
            PD_CUDA(cudaMemsetAsync(g->cols[(size_t)p], 0, slab_bytes(g), g->stream));
        }
    }
}

void init_geometry(pd_grid* g, int dims, int tbytes, const int64_t* size, const double* spacing,
                   int device) {
    if (dims != 2 && dims != 3) fail(PD_E_INPUT, "only 2-D and 3-D grids are supported");
    if (tbytes != 4 && tbytes != 8) fail(PD_E_INPUT, "scalar_bytes must be 4 or 8");
    g->dims = dims;
    g->tbytes = tbytes;
    g->V = dims == 3 ? 512 : 64;
    g->W = g->V / 64;
    g->device = device;
    g->cell_volume = 1.0;
    g->table_size = 1;
    for (int a = 0; a < dims; ++a) {
        if (size[a] < 1) fail(PD_E_INPUT, "grid size must be >= 1 along every axis");
        if (!(spacing[a] > 0.0)) fail(PD_E_INPUT, "grid spacing must be > 0 along every axis");
        g->size[a] = size[a];
        g->spacing[a] = spacing[a];
        g->cell_volume *= spacing[a];  // grid_geometry.hpp:105-109
        g->cc[a] = (size[a] + 7) / 8;
        g->table_size *= g->cc[a];
    }
}

void count_active(pd_grid* g) {
    unsigned long long* d_cnt = nullptr;
    PD_CUDA(pd_malloc(&d_cnt, sizeof(unsigned long long)));
    PD_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), g->stream));
    const int64_t words = g->n_chunks * g->W;
    if (words > 0) {
        const int blocks = (int)std::min<int64_t>(148 * 8, (words + 255) / 256);
        popcount_kernel<<<blocks, 256, 0, g->stream>>>(g->d_masks, words, d_cnt);
        PD_CUDA(cudaGetLastError());
    }
    unsigned long long h = 0;
    PD_CUDA(cudaMemcpyAsync(&h, d_cnt, sizeof h, cudaMemcpyDeviceToHost, g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    pd_free(d_cnt);
    g->active = (int64_t)h;
}

}  // namespace pdb

using namespace pdb;


namespace pdb {
// per chunk layer (z): allocated chunks and active nodes of a slot-mask pass
__global__ void layer_work_kernel(const uint64_t* __restrict__ slot_masks, const int32_t* __restrict__ slot_flag,
                                  int64_t per_layer, int64_t layers, unsigned long long* __restrict__ chunks,
                                  unsigned long long* __restrict__ active, unsigned long long* __restrict__ full) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= per_layer * layers) return;
    if (!slot_flag[slot]) return;
    const int64_t z = slot / per_layer;
    unsigned long long a = 0;
    for (int w = 0; w < 8; ++w) a += (unsigned long long)__popcll(slot_masks[slot * 8 + w]);
    atomicAdd(chunks + z, 1ull);
    atomicAdd(active + z, a);
    if (a == 512) atomicAdd(full + z, 1ull);
}
}  // namespace pdb

extern "C" {

const char* pd_last_error(void) { return t_err.c_str(); }

int pd_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

const char* pd_version(void) {
    return "porediff_b200 0.1 (sm_100a; fp64 parity + fp32; fused FTCS sparse-block step)";
}

int pd_grid_create(int dims, int scalar_bytes, const int64_t* size, const double* spacing,
                   int64_t n_chunks, const int32_t* keys, const uint64_t* masks, int n_props,
                   int device, pd_grid** out) {
    return guarded([&] {
        *out = nullptr;
        if (n_props < 1) fail(PD_E_INPUT, "sparse grid needs at least one property");
        if (n_chunks < 0) fail(PD_E_INPUT, "negative chunk count");
        auto* g = new pd_grid();
        try {
            init_geometry(g, dims, scalar_bytes, size, spacing, device);
            if (n_chunks > g->table_size)
                fail(PD_E_INPUT, "more chunks than the chunk table holds");
            // keys must be inside the chunk grid and strictly ascending in
            // linear index (sparse_block_grid.hpp:105-109,283-293)
            int64_t prev = -1;
            for (int64_t i = 0; i < n_chunks; ++i) {
                int64_t lin = 0;
                for (int a = dims - 1; a >= 0; --a) {
                    const int32_t k = keys[i * dims + a];
                    if (k < 0 || k >= g->cc[a]) fail(PD_E_BOUNDS, "chunk key outside grid");
                    lin = lin * g->cc[a] + k;
                }
                if (lin <= prev) fail(PD_E_INPUT, "chunk keys must be strictly ascending in linear index");
                prev = lin;
            }
            DeviceGuard dg(device);
            PD_CUDA(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
            g->stream = g->own_stream;
            g->n_chunks = n_chunks;
            PD_CUDA(pd_malloc(&g->d_table, sizeof(int32_t) * (size_t)g->table_size));
            PD_CUDA(cudaMemsetAsync(g->d_table, 0xff, sizeof(int32_t) * (size_t)g->table_size,
                                    g->stream));
            PD_CUDA(pd_malloc(&g->d_row, sizeof(double) * 4));
            if (n_chunks > 0) {
                PD_CUDA(pd_malloc(&g->d_keys, sizeof(int32_t) * (size_t)(n_chunks * dims)));
                PD_CUDA(pd_malloc(&g->d_masks, sizeof(uint64_t) * (size_t)(n_chunks * g->W)));
                PD_CUDA(cudaMemcpyAsync(g->d_keys, keys, sizeof(int32_t) * (size_t)(n_chunks * dims),
                                        cudaMemcpyHostToDevice, g->stream));
                PD_CUDA(cudaMemcpyAsync(g->d_masks, masks,
                                        sizeof(uint64_t) * (size_t)(n_chunks * g->W),
                                        cudaMemcpyHostToDevice, g->stream));
                const int blocks = (int)((n_chunks + 255) / 256);
                if (dims == 3)
                    build_table_kernel<3><<<blocks, 256, 0, g->stream>>>(g->d_keys, n_chunks, g->cc[0],
                                                                         g->cc[1], g->d_table);
                else
                    build_table_kernel<2><<<blocks, 256, 0, g->stream>>>(g->d_keys, n_chunks, g->cc[0],
                                                                         g->cc[1], g->d_table);
                PD_CUDA(cudaGetLastError());
            }
            alloc_columns(g, n_props);
            count_active(g);
            ensure_scratch(g);
        } catch (...) {
            pd_grid_destroy(g);
            throw;
        }
        *out = g;
    });
}

int pd_grid_destroy(pd_grid* g) {
    if (!g) return PD_OK;
    grid_release(g);
    return PD_OK;
}

extern "C++" void grid_release(pd_grid* g) {
    if (--g->refs > 0) return;
    {
        DeviceGuard dg(g->device);
        if (g->stream) cudaStreamSynchronize(g->stream);
        if (g->own_stream) cudaStreamSynchronize(g->own_stream);
        for (size_t i = 0; i < g->cols.size(); ++i) {
            if (i < g->col_ipc.size() && g->col_ipc[i])
                cudaFree(g->cols[i]);
            else
                pd_free(g->cols[i]);
        }
        pd_free(g->d_keys);
        pd_free(g->d_masks);
        pd_free(g->d_table);
        pd_free(g->d_row);
        for (int k = 0; k < 3; ++k) {
            pd_free(g->red.part[k]);
            pd_free(g->red.tmp_a[k]);
            pd_free(g->red.tmp_b[k]);
        }
        if (g->own_stream) cudaStreamDestroy(g->own_stream);
    }
    delete g;
}

int pd_grid_upload(pd_grid* g, int prop, const void* host_slabs) {
    return guarded([&] {
        note_write(g, prop);
        DeviceGuard dg(g->device);
        void* c = col_ptr(g, prop);
        if (g->n_chunks == 0) return;
        PD_CUDA(cudaMemcpyAsync(c, host_slabs, slab_bytes(g), cudaMemcpyHostToDevice, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_grid_upload_device(pd_grid* g, int prop, const void* dev_slabs) {
    return guarded([&] {
        note_write(g, prop);
        DeviceGuard dg(g->device);
        void* c = col_ptr(g, prop);
        if (g->n_chunks == 0) return;
        PD_CUDA(cudaMemcpyAsync(c, dev_slabs, slab_bytes(g), cudaMemcpyDeviceToDevice, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_grid_download(pd_grid* g, int prop, void* host_slabs) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        void* c = col_ptr(g, prop);
        if (g->n_chunks == 0) return;
        PD_CUDA(cudaMemcpyAsync(host_slabs, c, slab_bytes(g), cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_grid_set_stream(pd_grid* g, void* stream) {
    return guarded([&] { g->stream = stream ? (cudaStream_t)stream : g->own_stream; });
}

static int face_io(pd_grid* g, int prop, const int32_t* ords, int64_t n, int face, void* out,
                   const void* in, bool unpack) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        void* col = col_ptr(g, prop);
        if (face < 0 || face >= 2 * g->dims) fail(PD_E_INPUT, "face index out of range");
        if (n <= 0) return;
        const int fa = g->dims == 3 ? 64 : 8;
        const unsigned blocks = (unsigned)((n * fa + 255) / 256);
        dispatch(g, [&](auto tp, auto dc) {
            using T = std::remove_pointer_t<decltype(tp)>;
            constexpr int D = decltype(dc)::value;
            face_pack_kernel<T, D><<<blocks, 256, 0, g->stream>>>((const T*)col, ords, n, face, (T*)out,
                                                                  unpack, (const T*)in, (T*)col);
        });
        PD_CUDA(cudaGetLastError());
    });
}

int pd_grid_pack_face(pd_grid* g, int prop, const int32_t* ords, int64_t n, int face, void* out) {
    return face_io(g, prop, ords, n, face, out, nullptr, false);
}

int pd_grid_unpack_face(pd_grid* g, int prop, const int32_t* ords, int64_t n, int face,
                        const void* in) {
    return face_io(g, prop, ords, n, face, nullptr, in, true);
}

int pd_grid_swap(pd_grid* g, int a, int b) {
    return guarded([&] {
        check_prop(g, a);
        check_prop(g, b);
        std::swap(g->column_of[(size_t)a], g->column_of[(size_t)b]);
        note_write(g, a);
        note_write(g, b);
    });
}

int pd_grid_column_of(const pd_grid* g, int prop, int* column) {
    return guarded([&] {
        check_prop(g, prop);
        *column = g->column_of[(size_t)prop];
    });
}

int pd_grid_device_ptr(pd_grid* g, int prop, void** ptr) {
    return guarded([&] {
        note_write(g, prop); *ptr = col_ptr(g, prop); });
}

int pd_grid_info(const pd_grid* g, int64_t* n_chunks, int64_t* active_nodes) {
    if (n_chunks) *n_chunks = g->n_chunks;
    if (active_nodes) *active_nodes = g->active;
    return PD_OK;
}

int pd_grid_download_layout(const pd_grid* g, int32_t* keys, uint64_t* masks) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        if (g->n_chunks == 0) return;
        if (keys)
            PD_CUDA(cudaMemcpyAsync(keys, g->d_keys, sizeof(int32_t) * (size_t)(g->n_chunks * g->dims),
                                    cudaMemcpyDeviceToHost, g->stream));
        if (masks)
            PD_CUDA(cudaMemcpyAsync(masks, g->d_masks, sizeof(uint64_t) * (size_t)(g->n_chunks * g->W),
                                    cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_grid_total_mass(pd_grid* g, int prop, double* out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        void* c = col_ptr(g, prop);
        launch_chunk_stats(g, c, g->d_masks);
        launch_pairwise_finalize(g, g->d_row, nullptr);
        double row[3];
        PD_CUDA(cudaMemcpyAsync(row, g->d_row, sizeof row, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        *out = row[0];
    });
}

int pd_grid_minmax_active(pd_grid* g, int prop, double* mn, double* mx) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        void* c = col_ptr(g, prop);
        launch_chunk_stats(g, c, g->d_masks);
        launch_pairwise_finalize(g, g->d_row, nullptr);
        double row[3];
        PD_CUDA(cudaMemcpyAsync(row, g->d_row, sizeof row, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        *mn = row[1];
        *mx = row[2];
    });
}

int pd_grid_max_active(pd_grid* g, int prop, double* out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        void* c = col_ptr(g, prop);
        if (g->active == 0) {
            *out = 0.0;
            return;
        }
        launch_chunk_max(g, c);
        launch_pairwise_finalize(g, g->d_row, nullptr);
        double row[3];
        PD_CUDA(cudaMemcpyAsync(row, g->d_row, sizeof row, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        *out = row[2];
    });
}

int pd_grid_populate_diffusion(pd_grid* g, int prop_phi, int prop_d, double d_min, double d_max,
                               double gamma1, double gamma2) {
    return guarded([&] {
        note_write(g, prop_d);
        if (d_min < 0.0) fail(PD_E_INPUT, "d_min must be non-negative");
        if (!(d_max > 0.0)) fail(PD_E_INPUT, "d_max must be positive");
        DeviceGuard dg(g->device);
        const void* phi = col_ptr(g, prop_phi);
        void* d = col_ptr(g, prop_d);
        if (g->n_chunks == 0) return;
        dispatch(g, [&](auto tp, auto dc) {
            using T = std::remove_pointer_t<decltype(tp)>;
            constexpr int D = decltype(dc)::value;
            populate_d_kernel<T, D><<<(unsigned)g->n_chunks, Geo<D>::V, 0, g->stream>>>(
                (const T*)phi, (T*)d, g->d_masks, d_min, d_max, gamma1, gamma2);
        });
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_grid_fill_hash(pd_grid* g, int prop, uint64_t seed) {
    return guarded([&] {
        note_write(g, prop);
        DeviceGuard dg(g->device);
        void* x = col_ptr(g, prop);
        if (g->n_chunks == 0) return;
        dispatch(g, [&](auto tp, auto dc) {
            using T = std::remove_pointer_t<decltype(tp)>;
            constexpr int D = decltype(dc)::value;
            fill_hash_kernel<T, D><<<(unsigned)g->n_chunks, Geo<D>::V, 0, g->stream>>>(
                (T*)x, g->d_masks, g->d_keys, g->size[0], g->size[1], seed);
        });
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

__global__ void smooth_diffusion_kernel(const double* __restrict__ phi, double* __restrict__ out, int64_t n,
                                        double dmin, double dmax, double g1, double g2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = pd_smooth_diffusion(phi[i], dmin, dmax, g1, g2);
}

int pd_smooth_diffusion_coefficients(const double* phi, int64_t n, double d_min, double d_max,
                                     double gamma1, double gamma2, double* out, int device) {
    return guarded([&] {
        if (d_min < 0.0) fail(PD_E_INPUT, "d_min must be non-negative");
        if (!(d_max > 0.0)) fail(PD_E_INPUT, "d_max must be positive");
        if (n <= 0) return;
        DeviceGuard dg(device);
        double* buf = nullptr;
        PD_CUDA(cudaMalloc(&buf, 2 * n * sizeof(double)));
        struct Free { double* p; ~Free() { cudaFree(p); } } fr{buf};
        PD_CUDA(cudaMemcpy(buf, phi, n * sizeof(double), cudaMemcpyHostToDevice));
        smooth_diffusion_kernel<<<148 * 8, 256>>>(buf, buf + n, n, d_min, d_max, gamma1, gamma2);
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cudaMemcpy(out, buf + n, n * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int pd_grid_fill_const(pd_grid* g, int prop, double value) {
    return guarded([&] {
        note_write(g, prop);
        DeviceGuard dg(g->device);
        void* x = col_ptr(g, prop);
        if (g->n_chunks == 0) return;
        dispatch(g, [&](auto tp, auto dc) {
            using T = std::remove_pointer_t<decltype(tp)>;
            constexpr int D = decltype(dc)::value;
            fill_const_kernel<T, D><<<(unsigned)g->n_chunks, Geo<D>::V, 0, g->stream>>>(
                (T*)x, g->d_masks, value);
        });
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_build_sphere_pack_grid(int scalar_bytes, const int64_t* size, const double* spacing,
                              const double* origin, int64_t n_spheres, const double* centers,
                              const double* radii, double b_low, double b_up, int n_props,
                              int prop_phi, int device, pd_grid** out) {
    return pd_build_sphere_pack_region(scalar_bytes, size, spacing, origin, n_spheres, centers, radii,
                                       b_low, b_up, nullptr, nullptr, n_props, prop_phi, device, out);
}

/* Work per chunk layer of a sphere-pack domain without building it: the
 * band test of build_sparse_grid (same mask pass as the builder), reduced
 * to allocated chunks and active nodes per z chunk layer (cc[2] entries
 * each), for work-balanced z-slab cuts. */
int pd_sphere_pack_layer_work(int scalar_bytes, const int64_t* size, const double* spacing, const double* origin,
                              int64_t n_spheres, const double* centers, const double* radii, double b_low,
                              double b_up, int device, int64_t* chunks_per_layer, int64_t* active_per_layer) {
    return pd_sphere_pack_layer_cost(scalar_bytes, size, spacing, origin, n_spheres, centers, radii, b_low, b_up,
                                     device, chunks_per_layer, active_per_layer, nullptr);
}

int pd_sphere_pack_layer_cost(int scalar_bytes, const int64_t* size, const double* spacing, const double* origin,
                              int64_t n_spheres, const double* centers, const double* radii, double b_low,
                              double b_up, int device, int64_t* chunks_per_layer, int64_t* active_per_layer,
                              int64_t* full_per_layer) {
    return guarded([&] {
        pd_grid tmp;
        init_geometry(&tmp, 3, scalar_bytes, size, spacing, device);
        DeviceGuard dg(device);
        cudaStream_t st = nullptr;
        PD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        void *d_centers = nullptr, *d_radii = nullptr, *d_cnt = nullptr;
        uint64_t* slot_masks = nullptr;
        int32_t* slot_flag = nullptr;
        struct Free {
            std::vector<void*> p;
            cudaStream_t s;
            ~Free() {
                for (void* q : p) pd_free(q);
                if (s) cudaStreamDestroy(s);
            }
        } fr{{}, st};
        PackArgs p;
        int64_t slots = 1;
        for (int a = 0; a < 3; ++a) {
            p.size[a] = size[a];
            p.spacing[a] = spacing[a];
            p.origin[a] = origin[a];
            p.cc[a] = tmp.cc[a];
            p.rlo[a] = 0;
            p.rext[a] = tmp.cc[a];
            slots *= tmp.cc[a];
        }
        p.n_spheres = n_spheres;
        PD_CUDA(pd_malloc(&d_centers, sizeof(double) * (size_t)std::max<int64_t>(1, n_spheres * 3)));
        fr.p.push_back(d_centers);
        PD_CUDA(pd_malloc(&d_radii, sizeof(double) * (size_t)std::max<int64_t>(1, n_spheres)));
        fr.p.push_back(d_radii);
        if (n_spheres > 0) {
            PD_CUDA(cudaMemcpyAsync(d_centers, centers, sizeof(double) * (size_t)(n_spheres * 3),
                                    cudaMemcpyHostToDevice, st));
            PD_CUDA(cudaMemcpyAsync(d_radii, radii, sizeof(double) * (size_t)n_spheres, cudaMemcpyHostToDevice, st));
        }
        p.centers = (const double*)d_centers;
        p.radii = (const double*)d_radii;
        PD_CUDA(pd_malloc(&slot_masks, sizeof(uint64_t) * (size_t)slots * 8));
        fr.p.push_back(slot_masks);
        PD_CUDA(pd_malloc(&slot_flag, sizeof(int32_t) * (size_t)slots));
        fr.p.push_back(slot_flag);
        const int64_t layers = tmp.cc[2];
        PD_CUDA(pd_malloc(&d_cnt, sizeof(unsigned long long) * 3 * (size_t)layers));
        fr.p.push_back(d_cnt);
        PD_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 3 * (size_t)layers, st));
        if (scalar_bytes == 8) {
            const double eps = std::numeric_limits<double>::epsilon();
            pack_mask_kernel<double><<<(unsigned)slots, 512, 0, st>>>(p, b_low + eps, b_up - eps, slot_masks,
                                                                      slot_flag);
        } else {
            const float eps = std::numeric_limits<float>::epsilon();
            pack_mask_kernel<float><<<(unsigned)slots, 512, 0, st>>>(p, (float)b_low + eps, (float)b_up - eps,
                                                                     slot_masks, slot_flag);
        }
        auto* cnt = static_cast<unsigned long long*>(d_cnt);
        layer_work_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, st>>>(slot_masks, slot_flag, tmp.cc[0] * tmp.cc[1],
                                                                           layers, cnt, cnt + layers,
                                                                           cnt + 2 * layers);
        PD_CUDA(cudaGetLastError());
        std::vector<unsigned long long> h((size_t)(3 * layers));
        PD_CUDA(cudaMemcpyAsync(h.data(), d_cnt, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
        PD_CUDA(cudaStreamSynchronize(st));
        for (int64_t z = 0; z < layers; ++z) {
            if (chunks_per_layer) chunks_per_layer[z] = (int64_t)h[(size_t)z];
            if (active_per_layer) active_per_layer[z] = (int64_t)h[(size_t)(layers + z)];
            if (full_per_layer) full_per_layer[z] = (int64_t)h[(size_t)(2 * layers + z)];
        }
    });
}

int pd_build_sphere_pack_region(int scalar_bytes, const int64_t* size, const double* spacing,
                                const double* origin, int64_t n_spheres, const double* centers,
                                const double* radii, double b_low, double b_up,
                                const int64_t* chunk_lo, const int64_t* chunk_hi, int n_props,
                                int prop_phi, int device, pd_grid** out) {
    return guarded([&] {
        *out = nullptr;
        if (!(b_low < b_up))
            fail(PD_E_INPUT, "phase band is empty: lower bound must be below upper bound");
        if (n_props < 1 || prop_phi < 0 || prop_phi >= n_props)
            fail(PD_E_INPUT, "channel list must contain \"phi\" to receive the level set");
        auto* g = new pd_grid();
        void* d_centers = nullptr;
        void* d_radii = nullptr;
        uint64_t* slot_masks = nullptr;
        int32_t *slot_flag = nullptr, *ordinal = nullptr;
        void* cub_tmp = nullptr;
        try {
            init_geometry(g, 3, scalar_bytes, size, spacing, device);
            DeviceGuard dg(device);
            PD_CUDA(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
            g->stream = g->own_stream;
            PD_CUDA(pd_malloc(&g->d_row, sizeof(double) * 4));
            PackArgs p;
            int64_t slots = 1;
            for (int a = 0; a < 3; ++a) {
                p.size[a] = size[a];
                p.spacing[a] = spacing[a];
                p.origin[a] = origin[a];
                p.cc[a] = g->cc[a];
                const int64_t lo = chunk_lo ? std::max<int64_t>(0, chunk_lo[a]) : 0;
                const int64_t hi = chunk_hi ? std::min<int64_t>(g->cc[a], chunk_hi[a]) : g->cc[a];
                p.rlo[a] = lo;
                p.rext[a] = std::max<int64_t>(0, hi - lo);
                slots *= p.rext[a];
            }
            p.n_spheres = n_spheres;
            PD_CUDA(pd_malloc(&d_centers, sizeof(double) * (size_t)std::max<int64_t>(1, n_spheres * 3)));
            PD_CUDA(pd_malloc(&d_radii, sizeof(double) * (size_t)std::max<int64_t>(1, n_spheres)));
            if (n_spheres > 0) {
                PD_CUDA(cudaMemcpyAsync(d_centers, centers, sizeof(double) * (size_t)(n_spheres * 3),
                                        cudaMemcpyHostToDevice, g->stream));
                PD_CUDA(cudaMemcpyAsync(d_radii, radii, sizeof(double) * (size_t)n_spheres,
                                        cudaMemcpyHostToDevice, g->stream));
            }
            p.centers = (const double*)d_centers;
            p.radii = (const double*)d_radii;
            PD_CUDA(pd_malloc(&g->d_table, sizeof(int32_t) * (size_t)g->table_size));
            PD_CUDA(cudaMemsetAsync(g->d_table, 0xff, sizeof(int32_t) * (size_t)g->table_size, g->stream));
            if (slots == 0) {
                if (chunk_lo == nullptr)
                    fail(PD_E_INPUT, "no node lies inside the phase band: the grid would be empty");
                alloc_columns(g, n_props);
                ensure_scratch(g);
                PD_CUDA(cudaStreamSynchronize(g->stream));
                pd_free(d_centers);
                pd_free(d_radii);
                *out = g;
                return;
            }
            PD_CUDA(pd_malloc(&slot_masks, sizeof(uint64_t) * (size_t)slots * 8));
            PD_CUDA(pd_malloc(&slot_flag, sizeof(int32_t) * (size_t)slots));
            PD_CUDA(pd_malloc(&ordinal, sizeof(int32_t) * (size_t)slots));
            if (scalar_bytes == 8) {
                const double eps = std::numeric_limits<double>::epsilon();
                pack_mask_kernel<double><<<(unsigned)slots, 512, 0, g->stream>>>(
                    p, b_low + eps, b_up - eps, slot_masks, slot_flag);
            } else {
                const float eps = std::numeric_limits<float>::epsilon();
                pack_mask_kernel<float><<<(unsigned)slots, 512, 0, g->stream>>>(
                    p, (float)b_low + eps, (float)b_up - eps, slot_masks, slot_flag);
            }
            PD_CUDA(cudaGetLastError());
            size_t tmp_bytes = 0;
            PD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, slot_flag, ordinal,
                                                  (int)slots, g->stream));
            PD_CUDA(pd_malloc(&cub_tmp, tmp_bytes));
            PD_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, tmp_bytes, slot_flag, ordinal,
                                                  (int)slots, g->stream));
            int32_t last_ord = 0, last_flag = 0;
            PD_CUDA(cudaMemcpyAsync(&last_ord, ordinal + slots - 1, sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, g->stream));
            PD_CUDA(cudaMemcpyAsync(&last_flag, slot_flag + slots - 1, sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            g->n_chunks = (int64_t)last_ord + last_flag;
            if (g->n_chunks == 0 && chunk_lo == nullptr)
                fail(PD_E_INPUT, "no node lies inside the phase band: the grid would be empty");
            PD_CUDA(pd_malloc(&g->d_keys, sizeof(int32_t) * (size_t)(g->n_chunks * 3)));
            PD_CUDA(pd_malloc(&g->d_masks, sizeof(uint64_t) * (size_t)(g->n_chunks * 8)));
            alloc_columns(g, n_props);
            if (scalar_bytes == 8)
                pack_fill_kernel<double><<<(unsigned)slots, 512, 0, g->stream>>>(
                    p, slot_masks, slot_flag, ordinal, g->d_keys, g->d_masks, g->d_table,
                    (double*)g->cols[(size_t)prop_phi]);
            else
                pack_fill_kernel<float><<<(unsigned)slots, 512, 0, g->stream>>>(
                    p, slot_masks, slot_flag, ordinal, g->d_keys, g->d_masks, g->d_table,
                    (float*)g->cols[(size_t)prop_phi]);
            PD_CUDA(cudaGetLastError());
            PD_CUDA(cudaStreamSynchronize(g->stream));
            count_active(g);
            ensure_scratch(g);
        } catch (...) {
            pd_free(d_centers);
            pd_free(d_radii);
            pd_free(slot_masks);
            pd_free(slot_flag);
            pd_free(ordinal);
            pd_free(cub_tmp);
            pd_grid_destroy(g);
            throw;
        }
        pd_free(d_centers);
        pd_free(d_radii);
        pd_free(slot_masks);
        pd_free(slot_flag);
        pd_free(ordinal);
        pd_free(cub_tmp);
        *out = g;
    });
}

}  // extern "C"
