// Level-set geometry stage on the device (north_star subsystem 2; SURVEY.md
// §8f rows 1-2): dense fields, mask -> indicator, the thin-feature opening
// filter, Sussman redistancing, and band activation of a dense level set into
// the sparse block grid.
//
// Reference: geometry.hpp:67-176 (mask_to_indicator, box_filter_axis,
// filter_thin_features, build_sparse_grid), levelset.hpp:115-191
// (sussman_redistance). Bit-exactness: every node update mirrors the
// reference expression tree in T arithmetic (no contraction: --fmad=false;
// IEEE sqrt and division); the sweep's stopping residual is a max, which is
// order-independent, so the iteration count and every node value match.
//
// Layout: a dense field is one contiguous T array, axis 0 fastest
// (dense_field.hpp:12-82, grid_geometry.hpp:73-77).
#include <cub/device/device_scan.cuh>

#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <cstdlib>

#include "pd_internal.cuh"

namespace pdb {

struct FieldGeo {
    int64_t n[3];
    int64_t s1, s2;  // strides of axes 1 and 2
    int64_t total;
};

FieldGeo field_geo(const pd_field* f) {
    FieldGeo g;
    for (int a = 0; a < 3; ++a) g.n[a] = f->size[a];
    g.s1 = f->size[0];
    g.s2 = f->size[0] * f->size[1];
    g.total = f->n;
    return g;
}

// ---- mask -> indicator (geometry.hpp:67-77) -----------------------------
template <class T>
__global__ void indicator_kernel(const uint8_t* __restrict__ bits, int64_t n, T* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = bits[i] ? T(1) : T(-1);
}

// ---- opening filter (geometry.hpp:84-142) ---------------------------------
template <class T>
__global__ void cells_from_indicator(const T* __restrict__ v, int64_t n, uint8_t* __restrict__ c,
                                     int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const T x = v[i];
    if (x != T(1) && x != T(-1)) atomicOr(bad, 1);
    c[i] = x > T(0) ? 1 : 0;
}

// erode: AND of in[i .. i+w-1]; dilate: OR of in[i-w+1 .. i]; outside = false
__global__ void box_filter_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, FieldGeo g,
                                  int axis, int w, int erode) {
    const int64_t x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.n[0] || y >= g.n[1]) return;
    const int64_t f = x + y * g.s1 + z * g.s2;
    const int64_t stride = axis == 0 ? 1 : (axis == 1 ? g.s1 : g.s2);
    const int64_t i = axis == 0 ? x : (axis == 1 ? y : z);
    const int64_t na = g.n[axis];
    bool v = erode;
    for (int k = 0; k < w; ++k) {
        const int64_t j = i + (erode ? k : -k);
        const bool bit = j >= 0 && j < na && in[f + (j - i) * stride];
        v = erode ? (v && bit) : (v || bit);
    }
    out[f] = v ? 1 : 0;
}

template <class T>
__global__ void indicator_from_cells(const uint8_t* __restrict__ c, int64_t n, T* __restrict__ v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = c[i] ? T(1) : T(-1);
}

// ---- Sussman redistancing (levelset.hpp:115-191) --------------------------
template <class T>
__global__ void finite_crossing_kernel(const T* __restrict__ p, FieldGeo g, int dims, int* __restrict__ flags) {
    // flags[0] |= non-finite seen; flags[1] |= zero crossing seen
    const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (f >= g.total) return;
    const T v = p[f];
    if (!isfinite(v)) atomicOr(&flags[0], 1);
    const bool neg = v < T(0);
    const int64_t i0 = f % g.n[0], i1 = (f / g.s1) % g.n[1], i2 = f / g.s2;
    bool cross = false;
    if (g.n[0] > 1 && i0 + 1 < g.n[0]) cross = cross || (neg != (p[f + 1] < T(0)));
    if (dims >= 2 && g.n[1] > 1 && i1 + 1 < g.n[1]) cross = cross || (neg != (p[f + g.s1] < T(0)));
    if (dims == 3 && g.n[2] > 1 && i2 + 1 < g.n[2]) cross = cross || (neg != (p[f + g.s2] < T(0)));
    if (cross) atomicOr(&flags[1], 1);
}

template <class T>
__global__ void rescale_kernel(T* __restrict__ p, int64_t n, T h) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const T v = p[i];
        p[i] = v < T(0) ? -h : (v > T(0) ? h : T(0));
    }
}

template <class T>
__device__ __forceinline__ T max_ref(T a, T b) {  // std::max: (a < b) ? b : a
    return (a < b) ? b : a;
}
template <class T>
__device__ __forceinline__ T min_ref(T a, T b) {  // std::min: (b < a) ? b : a
    return (b < a) ? b : a;
}

// x, or 1 where `one` holds, through an opaque select (inline PTX): the
// compiler cannot fold it into the surrounding select, so a square root /
// division fed with it never sees the zero that sends the library routine
// down its out-of-line special-case path
__device__ __forceinline__ double or_one(double x, bool one) {
    double r;
    asm("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n selp.f64 %0, 0d3FF0000000000000, %1, p;\n}\n"
        : "=d"(r) : "d"(x), "r"((unsigned)one));
    return r;
}
__device__ __forceinline__ float or_one(float x, bool one) {
    float r;
    asm("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n selp.f32 %0, 0f3F800000, %1, p;\n}\n"
        : "=f"(r) : "f"(x), "r"((unsigned)one));
    return r;
}

// detail::godunov_axis_sq (levelset.hpp:43-53)
template <class T>
__device__ __forceinline__ T godunov_sq(T dm, T dp, bool pos) {
    T a, b;
    if (pos) {
        a = max_ref(dm, T(0));
        b = min_ref(dp, T(0));
    } else {
        a = min_ref(dm, T(0));
        b = max_ref(dp, T(0));
    }
    return max_ref(a * a, b * b);
}

template <class T>
struct SweepConsts {
    T inv_h[3];
    T h, dt, band, tol;
};

template <class T>
struct Bits;
template <>
struct Bits<double> {
    using U = unsigned long long;
    static __device__ U of(double x) { return (U)__double_as_longlong(x); }
    static __device__ double to(U u) { return __longlong_as_double((long long)u); }
};
template <>
struct Bits<float> {
    using U = unsigned int;
    static __device__ U of(float x) { return (U)__float_as_uint(x); }
    static __device__ float to(U u) { return __uint_as_float(u); }
};

// One Jacobi sweep: next = phi + dt * S(phi) * (1 - |grad phi|). Stops (no-op)
// once an earlier sweep of the batch converged. The band residual is an
// atomic max over the bit patterns of non-negative values (order-free).
template <class T, int D>
__global__ void __launch_bounds__(256)
    sussman_sweep_kernel(const T* __restrict__ phi, T* __restrict__ next, FieldGeo g, SweepConsts<T> K,
                         typename Bits<T>::U* __restrict__ res, const int* __restrict__ done) {
    if (*done) return;
    // 3-D launch: x = blockIdx.x*32 + tx, y = blockIdx.y*8 + ty, z = blockIdx.z
    const int64_t x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    const int64_t f = x + y * g.s1 + z * g.s2;
    T local = T(0);
    if (x < g.n[0] && y < g.n[1]) {
        const T c = phi[f];
        const int64_t idx[3] = {x, y, z};
        const int64_t stride[3] = {1, g.s1, g.s2};
        const bool pos = !(c < T(0));
        T sum = T(0);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const bool has_m = idx[a] > 0;
            const bool has_p = idx[a] + 1 < g.n[a];
            T dm = T(0), dp = T(0);
            if (has_m) dm = (c - phi[f - stride[a]]) * K.inv_h[a];
            if (has_p) dp = (phi[f + stride[a]] - c) * K.inv_h[a];
            if (!has_m) dm = dp;
            if (!has_p) dp = dm;
            sum += godunov_sq(dm, dp, pos);
        }
        // the zero cases are selected; the routines see a dummy 1 there (see
        // sussman_zmarch_kernel)
        const bool zs = sum == T(0), zc = c == T(0);
        const T grad = zs ? T(0) : sqrt(or_one(sum, zs));
        // smoothed_sign (levelset.hpp:30-34): phi / sqrt(phi^2 + |g|^2 h^2)
        const T ss = zc ? T(0) : c / sqrt(or_one(c * c + grad * grad * K.h * K.h, zc));
        const T update = K.dt * ss * (T(1) - grad);
        next[f] = c + update;
        if (fabs(c) <= K.band) local = fabs(update);
    }
    // warp max, then one atomic per warp
    typename Bits<T>::U b = Bits<T>::of(local);
    for (int o = 16; o; o >>= 1) {
        const typename Bits<T>::U other = __shfl_xor_sync(0xffffffffu, b, o);
        b = other > b ? other : b;
    }
    if (threadIdx.x == 0 && b) atomicMax(res, b);
}

// 3-D sweep as a z-march (same per-node expression tree as
// sussman_sweep_kernel, so the same bits): a 32 x 8 block owns an (x, y) tile
// and walks a segment of z; its own column values come through a register
// pipeline issued kAheadZ planes ahead, the tile's x / y neighbours through a
// shared-memory copy of the current plane (+ one halo cell per side, also
// prefetched), so every phi value is read from DRAM about once per sweep
// instead of once per neighbour use, and the loads are in flight while the
// previous planes compute. The band residual is folded per thread over the
// segment and reduced once per warp.
constexpr int kAheadZ = 3;

template <class T>
__device__ __forceinline__ T ld_or0(const T* __restrict__ p, int64_t i, bool ok) {
    return ok ? __ldg(p + i) : T(0);
}

template <class T>
__global__ void __launch_bounds__(256)
    sussman_zmarch_kernel(const T* __restrict__ phi, T* __restrict__ next, FieldGeo g, SweepConsts<T> K,
                          typename Bits<T>::U* __restrict__ res, const int* __restrict__ done, int zseg) {
    if (*done) return;
    __shared__ T tile[10][34];  // rows y-1..y+8 of the block, columns x-1..x+32
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t x = blockIdx.x * 32 + tx, y = blockIdx.y * 8 + ty;
    const int64_t nz = g.n[2];
    const int64_t z0 = (int64_t)blockIdx.z * zseg;
    const int64_t z1 = z0 + zseg < nz ? z0 + zseg : nz;
    const bool inb = x < g.n[0] && y < g.n[1];
    const int64_t col = x + y * g.s1;  // plane-0 index of the thread's own column
    // halo cell this thread stages (x halo for tx = 0 / 31, y halo for ty = 0 / 7)
    const bool hx = tx == 0 || tx == 31, hy = ty == 0 || ty == 7;
    const int64_t xh = tx == 0 ? x - 1 : x + 1, yh = ty == 0 ? y - 1 : y + 1;
    const bool hx_ok = hx && xh >= 0 && xh < g.n[0] && y < g.n[1];
    const bool hy_ok = hy && yh >= 0 && yh < g.n[1] && x < g.n[0];
    const int64_t hx_col = xh + y * g.s1, hy_col = x + yh * g.s1;
    // pipelines: q[k] = own value of plane z+k (k = -1 .. kAheadZ); hxq / hyq =
    // halo values of planes z .. z+kAheadZ-1
    T q[kAheadZ + 2];
    T hxq[kAheadZ], hyq[kAheadZ];
#pragma unroll
    for (int k = 0; k < kAheadZ + 2; ++k) {
        const int64_t z = z0 - 1 + k;
        q[k] = ld_or0(phi, col + z * g.s2, inb && z >= 0 && z < nz);
    }
#pragma unroll
    for (int k = 0; k < kAheadZ; ++k) {
        const int64_t z = z0 + k;
        hxq[k] = ld_or0(phi, hx_col + z * g.s2, hx_ok && z < nz);
        hyq[k] = ld_or0(phi, hy_col + z * g.s2, hy_ok && z < nz);
    }
    // residual as a max over bit patterns, like sussman_sweep_kernel (a NaN
    // update wins, exactly as there)
    typename Bits<T>::U lb = 0;
    const bool pos_x_m = x > 0, pos_x_p = x + 1 < g.n[0];
    const bool pos_y_m = y > 0, pos_y_p = y + 1 < g.n[1];
    // running pointers (no 64-bit index arithmetic per plane): the own column
    // kAheadZ+1 planes ahead, the halo columns kAheadZ ahead, the output plane
    const T* pq = phi + (inb ? col : 0) + (z0 + kAheadZ + 1) * g.s2;
    const T* phx = phi + (hx_ok ? hx_col : 0) + (z0 + kAheadZ) * g.s2;
    const T* phy = phi + (hy_ok ? hy_col : 0) + (z0 + kAheadZ) * g.s2;
    T* pn = next + (inb ? col : 0) + z0 * g.s2;
    const int64_t s2 = g.s2;
    int64_t left = nz - z0;  // planes from z to the box end
    for (int64_t z = z0; z < z1; ++z, pq += s2, phx += s2, phy += s2, pn += s2, --left) {
        const T c = q[1];
        __syncthreads();  // the previous plane's readers are done
        tile[ty + 1][tx + 1] = c;
        if (hx) tile[ty + 1][tx == 0 ? 0 : 33] = hxq[0];
        if (hy) tile[ty == 0 ? 0 : 9][tx + 1] = hyq[0];
        __syncthreads();
        // refill the pipelines (plane z+kAheadZ+1 own, z+kAheadZ halos)
        const T nq = (inb && left > kAheadZ + 1) ? __ldg(pq) : T(0);
        const T nhx = (hx_ok && left > kAheadZ) ? __ldg(phx) : T(0);
        const T nhy = (hy_ok && left > kAheadZ) ? __ldg(phy) : T(0);
        if (inb) {
            const bool pos = !(c < T(0));
            T sum = T(0);
            {  // axis 0
                T dm = T(0), dp = T(0);
                if (pos_x_m) dm = (c - tile[ty + 1][tx]) * K.inv_h[0];
                if (pos_x_p) dp = (tile[ty + 1][tx + 2] - c) * K.inv_h[0];
                if (!pos_x_m) dm = dp;
                if (!pos_x_p) dp = dm;
                sum += godunov_sq(dm, dp, pos);
            }
            {  // axis 1
                T dm = T(0), dp = T(0);
                if (pos_y_m) dm = (c - tile[ty][tx + 1]) * K.inv_h[1];
                if (pos_y_p) dp = (tile[ty + 2][tx + 1] - c) * K.inv_h[1];
                if (!pos_y_m) dm = dp;
                if (!pos_y_p) dp = dm;
                sum += godunov_sq(dm, dp, pos);
            }
            {  // axis 2
                const bool has_m = z > 0, has_p = z + 1 < nz;
                T dm = T(0), dp = T(0);
                if (has_m) dm = (c - q[0]) * K.inv_h[2];
                if (has_p) dp = (q[2] - c) * K.inv_h[2];
                if (!has_m) dm = dp;
                if (!has_p) dp = dm;
                sum += godunov_sq(dm, dp, pos);
            }
            // sqrt(+0) = +0 and smoothed_sign(0) = 0 are selected, and the
            // square roots / division then see a dummy 1 instead of the zero:
            // the library routines' special-case (out-of-line) path is never
            // taken for those nodes (a select alone still evaluates them)
            const bool zs = sum == T(0), zc = c == T(0);
            const T grad = zs ? T(0) : sqrt(or_one(sum, zs));
            // smoothed_sign (levelset.hpp:30-34): phi / sqrt(phi^2 + |g|^2 h^2)
            const T ss = zc ? T(0) : c / sqrt(or_one(c * c + grad * grad * K.h * K.h, zc));
            const T update = K.dt * ss * (T(1) - grad);
            *pn = c + update;
            if (fabs(c) <= K.band) {
                const typename Bits<T>::U ub = Bits<T>::of(fabs(update));
                lb = ub > lb ? ub : lb;
            }
        }
#pragma unroll
        for (int k = 0; k < kAheadZ + 1; ++k) q[k] = q[k + 1];
        q[kAheadZ + 1] = nq;
#pragma unroll
        for (int k = 0; k < kAheadZ - 1; ++k) {
            hxq[k] = hxq[k + 1];
            hyq[k] = hyq[k + 1];
        }
        hxq[kAheadZ - 1] = nhx;
        hyq[kAheadZ - 1] = nhy;
    }
    typename Bits<T>::U b = lb;
    for (int o = 16; o; o >>= 1) {
        const typename Bits<T>::U other = __shfl_xor_sync(0xffffffffu, b, o);
        b = other > b ? other : b;
    }
    if (tx == 0 && b) atomicMax(res, b);
}

// After sweep it (1-based): converged when residual < tol (levelset.hpp:183-187).
template <class T>
__global__ void sussman_check_kernel(const typename Bits<T>::U* __restrict__ res, int it, T tol,
                                     int* __restrict__ done, int* __restrict__ iters) {
    if (*done) return;
    *iters = it;
    if (Bits<T>::to(*res) < tol) *done = 1;
}

constexpr int kFieldThreads = 256;
inline unsigned blocks_for(int64_t n) { return (unsigned)((n + kFieldThreads - 1) / kFieldThreads); }
// 3-D launch over a field: 32 x 8 thread tiles of (x, y), one z per block row
inline dim3 grid3(const pd_field* f) {
    return dim3((unsigned)((f->size[0] + 31) / 32), (unsigned)((f->size[1] + 7) / 8), (unsigned)f->size[2]);
}
const dim3 kBlock3(32, 8, 1);

void check_field(const pd_field* f) {
    if (!f || !f->d) fail(PD_E_INPUT, "null field");
}

// ---- band activation of a dense level set (geometry.hpp:148-176) ---------
template <class T, int D>
__global__ void field_mask_kernel(const T* __restrict__ phi, FieldGeo g, int64_t cc0, int64_t cc1, T lo, T hi,
                                  uint64_t* __restrict__ slot_masks, int32_t* __restrict__ slot_flag) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t slot = blockIdx.x;
    const int off = threadIdx.x;
    const int64_t kx = slot % cc0, ky = (slot / cc0) % cc1, kz = D == 3 ? slot / (cc0 * cc1) : 0;
    const int64_t x = kx * 8 + (off & 7), y = ky * 8 + ((off >> 3) & 7), z = D == 3 ? kz * 8 + (off >> 6) : 0;
    bool act = false;
    if (x < g.n[0] && y < g.n[1] && (D == 2 || z < g.n[2])) {
        const T v = phi[x + y * g.s1 + z * g.s2];
        act = v > lo && v < hi;
    }
    const unsigned b = __ballot_sync(0xffffffffu, act);
    __shared__ unsigned words[V / 32];
    if ((off & 31) == 0) words[off >> 5] = b;
    __syncthreads();
    if (off < W) slot_masks[slot * W + off] = (uint64_t)words[2 * off] | ((uint64_t)words[2 * off + 1] << 32);
    if (off == 0) {
        int any = 0;
        for (int w = 0; w < V / 32; ++w) any |= words[w] != 0;
        slot_flag[slot] = any;
    }
}

template <class T, int D>
__global__ void field_fill_kernel(const T* __restrict__ phi, FieldGeo g, int64_t cc0, int64_t cc1,
                                  const uint64_t* __restrict__ slot_masks, const int32_t* __restrict__ slot_flag,
                                  const int32_t* __restrict__ ordinal, int32_t* __restrict__ keys,
                                  uint64_t* __restrict__ masks, int32_t* __restrict__ table, T* __restrict__ col) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    const int64_t slot = blockIdx.x;
    if (!slot_flag[slot]) return;
    const int64_t i = ordinal[slot];
    const int off = threadIdx.x;
    const int64_t kx = slot % cc0, ky = (slot / cc0) % cc1, kz = D == 3 ? slot / (cc0 * cc1) : 0;
    if (off == 0) {
        keys[i * D] = (int32_t)kx;
        keys[i * D + 1] = (int32_t)ky;
        if (D == 3) keys[i * D + 2] = (int32_t)kz;
        table[slot] = (int32_t)i;
    }
    if (off < W) masks[i * W + off] = slot_masks[slot * W + off];
    const bool act = (slot_masks[slot * W + (off >> 6)] >> (off & 63)) & 1u;
    T v = T(0);
    if (act) {
        const int64_t x = kx * 8 + (off & 7), y = ky * 8 + ((off >> 3) & 7), z = D == 3 ? kz * 8 + (off >> 6) : 0;
        v = phi[x + y * g.s1 + z * g.s2];
    }
    col[i * V + off] = v;
}

template <class T, int D>
void build_from_field(const pd_field* f, double b_low, double b_up, int n_props, int prop_phi, pd_grid* g) {
    const FieldGeo fg = field_geo(f);
    const int64_t slots = g->table_size;
    const int V = Geo<D>::V, W = Geo<D>::W;
    uint64_t* slot_masks = nullptr;
    int32_t *slot_flag = nullptr, *ordinal = nullptr;
    void* tmp = nullptr;
    try {
        PD_CUDA(pd_malloc(&slot_masks, sizeof(uint64_t) * (size_t)(slots * W)));
        PD_CUDA(pd_malloc(&slot_flag, sizeof(int32_t) * (size_t)slots));
        PD_CUDA(pd_malloc(&ordinal, sizeof(int32_t) * (size_t)slots));
        // eps = numeric_limits<T>::epsilon(); lo = T(b_low) + eps, hi = T(b_up) - eps
        const T eps = std::numeric_limits<T>::epsilon();
        const T lo = static_cast<T>(b_low) + eps;
        const T hi = static_cast<T>(b_up) - eps;
        field_mask_kernel<T, D><<<(unsigned)slots, V, 0, g->stream>>>((const T*)f->d, fg, g->cc[0], g->cc[1], lo,
                                                                      hi, slot_masks, slot_flag);
        PD_CUDA(cudaGetLastError());
        size_t tb = 0;
        PD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, slot_flag, ordinal, (int)slots, g->stream));
        PD_CUDA(pd_malloc(&tmp, tb));
        PD_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, slot_flag, ordinal, (int)slots, g->stream));
        int32_t last_ord = 0, last_flag = 0;
        PD_CUDA(cudaMemcpyAsync(&last_ord, ordinal + slots - 1, 4, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaMemcpyAsync(&last_flag, slot_flag + slots - 1, 4, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
        g->n_chunks = (int64_t)last_ord + last_flag;
        if (g->n_chunks == 0) fail(PD_E_INPUT, "no node lies inside the phase band: the grid would be empty");
        PD_CUDA(pd_malloc(&g->d_keys, sizeof(int32_t) * (size_t)(g->n_chunks * D)));
        PD_CUDA(pd_malloc(&g->d_masks, sizeof(uint64_t) * (size_t)(g->n_chunks * W)));
        alloc_columns(g, n_props);
        field_fill_kernel<T, D><<<(unsigned)slots, V, 0, g->stream>>>(
            (const T*)f->d, fg, g->cc[0], g->cc[1], slot_masks, slot_flag, ordinal, g->d_keys, g->d_masks,
            g->d_table, (T*)g->cols[(size_t)prop_phi]);
        PD_CUDA(cudaGetLastError());
        PD_CUDA(cudaStreamSynchronize(g->stream));
    } catch (...) {
        pd_free(slot_masks);
        pd_free(slot_flag);
        pd_free(ordinal);
        pd_free(tmp);
        throw;
    }
    pd_free(slot_masks);
    pd_free(slot_flag);
    pd_free(ordinal);
    pd_free(tmp);
}

template <class T>
void redistance(pd_field* f, const pd_levelset_options* o, pd_redistance_diag* out) {
    const FieldGeo g = field_geo(f);
    // levelset.hpp:127-131: h = T(min_spacing), dt = T(pseudo)*h, band, tol
    double hmin = f->spacing[0];
    for (int a = 1; a < f->dims; ++a) hmin = hmin < f->spacing[a] ? hmin : f->spacing[a];
    SweepConsts<T> K;
    K.h = static_cast<T>(hmin);
    K.dt = static_cast<T>(o->pseudo_time_step) * K.h;
    K.band = static_cast<T>(o->residual_band_width) * K.h;
    K.tol = static_cast<T>(o->tolerance) * K.h;
    for (int a = 0; a < 3; ++a) K.inv_h[a] = a < f->dims ? static_cast<T>(1.0 / f->spacing[a]) : T(0);
    if (o->rescale_initial)
        rescale_kernel<T><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>((T*)f->d, f->n, K.h);
    T* next = nullptr;
    typename Bits<T>::U* d_res = nullptr;
    int* d_state = nullptr;  // done, iters
    const int kSync = 32;    // sweeps per host check
    try {
        PD_CUDA(pd_malloc(&next, sizeof(T) * (size_t)f->n));
        PD_CUDA(pd_malloc(&d_res, sizeof(typename Bits<T>::U) * (size_t)(o->max_iterations + 1)));
        PD_CUDA(cudaMemsetAsync(d_res, 0, sizeof(typename Bits<T>::U) * (size_t)(o->max_iterations + 1), f->stream));
        PD_CUDA(pd_malloc(&d_state, 2 * sizeof(int)));
        PD_CUDA(cudaMemsetAsync(d_state, 0, 2 * sizeof(int), f->stream));
        T* bufs[2] = {(T*)f->d, next};
        int h_state[2] = {0, 0};
        // z-march segments: enough blocks for ~4 waves of the (x, y) tiles
        static const int zmarch = [] {
            const char* e = getenv("PD_SUSSMAN_ZMARCH");
            return e ? atoi(e) : 1;
        }();
        int sms = 148;
        PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, f->device));
        const int64_t tiles = ((f->size[0] + 31) / 32) * ((f->size[1] + 7) / 8);
        int64_t nseg = (int64_t)sms * 8 * 4 / (tiles > 0 ? tiles : 1);
        if (nseg < 1) nseg = 1;
        if (nseg > f->size[2]) nseg = f->size[2];
        const int zseg = (int)((f->size[2] + nseg - 1) / nseg);
        for (int it = 1; it <= o->max_iterations; ++it) {
            const T* src = bufs[(it - 1) & 1];
            T* dst = bufs[it & 1];
            if (f->dims == 3 && zmarch) {
                const dim3 gz((unsigned)((f->size[0] + 31) / 32), (unsigned)((f->size[1] + 7) / 8),
                              (unsigned)((f->size[2] + zseg - 1) / zseg));
                sussman_zmarch_kernel<T><<<gz, kBlock3, 0, f->stream>>>(src, dst, g, K, d_res + it, d_state, zseg);
            } else if (f->dims == 3)
                sussman_sweep_kernel<T, 3><<<grid3(f), kBlock3, 0, f->stream>>>(src, dst, g, K, d_res + it,
                                                                                   d_state);
            else
                sussman_sweep_kernel<T, 2><<<grid3(f), kBlock3, 0, f->stream>>>(src, dst, g, K, d_res + it,
                                                                                   d_state);
            sussman_check_kernel<T><<<1, 1, 0, f->stream>>>(d_res + it, it, K.tol, d_state, d_state + 1);
            if (it % kSync == 0 || it == o->max_iterations) {
                PD_CUDA(cudaMemcpyAsync(h_state, d_state, sizeof h_state, cudaMemcpyDeviceToHost, f->stream));
                PD_CUDA(cudaStreamSynchronize(f->stream));
                if (h_state[0]) break;
            }
        }
        PD_CUDA(cudaMemcpyAsync(h_state, d_state, sizeof h_state, cudaMemcpyDeviceToHost, f->stream));
        PD_CUDA(cudaStreamSynchronize(f->stream));
        const int iters = h_state[1];
        typename Bits<T>::U rbits = 0;
        PD_CUDA(cudaMemcpy(&rbits, d_res + iters, sizeof rbits, cudaMemcpyDeviceToHost));
        T resid;
        std::memcpy(&resid, &rbits, sizeof resid);
        // the final field is the output of sweep `iters` (std::swap per sweep)
        if (iters & 1) {
            PD_CUDA(cudaMemcpyAsync(f->d, next, sizeof(T) * (size_t)f->n, cudaMemcpyDeviceToDevice, f->stream));
            PD_CUDA(cudaStreamSynchronize(f->stream));
        }
        out->iterations = iters;
        out->final_residual = static_cast<double>(resid) / static_cast<double>(K.h);
        out->converged = h_state[0];
    } catch (...) {
        pd_free(next);
        pd_free(d_res);
        pd_free(d_state);
        throw;
    }
    pd_free(next);
    pd_free(d_res);
    pd_free(d_state);
}

}  // namespace pdb

using namespace pdb;

extern "C" {

int pd_field_create(int dims, int scalar_bytes, const int64_t* size, const double* spacing, const double* origin,
                    int device, pd_field** out) {
    return guarded([&] {
        *out = nullptr;
        if (dims != 2 && dims != 3) fail(PD_E_INPUT, "only 2-D and 3-D fields are supported");
        if (scalar_bytes != 4 && scalar_bytes != 8) fail(PD_E_INPUT, "scalar_bytes must be 4 or 8");
        auto* f = new pd_field();
        try {
            f->dims = dims;
            f->tbytes = scalar_bytes;
            f->device = device;
            f->n = 1;
            for (int a = 0; a < dims; ++a) {
                if (size[a] < 1) fail(PD_E_INPUT, "grid size must be >= 1 along every axis");
                if (!(spacing[a] > 0.0)) fail(PD_E_INPUT, "grid spacing must be > 0 along every axis");
                f->size[a] = size[a];
                f->spacing[a] = spacing[a];
                f->origin[a] = origin ? origin[a] : 0.0;
                f->n *= size[a];
            }
            DeviceGuard dg(device);
            PD_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
            PD_CUDA(pd_malloc(&f->d, (size_t)f->n * (size_t)scalar_bytes));
            PD_CUDA(cudaMemsetAsync(f->d, 0, (size_t)f->n * (size_t)scalar_bytes, f->stream));
            PD_CUDA(cudaStreamSynchronize(f->stream));
        } catch (...) {
            pd_field_destroy(f);
            throw;
        }
        *out = f;
    });
}

int pd_field_destroy(pd_field* f) {
    if (!f) return PD_OK;
    {
        DeviceGuard dg(f->device);
        if (f->stream) cudaStreamSynchronize(f->stream);
        pd_free(f->d);
        if (f->stream) cudaStreamDestroy(f->stream);
    }
    delete f;
    return PD_OK;
}

int pd_field_upload(pd_field* f, const void* host) {
    return guarded([&] {
        check_field(f);
        DeviceGuard dg(f->device);
        PD_CUDA(cudaMemcpyAsync(f->d, host, (size_t)f->n * (size_t)f->tbytes, cudaMemcpyHostToDevice, f->stream));
        PD_CUDA(cudaStreamSynchronize(f->stream));
    });
}

int pd_field_upload_device(pd_field* f, const void* dev) {
    return guarded([&] {
        check_field(f);
        DeviceGuard dg(f->device);
        PD_CUDA(cudaMemcpyAsync(f->d, dev, (size_t)f->n * (size_t)f->tbytes, cudaMemcpyDeviceToDevice, f->stream));
        PD_CUDA(cudaStreamSynchronize(f->stream));
    });
}

int pd_field_download(pd_field* f, void* host) {
    return guarded([&] {
        check_field(f);
        DeviceGuard dg(f->device);
        PD_CUDA(cudaMemcpyAsync(host, f->d, (size_t)f->n * (size_t)f->tbytes, cudaMemcpyDeviceToHost, f->stream));
        PD_CUDA(cudaStreamSynchronize(f->stream));
    });
}

int pd_field_device_ptr(pd_field* f, void** ptr) {
    *ptr = f ? f->d : nullptr;
    return PD_OK;
}

int pd_field_from_mask(pd_field* f, const uint8_t* host_bits, int64_t n_bits) {
    return guarded([&] {
        check_field(f);
        if (n_bits != f->n) fail(PD_E_INPUT, "mask bit count does not match voxel count");
        DeviceGuard dg(f->device);
        uint8_t* d_bits = nullptr;
        PD_CUDA(pd_malloc(&d_bits, (size_t)f->n));
        PD_CUDA(cudaMemcpyAsync(d_bits, host_bits, (size_t)f->n, cudaMemcpyHostToDevice, f->stream));
        if (f->tbytes == 8)
            indicator_kernel<double><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(d_bits, f->n, (double*)f->d);
        else
            indicator_kernel<float><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(d_bits, f->n, (float*)f->d);
        const cudaError_t e = cudaStreamSynchronize(f->stream);
        pd_free(d_bits);
        PD_CUDA(e);
    });
}

int pd_field_filter_thin(pd_field* f, int min_thickness_cells) {
    return guarded([&] {
        check_field(f);
        if (min_thickness_cells < 1) fail(PD_E_INPUT, "min_thickness_cells must be at least 1");
        DeviceGuard dg(f->device);
        const FieldGeo g = field_geo(f);
        uint8_t *a = nullptr, *b = nullptr;
        int* bad = nullptr;
        try {
            PD_CUDA(pd_malloc(&a, (size_t)f->n));
            PD_CUDA(pd_malloc(&b, (size_t)f->n));
            PD_CUDA(pd_malloc(&bad, sizeof(int)));
            PD_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), f->stream));
            if (f->tbytes == 8)
                cells_from_indicator<double><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>((const double*)f->d,
                                                                                              f->n, a, bad);
            else
                cells_from_indicator<float><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>((const float*)f->d,
                                                                                             f->n, a, bad);
            int h_bad = 0;
            PD_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, f->stream));
            PD_CUDA(cudaStreamSynchronize(f->stream));
            if (h_bad) fail(PD_E_INPUT, "indicator values must be exactly +1 or -1");
            // erode along every axis, then dilate along every axis (geometry.hpp:137-138)
            for (int pass = 0; pass < 2; ++pass)
                for (int ax = 0; ax < f->dims; ++ax) {
                    box_filter_kernel<<<grid3(f), kBlock3, 0, f->stream>>>(a, b, g, ax,
                                                                                       min_thickness_cells,
                                                                                       pass == 0);
                    std::swap(a, b);
                }
            if (f->tbytes == 8)
                indicator_from_cells<double><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(a, f->n,
                                                                                              (double*)f->d);
            else
                indicator_from_cells<float><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(a, f->n,
                                                                                             (float*)f->d);
            PD_CUDA(cudaGetLastError());
            PD_CUDA(cudaStreamSynchronize(f->stream));
        } catch (...) {
            pd_free(a);
            pd_free(b);
            pd_free(bad);
            throw;
        }
        pd_free(a);
        pd_free(b);
        pd_free(bad);
    });
}

int pd_field_redistance(pd_field* f, const pd_levelset_options* o, pd_redistance_diag* out) {
    return guarded([&] {
        check_field(f);
        // levelset.hpp:118-125, messages verbatim
        if (o->max_iterations < 1) fail(PD_E_INPUT, "max_iterations must be at least 1");
        if (!(o->tolerance > 0.0)) fail(PD_E_INPUT, "tolerance must be positive");
        if (!(o->pseudo_time_step > 0.0) || o->pseudo_time_step > 1.0)
            fail(PD_E_INPUT, "pseudo_time_step must lie in (0, 1] (units of h)");
        DeviceGuard dg(f->device);
        int* flags = nullptr;
        PD_CUDA(pd_malloc(&flags, 2 * sizeof(int)));
        int h[2] = {0, 0};
        try {
            PD_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), f->stream));
            const FieldGeo g = field_geo(f);
            if (f->tbytes == 8)
                finite_crossing_kernel<double><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(
                    (const double*)f->d, g, f->dims, flags);
            else
                finite_crossing_kernel<float><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(
                    (const float*)f->d, g, f->dims, flags);
            PD_CUDA(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, f->stream));
            PD_CUDA(cudaStreamSynchronize(f->stream));
        } catch (...) {
            pd_free(flags);
            throw;
        }
        pd_free(flags);
        if (h[0]) fail(PD_E_INPUT, "redistancing input contains non-finite values");
        if (!h[1]) fail(PD_E_INPUT, "no interface found: the field never changes sign");
        if (f->tbytes == 8)
            redistance<double>(f, o, out);
        else
            redistance<float>(f, o, out);
    });
}

int pd_build_grid_from_field(const pd_field* f, double b_low, double b_up, int n_props, int prop_phi,
                             pd_grid** out) {
    return guarded([&] {
        *out = nullptr;
        check_field(f);
        if (!(b_low < b_up)) fail(PD_E_INPUT, "phase band is empty: lower bound must be below upper bound");
        if (n_props < 1 || prop_phi < 0 || prop_phi >= n_props)
            fail(PD_E_INPUT, "channel list must contain \"phi\" to receive the level set");
        DeviceGuard dg(f->device);
        {  // all_finite (geometry.hpp:158)
            int* flags = nullptr;
            PD_CUDA(pd_malloc(&flags, 2 * sizeof(int)));
            int h[2] = {0, 0};
            PD_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), f->stream));
            const FieldGeo g = field_geo(f);
            if (f->tbytes == 8)
                finite_crossing_kernel<double><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(
                    (const double*)f->d, g, f->dims, flags);
            else
                finite_crossing_kernel<float><<<blocks_for(f->n), kFieldThreads, 0, f->stream>>>(
                    (const float*)f->d, g, f->dims, flags);
            const cudaError_t e1 = cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, f->stream);
            const cudaError_t e2 = cudaStreamSynchronize(f->stream);
            pd_free(flags);
            PD_CUDA(e1);
            PD_CUDA(e2);
            if (h[0]) fail(PD_E_INPUT, "level-set field contains non-finite values");
        }
        auto* g = new pd_grid();
        try {
            init_geometry(g, f->dims, f->tbytes, f->size, f->spacing, f->device);
            g->stream = f->stream;  // temporarily share the field's stream
            PD_CUDA(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
            PD_CUDA(pd_malloc(&g->d_row, sizeof(double) * 4));
            PD_CUDA(pd_malloc(&g->d_table, sizeof(int32_t) * (size_t)g->table_size));
            PD_CUDA(cudaMemsetAsync(g->d_table, 0xff, sizeof(int32_t) * (size_t)g->table_size, g->stream));
            if (f->tbytes == 8 && f->dims == 3)
                build_from_field<double, 3>(f, b_low, b_up, n_props, prop_phi, g);
            else if (f->tbytes == 8)
                build_from_field<double, 2>(f, b_low, b_up, n_props, prop_phi, g);
            else if (f->dims == 3)
                build_from_field<float, 3>(f, b_low, b_up, n_props, prop_phi, g);
            else
                build_from_field<float, 2>(f, b_low, b_up, n_props, prop_phi, g);
            g->stream = g->own_stream;
            count_active(g);
            ensure_scratch(g);
            PD_CUDA(cudaStreamSynchronize(g->stream));
        } catch (...) {
            g->stream = g->own_stream;
            pd_grid_destroy(g);
            throw;
        }
        *out = g;
    });
}

}  // extern "C"
