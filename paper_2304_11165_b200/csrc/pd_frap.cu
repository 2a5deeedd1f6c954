// FRAP experiment support on the device (reference
// analysis.hpp:147-225): the unobstructed free-box grid, the bleach initial
// condition, and the bleached-region mass observer.
//
// Parity: the reference observer sums u over the bleach box in lexicographic
// order, axis 0 fastest, skipping inactive nodes (analysis.hpp:108-125,
// 211-219) — a sequential double sum whose rounding depends on that order. It
// is reproduced exactly: one CTA gathers the box in 1024-node tiles (coalesced
// along x through the chunk table) and one thread folds each tile in order.
#include <algorithm>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {

constexpr int kBoxThreads = 256;
constexpr int kBoxTile = 1024;

struct BoxArgs {
    int64_t lo[3], n[3];  // box origin and extent (n[2] = 1 in 2-D)
    int64_t cc0, cc1;     // chunk-table extents (x, y)
    int64_t count;        // n0*n1*n2
};

template <class T, int D>
__global__ void __launch_bounds__(kBoxThreads)
    box_sum_kernel(const T* __restrict__ col, const uint64_t* __restrict__ masks,
                   const int32_t* __restrict__ table, BoxArgs b, double* __restrict__ out) {
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    __shared__ double val[kBoxTile];
    __shared__ unsigned char use[kBoxTile];
    double m = 0.0;  // thread 0's running sum (analysis.hpp:213)
    for (int64_t base = 0; base < b.count; base += kBoxTile) {
        for (int k = threadIdx.x; k < kBoxTile; k += kBoxThreads) {
            const int64_t f = base + k;
            bool act = false;
            double v = 0.0;
            if (f < b.count) {
                const int64_t x = b.lo[0] + f % b.n[0];
                const int64_t r = f / b.n[0];
                const int64_t y = b.lo[1] + r % b.n[1];
                const int64_t z = D == 3 ? b.lo[2] + r / b.n[1] : 0;
                int64_t lin = (y >> 3) * b.cc0 + (x >> 3);
                int off = (int)(((y & 7) << 3) | (x & 7));
                if (D == 3) {
                    lin += (z >> 3) * b.cc0 * b.cc1;
                    off |= (int)((z & 7) << 6);
                }
                const int32_t ord = table[lin];
                if (ord >= 0 && ((masks[(int64_t)ord * W + (off >> 6)] >> (off & 63)) & 1ull)) {
                    act = true;
                    v = (double)col[(int64_t)ord * V + off];
                }
            }
            val[k] = v;
            use[k] = act;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int lim = b.count - base < kBoxTile ? (int)(b.count - base) : kBoxTile;
            for (int k = 0; k < lim; ++k)
                if (use[k]) m += val[k];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = m;
}

template <class T, int D>
__global__ void __launch_bounds__(Geo<D>::V)
    frap_init_kernel(T* __restrict__ u, T* __restrict__ d, const uint64_t* __restrict__ masks,
                     const int32_t* __restrict__ keys, BoxArgs b, T dval,
                     unsigned long long* __restrict__ counts) {
    // analysis.hpp:179-186: u = in ? 0 : 1, D = T(d_molecular) on active nodes
    constexpr int V = Geo<D>::V, W = Geo<D>::W;
    __shared__ int s_region, s_phase;
    if (threadIdx.x == 0) s_region = s_phase = 0;
    __syncthreads();
    const int64_t i = blockIdx.x;
    const int off = threadIdx.x;
    if ((masks[i * W + (off >> 6)] >> (off & 63)) & 1ull) {
        const int64_t x = ((int64_t)keys[i * D] << 3) | (off & 7);
        const int64_t y = ((int64_t)keys[i * D + 1] << 3) | ((off >> 3) & 7);
        bool in = x >= b.lo[0] && x < b.lo[0] + b.n[0] && y >= b.lo[1] && y < b.lo[1] + b.n[1];
        if (D == 3) {
            const int64_t z = ((int64_t)keys[i * D + 2] << 3) | ((off >> 6) & 7);
            in = in && z >= b.lo[2] && z < b.lo[2] + b.n[2];
        }
        u[i * V + off] = in ? T(0) : T(1);
        d[i * V + off] = dval;
        if (in) atomicAdd(&s_region, 1);
        atomicAdd(&s_phase, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(&counts[0], (unsigned long long)s_region);
        atomicAdd(&counts[1], (unsigned long long)s_phase);
    }
}

BoxArgs box_args(const pd_grid* g, const int64_t* lo, const int64_t* hi) {
    BoxArgs b{};
    b.count = 1;
    for (int a = 0; a < 3; ++a) {
        if (a < g->dims) {
            b.lo[a] = lo[a];
            b.n[a] = std::max<int64_t>(0, hi[a] - lo[a]);
        } else {
            b.lo[a] = 0;
            b.n[a] = 1;
        }
        b.count *= b.n[a];
    }
    b.cc0 = g->cc[0];
    b.cc1 = g->cc[1];
    return b;
}

void launch_box_sum(pd_grid* g, const void* col, const int64_t* lo, const int64_t* hi, double* dst) {
    const BoxArgs b = box_args(g, lo, hi);
    if (g->tbytes == 8 && g->dims == 3)
        box_sum_kernel<double, 3><<<1, kBoxThreads, 0, g->stream>>>((const double*)col, g->d_masks,
                                                                    g->d_table, b, dst);
    else if (g->tbytes == 8)
        box_sum_kernel<double, 2><<<1, kBoxThreads, 0, g->stream>>>((const double*)col, g->d_masks,
                                                                    g->d_table, b, dst);
    else if (g->dims == 3)
        box_sum_kernel<float, 3><<<1, kBoxThreads, 0, g->stream>>>((const float*)col, g->d_masks,
                                                                   g->d_table, b, dst);
    else
        box_sum_kernel<float, 2><<<1, kBoxThreads, 0, g->stream>>>((const float*)col, g->d_masks,
                                                                   g->d_table, b, dst);
    PD_CUDA(cudaGetLastError());
}

void check_box(const pd_grid* g, const int64_t* lo, const int64_t* hi) {
    for (int a = 0; a < g->dims; ++a)
        if (lo[a] < 0 || hi[a] > g->size[a] || lo[a] > hi[a])
            fail(PD_E_BOUNDS, "box outside grid on axis " + std::to_string(a));
}

}  // namespace pdb

using namespace pdb;

extern "C" {

int pd_grid_box_sum(pd_grid* g, int prop, const int64_t* lo, const int64_t* hi, double* out) {
    return guarded([&] {
        if (prop < 0 || prop >= (int)g->column_of.size()) fail(PD_E_PROPERTY, "unknown property index");
        check_box(g, lo, hi);
        DeviceGuard dg(g->device);
        const void* col = g->cols[(size_t)g->column_of[(size_t)prop]];
        launch_box_sum(g, col, lo, hi, g->d_row + 3);
        PD_CUDA(cudaMemcpyAsync(out, g->d_row + 3, sizeof(double), cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int pd_grid_frap_init(pd_grid* g, int prop_u, int prop_d, const int64_t* lo, const int64_t* hi,
                      double d_molecular, int64_t* region, int64_t* phase) {
    return guarded([&] {
        for (int p : {prop_u, prop_d})
            if (p < 0 || p >= (int)g->column_of.size()) fail(PD_E_PROPERTY, "unknown property index");
        DeviceGuard dg(g->device);
        unsigned long long* d_counts = nullptr;
        PD_CUDA(pd_malloc(&d_counts, 2 * sizeof(unsigned long long)));
        try {
            PD_CUDA(cudaMemsetAsync(d_counts, 0, 2 * sizeof(unsigned long long), g->stream));
            const BoxArgs b = box_args(g, lo, hi);
            void* u = g->cols[(size_t)g->column_of[(size_t)prop_u]];
            void* d = g->cols[(size_t)g->column_of[(size_t)prop_d]];
            const unsigned nb = (unsigned)g->n_chunks;
            if (nb > 0) {
                if (g->tbytes == 8 && g->dims == 3)
                    frap_init_kernel<double, 3><<<nb, 512, 0, g->stream>>>((double*)u, (double*)d, g->d_masks,
                                                                          g->d_keys, b, d_molecular, d_counts);
                else if (g->tbytes == 8)
                    frap_init_kernel<double, 2><<<nb, 64, 0, g->stream>>>((double*)u, (double*)d, g->d_masks,
                                                                         g->d_keys, b, d_molecular, d_counts);
                else if (g->dims == 3)
                    frap_init_kernel<float, 3><<<nb, 512, 0, g->stream>>>((float*)u, (float*)d, g->d_masks,
                                                                         g->d_keys, b, (float)d_molecular,
                                                                         d_counts);
                else
                    frap_init_kernel<float, 2><<<nb, 64, 0, g->stream>>>((float*)u, (float*)d, g->d_masks,
                                                                        g->d_keys, b, (float)d_molecular,
                                                                        d_counts);
                PD_CUDA(cudaGetLastError());
            }
            unsigned long long h[2] = {0, 0};
            PD_CUDA(cudaMemcpyAsync(h, d_counts, sizeof h, cudaMemcpyDeviceToHost, g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            *region = (int64_t)h[0];
            *phase = (int64_t)h[1];
            note_write(g, -1);
        } catch (...) {
            pd_free(d_counts);
            throw;
        }
        pd_free(d_counts);
    });
}

int pd_grid_create_full(int dims, int scalar_bytes, const int64_t* size, const double* spacing, int n_props,
                        int prop_phi, double phi_value, int device, pd_grid** out) {
    return guarded([&] {
        *out = nullptr;
        if (dims != 2 && dims != 3) fail(PD_E_INPUT, "dims must be 2 or 3");
        // every node active (build_free_box_grid, analysis.hpp:147-153):
        // chunks in ascending linear index, partial chunks at the far faces
        int64_t cc[3] = {1, 1, 1};
        for (int a = 0; a < dims; ++a) {
            if (size[a] < 1) fail(PD_E_INPUT, "grid size must be positive");
            cc[a] = (size[a] + 7) / 8;
        }
        const int W = dims == 3 ? 8 : 1;
        const int64_t n = cc[0] * cc[1] * cc[2];
        std::vector<int32_t> keys((size_t)(n * dims));
        std::vector<uint64_t> masks((size_t)(n * W), 0ull);
        int64_t i = 0;
        for (int64_t kz = 0; kz < cc[2]; ++kz)
            for (int64_t ky = 0; ky < cc[1]; ++ky)
                for (int64_t kx = 0; kx < cc[0]; ++kx, ++i) {
                    keys[(size_t)(i * dims)] = (int32_t)kx;
                    keys[(size_t)(i * dims + 1)] = (int32_t)ky;
                    if (dims == 3) keys[(size_t)(i * dims + 2)] = (int32_t)kz;
                    const int V = dims == 3 ? 512 : 64;
                    for (int off = 0; off < V; ++off) {
                        const int64_t x = kx * 8 + (off & 7), y = ky * 8 + ((off >> 3) & 7);
                        const int64_t z = dims == 3 ? kz * 8 + (off >> 6) : 0;
                        if (x < size[0] && y < size[1] && (dims == 2 || z < size[2]))
                            masks[(size_t)(i * W + (off >> 6))] |= 1ull << (off & 63);
                    }
                }
        pd_grid* g = nullptr;
        int rc = pd_grid_create(dims, scalar_bytes, size, spacing, n, keys.data(), masks.data(), n_props, device, &g);
        if (rc != PD_OK) fail(rc, pd_last_error());
        if (prop_phi >= 0) {
            rc = pd_grid_fill_const(g, prop_phi, phi_value);
            if (rc != PD_OK) {
                const std::string m = pd_last_error();
                pd_grid_destroy(g);
                fail(rc, m);
            }
        }
        *out = g;
    });
}

}  // extern "C"
