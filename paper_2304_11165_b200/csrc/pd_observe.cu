// Steady-state observers of the FTCS stepper (north_star (3): "warp-level
// reductions feed the steady-state / convergence and flux norms used for
// effective diffusivity and tortuosity").
//
// The reference has no flux-based estimator (its only D_eff path is the FRAP
// fit, analysis.hpp:160-309), so these observers have no reference
// counterpart: they are checked against a NumPy restatement
// (tests/test_observe.py), "parity unpinned".
//
// * convergence norm: max over active nodes of |u_new - u_old| at a recorded
//   step. Non-negative doubles order like their bit patterns, so a warp
//   max-reduction plus one 64-bit atomicMax per warp is exact and order-free
//   (a NaN difference propagates as the largest pattern).
// * plane flux: the total diffusive flux through the plane between node
//   layers L and L+1 of an axis, with the reference's face coefficient
//   dh = (d_a + d_b) * T(0.5) in T arithmetic (solver.hpp:430-433): faces
//   whose far side is not fluid are substituted in the reference (no flux).
//   F = -sum_faces dh * (u_{L+1} - u_L) / h_axis * (area of one face); the
//   per-chunk face sums are folded sequentially in offset order and the
//   chunk sums pairwise on the host (fixed order: reproducible bits).
#include <algorithm>
#include <cstring>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {
namespace {

template <class T>
__global__ void __launch_bounds__(256) absdiff_max_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                          const uint64_t* __restrict__ masks, int64_t n_slots,
                                                          unsigned long long* __restrict__ out) {
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_slots;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!((masks[i >> 6] >> (i & 63)) & 1ull)) continue;
        const double d = fabs((double)a[i] - (double)b[i]);
        unsigned long long bits = (unsigned long long)__double_as_longlong(d);
        if (d != d) bits = 0x7FFFFFFFFFFFFFFFull;  // NaN: largest pattern
        best = best > bits ? best : bits;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
        best = best > v ? best : v;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

// One CTA per chunk crossing the plane: 64 threads, one per face (the other
// two coordinates), each computing its face term; thread 0 folds the 64 terms
// in ascending offset order.
template <class T, int D>
__global__ void plane_flux_kernel(const T* __restrict__ u, const T* __restrict__ d,
                                  const uint64_t* __restrict__ fluid, const int32_t* __restrict__ nbr,
                                  const int32_t* __restrict__ chunks, int64_t n, int axis, int local,
                                  double* __restrict__ part) {
    constexpr int V = D == 3 ? 512 : 64, W = V / 64, NF = D == 3 ? 64 : 8;
    __shared__ double terms[64];
    const int64_t k = blockIdx.x;
    if (k >= n) return;
    const int32_t c = chunks[k];
    const int t = threadIdx.x;
    double term = 0.0;
    if (t < NF) {
        // coordinates of face t: the two (one) other axes, ascending
        int idx[3] = {0, 0, 0};
        int r = t;
        for (int a = 0; a < D; ++a) {
            if (a == axis) continue;
            idx[a] = r & 7;
            r >>= 3;
        }
        idx[axis] = local;
        int off = 0;
        for (int a = D - 1; a >= 0; --a) off = (off << 3) | idx[a];
        const bool fa = (fluid[(int64_t)c * W + (off >> 6)] >> (off & 63)) & 1ull;
        int c2 = c, off2;
        if (local < 7) {
            off2 = off + (1 << (3 * axis));
        } else {
            c2 = nbr[(int64_t)c * 2 * D + 2 * axis + 1];
            off2 = off - 7 * (1 << (3 * axis));
        }
        const bool fb = c2 >= 0 && ((fluid[(int64_t)c2 * W + (off2 >> 6)] >> (off2 & 63)) & 1ull);
        if (fa && fb) {
            const T ua = u[(int64_t)c * V + off], ub = u[(int64_t)c2 * V + off2];
            const T da = d[(int64_t)c * V + off], db = d[(int64_t)c2 * V + off2];
            const T dh = (da + db) * T(0.5);
            term = (double)(dh * (ub - ua));
        }
    }
    if (t < 64) terms[t] = term;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int i = 0; i < NF; ++i) s += terms[i];
        part[k] = s;
    }
}

}  // namespace

void launch_absdiff_max(pd_grid* g, const void* a, const void* b, unsigned long long* out) {
    const int64_t slots = g->n_chunks * g->V;
    if (slots == 0) return;
    const unsigned blocks = (unsigned)std::min<int64_t>((slots + 255) / 256, 148 * 16);
    if (g->tbytes == 8)
        absdiff_max_kernel<double><<<blocks, 256, 0, g->stream>>>((const double*)a, (const double*)b, g->d_masks,
                                                                  slots, out);
    else
        absdiff_max_kernel<float><<<blocks, 256, 0, g->stream>>>((const float*)a, (const float*)b, g->d_masks,
                                                                 slots, out);
    PD_CUDA(cudaGetLastError());
}

// Sum of dh * (u_{L+1} - u_L) over the fluid faces between layers L, L+1 of
// `axis` (global layer index L in [0, size[axis] - 2]), pairwise over chunks
// in ordinal order; faces counted into *faces.
double plane_face_sum(pd_grid* g, const void* u, const void* d, const uint64_t* fluid, const int32_t* nbr,
                      int axis, int64_t layer, int64_t* faces) {
    std::vector<int32_t> keys((size_t)g->n_chunks * g->dims);
    if (g->n_chunks)
        PD_CUDA(cudaMemcpyAsync(keys.data(), g->d_keys, sizeof(int32_t) * keys.size(), cudaMemcpyDeviceToHost,
                                g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    std::vector<int32_t> sel;
    for (int64_t c = 0; c < g->n_chunks; ++c)
        if (keys[(size_t)(c * g->dims + axis)] == (int32_t)(layer >> 3)) sel.push_back((int32_t)c);
    *faces = 0;
    if (sel.empty()) return 0.0;
    int32_t* d_sel = nullptr;
    double* d_part = nullptr;
    PD_CUDA(pd_malloc(&d_sel, sizeof(int32_t) * sel.size()));
    struct Free {
        void* a;
        void* b;
        ~Free() {
            pd_free(a);
            pd_free(b);
        }
    } fr{d_sel, nullptr};
    PD_CUDA(pd_malloc(&d_part, sizeof(double) * sel.size()));
    fr.b = d_part;
    PD_CUDA(cudaMemcpyAsync(d_sel, sel.data(), sizeof(int32_t) * sel.size(), cudaMemcpyHostToDevice, g->stream));
    const int local = (int)(layer & 7);
    const unsigned nb = (unsigned)sel.size();
    if (g->tbytes == 8 && g->dims == 3)
        plane_flux_kernel<double, 3><<<nb, 64, 0, g->stream>>>((const double*)u, (const double*)d, fluid, nbr, d_sel,
                                                              (int64_t)nb, axis, local, d_part);
    else if (g->tbytes == 8)
        plane_flux_kernel<double, 2><<<nb, 64, 0, g->stream>>>((const double*)u, (const double*)d, fluid, nbr, d_sel,
                                                              (int64_t)nb, axis, local, d_part);
    else if (g->dims == 3)
        plane_flux_kernel<float, 3><<<nb, 64, 0, g->stream>>>((const float*)u, (const float*)d, fluid, nbr, d_sel,
                                                             (int64_t)nb, axis, local, d_part);
    else
        plane_flux_kernel<float, 2><<<nb, 64, 0, g->stream>>>((const float*)u, (const float*)d, fluid, nbr, d_sel,
                                                             (int64_t)nb, axis, local, d_part);
    PD_CUDA(cudaGetLastError());
    std::vector<double> part(sel.size());
    PD_CUDA(cudaMemcpyAsync(part.data(), d_part, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, g->stream));
    PD_CUDA(cudaStreamSynchronize(g->stream));
    // parallel.hpp:68-84's level-by-level pairwise tree (odd tail carried)
    while (part.size() > 1) {
        std::vector<double> nx((part.size() + 1) / 2);
        for (size_t i = 0; i + 1 < part.size(); i += 2) nx[i / 2] = part[i] + part[i + 1];
        if (part.size() & 1) nx.back() = part.back();
        part.swap(nx);
    }
    *faces = (int64_t)sel.size() * (g->dims == 3 ? 64 : 8);
    return part[0];
}

}  // namespace pdb
