// Fused multi-GPU halo exchange over peer memory (the
// reference paper's OpenFPM ghost_get). Rank r owns a z-slab of chunk layers
// plus one ghost layer per side. Instead of pack -> NCCL send/recv -> unpack
// after the step, the step kernel itself stores the new z=0 / z=7 plane of
// every boundary chunk into the neighbour's ghost chunk (ftcs_march14_kernel,
// push_pair14: NVLink P2P stores issued tile by tile while the rest of the
// slab is computed). Step ordering uses one counter per neighbour in the
// receiver's memory:
//
//   before step e:  wait until both neighbours have completed e steps — then
//                   the ghost u of step e has landed (their step e-1 pushes)
//                   and they no longer read the ghost column this step's
//                   pushes overwrite (their u of step e-1);
//   after step e:   __threadfence_system by every pushing thread (kernel end),
//                   then raise the neighbours' counters to e+1.
//
// Both sides swap u / u_next in lockstep, so the neighbour's u_next physical
// column has the same index as ours. Waits are bounded (30 s, then an error
// flag that pd_stepper_status reports) so a lost peer never hangs the device.
// Columns are moved to cudaMalloc allocations (IPC-exportable) for the
// cross-process case; within one process the raw pointers are used directly.
#include <cstring>

#include "pd_internal.cuh"

namespace pdb {

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
    return t;
}

// err[0]: timeout flag; err + 8 B: total wait ns and wait count (the per-step
// barrier time of the fused exchange, pd_stepper_peer_stats)
__global__ void peer_wait_kernel(const unsigned* sync, int need_lo, int need_hi, unsigned epoch, int* err) {
    const unsigned long long t0 = global_ns();
    for (int side = 0; side < 2; ++side) {
        if (!(side ? need_hi : need_lo)) continue;
        while ((int)(ld_acquire_sys(sync + side) - epoch) < 0) {
            __nanosleep(200);
            if (global_ns() - t0 > 30000000000ull) {
                atomicOr(err, 1);
                return;
            }
        }
    }
    unsigned long long* st = reinterpret_cast<unsigned long long*>(err) + 1;
    st[0] += global_ns() - t0;
    st[1] += 1;
}

__global__ void peer_signal_kernel(unsigned* lo, unsigned* hi, unsigned v) {
    __threadfence_system();
    if (lo) st_release_sys(lo, v);
    if (hi) st_release_sys(hi, v);
}

}  // namespace

void peer_wait(cudaStream_t st, const PeerState& p) {
    peer_wait_kernel<<<1, 1, 0, st>>>(p.d_sync, p.side[0], p.side[1], p.epoch, p.d_err);
    PD_CUDA(cudaGetLastError());
}

void peer_signal(cudaStream_t st, const PeerState& p) {
    // lower neighbour: its word 1 (written by its upper neighbour); upper: word 0
    peer_signal_kernel<<<1, 1, 0, st>>>(p.side[0] ? p.sync[0] + 1 : nullptr, p.side[1] ? p.sync[1] : nullptr,
                                        p.epoch + 1);
    PD_CUDA(cudaGetLastError());
}

}  // namespace pdb

using namespace pdb;

extern "C" {

int pd_grid_make_shareable(pd_grid* g) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        g->col_ipc.resize(g->cols.size(), 0);
        const size_t bytes = (size_t)std::max<int64_t>(1, g->n_chunks) * (size_t)g->V * (size_t)g->tbytes;
        for (size_t i = 0; i < g->cols.size(); ++i) {
            if (g->col_ipc[i]) continue;
            void* p = nullptr;
            PD_CUDA(cudaMalloc(&p, bytes));
            PD_CUDA(cudaMemcpyAsync(p, g->cols[i], bytes, cudaMemcpyDeviceToDevice, g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            pd_free(g->cols[i]);
            g->cols[i] = p;
            g->col_ipc[i] = 1;
        }
        g->generation++;  // same data, new addresses
    });
}

int pd_grid_ipc_handles(pd_grid* g, void* out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        for (size_t i = 0; i < g->cols.size(); ++i) {
            if (i >= g->col_ipc.size() || !g->col_ipc[i])
                fail(PD_E_INPUT, "grid columns are not shareable (call pd_grid_make_shareable)");
            cudaIpcMemHandle_t h;
            PD_CUDA(cudaIpcGetMemHandle(&h, g->cols[i]));
            std::memcpy(static_cast<char*>(out) + i * sizeof h, &h, sizeof h);
        }
    });
}

int pd_grid_column_ptrs(pd_grid* g, void** out) {
    return guarded([&] {
        for (size_t i = 0; i < g->cols.size(); ++i) out[i] = g->cols[i];
    });
}

int pd_ipc_open(const void* handle, int device, void** ptr) {
    return guarded([&] {
        DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        PD_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int pd_ipc_close(void* ptr, int device) {
    return guarded([&] {
        DeviceGuard dg(device);
        PD_CUDA(cudaIpcCloseMemHandle(ptr));
    });
}

int pd_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

}  // extern "C"
