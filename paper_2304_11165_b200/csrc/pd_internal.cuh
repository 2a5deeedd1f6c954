// Internal declarations shared by the porediff_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "porediff_b200.h"

namespace pdb {

// Device allocations come from the device's stream-ordered memory pool with
// an unlimited release threshold, so memory freed by one grid / stepper /
// temporary is reused by the next without returning to the driver (grids are
// created and destroyed per FRAP probe and per run_simulation call; plain
// cudaMalloc/cudaFree cost tens of milliseconds at these sizes and synchronise
// the device). The allocation is complete before pd_malloc returns; pd_free
// waits for outstanding device work first, as cudaFree does.
inline void pool_init_once() {
    static thread_local int done_for = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (done_for == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_for = dev;
}
template <class T>
inline cudaError_t pd_malloc(T** p, size_t n) {
    pool_init_once();
    void* v = nullptr;
    cudaError_t e = cudaMallocAsync(&v, n, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    *p = static_cast<T*>(v);
    return e;
}
inline cudaError_t pd_free(void* p) {
    if (!p) return cudaSuccess;
    cudaDeviceSynchronize();
    const cudaError_t e = cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    return e;
}

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define PD_CUDA(x)                                                                       \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess)                                                           \
            ::pdb::fail(PD_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

void set_error(const std::string& msg);

template <class F>
int guarded(F&& f) {
    try {
        f();
        set_error("");
        return PD_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return PD_E_CUDA;
    }
}

// Chunk geometry per dimensionality (sparse_block_grid.hpp:33-35).
template <int D>
struct Geo {
    static constexpr int V = D == 3 ? 512 : 64;  // nodes per chunk
    static constexpr int W = V / 64;             // mask words per chunk
    static constexpr int FA = D == 3 ? 64 : 8;   // nodes per chunk face
    static constexpr int NH = 2 * D * FA;        // halo cells (face layers)
    static constexpr int TE = 10;                // staged tile edge (8 + 2 halo)
    static constexpr int TV = D == 3 ? 1000 : 100;
};

// Partial-reduction scratch (per-chunk mass / min / max, then pairwise tree).
struct ReduceScratch {
    double* part[3] = {nullptr, nullptr, nullptr};
    double* tmp_a[3] = {nullptr, nullptr, nullptr};
    double* tmp_b[3] = {nullptr, nullptr, nullptr};
    int64_t cap = 0;
};

}  // namespace pdb

struct pd_grid {
    int dims = 3, tbytes = 8, V = 512, W = 8, device = 0;
    int64_t size[3] = {1, 1, 1};
    double spacing[3] = {1, 1, 1};
    double cell_volume = 1.0;
    int64_t cc[3] = {1, 1, 1};
    int64_t table_size = 1;
    int64_t n_chunks = 0, active = 0;
    int32_t* d_keys = nullptr;
    uint64_t* d_masks = nullptr;
    int32_t* d_table = nullptr;  // chunk linear index -> ordinal, -1 absent
    std::vector<void*> cols;     // physical columns
    std::vector<char> col_ipc;   // column allocated with cudaMalloc (IPC-exportable)
    std::vector<int> column_of;  // logical property -> physical column
    cudaStream_t stream = nullptr;      // stream all work is issued on
    cudaStream_t own_stream = nullptr;  // the grid's own stream
    pdb::ReduceScratch red;
    double* d_row = nullptr;  // 3 doubles: mass, min, max
    uint64_t generation = 0;  // bumped by every host-visible write to a column
    std::vector<uint64_t> prop_ver;  // per logical property: bumped by each write to it
    // owners: the handle returned to the caller plus one per live stepper, so
    // a stepper destroyed after its grid's handle (any finaliser order) still
    // finds the grid; the storage is released when the last owner goes
    int refs = 1;
};

// Drops one owner of g; frees it when none is left (pd_grid.cu).
void grid_release(pd_grid* g);

// Records a write to logical property `prop` (all properties if prop < 0):
// steppers compare the versions of phi and D before stepping and rebuild
// their static predicates / march plan when either changed.
inline void note_write(pd_grid* g, int prop) {
    g->generation++;
    if (g->prop_ver.size() < g->column_of.size()) g->prop_ver.resize(g->column_of.size(), 0);
    if (prop < 0)
        for (auto& v : g->prop_ver) ++v;
    else if ((size_t)prop < g->prop_ver.size())
        ++g->prop_ver[(size_t)prop];
}
inline uint64_t prop_version(const pd_grid* g, int prop) {
    return (size_t)prop < g->prop_ver.size() ? g->prop_ver[(size_t)prop] : 0;
}

// A dense field on the device (pd_levelset.cu, pd_snapshot.cu).
struct pd_field {
    int dims = 3, tbytes = 8, device = 0;
    int64_t size[3] = {1, 1, 1};
    double spacing[3] = {1, 1, 1}, origin[3] = {0, 0, 0};
    int64_t n = 0;
    void* d = nullptr;
    cudaStream_t stream = nullptr;
};

namespace pdb {

// Chunk-level reductions (pd_grid.cu).
void ensure_scratch(pd_grid* g);
// Per-chunk sequential mass + left-preference min/max of an active-masked
// column into red.part[0..2] (solver.hpp:158-171, 282-301).
void launch_chunk_stats(pd_grid* g, const void* col, const uint64_t* masks);
// pairwise_sum (parallel.hpp:68-84) of red.part[0] and min/max fold of
// part[1..2] over ordinals; writes {mass*cell_volume, min, max} to dst
// (device) and, when flags != nullptr, ORs 4 into *flags if the mass is not
// finite. Empty grids produce {0, +inf, -inf}.
void launch_pairwise_finalize(pd_grid* g, double* dst, int* flags, int64_t begin = 0,
                              int64_t count = -1);
// max over active nodes of a column (solver.hpp:139-154) into red.part.
void launch_chunk_max(pd_grid* g, const void* col);

int device_of(const pd_grid* g);

// Arguments of one FTCS step launch (all pointers are device pointers).
template <class T>
struct StepArgs {
    const T* __restrict__ u;
    T* __restrict__ un;
    const T* __restrict__ d;
    const T* __restrict__ src;
    const uint64_t* __restrict__ active;
    const uint64_t* __restrict__ fluid;
    const uint64_t* __restrict__ sink;
    const int32_t* __restrict__ nbr;
    const int32_t* __restrict__ keys;
    int64_t size[3];
    T inv_dx2[3];
    T dt, neg_k, src_factor;
    T bcv[6];
    int dirichlet;  // bit (axis*2+side)
    int reaction;   // PD_REACTION_*
    double* p_mass;
    double* p_mn;
    double* p_mx;
    unsigned long long* bad_key;  // (ordinal << 10) | offset, atomicMin
    int* flags;                   // per step of the batch: 1 bad, 2 huge, 4 mass
    // "huge": |u_next| >= 2^e_huge, below which the step's total mass
    // (pairwise_sum * cell_volume over <= n_slots values) cannot overflow;
    // e_huge = 1022 - ceil(log2 n_slots) - max(0, ceil(log2 cell_volume))
    // (huge_hi: the same as a high-word threshold on the absolute value)
    double huge_abs;
    uint32_t huge_hi;
    int k;                        // step index within the batch
    int64_t ord0;                 // first chunk ordinal of the launch
};

// Warp-specialized march plan of the 3-D FP64 fast path (pd_march.cu).
struct MarchPlan {
    int32_t* d_stream = nullptr;   // owned chunk ordinals in schedule order
    int32_t* d_desc = nullptr;     // 8 ints per chunk: nbr[0..5], packed key, flags
    void* d_deff = nullptr;        // D (grid scalar type) on fluid nodes, -inf elsewhere (static per run)
    void* d_dv = nullptr;          // per chunk: uniform D_eff of kFlagUnif chunks (grid scalar type)
    int* d_counter = nullptr;      // per-step dynamic batch counters
    uint32_t* d_lm = nullptr;      // per chunk and lane: active / sink bits [c][32]
    uint32_t* d_ctx = nullptr;     // v30: packed chunk record [c][44]: lm[32] | desc[8] | dv | pad
    // v30: schedules with bit 31 set on uniform chunks (keyed by the plain schedule)
    std::vector<std::pair<const int32_t*, int32_t*>> flagged;
    int grid = 0;
    int64_t n = 0;
    bool ready = false;
    bool half = false;             // D_eff stored halved (face coefficient h_a + h_b, pd_march*.cu)
    struct Sub {  // sub-range schedules (overlapped multi-GPU stepping)
        int64_t begin = 0, end = 0, n = 0;
        int32_t* d_stream = nullptr;
        int* d_counter = nullptr;
    };
    std::vector<Sub> subs;
};
void march_build(pd_grid* g, const int32_t* d_nbr, const uint64_t* d_fluid, const uint64_t* d_sink,
                 const void* d_dcol, int dirichlet, int64_t begin, int64_t end, MarchPlan* plan);
int march_counters_per_step();
void march_free(MarchPlan* plan);
// fused halo push targets of one launch (pd_peer.cu)
struct PeerLaunch {
    double* un[2];         // lower / upper peer's u_next column base (null: none)
    const int32_t* ord;    // [n_chunks][2] peer ghost ordinal, -1 none
};
void march_launch(pd_grid* g, MarchPlan& plan, const StepArgs<double>& a, int reaction,
                  const PeerLaunch* pl = nullptr);
void march_push_flags(pd_grid* g, MarchPlan& p, const int32_t* d_ord);
// 3-D FP32 grids (pd_march32.cu)
bool march32_deff(pd_grid* g, const void* d_dcol, const uint64_t* d_fluid, void** out, bool* half);
void march32_launch(pd_grid* g, MarchPlan& p, const StepArgs<float>& a, int reaction);
// chunk schedule with bit 31 set on uniform chunks (pd_march.cu; built once per schedule)
const int32_t* march_flagged_schedule(pd_grid* g, MarchPlan& p, const int32_t* sched, int64_t n);
void march32_launch_sched(pd_grid* g, MarchPlan& p, const StepArgs<float>& a, int reaction, const int32_t* sched,
                          int64_t n, int* counter);
int32_t* march_schedule(pd_grid* g, int64_t begin, int64_t end);
MarchPlan::Sub& march_sub(pd_grid* g, MarchPlan& p, int64_t begin, int64_t end);
void march_launch_sched(pd_grid* g, MarchPlan& p, const StepArgs<double>& a, int reaction, const int32_t* sched,
                        int64_t n, int* counter, const PeerLaunch* pl = nullptr);

// Multi-GPU peer exchange state of a stepper (pd_peer.cu, pd_ftcs.cu): the
// step kernel pushes the boundary planes straight into the neighbours' ghost
// chunks; per-neighbour step counters in peer memory order the steps.
struct PeerState {
    bool on = false;
    bool side[2] = {false, false};   // lower / upper neighbour present
    void* cols[2][16] = {};          // neighbour's physical column bases
    unsigned* sync[2] = {};          // neighbour's counter words
    unsigned* d_sync = nullptr;      // own counters: [0] written by the lower, [1] by the upper neighbour
    int* d_err = nullptr;            // wait timed out
    int32_t* d_ord = nullptr;        // [n_chunks][2] neighbour ghost ordinal, -1 none
    uint32_t epoch = 0;              // steps taken since the handshake
    bool flags_dirty = false;
};
void peer_wait(cudaStream_t st, const PeerState& p);
void peer_signal(cudaStream_t st, const PeerState& p);
// pairwise_sum + left-preference min/max fold of caller arrays (n leaves)
// into dst[0..2] = {sum*cell_volume, min, max} (pd_grid.cu).
void launch_pairwise_arrays(pd_grid* g, const double* m, const double* a, const double* b, int64_t n,
                            double* dst, double* scratch);

// Grid construction helpers (pd_grid.cu).
void init_geometry(pd_grid* g, int dims, int tbytes, const int64_t* size, const double* spacing, int device);
void alloc_columns(pd_grid* g, int n_props);
void count_active(pd_grid* g);

// Sequential lexicographic (axis 0 fastest) double sum of the active nodes of
// a column inside the box [lo, hi) into *dst (device) — the run_frap region
// observer (analysis.hpp:211-219), pd_frap.cu.
void launch_box_sum(pd_grid* g, const void* col, const int64_t* lo, const int64_t* hi, double* dst);
void check_box(const pd_grid* g, const int64_t* lo, const int64_t* hi);

// Steady-state observers (pd_observe.cu).
void launch_absdiff_max(pd_grid* g, const void* a, const void* b, unsigned long long* out);
double plane_face_sum(pd_grid* g, const void* u, const void* d, const uint64_t* fluid, const int32_t* nbr,
                      int axis, int64_t layer, int64_t* faces);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace pdb
