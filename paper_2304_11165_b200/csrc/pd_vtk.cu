// Legacy ASCII VTK export streamed from the device (
// reference vtk.hpp:57-143, scalar_text.hpp:20-28). Byte-identical to the
// reference writer: the same header lines, then every point-data array as one
// format_scalar text per node ("%.17g" / "%.9g", "nan") and the int mask.
//
// The text is produced on the device in batches of lattice nodes:
//   vtk_format_kernel   one thread per node: fetch the value (dense array, or
//                       the sparse grid's chunk table + mask + column for
//                       vtk_from_sparse, blank for inactive nodes), format it
//                       exactly (pd_format.cuh) into a 32-B slot + length
//   cub ExclusiveSum    byte offsets of the node texts
//   vtk_compact_kernel  slots -> contiguous text
// and the batch's text is copied to a pinned buffer and written by the host
// while the device formats the next batch (two buffers, one event each).
#include <cub/device/device_scan.cuh>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pd_format.cuh"
#include "pd_internal.cuh"

namespace pdb {

namespace {

constexpr int kSlot = 32;
constexpr int64_t kVtkBatch = int64_t{1} << 22;  // lattice nodes per batch

enum VtkKind { kDense = 0, kSparse = 1, kSparseMask = 2, kDenseInt = 3 };

struct VtkSrc {
    int kind = kDense;
    int tbytes = 8;
    const void* p = nullptr;  // dense values (p[f - base]) or the sparse column
    int64_t base = 0;
    const int32_t* table = nullptr;
    const uint64_t* masks = nullptr;
    int64_t size0 = 1, size1 = 1, cc0 = 1, cc1 = 1;
    int dims = 3;
    double blank = 0.0;
};

// vtk_from_sparse's lookup (sparse_block_grid.hpp:93-109 key / offset rules):
// slot of lattice node f, false if the node is not active.
__device__ __forceinline__ bool sparse_slot(const VtkSrc& s, int64_t f, int64_t& slot) {
    const int64_t x = f % s.size0;
    const int64_t r = f / s.size0;
    int64_t y, z, lin;
    int off;
    if (s.dims == 3) {
        y = r % s.size1;
        z = r / s.size1;
        lin = (x >> 3) + s.cc0 * ((y >> 3) + s.cc1 * (z >> 3));
        off = (int)(((z & 7) << 6) | ((y & 7) << 3) | (x & 7));
    } else {
        y = r;
        lin = (x >> 3) + s.cc0 * (y >> 3);
        off = (int)(((y & 7) << 3) | (x & 7));
    }
    const int32_t ord = s.table[lin];
    if (ord < 0) return false;
    const int W = s.dims == 3 ? 8 : 1, V = s.dims == 3 ? 512 : 64;
    if (!((s.masks[(int64_t)ord * W + (off >> 6)] >> (off & 63)) & 1u)) return false;
    slot = (int64_t)ord * V + off;
    return true;
}

__device__ __forceinline__ double load_t(const void* p, int64_t i, int tbytes) {
    return tbytes == 8 ? static_cast<const double*>(p)[i] : (double)static_cast<const float*>(p)[i];
}

__global__ void vtk_format_kernel(VtkSrc s, int64_t f0, int64_t n, char* __restrict__ slots,
                                  uint32_t* __restrict__ lens) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t f = f0 + i;
    union {
        char c[kSlot];
        uint4 v[2];
    } t;
    int len;
    const int P = s.tbytes == 8 ? 17 : 9;
    switch (s.kind) {
        case kDense:
            len = fmt::format_g(load_t(s.p, f - s.base, s.tbytes), P, t.c);
            break;
        case kSparse: {
            int64_t slot;
            double v = s.tbytes == 8 ? s.blank : (double)(float)s.blank;
            if (sparse_slot(s, f, slot)) v = load_t(s.p, slot, s.tbytes);
            len = fmt::format_g(v, P, t.c);
            break;
        }
        case kSparseMask: {
            int64_t slot;
            t.c[0] = sparse_slot(s, f, slot) ? '1' : '0';
            len = 1;
            break;
        }
        default:
            len = fmt::format_int(static_cast<const int32_t*>(s.p)[f - s.base], t.c);
            break;
    }
    t.c[len++] = '\n';
    uint4* d = reinterpret_cast<uint4*>(slots + i * kSlot);
    d[0] = t.v[0];
    d[1] = t.v[1];
    lens[i] = (uint32_t)len;
}

__global__ void vtk_compact_kernel(const char* __restrict__ slots, const uint32_t* __restrict__ lens,
                                   const uint32_t* __restrict__ offs, int64_t n, char* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const char* s = slots + i * kSlot;
    char* o = out + offs[i];
    const int len = (int)lens[i];
    for (int k = 0; k < len; ++k) o[k] = s[k];
}

// densify one property (vtk_from_sparse, vtk.hpp:115-143) into a device array
__global__ void vtk_densify_kernel(VtkSrc s, int64_t n, void* __restrict__ values, int32_t* __restrict__ mask) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n) return;
    int64_t slot;
    const bool act = sparse_slot(s, f, slot);
    if (values) {
        if (s.tbytes == 8)
            static_cast<double*>(values)[f] = act ? static_cast<const double*>(s.p)[slot] : s.blank;
        else
            static_cast<float*>(values)[f] = act ? static_cast<const float*>(s.p)[slot] : (float)s.blank;
    }
    if (mask) mask[f] = act ? 1 : 0;
}

std::string fmt_host(double v, int P) {
    char b[kSlot];
    const int n = fmt::format_g(v, P, b);
    return std::string(b, (size_t)n);
}

// write_vtk's dataset checks that the C ABI can see (vtk.hpp:46-75)
void check_names(const char* const* names, int n_arrays, bool has_mask) {
    if (n_arrays == 0 && !has_mask) fail(PD_E_INPUT, "VTK dataset has no arrays to write");
    for (int i = 0; i < n_arrays; ++i) {
        const std::string nm = names[i] ? names[i] : "";
        if (nm.empty()) fail(PD_E_INPUT, "VTK array name must not be empty");
        for (char c : nm)
            if (c == ' ' || c == '\t' || c == '\n' || c == '\r')
                fail(PD_E_INPUT, "VTK array name '" + nm + "' contains whitespace");
    }
    for (int i = 0; i < n_arrays; ++i)
        for (int k = i + 1; k < n_arrays; ++k)
            if (std::strcmp(names[i], names[k]) == 0)
                fail(PD_E_INPUT, "duplicate VTK array name '" + std::string(names[i]) + "'");
}

class VtkStream {
  public:
    VtkStream(const char* path, int64_t nodes, cudaStream_t st) : path_(path), n_(nodes), st_(st) {
        f_ = std::fopen(path, "wb");
        if (!f_) fail(PD_E_IO, "cannot open '" + path_ + "' for writing");
        nb_ = std::max<int64_t>(1, std::min<int64_t>(kVtkBatch, n_));
        PD_CUDA(pd_malloc(&slots_, (size_t)nb_ * kSlot));
        PD_CUDA(pd_malloc(&lens_, (size_t)nb_ * 4));
        PD_CUDA(pd_malloc(&offs_, (size_t)nb_ * 4));
        PD_CUDA(pd_malloc(&out_, (size_t)nb_ * fmt::kMaxText));
        PD_CUDA(pd_malloc(&stage_, (size_t)nb_ * 8));
        PD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes_, lens_, offs_, (int)nb_, st_));
        PD_CUDA(pd_malloc(&tmp_, std::max<size_t>(tmp_bytes_, 16)));
        for (int k = 0; k < 2; ++k) {
            PD_CUDA(cudaMallocHost(&host_[k], (size_t)nb_ * fmt::kMaxText));
            PD_CUDA(cudaEventCreateWithFlags(&ev_[k], cudaEventDisableTiming));
        }
        PD_CUDA(cudaMallocHost(&tot_, 4 * sizeof(uint32_t)));
    }
    ~VtkStream() {
        if (f_) std::fclose(f_);
        cudaStreamSynchronize(st_);
        for (void* p : {(void*)slots_, (void*)lens_, (void*)offs_, (void*)out_, (void*)stage_, tmp_}) pd_free(p);
        for (int k = 0; k < 2; ++k) {
            if (host_[k]) cudaFreeHost(host_[k]);
            if (ev_[k]) cudaEventDestroy(ev_[k]);
        }
        if (tot_) cudaFreeHost(tot_);
    }

    void text(const std::string& s) {
        flush();
        put(s.data(), s.size());
    }

    // one point-data array over the lattice; host_values: stage from the host
    void array(VtkSrc s, const void* host_values, int elem_bytes) {
        for (int64_t f0 = 0; f0 < n_; f0 += nb_) {
            const int64_t nb = std::min(nb_, n_ - f0);
            const int k = batch_++ & 1;
            VtkSrc b = s;
            if (host_values) {
                PD_CUDA(cudaMemcpyAsync(stage_, static_cast<const char*>(host_values) + f0 * elem_bytes,
                                        (size_t)(nb * elem_bytes), cudaMemcpyHostToDevice, st_));
                b.p = stage_;
                b.base = f0;
            }
            const unsigned blocks = (unsigned)((nb + 255) / 256);
            vtk_format_kernel<<<blocks, 256, 0, st_>>>(b, f0, nb, slots_, lens_);
            PD_CUDA(cudaGetLastError());
            PD_CUDA(cub::DeviceScan::ExclusiveSum(tmp_, tmp_bytes_, lens_, offs_, (int)nb, st_));
            vtk_compact_kernel<<<blocks, 256, 0, st_>>>(slots_, lens_, offs_, nb, out_);
            PD_CUDA(cudaGetLastError());
            // wait for the previous batch's host write before reusing its buffer
            flush();
            PD_CUDA(cudaMemcpyAsync(tot_ + 2 * k, offs_ + nb - 1, 4, cudaMemcpyDeviceToHost, st_));
            PD_CUDA(cudaMemcpyAsync(tot_ + 2 * k + 1, lens_ + nb - 1, 4, cudaMemcpyDeviceToHost, st_));
            PD_CUDA(cudaMemcpyAsync(host_[k], out_, (size_t)nb * fmt::kMaxText, cudaMemcpyDeviceToHost, st_));
            PD_CUDA(cudaEventRecord(ev_[k], st_));
            pending_ = k;
        }
    }

    void finish() {
        flush();
        if (std::fflush(f_) != 0) fail(PD_E_IO, "write to '" + path_ + "' failed");
    }

  private:
    void put(const void* p, size_t n) {
        if (n && std::fwrite(p, 1, n, f_) != n) fail(PD_E_IO, "write to '" + path_ + "' failed");
    }
    void flush() {
        if (pending_ < 0) return;
        const int k = pending_;
        pending_ = -1;
        PD_CUDA(cudaEventSynchronize(ev_[k]));
        put(host_[k], (size_t)tot_[2 * k] + tot_[2 * k + 1]);
    }

    std::string path_;
    int64_t n_, nb_ = 1;
    cudaStream_t st_;
    FILE* f_ = nullptr;
    char* slots_ = nullptr;
    uint32_t* lens_ = nullptr;
    uint32_t* offs_ = nullptr;
    char* out_ = nullptr;
    void* stage_ = nullptr;
    void* tmp_ = nullptr;
    size_t tmp_bytes_ = 0;
    char* host_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    uint32_t* tot_ = nullptr;
    int pending_ = -1;
    int64_t batch_ = 0;
};

// header lines (vtk.hpp:80-97)
std::string vtk_header(const char* title, int dims, const int64_t* size, const double* spacing,
                       const double* origin, int64_t n) {
    int64_t d[3] = {1, 1, 1};
    double o[3] = {0.0, 0.0, 0.0}, h[3] = {1.0, 1.0, 1.0};
    for (int a = 0; a < dims; ++a) {
        d[a] = size[a];
        o[a] = origin[a];
        h[a] = spacing[a];
    }
    std::string s = "# vtk DataFile Version 3.0\n";
    s += (title ? title : "porediff field export");
    s += "\nASCII\nDATASET STRUCTURED_POINTS\n";
    s += "DIMENSIONS " + std::to_string(d[0]) + ' ' + std::to_string(d[1]) + ' ' + std::to_string(d[2]) + '\n';
    s += "ORIGIN " + fmt_host(o[0], 17) + ' ' + fmt_host(o[1], 17) + ' ' + fmt_host(o[2], 17) + '\n';
    s += "SPACING " + fmt_host(h[0], 17) + ' ' + fmt_host(h[1], 17) + ' ' + fmt_host(h[2], 17) + '\n';
    s += "POINT_DATA " + std::to_string(n) + '\n';
    return s;
}

std::string scalars_line(const std::string& name, int tbytes) {
    return "SCALARS " + name + (tbytes == 4 ? " float" : " double") + " 1\nLOOKUP_TABLE default\n";
}

const char* kMaskLines = "SCALARS mask int 1\nLOOKUP_TABLE default\n";

}  // namespace

}  // namespace pdb

using namespace pdb;

extern "C" {

int pd_format_scalar(double v, int scalar_bytes, char* buf, size_t cap, int* len) {
    return guarded([&] {
        if (scalar_bytes != 4 && scalar_bytes != 8) fail(PD_E_INPUT, "scalar_bytes must be 4 or 8");
        char b[kSlot];
        const int n = fmt::format_g(v, scalar_bytes == 8 ? 17 : 9, b);
        if (cap < (size_t)n + 1) fail(PD_E_INPUT, "format buffer too small");
        std::memcpy(buf, b, (size_t)n);
        buf[n] = '\0';
        if (len) *len = n;
    });
}

int pd_write_vtk(const char* path, const char* title, int dims, const int64_t* size, const double* spacing,
                 const double* origin, int scalar_bytes, int n_arrays, const char* const* names,
                 const void* const* values, int values_on_device, const int32_t* mask, int device) {
    return guarded([&] {
        if (dims != 2 && dims != 3) fail(PD_E_INPUT, "dims must be 2 or 3");
        if (scalar_bytes != 4 && scalar_bytes != 8) fail(PD_E_INPUT, "scalar_bytes must be 4 or 8");
        check_names(names, n_arrays, mask != nullptr);
        int64_t n = 1;
        for (int a = 0; a < dims; ++a) n *= size[a];
        DeviceGuard dg(device);
        cudaStream_t st = nullptr;
        PD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        std::unique_ptr<CUstream_st, cudaError_t (*)(cudaStream_t)> sguard(st, cudaStreamDestroy);
        VtkStream w(path, n, st);
        w.text(vtk_header(title, dims, size, spacing, origin, n));
        for (int i = 0; i < n_arrays; ++i) {
            w.text(scalars_line(names[i], scalar_bytes));
            VtkSrc s;
            s.kind = kDense;
            s.tbytes = scalar_bytes;
            s.p = values[i];
            w.array(s, values_on_device ? nullptr : values[i], scalar_bytes);
        }
        if (mask) {
            w.text(kMaskLines);
            VtkSrc s;
            s.kind = kDenseInt;
            s.p = mask;
            w.array(s, values_on_device ? nullptr : mask, 4);
        }
        w.finish();
    });
}

int pd_grid_write_vtk(pd_grid* g, const char* path, const char* title, const int* props, const char* const* names,
                      int n_sel, double blank, const double* origin) {
    return guarded([&] {
        for (int i = 0; i < n_sel; ++i)
            if (props[i] < 0 || props[i] >= (int)g->column_of.size()) fail(PD_E_PROPERTY, "unknown property index");
        check_names(names, n_sel, true);
        int64_t n = 1;
        for (int a = 0; a < g->dims; ++a) n *= g->size[a];
        DeviceGuard dg(g->device);
        VtkSrc s;
        s.tbytes = g->tbytes;
        s.table = g->d_table;
        s.masks = g->d_masks;
        s.size0 = g->size[0];
        s.size1 = g->size[1];
        s.cc0 = g->cc[0];
        s.cc1 = g->cc[1];
        s.dims = g->dims;
        s.blank = blank;
        VtkStream w(path, n, g->stream);
        w.text(vtk_header(title, g->dims, g->size, g->spacing, origin, n));
        for (int i = 0; i < n_sel; ++i) {
            w.text(scalars_line(names[i], g->tbytes));
            VtkSrc a = s;
            a.kind = kSparse;
            a.p = g->cols[(size_t)g->column_of[(size_t)props[i]]];
            w.array(a, nullptr, 0);
        }
        w.text(kMaskLines);
        VtkSrc m = s;
        m.kind = kSparseMask;
        w.array(m, nullptr, 0);
        w.finish();
    });
}

int pd_grid_densify(pd_grid* g, int prop, double blank, void* host_values, int32_t* host_mask) {
    return guarded([&] {
        if (host_values && (prop < 0 || prop >= (int)g->column_of.size()))
            fail(PD_E_PROPERTY, "unknown property index");
        int64_t n = 1;
        for (int a = 0; a < g->dims; ++a) n *= g->size[a];
        DeviceGuard dg(g->device);
        VtkSrc s;
        s.tbytes = g->tbytes;
        s.table = g->d_table;
        s.masks = g->d_masks;
        s.size0 = g->size[0];
        s.size1 = g->size[1];
        s.cc0 = g->cc[0];
        s.cc1 = g->cc[1];
        s.dims = g->dims;
        s.blank = blank;
        if (host_values) s.p = g->cols[(size_t)g->column_of[(size_t)prop]];
        void* dv = nullptr;
        int32_t* dm = nullptr;
        if (host_values) PD_CUDA(pd_malloc(&dv, (size_t)n * g->tbytes));
        if (host_mask) PD_CUDA(pd_malloc(&dm, (size_t)n * 4));
        struct Free {
            void* a;
            void* b;
            ~Free() {
                pd_free(a);
                pd_free(b);
            }
        } fr{dv, dm};
        if (n > 0) {
            vtk_densify_kernel<<<(unsigned)((n + 255) / 256), 256, 0, g->stream>>>(s, n, dv, dm);
            PD_CUDA(cudaGetLastError());
        }
        if (host_values)
            PD_CUDA(cudaMemcpyAsync(host_values, dv, (size_t)n * g->tbytes, cudaMemcpyDeviceToHost, g->stream));
        if (host_mask) PD_CUDA(cudaMemcpyAsync(host_mask, dm, (size_t)n * 4, cudaMemcpyDeviceToHost, g->stream));
        PD_CUDA(cudaStreamSynchronize(g->stream));
    });
}

}  // extern "C"
