// SBGR / SBGD snapshots streamed from / to the device (
// reference snapshot.hpp:195-348). Byte-identical to the reference writer:
// little-endian header (magic, version 1, scalar bits, dims, size, spacing,
// origin), the property-name table, then one record per chunk in ascending
// linear index — key, occupancy mask, the full slab of every property in
// registration order (inactive slots included, regardless of u/u_next swaps).
//
// Records are assembled on the device (record_pack_kernel: chunk-major
// key|mask|slabs from the property-major columns) in batches and written
// through a pinned staging buffer; reading parses batches into the same
// staging buffer and scatters them into the columns (record_unpack_kernel).
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "pd_internal.cuh"

namespace pdb {

constexpr uint32_t kSnapVersion = 1;
constexpr int64_t kSnapBatch = 8192;  // chunks per staging batch

struct ColPtrs {
    const unsigned char* col[16];
};

// record = key (dims int32) | mask (W uint64) | n_props slabs of V*tbytes
__global__ void record_pack_kernel(const int32_t* __restrict__ keys, const uint64_t* __restrict__ masks, ColPtrs cols,
                                   int n_props, int dims, int W, int64_t slab_bytes, int64_t rec_bytes, int64_t c0,
                                   int64_t n, unsigned char* __restrict__ out) {
    const int64_t j = blockIdx.x;
    if (j >= n) return;
    const int64_t c = c0 + j;
    unsigned char* r = out + j * rec_bytes;
    const int head = 4 * dims + 8 * W;
    for (int b = threadIdx.x; b < head; b += blockDim.x) {
        if (b < 4 * dims)
            r[b] = reinterpret_cast<const unsigned char*>(keys + c * dims)[b];
        else
            r[b] = reinterpret_cast<const unsigned char*>(masks + c * W)[b - 4 * dims];
    }
    for (int p = 0; p < n_props; ++p) {
        const uint32_t* s = reinterpret_cast<const uint32_t*>(cols.col[p] + c * slab_bytes);
        unsigned char* d = r + head + p * slab_bytes;
        for (int64_t w = threadIdx.x; w < slab_bytes / 4; w += blockDim.x) {
            const uint32_t v = s[w];
            std::memcpy(d + 4 * w, &v, 4);  // records are only 4-B aligned
        }
    }
}

__global__ void record_unpack_kernel(const unsigned char* __restrict__ in, int n_props, int dims, int W,
                                     int64_t slab_bytes, int64_t rec_bytes, int64_t c0, int64_t n, ColPtrs cols) {
    const int64_t j = blockIdx.x;
    if (j >= n) return;
    const int64_t c = c0 + j;
    const unsigned char* r = in + j * rec_bytes + 4 * dims + 8 * W;
    for (int p = 0; p < n_props; ++p) {
        uint32_t* d = reinterpret_cast<uint32_t*>(const_cast<unsigned char*>(cols.col[p]) + c * slab_bytes);
        for (int64_t w = threadIdx.x; w < slab_bytes / 4; w += blockDim.x) {
            uint32_t v;
            std::memcpy(&v, r + p * slab_bytes + 4 * w, 4);
            d[w] = v;
        }
    }
}

struct File {
    FILE* f = nullptr;
    std::string path;
    File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)), path(p) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

template <class V>
void put(File& w, V v) {
    if (std::fwrite(&v, sizeof v, 1, w.f) != 1) fail(PD_E_IO, "write to '" + w.path + "' failed");
}
void put_bytes(File& w, const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, w.f) != n) fail(PD_E_IO, "write to '" + w.path + "' failed");
}
void get_bytes(File& r, void* p, size_t n) {
    if (n && std::fread(p, 1, n, r.f) != n) fail(PD_E_IO, "'" + r.path + "' is truncated");
}
template <class V>
V get(File& r) {
    V v;
    get_bytes(r, &v, sizeof v);
    return v;
}
void expect_eof(File& r) {
    if (std::fgetc(r.f) != EOF) fail(PD_E_IO, "'" + r.path + "' has trailing bytes after the payload");
}

void write_header(File& w, const char* magic, int tbytes, int dims, const int64_t* size, const double* spacing,
                  const double* origin) {
    put_bytes(w, magic, 4);
    put<uint32_t>(w, kSnapVersion);
    put<uint32_t>(w, (uint32_t)(tbytes * 8));
    put<uint32_t>(w, (uint32_t)dims);
    for (int a = 0; a < dims; ++a) put<uint64_t>(w, (uint64_t)size[a]);
    for (int a = 0; a < dims; ++a) put<double>(w, spacing[a]);
    for (int a = 0; a < dims; ++a) put<double>(w, origin[a]);
}

// read_common_header (snapshot.hpp:147-179), messages verbatim
void read_header(File& r, const char* magic, int tbytes, int dims, int64_t* size, double* spacing, double* origin) {
    char m[4];
    get_bytes(r, m, 4);
    if (std::memcmp(m, magic, 4) != 0)
        fail(PD_E_IO, "'" + r.path + "' is not a " + std::string(magic, 4) + " snapshot (magic mismatch)");
    const uint32_t version = get<uint32_t>(r);
    if (version != kSnapVersion) fail(PD_E_IO, "'" + r.path + "': unsupported format version " + std::to_string(version));
    const uint32_t bits = get<uint32_t>(r);
    if (bits != (uint32_t)(tbytes * 8))
        fail(PD_E_IO, "'" + r.path + "' stores " + std::to_string(bits) + "-bit scalars, expected " +
                          std::to_string(tbytes * 8));
    const uint32_t d = get<uint32_t>(r);
    if (d != (uint32_t)dims)
        fail(PD_E_IO, "'" + r.path + "' is " + std::to_string(d) + "-dimensional, expected " + std::to_string(dims));
    for (int a = 0; a < dims; ++a) {
        const uint64_t n = get<uint64_t>(r);
        if (n == 0 || n > (uint64_t)std::numeric_limits<int32_t>::max())
            fail(PD_E_IO, "'" + r.path + "': axis extent " + std::to_string(n) + " out of range");
        size[a] = (int64_t)n;
    }
    for (int a = 0; a < dims; ++a) spacing[a] = get<double>(r);
    for (int a = 0; a < dims; ++a) origin[a] = get<double>(r);
}

struct Pinned {
    unsigned char* p = nullptr;
    explicit Pinned(size_t n) { PD_CUDA(cudaMallocHost(&p, n)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};
struct DevBuf {
    unsigned char* p = nullptr;
    explicit DevBuf(size_t n) { PD_CUDA(pd_malloc(&p, n)); }
    ~DevBuf() {
        if (p) pd_free(p);
    }
};

}  // namespace pdb

using namespace pdb;

extern "C" {

int pd_grid_write_snapshot(pd_grid* g, const char* path, const char* const* names, int n_names,
                           const double* origin) {
    return guarded([&] {
        if (n_names != (int)g->column_of.size()) fail(PD_E_INPUT, "one name per grid property is required");
        if (n_names > 16) fail(PD_E_INPUT, "at most 16 properties per snapshot");
        DeviceGuard dg(g->device);
        File w(path, "wb");
        if (!w.f) fail(PD_E_IO, "cannot open '" + std::string(path) + "' for writing");
        write_header(w, "SBGR", g->tbytes, g->dims, g->size, g->spacing, origin);
        put<uint32_t>(w, (uint32_t)n_names);
        for (int i = 0; i < n_names; ++i) {
            const uint32_t len = (uint32_t)std::strlen(names[i]);
            put<uint32_t>(w, len);
            put_bytes(w, names[i], len);
        }
        put<uint64_t>(w, (uint64_t)g->n_chunks);
        const int64_t slab = (int64_t)g->V * g->tbytes;
        const int64_t rec = 4 * g->dims + 8 * g->W + (int64_t)n_names * slab;
        const int64_t batch = std::min<int64_t>(kSnapBatch, std::max<int64_t>(1, g->n_chunks));
        ColPtrs cols{};
        for (int p = 0; p < n_names; ++p)  // logical order: registration order regardless of swaps
            cols.col[p] = (const unsigned char*)g->cols[(size_t)g->column_of[(size_t)p]];
        DevBuf dbuf((size_t)(batch * rec));
        Pinned hbuf((size_t)(batch * rec));
        for (int64_t c0 = 0; c0 < g->n_chunks; c0 += batch) {
            const int64_t n = std::min<int64_t>(batch, g->n_chunks - c0);
            record_pack_kernel<<<(unsigned)n, 256, 0, g->stream>>>(g->d_keys, g->d_masks, cols, n_names, g->dims,
                                                                   g->W, slab, rec, c0, n, dbuf.p);
            PD_CUDA(cudaGetLastError());
            PD_CUDA(cudaMemcpyAsync(hbuf.p, dbuf.p, (size_t)(n * rec), cudaMemcpyDeviceToHost, g->stream));
            PD_CUDA(cudaStreamSynchronize(g->stream));
            put_bytes(w, hbuf.p, (size_t)(n * rec));
        }
        if (std::fflush(w.f) != 0) fail(PD_E_IO, "write to '" + std::string(path) + "' failed");
    });
}

int pd_grid_read_snapshot(const char* path, int dims, int scalar_bytes, int device, pd_grid** out,
                          double* origin, char* names_buf, size_t names_cap, int* n_names) {
    return guarded([&] {
        *out = nullptr;
        File r(path, "rb");
        if (!r.f) fail(PD_E_IO, "cannot open '" + std::string(path) + "' for reading");
        int64_t size[3] = {1, 1, 1};
        double spacing[3] = {1, 1, 1}, org[3] = {0, 0, 0};
        read_header(r, "SBGR", scalar_bytes, dims, size, spacing, org);
        const uint32_t np = get<uint32_t>(r);
        if (np == 0 || np > 4096)
            fail(PD_E_IO, "'" + r.path + "': property count " + std::to_string(np) + " out of range");
        std::string all;
        for (uint32_t i = 0; i < np; ++i) {
            const uint32_t len = get<uint32_t>(r);
            if (len == 0 || len > 4096)
                fail(PD_E_IO, "'" + r.path + "': property name length " + std::to_string(len) + " out of range");
            std::string s(len, '\0');
            get_bytes(r, s.data(), len);
            all += s;
            all.push_back('\0');
        }
        if (np > 16) fail(PD_E_INPUT, "at most 16 properties per snapshot");
        const int V = dims == 3 ? 512 : 64, W = V / 64;
        int64_t cc[3] = {1, 1, 1}, maxc = 1;
        for (int a = 0; a < dims; ++a) {
            cc[a] = (size[a] + 7) / 8;
            maxc *= cc[a];
        }
        const uint64_t nch = get<uint64_t>(r);
        if (nch > (uint64_t)maxc)
            fail(PD_E_IO, "'" + r.path + "': chunk count " + std::to_string(nch) + " exceeds the geometry's chunk table");
        const int64_t slab = (int64_t)V * scalar_bytes;
        const int64_t rec = 4 * dims + 8 * W + (int64_t)np * slab;
        // pass 1 (host): keys and masks, validated like read_sparse_snapshot
        // (snapshot.hpp:270-297); the slabs stay in the file and are streamed in
        // pass 2
        std::vector<int32_t> keys((size_t)nch * dims);
        std::vector<uint64_t> masks((size_t)nch * W);
        const long data0 = std::ftell(r.f);
        int64_t prev = -1;
        std::vector<unsigned char> rb((size_t)rec);
        for (uint64_t i = 0; i < nch; ++i) {
            get_bytes(r, rb.data(), (size_t)rec);
            int64_t lin = 0;
            int32_t k[3];
            std::memcpy(k, rb.data(), 4 * dims);
            for (int a = 0; a < dims; ++a)
                if (k[a] < 0 || k[a] >= cc[a]) fail(PD_E_IO, "'" + r.path + "': chunk key outside the geometry");
            for (int a = dims - 1; a >= 0; --a) lin = lin * cc[a] + k[a];
            if (lin <= prev) fail(PD_E_IO, "'" + r.path + "': chunk records out of order");
            prev = lin;
            std::memcpy(&keys[i * dims], k, 4 * dims);
            std::memcpy(&masks[i * W], rb.data() + 4 * dims, 8 * W);
            bool any = false;
            for (int w = 0; w < W; ++w) any = any || masks[i * W + w] != 0;
            if (!any) fail(PD_E_IO, "'" + r.path + "': chunk record with empty occupancy mask");
        }
        expect_eof(r);
        pd_grid* g = nullptr;
        int rc = pd_grid_create(dims, scalar_bytes, size, spacing, (int64_t)nch, keys.data(), masks.data(), (int)np,
                                device, &g);
        if (rc != PD_OK) fail(rc, pd_last_error());
        std::unique_ptr<pd_grid, int (*)(pd_grid*)> guard(g, pd_grid_destroy);
        DeviceGuard dg(device);
        // pass 2: slabs, batch by batch through the pinned staging buffer
        std::fseek(r.f, data0, SEEK_SET);
        const int64_t batch = std::min<int64_t>(kSnapBatch, std::max<int64_t>(1, (int64_t)nch));
        DevBuf dbuf((size_t)(batch * rec));
        Pinned hbuf((size_t)(batch * rec));
        ColPtrs cols{};
        for (uint32_t p = 0; p < np; ++p) cols.col[p] = (const unsigned char*)g->cols[(size_t)g->column_of[p]];
        for (int64_t c0 = 0; c0 < (int64_t)nch; c0 += batch) {
            const int64_t n = std::min<int64_t>(batch, (int64_t)nch - c0);
            get_bytes(r, hbuf.p, (size_t)(n * rec));
            PD_CUDA(cudaMemcpyAsync(dbuf.p, hbuf.p, (size_t)(n * rec), cudaMemcpyHostToDevice, g->stream));
            record_unpack_kernel<<<(unsigned)n, 256, 0, g->stream>>>(dbuf.p, (int)np, dims, W, slab, rec, c0, n, cols);
            PD_CUDA(cudaGetLastError());
            PD_CUDA(cudaStreamSynchronize(g->stream));
        }
        for (int a = 0; a < dims; ++a) origin[a] = org[a];
        *n_names = (int)np;
        if (names_buf) {
            if (all.size() > names_cap) fail(PD_E_INPUT, "property-name buffer too small");
            std::memcpy(names_buf, all.data(), all.size());
        }
        *out = guard.release();
    });
}

int pd_field_write_snapshot(pd_field* f, const char* path) {
    return guarded([&] {
        DeviceGuard dg(f->device);
        File w(path, "wb");
        if (!w.f) fail(PD_E_IO, "cannot open '" + std::string(path) + "' for writing");
        write_header(w, "SBGD", f->tbytes, f->dims, f->size, f->spacing, f->origin);
        const size_t chunk = (size_t)64 << 20;
        const size_t total = (size_t)f->n * (size_t)f->tbytes;
        Pinned hbuf(std::min(chunk, std::max<size_t>(1, total)));
        for (size_t o = 0; o < total; o += chunk) {
            const size_t n = std::min(chunk, total - o);
            PD_CUDA(cudaMemcpyAsync(hbuf.p, (const unsigned char*)f->d + o, n, cudaMemcpyDeviceToHost, f->stream));
            PD_CUDA(cudaStreamSynchronize(f->stream));
            put_bytes(w, hbuf.p, n);
        }
        if (std::fflush(w.f) != 0) fail(PD_E_IO, "write to '" + std::string(path) + "' failed");
    });
}

int pd_field_read_snapshot(const char* path, int dims, int scalar_bytes, int device, pd_field** out) {
    return guarded([&] {
        *out = nullptr;
        File r(path, "rb");
        if (!r.f) fail(PD_E_IO, "cannot open '" + std::string(path) + "' for reading");
        int64_t size[3] = {1, 1, 1};
        double spacing[3] = {1, 1, 1}, org[3] = {0, 0, 0};
        read_header(r, "SBGD", scalar_bytes, dims, size, spacing, org);
        pd_field* f = nullptr;
        int rc = pd_field_create(dims, scalar_bytes, size, spacing, org, device, &f);
        if (rc != PD_OK) fail(rc, pd_last_error());
        std::unique_ptr<pd_field, int (*)(pd_field*)> guard(f, pd_field_destroy);
        DeviceGuard dg(device);
        const size_t chunk = (size_t)64 << 20;
        const size_t total = (size_t)f->n * (size_t)f->tbytes;
        Pinned hbuf(std::min(chunk, std::max<size_t>(1, total)));
        for (size_t o = 0; o < total; o += chunk) {
            const size_t n = std::min(chunk, total - o);
            get_bytes(r, hbuf.p, n);
            PD_CUDA(cudaMemcpyAsync((unsigned char*)f->d + o, hbuf.p, n, cudaMemcpyHostToDevice, f->stream));
            PD_CUDA(cudaStreamSynchronize(f->stream));
        }
        expect_eof(r);
        *out = guard.release();
    });
}

int pd_peek_snapshot(const char* path, pd_snapshot_info* info, char* names_buf, size_t names_cap) {
    return guarded([&] {
        File r(path, "rb");
        if (!r.f) fail(PD_E_IO, "cannot open '" + std::string(path) + "' for reading");
        char m[4];
        get_bytes(r, m, 4);
        const std::string magic(m, 4);
        if (magic != "SBGD" && magic != "SBGR")
            fail(PD_E_IO, "'" + r.path + "' is not a snapshot file (magic '" + magic + "')");
        std::memcpy(info->magic, m, 4);
        info->magic[4] = '\0';
        info->version = get<uint32_t>(r);
        if (info->version != kSnapVersion)
            fail(PD_E_IO, "'" + r.path + "': unsupported format version " + std::to_string(info->version));
        info->scalar_bits = get<uint32_t>(r);
        info->dims = get<uint32_t>(r);
        if (info->dims < 2 || info->dims > 3)
            fail(PD_E_IO, "'" + r.path + "': rank " + std::to_string(info->dims) + " out of range");
        for (uint32_t a = 0; a < info->dims; ++a) info->size[a] = get<uint64_t>(r);
        for (uint32_t a = 0; a < info->dims; ++a) info->spacing[a] = get<double>(r);
        for (uint32_t a = 0; a < info->dims; ++a) info->origin[a] = get<double>(r);
        info->n_properties = 0;
        if (magic == "SBGR") {
            const uint32_t np = get<uint32_t>(r);
            if (np == 0 || np > 4096)
                fail(PD_E_IO, "'" + r.path + "': property count " + std::to_string(np) + " out of range");
            std::string all;
            for (uint32_t i = 0; i < np; ++i) {
                const uint32_t len = get<uint32_t>(r);
                if (len == 0 || len > 4096)
                    fail(PD_E_IO, "'" + r.path + "': property name length " + std::to_string(len) + " out of range");
                std::string s(len, '\0');
                get_bytes(r, s.data(), len);
                all += s;
                all.push_back('\0');
            }
            info->n_properties = np;
            if (names_buf) {
                if (all.size() > names_cap) fail(PD_E_INPUT, "property-name buffer too small");
                std::memcpy(names_buf, all.data(), all.size());
            }
        }
    });
}

}  // extern "C"
