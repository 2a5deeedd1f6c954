// porediff drop-in: SBGD / SBGR snapshot containers (reference
// snapshot.hpp:33-348), routed through the B200 C ABI: the sparse writer
// streams records assembled on the device from the grid's device mirror
// (pd_grid_write_snapshot), the readers parse and validate through
// pd_*_read_snapshot (the reference's checks and messages) and hand the
// payload back to host containers. Files are byte-identical to the
// reference's (tests/test_snapshot.py; io_test.cpp via cpp/Makefile).
#pragma once

#include <cstdint>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "porediff/b200.hpp"
#include "porediff/dense_field.hpp"
#include "porediff/sparse_block_grid.hpp"

namespace porediff {

/// Header summary (snapshot.hpp:41-50).
struct SnapshotInfo {
    std::string magic;
    std::uint32_t version = 0;
    std::uint32_t scalar_bits = 0;
    std::uint32_t dims = 0;
    std::vector<std::uint64_t> size;
    std::vector<double> spacing;
    std::vector<double> origin;
    std::vector<std::string> properties;
};

namespace detail {

struct FieldHandle {
    pd_field* f = nullptr;
    ~FieldHandle() {
        if (f) pd_field_destroy(f);
    }
};
struct GridHandle {
    pd_grid* g = nullptr;
    ~GridHandle() {
        if (g) pd_grid_destroy(g);
    }
};

inline std::vector<std::string> split_names(const std::vector<char>& buf, int n) {
    std::vector<std::string> out;
    const char* p = buf.data();
    for (int i = 0; i < n; ++i) {
        out.emplace_back(p);
        p += out.back().size() + 1;
    }
    return out;
}

template <int Dims>
GridGeometry<Dims> geometry_of(const SnapshotInfo& info) {
    std::array<std::int64_t, Dims> n{};
    std::array<double, Dims> h{}, o{};
    for (int a = 0; a < Dims; ++a) {
        n[a] = static_cast<std::int64_t>(info.size[static_cast<std::size_t>(a)]);
        h[a] = info.spacing[static_cast<std::size_t>(a)];
        o[a] = info.origin[static_cast<std::size_t>(a)];
    }
    return GridGeometry<Dims>::make(n, h, o);
}

template <int Dims>
void lattice_arrays(const GridGeometry<Dims>& g, std::int64_t* n, double* h, double* o) {
    for (int a = 0; a < 3; ++a) {
        n[a] = a < Dims ? g.size[a] : 1;
        h[a] = a < Dims ? g.spacing[a] : 1.0;
        o[a] = a < Dims ? g.origin[a] : 0.0;
    }
}

}  // namespace detail

/// peek_snapshot (snapshot.hpp:303-346).
inline SnapshotInfo peek_snapshot(const std::filesystem::path& path) {
    pd_snapshot_info c{};
    std::vector<char> names(1 << 20);
    b200::check(pd_peek_snapshot(path.string().c_str(), &c, names.data(), names.size()));
    SnapshotInfo info;
    info.magic = c.magic;
    info.version = c.version;
    info.scalar_bits = c.scalar_bits;
    info.dims = c.dims;
    for (std::uint32_t a = 0; a < c.dims; ++a) {
        info.size.push_back(c.size[a]);
        info.spacing.push_back(c.spacing[a]);
        info.origin.push_back(c.origin[a]);
    }
    info.properties = detail::split_names(names, static_cast<int>(c.n_properties));
    return info;
}

/// write_dense_snapshot (snapshot.hpp:194-201).
template <typename T, int Dims>
void write_dense_snapshot(const DenseField<T, Dims>& field, const std::filesystem::path& path) {
    std::int64_t n[3];
    double h[3], o[3];
    detail::lattice_arrays(field.geometry(), n, h, o);
    detail::FieldHandle f;
    b200::check(pd_field_create(Dims, static_cast<int>(sizeof(T)), n, h, o, b200::default_device(), &f.f));
    b200::check(pd_field_upload(f.f, field.data()));
    b200::check(pd_field_write_snapshot(f.f, path.string().c_str()));
}

/// read_dense_snapshot (snapshot.hpp:204-212).
template <typename T, int Dims>
DenseField<T, Dims> read_dense_snapshot(const std::filesystem::path& path) {
    detail::FieldHandle f;
    b200::check(pd_field_read_snapshot(path.string().c_str(), Dims, static_cast<int>(sizeof(T)),
                                       b200::default_device(), &f.f));
    DenseField<T, Dims> field(detail::geometry_of<Dims>(peek_snapshot(path)));
    b200::check(pd_field_download(f.f, field.data()));
    return field;
}

/// write_sparse_snapshot (snapshot.hpp:218-241): records assembled on the
/// device from the grid's mirror, payloads in registration order.
template <typename T, int Dims>
void write_sparse_snapshot(const SparseBlockGrid<T, Dims>& grid, const std::filesystem::path& path) {
    auto& g = const_cast<SparseBlockGrid<T, Dims>&>(grid);  // the mirror is a cache
    pd_grid* dev = g.device_grid();
    std::vector<const char*> names;
    for (const std::string& s : grid.property_names()) names.push_back(s.c_str());
    std::int64_t n[3];
    double h[3], o[3];
    detail::lattice_arrays(grid.geometry(), n, h, o);
    b200::check(pd_grid_write_snapshot(dev, path.string().c_str(), names.data(), static_cast<int>(names.size()), o));
}

/// read_sparse_snapshot (snapshot.hpp:245-297): validated and loaded on the
/// device; the host grid adopts it (slabs fetched on first host access).
template <typename T, int Dims>
SparseBlockGrid<T, Dims> read_sparse_snapshot(const std::filesystem::path& path) {
    using Grid = SparseBlockGrid<T, Dims>;
    detail::GridHandle h;
    double origin[3] = {0, 0, 0};
    std::vector<char> buf(1 << 20);
    int n_names = 0;
    b200::check(pd_grid_read_snapshot(path.string().c_str(), Dims, static_cast<int>(sizeof(T)),
                                      b200::default_device(), &h.g, origin, buf.data(), buf.size(), &n_names));
    Grid grid(detail::geometry_of<Dims>(peek_snapshot(path)), detail::split_names(buf, n_names));
    // the host grid adopts the device grid as its mirror: layout now, slabs
    // on first host access
    std::vector<int> all(static_cast<std::size_t>(n_names));
    for (int p = 0; p < n_names; ++p) all[static_cast<std::size_t>(p)] = p;
    pd_grid* g = h.g;
    h.g = nullptr;
    grid.adopt_device(g, b200::default_device(), all);
    return grid;
}

}  // namespace porediff
