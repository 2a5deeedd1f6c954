// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper that compiles the UNMODIFIED reference headers
// (/root/reference/proj/include/porediff, included in place — nothing is
// copied) into oracle/_ref/libporediff_ref.so, so the parity tests, the golden
// generator and bench.py's cpu_baseline/--impl reference leg can call the
// reference's own run_simulation / build_sparse_grid / run_frap on identical
// inputs. Build recipe: oracle/Makefile (g++ -std=c++20 -O3 -ffp-contract=off,
// the reference's Release flags, CMakeLists.txt:11-14).
//
// Only tests/, __graft_entry__.smoke() and bench.py may load this library.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "porediff/analysis.hpp"
#include "porediff/geometry.hpp"
#include "porediff/parallel.hpp"
#include "porediff/solver.hpp"
#include "porediff/sparse_block_grid.hpp"
#include "porediff/synthetic.hpp"
#include "porediff/config.hpp"
#include "porediff/levelset.hpp"
#include "porediff/snapshot.hpp"
#include "porediff/vtk.hpp"

#include "porediff_b200.h"  // pd_sim_config / pd_diag layouts only

namespace pd = porediff;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const pd::input_error*>(&e)) return PD_E_INPUT;
    if (dynamic_cast<const pd::bounds_error*>(&e)) return PD_E_BOUNDS;
    if (dynamic_cast<const pd::property_error*>(&e)) return PD_E_PROPERTY;
    if (dynamic_cast<const pd::io_error*>(&e)) return PD_E_IO;
    if (dynamic_cast<const pd::stability_error*>(&e)) return PD_E_STABILITY;
    if (dynamic_cast<const pd::numeric_error*>(&e)) return PD_E_NUMERIC;
    return 99;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

typedef double (*time_factor_fn)(double);

struct RefGridBase {
    virtual ~RefGridBase() = default;
    virtual int64_t chunk_count() const = 0;
    virtual int64_t active_count() const = 0;
    virtual void export_layout(int32_t* keys, uint64_t* masks) const = 0;
    virtual void export_prop(int prop, void* slabs) const = 0;
    virtual void import_prop(int prop, const void* slabs) = 0;
    virtual void populate_d(double dmin, double dmax, double g1, double g2) = 0;
    virtual void fill_hash(int prop, uint64_t seed) = 0;
    virtual void run(const pd_sim_config* c, time_factor_fn tf, pd_diag* rows,
                     int64_t* n_rows) = 0;
    virtual double total_mass(int prop) const = 0;
    virtual double max_diffusivity(int prop) const = 0;
    virtual void write_snapshot(const char* path) const = 0;
    virtual void write_vtk(const char* path, const char* channels, double blank, const double* origin) const = 0;
};

template <typename T, int D>
struct RefGrid : RefGridBase {
    using G = pd::SparseBlockGrid<T, D>;
    static constexpr int V = G::chunk_volume;
    static constexpr int W = G::mask_words;
    G g;
    explicit RefGrid(G&& grid) : g(std::move(grid)) {}

    int64_t chunk_count() const override { return g.chunk_count(); }
    int64_t active_count() const override { return g.active_node_count(); }
    void write_snapshot(const char* path) const override { pd::write_sparse_snapshot(g, path); }
    // write_vtk(vtk_from_sparse(g, channels, blank)); channels: '\n'-joined,
    // empty = every property; origin overrides the grid's when non-null
    void write_vtk(const char* path, const char* channels, double blank, const double* origin) const override {
        std::vector<std::string> ch;
        std::string cur;
        for (const char* c = channels; *c; ++c) {
            if (*c == '\n') {
                ch.push_back(cur);
                cur.clear();
            } else {
                cur.push_back(*c);
            }
        }
        if (!cur.empty()) ch.push_back(cur);
        auto ds = pd::vtk_from_sparse(g, ch, static_cast<T>(blank));
        if (origin)
            for (int a = 0; a < D; ++a) ds.geometry.origin[a] = origin[a];
        pd::write_vtk(ds, path);
    }

    void export_layout(int32_t* keys, uint64_t* masks) const override {
        int64_t i = 0;
        g.for_each_chunk([&](const typename G::Chunk& c) {
            for (int a = 0; a < D; ++a) keys[i * D + a] = c.key[a];
            for (int w = 0; w < W; ++w) masks[i * W + w] = c.mask[w];
            ++i;
        });
    }
    void export_prop(int prop, void* slabs) const override {
        T* out = static_cast<T*>(slabs);
        int64_t i = 0;
        g.for_each_chunk([&](const typename G::Chunk& c) {
            std::memcpy(out + i * V, g.channel_data(c, prop), sizeof(T) * V);
            ++i;
        });
    }
    void import_prop(int prop, const void* slabs) override {
        const T* in = static_cast<const T*>(slabs);
        int64_t i = 0;
        g.for_each_chunk([&](typename G::Chunk& c) {
            std::memcpy(g.channel_data(c, prop), in + i * V, sizeof(T) * V);
            ++i;
        });
    }
    void populate_d(double dmin, double dmax, double g1, double g2) override {
        pd::populate_diffusion_channel(g, pd::DiffusionProfile{dmin, dmax, g1, g2});
    }
    void fill_hash(int prop, uint64_t seed) override {
        const auto names = g.property_names();
        const std::string name(names[static_cast<std::size_t>(prop)]);
        const auto& geom = g.geometry();
        g.for_each_active([&](const pd::NodeIndex<D>& idx, const auto&, int) {
            g.set(idx, name,
                  static_cast<T>(pd::hash_unit_value(
                      seed, static_cast<std::uint64_t>(geom.flat_index(idx)))));
        });
    }
    void run(const pd_sim_config* c, time_factor_fn tf, pd_diag* rows,
             int64_t* n_rows) override {
        pd::SimulationConfig cfg;
        cfg.dt = c->dt;
        cfg.n_steps = c->n_steps;
        cfg.phase_band = pd::PhaseBand{c->b_low, c->b_up};
        cfg.boundary_epsilon = c->boundary_epsilon;
        if (c->reaction_kind == PD_REACTION_SURFACE_SINK) {
            cfg.reaction = pd::ReactionSpec::surface_sink(c->rate, c->band_half_width);
        } else if (c->reaction_kind == PD_REACTION_VOLUMETRIC) {
            const auto names = g.property_names();
            std::string ch = c->source_prop >= 0 &&
                                     c->source_prop < static_cast<int>(names.size())
                                 ? std::string(names[static_cast<std::size_t>(c->source_prop)])
                                 : std::string("missing");
            std::function<double(double)> f;
            if (tf) f = [tf](double t) { return tf(t); };
            cfg.reaction = pd::ReactionSpec::volumetric(ch, f);
        }
        for (int i = 0; i < 6; ++i)
            cfg.outer_bc[static_cast<std::size_t>(i)] =
                c->bc_type[i] == PD_BC_DIRICHLET ? pd::FaceBc::dirichlet(c->bc_value[i])
                                                 : pd::FaceBc::no_flux();
        cfg.record_every = c->record_every;
        cfg.enforce_stability = c->enforce_stability != 0;
        const auto r = pd::run_simulation(g, cfg);
        int64_t k = 0;
        for (const auto& d : r.diagnostics) {
            rows[k].step = d.step;
            rows[k].time = d.time;
            rows[k].total_mass = d.total_mass;
            rows[k].min_u = d.min_u;
            rows[k].max_u = d.max_u;
            ++k;
        }
        *n_rows = k;
    }
    double total_mass(int prop) const override {
        const auto names = g.property_names();
        return pd::total_mass(g, names[static_cast<std::size_t>(prop)]);
    }
    double max_diffusivity(int prop) const override {
        const auto names = g.property_names();
        return pd::max_diffusivity(g, names[static_cast<std::size_t>(prop)]);
    }
};

template <int D>
pd::GridGeometry<D> geom_of(const int64_t* size, const double* spacing, const double* origin) {
    std::array<std::int64_t, D> s{};
    std::array<double, D> h{}, o{};
    for (int a = 0; a < D; ++a) {
        s[a] = size[a];
        h[a] = spacing[a];
        o[a] = origin ? origin[a] : 0.0;
    }
    return pd::GridGeometry<D>::make(s, h, o);
}

std::vector<std::string> names_of(int n, const char* const* names) {
    std::vector<std::string> v;
    for (int i = 0; i < n; ++i) v.emplace_back(names[i]);
    return v;
}

template <typename T, int D>
RefGridBase* from_sdf(const int64_t* size, const double* spacing, const double* origin,
                      const double* sdf, double b_low, double b_up, int n,
                      const char* const* names) {
    auto geom = geom_of<D>(size, spacing, origin);
    pd::DenseField<T, D> field(geom);
    for (int64_t f = 0; f < geom.node_count(); ++f) field[f] = static_cast<T>(sdf[f]);
    return new RefGrid<T, D>(
        pd::build_sparse_grid(field, pd::PhaseBand{b_low, b_up}, names_of(n, names)));
}

template <typename T, int D>
RefGridBase* from_chunks(const int64_t* size, const double* spacing, const double* origin,
                         int n, const char* const* names, int64_t n_chunks,
                         const int32_t* keys, const uint64_t* masks) {
    using G = pd::SparseBlockGrid<T, D>;
    G g(geom_of<D>(size, spacing, origin), names_of(n, names));
    for (int64_t i = 0; i < n_chunks; ++i) {
        typename G::Key key{};
        for (int a = 0; a < D; ++a) key[a] = keys[i * D + a];
        for (int off = 0; off < G::chunk_volume; ++off)
            if ((masks[i * G::mask_words + (off >> 6)] >> (off & 63)) & 1u)
                g.insert(G::node_index(key, off));
    }
    return new RefGrid<T, D>(std::move(g));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_worker_count(int n) { pd::set_worker_count(n); }
int ref_worker_count(void) { return pd::worker_count(); }

double ref_hash_unit_value(uint64_t seed, uint64_t key) { return pd::hash_unit_value(seed, key); }

double ref_pairwise_sum(const double* v, int64_t n) {
    return pd::pairwise_sum(std::vector<double>(v, v + n));
}

double ref_stability_dt(int dims, const double* spacing, double d_max, int* code) {
    double out = 0.0;
    *code = guarded([&] {
        double sp[3] = {spacing[0], spacing[1], dims == 3 ? spacing[2] : 1.0};
        int64_t sz[3] = {1, 1, 1};
        if (dims == 2)
            out = pd::stability_dt(geom_of<2>(sz, sp, nullptr), d_max);
        else
            out = pd::stability_dt(geom_of<3>(sz, sp, nullptr), d_max);
    });
    return out;
}

/* synthetic::SpherePacking::random (synthetic.hpp:42-55) */
void ref_sphere_packing(const double* lo, const double* hi, int count, double r_min,
                        double r_max, uint32_t seed, double* centers, double* radii) {
    const auto p = pd::synthetic::SpherePacking::random({lo[0], lo[1], lo[2]},
                                                        {hi[0], hi[1], hi[2]}, count,
                                                        r_min, r_max, seed);
    for (int i = 0; i < count; ++i) {
        for (int a = 0; a < 3; ++a) centers[i * 3 + a] = p.centers[i][a];
        radii[i] = p.radii[i];
    }
}

/* field_from(geom, pack.fluid_sdf) into a dense double array (flat order). */
void ref_field_sphere_pack(const int64_t* size, const double* spacing, const double* origin,
                           int count, const double* centers, const double* radii,
                           double* out) {
    pd::synthetic::SpherePacking p;
    for (int i = 0; i < count; ++i) {
        p.centers.push_back({centers[i * 3], centers[i * 3 + 1], centers[i * 3 + 2]});
        p.radii.push_back(radii[i]);
    }
    auto geom = geom_of<3>(size, spacing, origin);
    auto f = pd::synthetic::field_from<double, 3>(
        geom, [&](const std::array<double, 3>& x) { return p.fluid_sdf(x); });
    std::memcpy(out, f.data(), sizeof(double) * static_cast<std::size_t>(geom.node_count()));
}

/* field_from(geom, sign * ball_sdf(x, c, r)) */
void ref_field_ball(int dims, const int64_t* size, const double* spacing, const double* origin,
                    const double* center, double radius, double sign, double* out) {
    if (dims == 2) {
        auto geom = geom_of<2>(size, spacing, origin);
        auto f = pd::synthetic::field_from<double, 2>(geom, [&](const std::array<double, 2>& x) {
            return sign * pd::synthetic::ball_sdf<2>(x, {center[0], center[1]}, radius);
        });
        std::memcpy(out, f.data(), sizeof(double) * static_cast<std::size_t>(geom.node_count()));
    } else {
        auto geom = geom_of<3>(size, spacing, origin);
        auto f = pd::synthetic::field_from<double, 3>(geom, [&](const std::array<double, 3>& x) {
            return sign * pd::synthetic::ball_sdf<3>(x, {center[0], center[1], center[2]},
                                                     radius);
        });
        std::memcpy(out, f.data(), sizeof(double) * static_cast<std::size_t>(geom.node_count()));
    }
}

void* ref_grid_from_sdf(int dims, int tbytes, const int64_t* size, const double* spacing,
                        const double* origin, const double* sdf, double b_low, double b_up,
                        int n_props, const char* const* names, int* code) {
    RefGridBase* h = nullptr;
    *code = guarded([&] {
        if (dims == 2 && tbytes == 8)
            h = from_sdf<double, 2>(size, spacing, origin, sdf, b_low, b_up, n_props, names);
        else if (dims == 3 && tbytes == 8)
            h = from_sdf<double, 3>(size, spacing, origin, sdf, b_low, b_up, n_props, names);
        else if (dims == 2)
            h = from_sdf<float, 2>(size, spacing, origin, sdf, b_low, b_up, n_props, names);
        else
            h = from_sdf<float, 3>(size, spacing, origin, sdf, b_low, b_up, n_props, names);
    });
    return h;
}

void* ref_grid_from_chunks(int dims, int tbytes, const int64_t* size, const double* spacing,
                           const double* origin, int n_props, const char* const* names,
                           int64_t n_chunks, const int32_t* keys, const uint64_t* masks,
                           int* code) {
    RefGridBase* h = nullptr;
    *code = guarded([&] {
        if (dims == 2 && tbytes == 8)
            h = from_chunks<double, 2>(size, spacing, origin, n_props, names, n_chunks, keys, masks);
        else if (dims == 3 && tbytes == 8)
            h = from_chunks<double, 3>(size, spacing, origin, n_props, names, n_chunks, keys, masks);
        else if (dims == 2)
            h = from_chunks<float, 2>(size, spacing, origin, n_props, names, n_chunks, keys, masks);
        else
            h = from_chunks<float, 3>(size, spacing, origin, n_props, names, n_chunks, keys, masks);
    });
    return h;
}

void ref_grid_free(void* h) { delete static_cast<RefGridBase*>(h); }
int64_t ref_grid_chunk_count(void* h) { return static_cast<RefGridBase*>(h)->chunk_count(); }
int64_t ref_grid_active_count(void* h) { return static_cast<RefGridBase*>(h)->active_count(); }
void ref_grid_export_layout(void* h, int32_t* keys, uint64_t* masks) {
    static_cast<RefGridBase*>(h)->export_layout(keys, masks);
}
void ref_grid_export_prop(void* h, int prop, void* slabs) {
    static_cast<RefGridBase*>(h)->export_prop(prop, slabs);
}
void ref_grid_import_prop(void* h, int prop, const void* slabs) {
    static_cast<RefGridBase*>(h)->import_prop(prop, slabs);
}
int ref_grid_populate_diffusion(void* h, double dmin, double dmax, double g1, double g2) {
    return guarded([&] { static_cast<RefGridBase*>(h)->populate_d(dmin, dmax, g1, g2); });
}
int ref_grid_fill_hash(void* h, int prop, uint64_t seed) {
    return guarded([&] { static_cast<RefGridBase*>(h)->fill_hash(prop, seed); });
}
double ref_grid_total_mass(void* h, int prop) {
    return static_cast<RefGridBase*>(h)->total_mass(prop);
}
double ref_grid_max_diffusivity(void* h, int prop) {
    return static_cast<RefGridBase*>(h)->max_diffusivity(prop);
}

/* run_simulation (solver.hpp:489-519); rows must hold n_steps/record_every+2. */
int ref_run_simulation(void* h, const pd_sim_config* cfg, time_factor_fn tf, pd_diag* rows,
                       int64_t* n_rows) {
    *n_rows = 0;
    return guarded([&] { static_cast<RefGridBase*>(h)->run(cfg, tf, rows, n_rows); });
}

/* ---- FRAP / D_eff (analysis.hpp:160-309), 3-D double ---------------------- */

/* run_frap on a sphere-pack grid + fit_effective_D against free-box runs.
 * Returns d_eff/tau and the reference curve (times, recovery). */
int ref_frap_fit(void* h, double bleach_fraction, double d_molecular, double t_final,
                 int n_samples, double dt, double d_lo, double d_hi, double rel_tol,
                 double* d_eff, double* tau, double* residual, double* curve_t,
                 double* curve_r, int64_t* curve_n) {
    return guarded([&] {
        auto* rg = dynamic_cast<RefGrid<double, 3>*>(static_cast<RefGridBase*>(h));
        if (!rg) throw pd::input_error("ref_frap_fit needs a 3-D double grid");
        const auto& geom = rg->g.geometry();
        const auto box = pd::central_bleach_box(geom, bleach_fraction);
        pd::FrapSchedule s;
        s.t_final = t_final;
        s.n_samples = n_samples;
        s.dt = dt;
        const auto exp = pd::run_frap(rg->g, box, d_molecular, s);
        *curve_n = static_cast<int64_t>(exp.curve.size());
        if (curve_t)
            for (std::size_t i = 0; i < exp.curve.size(); ++i) {
                curve_t[i] = exp.curve[i].time;
                curve_r[i] = exp.curve[i].recovery;
            }
        if (d_lo > 0.0) {
            pd::FitOptions o;
            o.dt = dt;
            o.rel_tol = rel_tol;
            const auto fit = pd::fit_effective_D(exp, geom, box, d_lo, d_hi, o);
            *d_eff = fit.d_eff;
            *tau = fit.tau_d;
            *residual = fit.fit_residual;
        }
    });
}

/* ---- level-set stage (levelset.hpp:115-191, geometry.hpp:121-142), dense
 *      fields in place ------------------------------------------------------- */

}  // extern "C"

namespace {
template <class T, int D, class F>
int with_field(const int64_t* size, const double* spacing, void* data, F&& f) {
    return guarded([&] {
        auto geom = geom_of<D>(size, spacing, nullptr);
        pd::DenseField<T, D> field(geom);
        std::memcpy(field.data(), data, sizeof(T) * (size_t)geom.node_count());
        f(field);
        std::memcpy(data, field.data(), sizeof(T) * (size_t)geom.node_count());
    });
}
template <class F>
int dispatch_field(int dims, int tbytes, const int64_t* size, const double* spacing, void* data, F&& f) {
    if (dims == 3 && tbytes == 8) return with_field<double, 3>(size, spacing, data, f);
    if (dims == 2 && tbytes == 8) return with_field<double, 2>(size, spacing, data, f);
    if (dims == 3) return with_field<float, 3>(size, spacing, data, f);
    return with_field<float, 2>(size, spacing, data, f);
}
}  // namespace

extern "C" {

int ref_field_redistance(int dims, int tbytes, const int64_t* size, const double* spacing, void* data,
                         const pd_levelset_options* o, pd_redistance_diag* out) {
    return dispatch_field(dims, tbytes, size, spacing, data, [&](auto& field) {
        pd::LevelSetOptions opts;
        opts.max_iterations = o->max_iterations;
        opts.tolerance = o->tolerance;
        opts.pseudo_time_step = o->pseudo_time_step;
        opts.band_width_for_error = o->band_width_for_error;
        opts.residual_band_width = o->residual_band_width;
        opts.rescale_initial = o->rescale_initial != 0;
        const auto d = pd::sussman_redistance(field, opts);
        out->iterations = d.iterations;
        out->final_residual = d.final_residual;
        out->converged = d.converged;
    });
}

int ref_field_filter_thin(int dims, int tbytes, const int64_t* size, const double* spacing, void* data,
                          int min_thickness_cells) {
    return dispatch_field(dims, tbytes, size, spacing, data, [&](auto& field) {
        field = pd::filter_thin_features(field, min_thickness_cells);
    });
}

/* ---- snapshots (snapshot.hpp) -------------------------------------------- */

int ref_grid_write_snapshot(void* h, const char* path) {
    return guarded([&] { static_cast<RefGridBase*>(h)->write_snapshot(path); });
}

/* read_sparse_snapshot into a reference grid handle (3-D double only). */
void* ref_grid_read_snapshot(const char* path, int* code) {
    void* out = nullptr;
    *code = guarded([&] { out = new RefGrid<double, 3>(pd::read_sparse_snapshot<double, 3>(path)); });
    return out;
}

int ref_field_write_snapshot(int dims, int tbytes, const int64_t* size, const double* spacing, const double* origin,
                             const void* data, const char* path) {
    return guarded([&] {
        auto go = [&](auto tag, auto dc) {
            using T = decltype(tag);
            constexpr int D = decltype(dc)::value;
            pd::DenseField<T, D> f(geom_of<D>(size, spacing, origin));
            std::memcpy(f.data(), data, sizeof(T) * (size_t)f.node_count());
            pd::write_dense_snapshot(f, path);
        };
        if (dims == 3 && tbytes == 8) go(double{}, std::integral_constant<int, 3>{});
        else if (dims == 2 && tbytes == 8) go(double{}, std::integral_constant<int, 2>{});
        else if (dims == 3) go(float{}, std::integral_constant<int, 3>{});
        else go(float{}, std::integral_constant<int, 2>{});
    });
}

/* ---- VTK (vtk.hpp) ------------------------------------------------------- */

int ref_grid_write_vtk(void* h, const char* path, const char* channels, double blank, const double* origin) {
    return guarded([&] { static_cast<RefGridBase*>(h)->write_vtk(path, channels, blank, origin); });
}

/* write_vtk of a dense dataset: n_arrays arrays (names '\n'-joined), optional
 * int32 mask (NULL = none). */
int ref_write_vtk(const char* path, const char* title, int dims, int tbytes, const int64_t* size,
                  const double* spacing, const double* origin, int n_arrays, const char* names,
                  const void* const* values, const int32_t* mask, int64_t mask_len) {
    return guarded([&] {
        std::vector<std::string> nm;
        std::string cur;
        for (const char* c = names; *c; ++c) {
            if (*c == '\n') {
                nm.push_back(cur);
                cur.clear();
            } else {
                cur.push_back(*c);
            }
        }
        nm.push_back(cur);
        auto go = [&](auto tag, auto dc) {
            using T = decltype(tag);
            constexpr int D = decltype(dc)::value;
            pd::VtkDataset<T, D> ds;
            ds.geometry = geom_of<D>(size, spacing, origin);
            const size_t n = (size_t)ds.geometry.node_count();
            for (int i = 0; i < n_arrays; ++i) {
                const T* v = static_cast<const T*>(values[i]);
                ds.add_scalar(nm[(size_t)i], std::vector<T>(v, v + n));
            }
            if (mask) ds.mask.assign(mask, mask + mask_len);
            pd::write_vtk(ds, path, title);
        };
        if (dims == 3 && tbytes == 8) go(double{}, std::integral_constant<int, 3>{});
        else if (dims == 2 && tbytes == 8) go(double{}, std::integral_constant<int, 2>{});
        else if (dims == 3) go(float{}, std::integral_constant<int, 3>{});
        else go(float{}, std::integral_constant<int, 2>{});
    });
}

}  // extern "C"
