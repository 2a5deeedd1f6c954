// porediff drop-in: the FTCS reaction-diffusion stepper (reference
// solver.hpp:36-519) with the step executed on the B200.
//
// Same types, names, validation order, messages and results as the
// reference; the hot loop (process_chunk / gather, solver.hpp:360-455) and
// the per-step diagnostics (solver.hpp:262-278) run in the CUDA kernels of
// libporediff_b200.so through the C ABI (include/porediff_b200.h). The host
// SparseBlockGrid stays the source of truth; its device mirror is refreshed
// lazily (sparse_block_grid.hpp here), so a run_simulation over n steps moves
// the grid to the GPU once and u back only when the host reads it.
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "porediff/b200.hpp"
#include "porediff/errors.hpp"
#include "porediff/geometry.hpp"
#include "porediff/parallel.hpp"
#include "porediff/scalar_text.hpp"
#include "porediff/sparse_block_grid.hpp"

namespace porediff {

struct ReactionSpec {
    enum class Kind { none, surface_sink, volumetric };

    Kind kind = Kind::none;
    double rate = 0.0;             // surface_sink k >= 0: -k*u on |phi| <= w*h_min
    double band_half_width = 1.0;  // surface_sink w > 0
    std::string source_channel;    // volumetric f(x)
    std::function<double(double)> time_factor;  // volumetric g(t), optional

    static ReactionSpec none() { return {}; }
    static ReactionSpec surface_sink(double k, double w = 1.0) {
        ReactionSpec r;
        r.kind = Kind::surface_sink;
        r.rate = k;
        r.band_half_width = w;
        return r;
    }
    static ReactionSpec volumetric(std::string channel, std::function<double(double)> g = {}) {
        ReactionSpec r;
        r.kind = Kind::volumetric;
        r.source_channel = std::move(channel);
        r.time_factor = std::move(g);
        return r;
    }
};

struct FaceBc {
    enum class Type { no_flux, dirichlet };
    Type type = Type::no_flux;
    double value = 0.0;

    static FaceBc no_flux() { return {}; }
    static FaceBc dirichlet(double v) { return {Type::dirichlet, v}; }
};

struct SimulationConfig {
    double dt = 0.0;
    std::int64_t n_steps = 1;
    PhaseBand phase_band{};
    double boundary_epsilon = 0.0;
    ReactionSpec reaction{};
    std::array<FaceBc, 6> outer_bc{};  // [axis*2 + side]
    std::int64_t record_every = 1;
    bool enforce_stability = true;
};

struct StepDiagnostics {
    std::int64_t step = 0;
    double time = 0.0;
    double total_mass = 0.0;
    double min_u = 0.0;
    double max_u = 0.0;
    double wall_seconds = 0.0;
};

/// dt_max = 1 / (2 D_max) / sum_a h_a^-2 (strict bound; reference solver.hpp:103-115).
template <int Dims>
double stability_dt(const GridGeometry<Dims>& geometry, double d_max) {
    if (!(d_max > 0.0)) throw input_error("stability bound needs D_max > 0");
    double inv_sum = 0.0;
    for (int a = 0; a < Dims; ++a) inv_sum += 1.0 / (geometry.spacing[a] * geometry.spacing[a]);
    return 1.0 / (2.0 * d_max) / inv_sum;
}

/// Pointwise reaction rate before the dt factor (reference solver.hpp:120-134).
inline double apply_reaction(double u, double phi, const ReactionSpec& spec, double h_min, double time,
                             double source_value = 0.0) {
    if (spec.kind == ReactionSpec::Kind::surface_sink)
        return std::abs(phi) <= spec.band_half_width * h_min ? -spec.rate * u : 0.0;
    if (spec.kind == ReactionSpec::Kind::volumetric)
        return spec.time_factor ? source_value * spec.time_factor(time) : source_value;
    return 0.0;
}

/// Max of a channel over active nodes, 0 on an empty grid (solver.hpp:139-154).
/// Evaluated on the device mirror (pd_grid_max_active; the max is
/// order-free, so the fold order does not matter).
template <typename T, int Dims>
double max_diffusivity(const SparseBlockGrid<T, Dims>& grid, std::string_view channel = "D") {
    const int prop = grid.property_index(channel);
    double out = 0.0;
    b200::check(pd_grid_max_active(const_cast<SparseBlockGrid<T, Dims>&>(grid).device_grid(), prop, &out));
    return out;
}

/// sum(u) * cell volume: per-chunk sequential sums, pairwise over chunks
/// (solver.hpp:158-171), on the device mirror (pd_grid_total_mass keeps the
/// reference's summation order, so the bits are the same).
template <typename T, int Dims>
double total_mass(const SparseBlockGrid<T, Dims>& grid, std::string_view channel = "u") {
    const int prop = grid.property_index(channel);
    double out = 0.0;
    b200::check(pd_grid_total_mass(const_cast<SparseBlockGrid<T, Dims>&>(grid).device_grid(), prop, &out));
    return out;
}

inline constexpr const char* scratch_channel = "u_next";

inline std::vector<std::string> solver_channels() { return {"phi", "u", "D", scratch_channel}; }

/// FtcsStepper<T,Dims> (reference solver.hpp:183-467) bound to a grid; the
/// step runs on the grid's B200 mirror. Construction validates exactly like
/// the reference and creates the device stepper (neighbour table, march
/// schedule) once.
template <typename T, int Dims>
class FtcsStepper {
  public:
    using Grid = SparseBlockGrid<T, Dims>;
    using Chunk = typename Grid::Chunk;
    static constexpr int volume = Grid::chunk_volume;

    FtcsStepper(Grid& grid, const SimulationConfig& config) : grid_(grid), cfg_(config) {
        validate();
        i_phi_ = grid_.property_index("phi");
        i_u_ = grid_.property_index("u");
        i_d_ = grid_.property_index("D");
        i_next_ = grid_.property_index(scratch_channel);
        i_src_ = cfg_.reaction.kind == ReactionSpec::Kind::volumetric
                     ? grid_.property_index(cfg_.reaction.source_channel)
                     : -1;
        c_.dt = cfg_.dt;
        c_.n_steps = cfg_.n_steps;
        c_.b_low = cfg_.phase_band.b_low;
        c_.b_up = cfg_.phase_band.b_up;
        c_.boundary_epsilon = cfg_.boundary_epsilon;
        c_.reaction_kind = cfg_.reaction.kind == ReactionSpec::Kind::surface_sink ? PD_REACTION_SURFACE_SINK
                           : cfg_.reaction.kind == ReactionSpec::Kind::volumetric ? PD_REACTION_VOLUMETRIC
                                                                                   : PD_REACTION_NONE;
        c_.source_prop = i_src_;
        c_.rate = cfg_.reaction.rate;
        c_.band_half_width = cfg_.reaction.band_half_width;
        for (int f = 0; f < 6; ++f) {
            c_.bc_type[f] = cfg_.outer_bc[f].type == FaceBc::Type::dirichlet ? PD_BC_DIRICHLET : PD_BC_NO_FLUX;
            c_.bc_value[f] = cfg_.outer_bc[f].value;
        }
        c_.record_every = cfg_.record_every;
        c_.enforce_stability = cfg_.enforce_stability ? 1 : 0;
        c_.has_time_factor = cfg_.reaction.time_factor ? 1 : 0;
        bind();
    }

    FtcsStepper(const FtcsStepper&) = delete;
    FtcsStepper& operator=(const FtcsStepper&) = delete;
    ~FtcsStepper() {
        if (st_) pd_stepper_destroy(st_);
    }

    const SimulationConfig& config() const { return cfg_; }

    /// stability_dt(max D over active nodes), or +inf if that max is <= 0
    /// (solver.hpp:220-224), evaluated by the device stepper.
    double stability_bound() const {
        const_cast<FtcsStepper*>(this)->bind();
        double out = 0.0;
        b200::check(pd_stepper_stability_bound(st_, &out));
        return out;
    }

    /// One step from state u(step_index*dt) (reference solver.hpp:228-279).
    /// A non-finite node throws numeric_error; a non-finite total mass is
    /// returned in the row (run_simulation checks it, solver.hpp:514-515).
    StepDiagnostics step(std::int64_t step_index) {
        const auto t0 = std::chrono::steady_clock::now();
        bind();
        double factor = 1.0;
        if (cfg_.reaction.kind == ReactionSpec::Kind::volumetric && cfg_.reaction.time_factor)
            factor = static_cast<double>(
                static_cast<T>(cfg_.reaction.time_factor(static_cast<double>(step_index) * cfg_.dt)));
        int col_before = 0, col_after = 0;
        b200::check(pd_grid_column_of(dev_.get(), i_u_, &col_before));
        pd_diag d{};
        const int rc = pd_stepper_step(st_, step_index, factor, &d);
        const std::string err = rc == PD_OK ? std::string() : std::string(pd_last_error());
        b200::check(pd_grid_column_of(dev_.get(), i_u_, &col_after));
        if (col_after != col_before)
            grid_.note_device_swap(i_u_, i_next_);
        else {
            grid_.mark_device_newer(i_u_);
            grid_.mark_device_newer(i_next_);
        }
        if (rc != PD_OK) b200::raise(rc, err);
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return {d.step, d.time, d.total_mass, d.min_u, d.max_u, wall};
    }

    /// `n` consecutive steps in one device call; returns the rows
    /// run_simulation records ((s+1) % record_every == 0 or s+1 == final_step).
    /// Equivalent to n calls of step() plus run_simulation's per-step
    /// non-finite-mass check.
    std::vector<StepDiagnostics> advance(std::int64_t step0, std::int64_t n, std::int64_t final_step) {
        const auto t0 = std::chrono::steady_clock::now();
        bind();
        std::vector<double> factors;
        if (cfg_.reaction.kind == ReactionSpec::Kind::volumetric && cfg_.reaction.time_factor) {
            factors.resize(static_cast<std::size_t>(n));
            for (std::int64_t k = 0; k < n; ++k)
                factors[static_cast<std::size_t>(k)] =
                    static_cast<double>(static_cast<T>(cfg_.reaction.time_factor(static_cast<double>(step0 + k) * cfg_.dt)));
        }
        int col_before = 0, col_after = 0;
        b200::check(pd_grid_column_of(dev_.get(), i_u_, &col_before));
        std::vector<pd_diag> rows(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
        std::int64_t n_rows = 0;
        const int rc = pd_stepper_run(st_, step0, n, final_step, factors.empty() ? nullptr : factors.data(),
                                      rows.data(), &n_rows);
        const std::string err = rc == PD_OK ? std::string() : std::string(pd_last_error());
        // the device swapped u/u_next once per completed step; mirror the parity
        b200::check(pd_grid_column_of(dev_.get(), i_u_, &col_after));
        if (col_after != col_before)
            grid_.note_device_swap(i_u_, i_next_);
        else {
            grid_.mark_device_newer(i_u_);
            grid_.mark_device_newer(i_next_);
        }
        if (rc != PD_OK) b200::raise(rc, err);
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::vector<StepDiagnostics> out;
        out.reserve(static_cast<std::size_t>(n_rows));
        for (std::int64_t r = 0; r < n_rows; ++r) {
            const pd_diag& d = rows[static_cast<std::size_t>(r)];
            out.push_back({d.step, d.time, d.total_mass, d.min_u, d.max_u, wall / static_cast<double>(n)});
        }
        return out;
    }

    /// Step-0 row: mass / min / max of the current u (solver.hpp:282-301).
    StepDiagnostics snapshot_diagnostics() const {
        const_cast<FtcsStepper*>(this)->bind();
        pd_diag d{};
        b200::check(pd_stepper_snapshot_diag(st_, &d));
        StepDiagnostics s;
        s.total_mass = d.total_mass;
        s.min_u = d.min_u;
        s.max_u = d.max_u;
        return s;
    }

    /// Attaches the device region-mass observer (run_frap): every recorded
    /// step of advance() also yields the lexicographic sum of u over [lo, hi).
    void set_region(const NodeIndex<Dims>& lo, const NodeIndex<Dims>& hi) {
        bind();
        region_ = true;
        lo_ = lo;
        hi_ = hi;
        std::int64_t a[3] = {0, 0, 0}, b[3] = {1, 1, 1};
        for (int k = 0; k < Dims; ++k) {
            a[k] = lo[k];
            b[k] = hi[k];
        }
        b200::check(pd_stepper_set_region(st_, a, b));
    }

    /// Region sums of the rows of the last advance() (row order).
    std::vector<double> region_sums() const {
        std::int64_t n = 0;
        b200::check(pd_stepper_region_sums(st_, nullptr, 0, &n));
        std::vector<double> out(static_cast<std::size_t>(n));
        b200::check(pd_stepper_region_sums(st_, out.data(), n, &n));
        return out;
    }

    /// Region sum of the current u (the step-0 row).
    double region_sum_now() const {
        std::int64_t a[3] = {0, 0, 0}, b[3] = {1, 1, 1};
        for (int k = 0; k < Dims; ++k) {
            a[k] = lo_[k];
            b[k] = hi_[k];
        }
        double m = 0.0;
        b200::check(pd_grid_box_sum(dev_.get(), i_u_, a, b, &m));
        return m;
    }

    /// Device time of the last advance()'s step kernels (CUDA events).
    double last_device_ms() const {
        double ms = 0.0;
        b200::check(pd_stepper_last_ms(st_, &ms));
        return ms;
    }

  private:
    // Reference solver.hpp:304-330, same order and messages.
    void validate() const {
        if (!(cfg_.dt > 0.0) || !std::isfinite(cfg_.dt)) throw input_error("time step must be positive and finite");
        if (cfg_.n_steps < 1) throw input_error("step count must be at least 1");
        if (cfg_.record_every < 1) throw input_error("record_every must be at least 1");
        if (!(cfg_.phase_band.b_low < cfg_.phase_band.b_up))
            throw input_error("phase band is empty (b_low must be < b_up)");
        if (cfg_.boundary_epsilon < 0.0 || !std::isfinite(cfg_.boundary_epsilon))
            throw input_error("boundary_epsilon must be finite and >= 0");
        if (cfg_.reaction.kind == ReactionSpec::Kind::surface_sink) {
            if (cfg_.reaction.rate < 0.0) throw input_error("surface sink rate must be >= 0");
            if (!(cfg_.reaction.band_half_width > 0.0))
                throw input_error("surface sink band half-width must be > 0");
        }
        for (const std::string& ch : solver_channels()) {
            const auto names = grid_.property_names();
            if (std::find(names.begin(), names.end(), ch) == names.end())
                throw input_error("grid lacks the '" + ch +
                                  "' channel; build simulation grids with channels {phi, u, D, u_next}");
        }
        if (cfg_.reaction.kind == ReactionSpec::Kind::volumetric)
            (void)grid_.property_index(cfg_.reaction.source_channel);
    }

    /// (Re)creates the device stepper when the grid's mirror changed (first
    /// use, or the host inserted nodes since).
    void bind() {
        auto dev = grid_.device_grid_shared();
        if (st_ && dev.get() == dev_.get()) return;
        if (st_) pd_stepper_destroy(st_);
        st_ = nullptr;
        dev_ = std::move(dev);
        b200::check(pd_stepper_create(dev_.get(), &c_, i_phi_, i_u_, i_d_, i_next_, &st_));
        if (region_) set_region(lo_, hi_);
    }

    Grid& grid_;
    SimulationConfig cfg_;
    pd_sim_config c_{};
    int i_phi_ = -1, i_u_ = -1, i_d_ = -1, i_next_ = -1, i_src_ = -1;
    std::shared_ptr<pd_grid> dev_;
    pd_stepper* st_ = nullptr;
    bool region_ = false;
    NodeIndex<Dims> lo_{}, hi_{};
};

template <typename T, int Dims>
StepDiagnostics ftcs_step(SparseBlockGrid<T, Dims>& grid, const SimulationConfig& config,
                          std::int64_t step_index = 0) {
    FtcsStepper<T, Dims> stepper(grid, config);
    return stepper.step(step_index);
}

template <typename T, int Dims>
using SimulationObserver = std::function<void(const SparseBlockGrid<T, Dims>&, const StepDiagnostics&)>;

struct SimulationResult {
    std::vector<StepDiagnostics> diagnostics;  // step 0 plus every recorded step
};

namespace detail {

/// run_simulation core; with `region` (lo, hi) the device region-mass
/// observer of run_frap is attached and its per-row sums appended to `sums`.
template <typename T, int Dims>
SimulationResult run_simulation_impl(SparseBlockGrid<T, Dims>& grid, const SimulationConfig& config,
                                     const std::vector<SimulationObserver<T, Dims>>& observers,
                                     const NodeIndex<Dims>* region, std::vector<double>* sums) {
    FtcsStepper<T, Dims> stepper(grid, config);
    if (config.enforce_stability) {
        const double bound = stepper.stability_bound();
        if (!(config.dt < bound))
            throw stability_error("time step " + format_scalar(config.dt) + " violates the explicit stability bound " +
                                  format_scalar(bound) + " (dt must be strictly below it; max D = " +
                                  format_scalar(max_diffusivity(grid)) + ")");
    }
    if (region) stepper.set_region(region[0], region[1]);
    SimulationResult result;
    auto record = [&](const StepDiagnostics& d) {
        result.diagnostics.push_back(d);
        for (const auto& obs : observers) obs(grid, d);
    };
    record(stepper.snapshot_diagnostics());
    if (region) sums->push_back(stepper.region_sum_now());
    const std::int64_t n = config.n_steps;
    if (observers.empty()) {
        for (const auto& d : stepper.advance(0, n, n)) result.diagnostics.push_back(d);
        if (region)
            for (double m : stepper.region_sums()) sums->push_back(m);
        return result;
    }
    for (std::int64_t s = 0; s < n;) {
        const std::int64_t next = std::min(n, (s / config.record_every + 1) * config.record_every);
        for (const auto& d : stepper.advance(s, next - s, n)) record(d);
        if (region)
            for (double m : stepper.region_sums()) sums->push_back(m);
        s = next;
    }
    return result;
}

}  // namespace detail

/// Reference solver.hpp:489-519. Without observers the whole run is one
/// device call; with observers the run is split at record points so each
/// observer sees the grid at exactly the recorded step.
template <typename T, int Dims>
SimulationResult run_simulation(SparseBlockGrid<T, Dims>& grid, const SimulationConfig& config,
                                const std::vector<SimulationObserver<T, Dims>>& observers = {}) {
    return detail::run_simulation_impl(grid, config, observers, nullptr, nullptr);
}

}  // namespace porediff
