// porediff drop-in: level-set redistancing (reference levelset.hpp:13-228).
//
// sussman_redistance runs on the B200 (pd_field_redistance: bit-exact Jacobi
// sweeps, same stopping rule and iteration count); the DenseField stays the
// caller's host container and is copied in and out around the device call.
// The scalar building blocks and the verification norm are host functions
// with the reference's semantics (they are queried per node by tests and
// reports, never in a loop over the grid).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>

#include "porediff/b200.hpp"
#include "porediff/dense_field.hpp"
#include "porediff/errors.hpp"

namespace porediff {

struct LevelSetOptions {
    int max_iterations = 1000;
    double tolerance = 1e-3;          ///< stop when the max band update < tolerance * h
    double pseudo_time_step = 0.5;    ///< in units of h
    double band_width_for_error = 4.0;
    double residual_band_width = 6.0; ///< |phi| <= width*h nodes feed the stopping rule
    bool rescale_initial = true;      ///< start from sign(phi)*h
};

struct RedistanceDiagnostics {
    int iterations = 0;
    double final_residual = 0.0;  ///< last max band update / h
    bool converged = false;
};

/// phi / sqrt(phi^2 + |grad|^2 h^2); exactly 0 at phi = 0.
template <typename T>
T smoothed_sign(T phi, T grad_mag, T h) {
    if (phi == T{0}) return T{0};
    const T denom2 = phi * phi + grad_mag * grad_mag * h * h;
    return phi / std::sqrt(denom2);
}

namespace detail {

/// Squared one-axis Godunov term: for a non-negative sign the admissible
/// differences are the positive backward and the negative forward one,
/// mirrored for a negative sign; the larger square wins.
template <typename T>
T godunov_axis_sq(T d_minus, T d_plus, int sign) {
    const bool up = sign >= 0;
    const T back = up ? std::max(d_minus, T{0}) : std::min(d_minus, T{0});
    const T fwd = up ? std::min(d_plus, T{0}) : std::max(d_plus, T{0});
    return std::max(back * back, fwd * fwd);
}

}  // namespace detail

/// Godunov upwind |grad phi| at one node; a missing one-sided difference at
/// a box face is replaced by the other one.
template <typename T, int Dims>
T upwind_gradient_magnitude(const DenseField<T, Dims>& phi, const NodeIndex<Dims>& idx, int sign_at_index) {
    const auto& g = phi.geometry();
    if (!g.contains(idx)) throw bounds_error("upwind gradient queried outside grid");
    const std::int64_t f = g.flat_index(idx);
    std::int64_t stride = 1;
    T acc{0};
    for (int a = 0; a < Dims; ++a) {
        const T inv_h = static_cast<T>(1.0 / g.spacing[a]);
        const bool lo = idx[a] > 0, hi = idx[a] + 1 < g.size[a];
        T back{0}, fwd{0};
        if (lo) back = (phi[f] - phi[f - stride]) * inv_h;
        if (hi) fwd = (phi[f + stride] - phi[f]) * inv_h;
        if (!lo) back = fwd;
        if (!hi) fwd = back;
        acc += detail::godunov_axis_sq(back, fwd, sign_at_index);
        stride *= g.size[a];
    }
    return std::sqrt(acc);
}

/// True when some pair of axis-neighbours has opposite signs (one < 0).
template <typename T, int Dims>
bool has_zero_crossing(const DenseField<T, Dims>& phi) {
    const auto& g = phi.geometry();
    bool found = false;
    std::int64_t stride = 1;
    for (int a = 0; a < Dims && !found; ++a) {
        if (g.size[a] > 1)
            phi.for_each_index([&](const NodeIndex<Dims>& idx, std::int64_t f) {
                if (!found && idx[a] + 1 < g.size[a] && ((phi[f] < T{0}) != (phi[f + stride] < T{0})))
                    found = true;
            });
        stride *= g.size[a];
    }
    return found;
}

/// Redistancing toward |grad phi| = 1 on the device (pd_field_redistance).
template <typename T, int Dims>
RedistanceDiagnostics sussman_redistance(DenseField<T, Dims>& phi, const LevelSetOptions& opts = {}) {
    const auto& g = phi.geometry();
    std::int64_t size[3] = {1, 1, 1};
    double spacing[3] = {1, 1, 1}, origin[3] = {0, 0, 0};
    for (int a = 0; a < Dims; ++a) {
        size[a] = g.size[a];
        spacing[a] = g.spacing[a];
        origin[a] = g.origin[a];
    }
    pd_field* raw = nullptr;
    b200::check(pd_field_create(Dims, static_cast<int>(sizeof(T)), size, spacing, origin, b200::default_device(),
                                &raw));
    std::unique_ptr<pd_field, int (*)(pd_field*)> field(raw, pd_field_destroy);
    b200::check(pd_field_upload(field.get(), phi.data()));
    pd_levelset_options o{};
    o.max_iterations = opts.max_iterations;
    o.tolerance = opts.tolerance;
    o.pseudo_time_step = opts.pseudo_time_step;
    o.band_width_for_error = opts.band_width_for_error;
    o.residual_band_width = opts.residual_band_width;
    o.rescale_initial = opts.rescale_initial ? 1 : 0;
    pd_redistance_diag d{};
    b200::check(pd_field_redistance(field.get(), &o, &d));
    b200::check(pd_field_download(field.get(), phi.data()));
    RedistanceDiagnostics out;
    out.iterations = d.iterations;
    out.final_residual = d.final_residual;
    out.converged = d.converged != 0;
    return out;
}

struct BandErrorNorms {
    double l2 = 0.0;    ///< RMS absolute error over band nodes
    double linf = 0.0;  ///< max absolute error over band nodes
    std::int64_t count = 0;
};

/// Error norms against an exact functor of position over |exact| <= w*h.
template <typename T, int Dims, class ExactFn>
BandErrorNorms band_error_norms(const DenseField<T, Dims>& phi, ExactFn&& exact, double band_width) {
    const auto& g = phi.geometry();
    const double band = band_width * g.min_spacing();
    BandErrorNorms r;
    double sq = 0.0;
    phi.for_each_index([&](const NodeIndex<Dims>& idx, std::int64_t f) {
        const double e = exact(g.position(idx));
        if (std::abs(e) > band) return;
        const double err = std::abs(static_cast<double>(phi[f]) - e);
        sq += err * err;
        r.linf = std::max(r.linf, err);
        ++r.count;
    });
    if (r.count == 0) throw input_error("error band is empty: no node satisfies |exact| <= band_width*h");
    r.l2 = std::sqrt(sq / static_cast<double>(r.count));
    return r;
}

}  // namespace porediff
