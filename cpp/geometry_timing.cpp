// Times the reference-API geometry stage through the drop-in headers at
// large sizes: mask_to_indicator -> filter_thin_features
// -> build_sparse_grid -> populate_diffusion_channel -> FTCS steps, every
// node pass on the B200. The mask is a thresholded trigonometric field made on
// the host (the caller's input, untimed).
//   build/cpp/geometry_timing [n=1024] [steps=20]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "porediff/geometry.hpp"
#include "porediff/solver.hpp"

using namespace porediff;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); }

int main(int argc, char** argv) {
    const std::int64_t n = argc > 1 ? std::atoll(argv[1]) : 1024;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 20;
    const double h = 1.0 / static_cast<double>(n);
    std::vector<std::uint8_t> bits(static_cast<std::size_t>(n * n * n));
    for (std::int64_t z = 0; z < n; ++z)
        for (std::int64_t y = 0; y < n; ++y)
            for (std::int64_t x = 0; x < n; ++x) {
                const double px = 6.2831853 * 3 * (x + 0.5) * h, py = 6.2831853 * 3 * (y + 0.5) * h,
                             pz = 6.2831853 * 3 * (z + 0.5) * h;
                const double g = std::sin(px) * std::cos(py) + std::sin(py) * std::cos(pz) + std::sin(pz) * std::cos(px);
                bits[static_cast<std::size_t>((z * n + y) * n + x)] = g > 0.2;  // gyroid-like pore space
            }
    auto mask = VoxelMask<3>::make({n, n, n}, {h, h, h}, std::move(bits));
    auto t = clk::now();
    auto ind = mask_to_indicator<double, 3>(mask);
    const double t_ind = secs(t);
    t = clk::now();
    auto opened = filter_thin_features(ind, 2);
    const double t_open = secs(t);
    t = clk::now();
    auto grid = build_sparse_grid(opened, PhaseBand{0.0, std::numeric_limits<double>::infinity()}, solver_channels());
    const double t_build = secs(t);
    t = clk::now();
    populate_diffusion_channel(grid, DiffusionProfile{0.05, 1.0, 0.0, 4.0 / h});
    const double t_d = secs(t);
    SimulationConfig cfg;
    t = clk::now();
    cfg.dt = 0.4 * stability_dt(grid.geometry(), max_diffusivity(grid));
    const double t_max = secs(t);
    cfg.n_steps = steps;
    cfg.record_every = steps;
    cfg.reaction = ReactionSpec::surface_sink(1.0, 1.0);
    t = clk::now();
    const auto r = run_simulation(grid, cfg);
    const double t_run = secs(t);
    std::printf("n=%lld chunks=%lld active=%lld\n", (long long)n, (long long)grid.chunk_count(),
                (long long)grid.active_node_count());
    std::printf("mask_to_indicator %.3f s, filter_thin_features %.3f s, build_sparse_grid %.3f s, "
                "populate_diffusion_channel %.3f s, max_diffusivity %.3f s, run_simulation(%d steps, incl. "
                "upload) %.3f s, final mass %.17g\n",
                t_ind, t_open, t_build, t_d, t_max, steps, t_run, r.diagnostics.back().total_mass);
    return 0;
}
