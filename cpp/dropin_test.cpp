// Coherence tests of the drop-in's host grid <-> B200 mirror (include/porediff):
// a run split into any sequence of device calls, interleaved with host reads,
// host writes, channel swaps, copies and re-layouts, must give the same bits
// as one uninterrupted run.
#include <gtest/gtest.h>

#include <bit>
#include <cstdint>
#include <vector>

#include "porediff/geometry.hpp"
#include "porediff/solver.hpp"
#include "porediff/synthetic.hpp"

namespace pd = porediff;
using Grid = pd::SparseBlockGrid<double, 3>;

namespace {

Grid ball_grid(std::int64_t n) {
    const auto geom = pd::GridGeometry<3>::cell_centered_box(n, 0.0, 1.0);
    const auto sdf = pd::synthetic::field_from<double, 3>(geom, [](const std::array<double, 3>& x) {
        return pd::synthetic::ball_sdf<3>(x, {0.5, 0.5, 0.5}, 0.41);
    });
    auto grid = pd::build_sparse_grid(sdf, pd::PhaseBand{}, pd::solver_channels());
    pd::populate_diffusion_channel(grid, pd::DiffusionProfile::anchored(0.1, 1.0, 30.0, 0.05));
    grid.for_each_active([&](const Grid::Index& idx, const Grid::Chunk&, int) {
        grid.set(idx, "u", static_cast<double>((idx[0] * 7 + idx[1] * 3 + idx[2]) % 11) / 11.0);
    });
    return grid;
}

pd::SimulationConfig cfg_for(const Grid& g, std::int64_t steps) {
    pd::SimulationConfig c;
    c.dt = 0.45 * pd::stability_dt(g.geometry(), pd::max_diffusivity(g));
    c.n_steps = steps;
    c.record_every = 3;
    c.reaction = pd::ReactionSpec::surface_sink(1.5, 1.0);
    c.outer_bc[4] = pd::FaceBc::dirichlet(0.25);
    return c;
}

std::vector<std::uint64_t> bits_of(const Grid& g, const char* ch) {
    std::vector<std::uint64_t> out;
    g.for_each_active([&](const Grid::Index& idx, const Grid::Chunk&, int) {
        out.push_back(std::bit_cast<std::uint64_t>(*g.get(idx, ch)));
    });
    return out;
}

}  // namespace

TEST(DropIn, OneCallEqualsStepwiseCalls) {
    Grid a = ball_grid(24), b = ball_grid(24);
    const auto cfg = cfg_for(a, 10);
    const auto res = pd::run_simulation(a, cfg);
    for (std::int64_t s = 0; s < 10; ++s) {
        const auto d = pd::ftcs_step(b, cfg, s);
        if ((s + 1) % 3 == 0 || s == 9) {
            const auto& r = res.diagnostics[static_cast<std::size_t>((s + 1) / 3 + (s == 9 ? 1 : 0))];
            EXPECT_EQ(std::bit_cast<std::uint64_t>(r.total_mass), std::bit_cast<std::uint64_t>(d.total_mass));
            EXPECT_EQ(r.step, d.step);
        }
    }
    EXPECT_EQ(bits_of(a, "u"), bits_of(b, "u"));
    EXPECT_EQ(bits_of(a, "u_next"), bits_of(b, "u_next"));
}

TEST(DropIn, ObserversSeeTheRecordedState) {
    Grid a = ball_grid(20), b = ball_grid(20);
    const auto cfg = cfg_for(a, 8);
    std::vector<double> seen;
    std::vector<pd::SimulationObserver<double, 3>> obs = {
        [&](const Grid& g, const pd::StepDiagnostics&) { seen.push_back(pd::total_mass(g)); }};
    const auto with = pd::run_simulation(a, cfg, obs);
    const auto without = pd::run_simulation(b, cfg);
    ASSERT_EQ(with.diagnostics.size(), without.diagnostics.size());
    ASSERT_EQ(seen.size(), with.diagnostics.size());
    for (std::size_t i = 0; i < seen.size(); ++i) {
        EXPECT_EQ(std::bit_cast<std::uint64_t>(with.diagnostics[i].total_mass),
                  std::bit_cast<std::uint64_t>(without.diagnostics[i].total_mass));
        EXPECT_EQ(std::bit_cast<std::uint64_t>(seen[i]), std::bit_cast<std::uint64_t>(with.diagnostics[i].total_mass));
    }
    EXPECT_EQ(bits_of(a, "u"), bits_of(b, "u"));
}

TEST(DropIn, HostWritesBetweenRunsReachTheDevice) {
    Grid a = ball_grid(20), b = ball_grid(20);
    auto cfg = cfg_for(a, 4);
    pd::run_simulation(a, cfg);
    pd::run_simulation(b, cfg);
    const Grid::Index probe{10, 10, 10};
    a.set(probe, "u", 3.0);
    b.set(probe, "u", 3.0);
    Grid c = b;  // host copy made after the write carries it to its own mirror
    pd::run_simulation(a, cfg);
    pd::run_simulation(c, cfg);
    EXPECT_EQ(bits_of(a, "u"), bits_of(c, "u"));
    EXPECT_NE(bits_of(a, "u"), bits_of(b, "u"));
}

TEST(DropIn, SwapAndRelayoutKeepTheMirrorCoherent) {
    Grid a = ball_grid(20), b = ball_grid(20);
    auto cfg = cfg_for(a, 5);
    pd::run_simulation(a, cfg);
    pd::run_simulation(b, cfg);
    a.swap_channels("u", "u_next");  // device-side O(1) swap, no transfer
    b.swap_channels("u", "u_next");
    (void)bits_of(b, "u");           // force b's host copy current before inserting
    EXPECT_EQ(bits_of(a, "u"), bits_of(b, "u"));
    // a node in a new chunk changes the layout: the mirror is rebuilt
    const Grid::Index far{0, 0, 0};
    ASSERT_FALSE(a.is_active(far));
    const std::vector<double> vals = {1e-3, 0.5, 1.0, 0.0};
    a.insert(far, vals);
    b.insert(far, vals);
    pd::run_simulation(a, cfg);
    pd::FtcsStepper<double, 3> st(b, cfg);
    for (std::int64_t s = 0; s < 5; ++s) st.step(s);
    EXPECT_EQ(bits_of(a, "u"), bits_of(b, "u"));
    EXPECT_EQ(a.active_node_count(), b.active_node_count());
}

TEST(DropIn, NumericErrorLeavesReferenceState) {
    Grid a = ball_grid(16);
    auto cfg = cfg_for(a, 3);
    cfg.enforce_stability = false;
    cfg.dt *= 1e300;
    try {
        pd::run_simulation(a, cfg);
        FAIL() << "expected numeric_error";
    } catch (const pd::numeric_error& e) {
        EXPECT_NE(std::string(e.what()).find("at step"), std::string::npos);
    }
}
