"""The reference's own solver known-answer tests (solver_test.cpp), restated
through the Python mirror of the porediff API and run on the B200."""
import math

import numpy as np
import pytest

from cases import solver_test_hash

pytestmark = pytest.mark.gpu
INF = math.inf


def bits_equal(a, b):
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


def disk_grid(n, radius=0.8):
    """solver_test.cpp:40-53"""
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import ball_sdf_field
    geom = pd.GridGeometry.cell_centered_box(n, -1.0, 1.0, 2)
    sdf = ball_sdf_field(geom, (0.0, 0.0), radius)
    grid = pd.build_sparse_grid(sdf, geom, pd.PhaseBand(0.0, INF), pd.solver_channels())
    pd.populate_diffusion_channel(grid, pd.DiffusionProfile(0.05, 1.0, 0.0, 16.0))
    u = grid.channel_data("u", writable=True)
    act = grid.active_bool()
    idx = grid.node_indices()
    for j, off in zip(*np.nonzero(act)):
        u[j, off] = solver_test_hash(int(idx[j, off, 0]), int(idx[j, off, 1]), 0, 0.0, 1.0)
    return grid


def row_grid(n, h, channels=None):
    """solver_test.cpp:57-68"""
    from paper_2304_11165_b200 import porediff as pd
    channels = channels or pd.solver_channels()
    geom = pd.GridGeometry.make((n, 3), (h, h))
    grid = pd.SparseBlockGrid(geom, channels)
    for x in range(n):
        grid.insert((x, 1))
        grid.set((x, 1), "phi", 1.0)
        grid.set((x, 1), "D", 1.0)
    return grid


def basic_config(dt, steps=1):
    from paper_2304_11165_b200 import porediff as pd
    return pd.SimulationConfig(dt=dt, n_steps=steps)


def test_hand_evaluated_three_point_stencil(cuda):
    from paper_2304_11165_b200 import porediff as pd
    h, dt = 0.5, 1.0 / 64
    grid = row_grid(3, h)
    grid.set((1, 1), "u", 1.0)
    diag = pd.ftcs_step(grid, basic_config(dt))
    q = dt / (h * h)
    assert grid.get((0, 1), "u") == q
    assert grid.get((1, 1), "u") == 1.0 - 2.0 * q
    assert grid.get((2, 1), "u") == q
    assert diag.total_mass == 1.0 * h * h
    assert diag.step == 1 and diag.time == dt
    assert diag.min_u == q and diag.max_u == 1.0 - 2.0 * q


def test_cross_chunk_neighbors_match_in_chunk_arithmetic(cuda):
    from paper_2304_11165_b200 import porediff as pd
    h, dt = 0.5, 1.0 / 64
    grid = row_grid(12, h)
    grid.set((7, 1), "u", 1.0)
    pd.ftcs_step(grid, basic_config(dt))
    q = dt / (h * h)
    assert grid.get((6, 1), "u") == q
    assert grid.get((7, 1), "u") == 1.0 - 2.0 * q
    assert grid.get((8, 1), "u") == q
    assert grid.get((9, 1), "u") == 0.0


def test_three_dimensional_pulse_splits_six_ways(cuda):
    from paper_2304_11165_b200 import porediff as pd
    h, dt = 0.5, 1.0 / 64
    geom = pd.GridGeometry.make((8, 8, 8), (h, h, h))
    grid = pd.SparseBlockGrid(geom, pd.solver_channels())
    c = (4, 4, 4)
    nbrs = [(3, 4, 4), (5, 4, 4), (4, 3, 4), (4, 5, 4), (4, 4, 3), (4, 4, 5)]
    for idx in [c] + nbrs:
        grid.insert(idx)
        grid.set(idx, "phi", 1.0)
        grid.set(idx, "D", 1.0)
    grid.set(c, "u", 1.0)
    diag = pd.ftcs_step(grid, basic_config(dt))
    q = dt / (h * h)
    assert grid.get(c, "u") == 1.0 - 6.0 * q
    for idx in nbrs:
        assert grid.get(idx, "u") == q
    assert diag.total_mass == h * h * h


def test_uniform_field_is_an_exact_fixed_point(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(24)
    grid.channel_data("u", writable=True)[grid.active_bool()] = 5.0
    cfg = basic_config(0.3 * pd.stability_dt(grid.geom, pd.max_diffusivity(grid)), 10)
    res = pd.run_simulation(grid, cfg)
    assert np.all(grid.channel_data("u")[grid.active_bool()] == 5.0)
    for d in res.diagnostics:
        assert d.min_u == 5.0 and d.max_u == 5.0
        assert d.total_mass == res.diagnostics[0].total_mass


def test_solid_phase_neighbor_blocks_flux_exactly(cuda):
    from paper_2304_11165_b200 import porediff as pd
    h = 0.5
    geom = pd.GridGeometry.make((4, 3), (h, h))
    grid = pd.SparseBlockGrid(geom, pd.solver_channels())
    grid.insert((1, 1), [1.0, 1.0, 1.0, 0.0])
    grid.insert((2, 1), [0.0, 0.25, 7.0, 0.0])
    diag = pd.ftcs_step(grid, basic_config(1.0 / 64))
    assert grid.get((1, 1), "u") == 1.0
    assert grid.get((2, 1), "u") == 0.25
    assert diag.total_mass == (1.0 + 0.25) * h * h


def test_dirichlet_face_acts_as_fixed_halo(cuda):
    from paper_2304_11165_b200 import porediff as pd
    h, dt = 0.5, 1.0 / 64
    grid = row_grid(12, h)
    cfg = basic_config(dt)
    cfg.outer_bc[0] = pd.FaceBc.dirichlet(1.0)
    pd.ftcs_step(grid, cfg)
    q = dt / (h * h)
    assert grid.get((0, 1), "u") == q
    for x in range(1, 12):
        assert grid.get((x, 1), "u") == 0.0
    grid2 = row_grid(12, h)
    cfg2 = basic_config(dt, 400)
    cfg2.outer_bc[0] = pd.FaceBc.dirichlet(1.0)
    cfg2.record_every = 25
    prev = [0.0] * 12

    def obs(g, d):
        for x in range(12):
            u = g.get((x, 1), "u")
            assert u >= prev[x] - 1e-13
            prev[x] = u

    pd.run_simulation(grid2, cfg2, [obs])
    assert prev[11] > 0.0 and prev[11] < prev[0]


def test_volumetric_source_uses_channel_and_time_factor(cuda):
    from paper_2304_11165_b200 import porediff as pd
    h, dt = 0.5, 1.0 / 32
    grid = row_grid(3, h, pd.solver_channels() + ["f"])
    for x in range(3):
        grid.set((x, 1), "D", 0.0)
        grid.set((x, 1), "f", 0.5 + x)
    cfg = basic_config(dt, 2)
    cfg.reaction = pd.ReactionSpec.volumetric("f", lambda t: math.exp(-t))
    pd.run_simulation(grid, cfg)
    for x in range(3):
        f = 0.5 + x
        expect = dt * f * 1.0 + dt * f * math.exp(-dt)
        assert math.isclose(grid.get((x, 1), "u"), expect, rel_tol=4 * 2.2e-16)


def test_sparse_dense_bit_identical_after_two_hundred_steps(cuda):
    """solver_test.cpp:339-400"""
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import ball_sdf_field
    n = 32
    geom = pd.GridGeometry.cell_centered_box(n, -1.0, 1.0, 2)
    sdf = ball_sdf_field(geom, (0.15, -0.1), 0.7)
    sparse = pd.build_sparse_grid(sdf, geom, pd.PhaseBand(0.0, INF), pd.solver_channels())
    pd.populate_diffusion_channel(sparse, pd.DiffusionProfile(0.05, 1.0, 0.0, 16.0))
    su = sparse.channel_data("u", writable=True)
    idx = sparse.node_indices()
    act = sparse.active_bool()
    for j, off in zip(*np.nonzero(act)):
        su[j, off] = solver_test_hash(int(idx[j, off, 0]), int(idx[j, off, 1]), 1, 0.0, 1.0)
    dense = pd.build_sparse_grid(np.full(n * n, 1.0), geom, pd.PhaseBand(-INF, INF), pd.solver_channels())
    dphi = dense.channel_data("phi", writable=True)
    didx = dense.node_indices()
    flat = didx[..., 0] + n * didx[..., 1]
    inb = (didx[..., 0] < n) & (didx[..., 1] < n)
    dphi[inb] = sdf[flat[inb]]
    du = dense.channel_data("u", writable=True)
    dd = dense.channel_data("D", writable=True)
    du[inb] = 123.0
    dd[inb] = 0.3
    sparse_vals = {}
    sidx = sparse.node_indices()
    for j, off in zip(*np.nonzero(act)):
        sparse_vals[(int(sidx[j, off, 0]), int(sidx[j, off, 1]))] = (su[j, off], sparse.channel_data("D")[j, off])
    for j, off in zip(*np.nonzero(dense.active_bool())):
        key = (int(didx[j, off, 0]), int(didx[j, off, 1]))
        if key in sparse_vals:
            du[j, off], dd[j, off] = sparse_vals[key]
    assert dense.active_node_count() == n * n
    cfg = basic_config(0.45 * pd.stability_dt(geom, pd.max_diffusivity(sparse)), 200)
    cfg.boundary_epsilon = np.finfo(np.float64).eps
    pd.run_simulation(sparse, cfg)
    pd.run_simulation(dense, cfg)
    compared = 0
    for key in sparse_vals:
        assert bits_equal(sparse.get(key, "u"), dense.get(key, "u")), key
        compared += 1
    assert compared > 300
    for j, off in zip(*np.nonzero(dense.active_bool())):
        key = (int(didx[j, off, 0]), int(didx[j, off, 1]))
        if key not in sparse_vals:
            assert dense.channel_data("u")[j, off] == 123.0


def test_mirror_symmetric_problem_stays_bitwise_symmetric(cuda):
    """solver_test.cpp:406-425"""
    from paper_2304_11165_b200 import porediff as pd
    n = 32
    grid = disk_grid(n)
    u = grid.channel_data("u", writable=True)
    idx = grid.node_indices()
    for j, off in zip(*np.nonzero(grid.active_bool())):
        x = grid.geom.position((int(idx[j, off, 0]), int(idx[j, off, 1])))
        u[j, off] = math.cos(x[1]) + x[0] * x[0]
    cfg = basic_config(0.45 * pd.stability_dt(grid.geom, pd.max_diffusivity(grid)), 100)
    pd.run_simulation(grid, cfg)
    for j, off in zip(*np.nonzero(grid.active_bool())):
        i0, i1 = int(idx[j, off, 0]), int(idx[j, off, 1])
        assert bits_equal(grid.get((i0, i1), "u"), grid.get((n - 1 - i0, i1), "u"))


def test_records_baseline_every_kth_and_final_step(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(16)
    cfg = basic_config(0.3 * pd.stability_dt(grid.geom, pd.max_diffusivity(grid)), 10)
    cfg.record_every = 4
    observed = []
    res = pd.run_simulation(grid, cfg, [lambda g, d: observed.append(d.step)])
    assert [d.step for d in res.diagnostics] == [0, 4, 8, 10]
    assert observed == [0, 4, 8, 10]
    assert res.diagnostics[0].time == 0.0
    assert math.isclose(res.diagnostics[-1].time, 10 * cfg.dt, rel_tol=1e-15)


def test_stability_gate_rejects_and_reports_the_bound(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(16)
    bound = pd.stability_dt(grid.geom, pd.max_diffusivity(grid))
    cfg = basic_config(10.0 * bound, 5)
    with pytest.raises(pd.StabilityError) as ei:
        pd.run_simulation(grid, cfg)
    assert pd.format_scalar(bound) in str(ei.value)
    cfg.dt = bound
    with pytest.raises(pd.StabilityError):
        pd.run_simulation(grid, cfg)
    cfg.dt = 1.01 * bound
    cfg.enforce_stability = False
    cfg.n_steps = 1
    pd.run_simulation(grid, cfg)


def test_non_finite_values_abort_with_step_and_node(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(16)
    grid.set((8, 8), "u", INF)
    cfg = basic_config(0.3 * pd.stability_dt(grid.geom, pd.max_diffusivity(grid)), 5)
    with pytest.raises(pd.NumericError) as ei:
        pd.run_simulation(grid, cfg)
    assert "step 1" in str(ei.value) and "node (" in str(ei.value)


def test_validates_configuration_and_channels(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(16)
    for cfg in [basic_config(0.0), basic_config(-1.0)]:
        with pytest.raises(pd.InputError):
            pd.run_simulation(grid, cfg)
    bad = [dict(n_steps=0), dict(record_every=0), dict(phase_band=pd.PhaseBand(2.0, 1.0)),
           dict(boundary_epsilon=-1.0), dict(reaction=pd.ReactionSpec.surface_sink(-0.1)),
           dict(reaction=pd.ReactionSpec.surface_sink(0.1, 0.0))]
    for kw in bad:
        cfg = basic_config(1e-6)
        for k, v in kw.items():
            setattr(cfg, k, v)
        with pytest.raises(pd.InputError):
            pd.run_simulation(grid, cfg)
    cfg = basic_config(1e-6)
    cfg.reaction = pd.ReactionSpec.volumetric("missing")
    with pytest.raises(pd.PropertyError):
        pd.run_simulation(grid, cfg)
    geom = pd.GridGeometry.make((8, 8), (0.1, 0.1))
    bare = pd.SparseBlockGrid(geom, ["phi", "u", "D"])
    bare.insert((4, 4), [1.0, 0.0, 1.0])
    with pytest.raises(pd.InputError) as ei:
        pd.run_simulation(bare, basic_config(1e-6))
    assert "u_next" in str(ei.value)


def test_mass_matches_standalone_total_mass(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(20)
    direct = pd.total_mass(grid)
    cfg = basic_config(0.3 * pd.stability_dt(grid.geom, pd.max_diffusivity(grid)), 3)
    res = pd.run_simulation(grid, cfg)
    assert bits_equal(res.diagnostics[0].total_mass, direct)
    assert bits_equal(res.diagnostics[-1].total_mass, pd.total_mass(grid))
    geom = pd.GridGeometry.make((4, 4, 4), (0.5, 0.5, 0.5))
    tiny = pd.SparseBlockGrid(geom, pd.solver_channels())
    tiny.insert((1, 2, 3), [1.0, 1.0, 1.0, 0.0])
    assert pd.total_mass(tiny) == 0.125
    tiny.set((1, 2, 3), "u", 0.0)
    assert pd.total_mass(tiny) == 0.0


def test_conservation_ten_thousand_steps(cuda):
    """solver_test.cpp:292-313 (drift <= 1e-12 per step, <= 1e-7 total)."""
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(32)
    cfg = basic_config(0.4 * pd.stability_dt(grid.geom, pd.max_diffusivity(grid)), 10000)
    cfg.record_every = 1
    res = pd.run_simulation(grid, cfg)
    m = np.array([d.total_mass for d in res.diagnostics])
    assert len(m) == 10001
    assert np.max(np.abs(np.diff(m))) / m[0] <= 1e-12
    assert abs(m[-1] - m[0]) / m[0] <= 1e-7


def test_surface_sink_drains_mass_monotonically(cuda):
    from paper_2304_11165_b200 import porediff as pd
    grid = disk_grid(24)
    grid.channel_data("u", writable=True)[grid.active_bool()] = 1.0
    bound = pd.stability_dt(grid.geom, pd.max_diffusivity(grid))
    cfg = basic_config(0.5 * bound, 400)
    cfg.reaction = pd.ReactionSpec.surface_sink(0.2 / cfg.dt * 0.01, 2.0)
    cfg.record_every = 20
    res = pd.run_simulation(grid, cfg)
    d = res.diagnostics
    for i in range(1, len(d)):
        assert d[i].total_mass <= d[i - 1].total_mass * (1.0 + 1e-14)
    assert d[-1].total_mass < d[0].total_mass * 0.999
    assert all(x.min_u >= 0.0 for x in d)
