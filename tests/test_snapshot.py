"""SBGR / SBGD snapshots (reference snapshot.hpp):
files written from the device are byte-identical to the reference writer's
on the same state (including the u/u_next swap parity and inactive slots),
reference-written files read back into device grids bit for bit, and I/O
errors carry the reference's messages."""
from pathlib import Path

import numpy as np
import pytest

from paper_2304_11165_b200 import porediff as pd

pytestmark = pytest.mark.gpu


def _pack_case(ref, n=24, steps=7):
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import synthetic as sy
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = sy.SpherePacking.random((0, 0, 0), (1, 1, 1), 12, 0.1, 0.2, 3)
    sdf = pack.fluid_sdf_field(geom)
    grid = pd.build_sparse_grid(sdf, geom, pd.PhaseBand(), pd.solver_channels())
    pd.populate_diffusion_channel(grid, pd.DiffusionProfile(0.05, 1.0, 0.0, 4.0 * n))
    u = grid.channel_data("u", writable=True)
    act = grid.active_bool()
    u[act] = np.array([pd.hash_unit_value(2, int(f)) for f in grid.flat_indices()[act]])
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, pd.max_diffusivity(grid)), n_steps=steps,
                              record_every=steps)
    pd.run_simulation(grid, cfg)  # odd step count: u / u_next columns swapped
    rg = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf)
    rg.populate_diffusion(0.05, 1.0, 0.0, 4.0 * n)
    rg.fill_hash("u", 2)
    code, msg, _ = rg.run(make_config(cfg.dt, steps, record_every=steps))
    assert code == 0, msg
    return geom, grid, rg


def test_sparse_snapshot_bytes_identical_and_round_trip(ref, cuda, tmp_path):
    from paper_2304_11165_b200 import snapshot as sn
    geom, grid, rg = _pack_case(ref)
    ours, theirs = tmp_path / "ours.sbgr", tmp_path / "ref.sbgr"
    sn.write_sparse_snapshot(grid, ours)
    code, msg = rg.write_snapshot(theirs)
    assert code == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()
    info = sn.peek_snapshot(theirs)
    assert (info.magic, info.version, info.scalar_bits, info.dims) == ("SBGR", 1, 64, 3)
    assert info.properties == pd.solver_channels() and info.size == [24, 24, 24]
    back = sn.read_sparse_snapshot(theirs)
    assert np.array_equal(back.keys(), grid.keys()) and np.array_equal(back.masks(), grid.masks())
    for p in pd.solver_channels():
        assert np.array_equal(back.channel_data(p).view(np.uint64), grid.channel_data(p).view(np.uint64)), p
    # resume: one more step from the snapshot equals one more step of the live grid
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, pd.max_diffusivity(grid)), n_steps=1)
    pd.run_simulation(grid, cfg)
    pd.run_simulation(back, cfg)
    assert np.array_equal(back.channel_data("u").view(np.uint64), grid.channel_data("u").view(np.uint64))


def test_dense_snapshot_bytes_identical(ref, cuda, tmp_path):
    from paper_2304_11165_b200 import levelset as ls
    from paper_2304_11165_b200 import snapshot as sn
    from paper_2304_11165_b200.synthetic import ball_sdf_field
    geom = pd.GridGeometry.make((20, 18, 16), (0.05, 0.05, 0.06), (-0.5, -0.4, -0.45))
    f = ls.DeviceField.from_host(geom, ball_sdf_field(geom, (0.0, 0.0, 0.0), 0.3))
    ls.sussman_redistance(f)
    ours, theirs = tmp_path / "ours.sbgd", tmp_path / "ref.sbgd"
    sn.write_dense_snapshot(f, ours)
    code, msg = ref.write_dense_snapshot(geom.size, geom.spacing, geom.origin, f.download(), theirs)
    assert code == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()
    back = sn.read_dense_snapshot(theirs)
    assert np.array_equal(back.download().view(np.uint64), f.download().view(np.uint64))
    assert back.geom.origin == geom.origin and back.geom.spacing == geom.spacing


def test_snapshot_errors(ref, cuda, tmp_path):
    from paper_2304_11165_b200 import snapshot as sn
    geom, grid, rg = _pack_case(ref, n=16, steps=2)
    good = tmp_path / "g.sbgr"
    sn.write_sparse_snapshot(grid, good)
    data = good.read_bytes()
    (tmp_path / "trunc.sbgr").write_bytes(data[:-9])
    with pytest.raises(pd.IoError, match="is truncated"):
        sn.read_sparse_snapshot(tmp_path / "trunc.sbgr")
    (tmp_path / "trail.sbgr").write_bytes(data + b"x")
    with pytest.raises(pd.IoError, match="trailing bytes"):
        sn.read_sparse_snapshot(tmp_path / "trail.sbgr")
    with pytest.raises(pd.IoError, match="stores 64-bit scalars, expected 32"):
        sn.read_sparse_snapshot(good, dtype=np.float32)
    with pytest.raises(pd.IoError, match="magic mismatch"):
        sn.read_dense_snapshot(good)
    with pytest.raises(pd.IoError, match="cannot open"):
        sn.read_sparse_snapshot(tmp_path / "missing.sbgr")
    # the reference reads our file too
    code, msg, rback = ref.read_sparse_snapshot(good)
    assert code == 0, msg
    assert np.array_equal(rback.prop("u").view(np.uint64), grid.channel_data("u").view(np.uint64))
