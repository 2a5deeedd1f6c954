"""VTK export (reference vtk.hpp, scalar_text.hpp).

CPU: the exact "%.17g" / "%.9g" formatter the device runs (pd_format_scalar,
the same pd_format.cuh code compiled for the host) against Python's correctly
rounded printf on random bit patterns, ties and edge values; the reader on
reference-written files.
GPU: whole files written from the device are byte-identical to the reference
writer's (dense datasets of random bit patterns with NaN / inf / denormals,
FP64 and FP32, 2-D and 3-D; sparse grids after stepping, default and chosen
channels, custom blank; a multi-batch lattice), and errors match."""
import math
import random
import struct

import numpy as np
import pytest

from paper_2304_11165_b200 import porediff as pd


def _bits_f64(rng, n):
    return np.frombuffer(rng.bytes(8 * n), np.float64).copy()


def _bits_f32(rng, n):
    return np.frombuffer(rng.bytes(4 * n), np.float32).copy()


def _py17(v):
    return "nan" if math.isnan(v) else "%.17g" % v


def _py9(v):
    return "nan" if math.isnan(v) else "%.9g" % float(v)


def test_format_scalar_matches_printf_random_bits():
    from paper_2304_11165_b200.vtk import format_scalar
    rng = np.random.default_rng(11)
    for v in _bits_f64(rng, 40000):
        assert format_scalar(v) == _py17(float(v)), float(v).hex()
    for v in _bits_f32(rng, 20000):
        assert format_scalar(float(v), np.float32) == _py9(float(v)), float(v).hex()


def test_format_scalar_edges_and_ties():
    from paper_2304_11165_b200.vtk import format_scalar
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 1e-5, 1e-4, 9.9999999999999999e-5, 1e16, 1e17, 1e22, 1e23,
            123456789012345678.0, 1.7976931348623157e308, 2.2250738585072014e-308, 5e-324, -5e-324,
            2251799813685246.25, 2251799813685247.75, 0.5, 2.5, math.inf, -math.inf, math.nan, -math.nan]
    for e in range(-1075, 1024, 7):
        x = math.ldexp(1.0, e)
        vals += [x, math.nextafter(x, 0.0), math.nextafter(x, math.inf)]
    for p in range(-325, 309, 3):
        x = float(f"1e{p}")
        vals += [x, math.nextafter(x, 0.0), math.nextafter(x, math.inf)]
    r = random.Random(5)
    for _ in range(3000):  # exact halfway cases: 18 significant digits ending in 5
        vals.append(math.ldexp(float(r.getrandbits(53) | 1), -r.randint(1, 6)))
    for v in vals:
        assert format_scalar(v) == _py17(v), float(v).hex()
        f = struct.unpack("f", struct.pack("f", v))[0] if abs(v) < 3.4e38 or math.isinf(v) or math.isnan(v) else None
        if f is not None:
            assert format_scalar(f, np.float32) == _py9(f), float(f).hex()


def test_reader_parses_reference_file(ref, tmp_path):
    from paper_2304_11165_b200 import vtk
    rng = np.random.default_rng(3)
    u = _bits_f64(rng, 12)
    u[~np.isfinite(u)] = 1.0
    u[3] = np.nan
    p = tmp_path / "r.vtk"
    code, msg = ref.write_vtk(p, (3, 2, 2), (0.1, 0.2, 0.3), (-0.5, 0.25, 1.0), [("u", u)],
                              mask=np.array([1] * 3 + [0] + [1] * 8, np.int32))
    assert code == 0, msg
    f = vtk.read_vtk(p)
    assert f.dimensions == [3, 2, 2] and f.origin == [-0.5, 0.25, 1.0] and f.spacing == [0.1, 0.2, 0.3]
    back = f.array("u").as_(np.float64)
    ok = ~np.isnan(u)
    assert np.array_equal(back[ok].view(np.uint64), u[ok].view(np.uint64)) and np.isnan(back[3])
    assert list(f.array("mask").as_(np.int32)) == [1, 1, 1, 0] + [1] * 8
    with pytest.raises(pd.InputError, match="no array named 'missing'"):
        f.array("missing")
    bad = tmp_path / "bad.vtk"
    bad.write_text("# vtk DataFile Version 3.0\nt\nBINARY\n")
    with pytest.raises(pd.InputError, match="only ASCII format is supported"):
        vtk.read_vtk(bad)


# ---- device writers vs the reference writer (byte-identical) -------------

@pytest.mark.gpu
@pytest.mark.parametrize("dims,dtype", [(3, np.float64), (2, np.float64), (3, np.float32), (2, np.float32)])
def test_dense_dataset_bytes_identical(ref, cuda, tmp_path, dims, dtype):
    from paper_2304_11165_b200 import vtk
    size = (13, 7, 5)[:dims]
    geom = pd.GridGeometry.make(size, (0.1, 0.2, 0.3)[:dims], (-0.5, 0.25, 1.0)[:dims])
    n = geom.node_count()
    rng = np.random.default_rng(dims * 10 + np.dtype(dtype).itemsize)
    mk = _bits_f64 if dtype == np.float64 else _bits_f32
    u, d = mk(rng, n), mk(rng, n)
    u[:4] = [np.nan, np.inf, -np.inf, 0.0]
    mask = rng.integers(-3, 3, n).astype(np.int32)
    mask[0] = np.iinfo(np.int32).min
    ds = vtk.VtkDataset(geom, dtype=np.dtype(dtype))
    ds.add_scalar("u", u)
    ds.add_scalar("D", d)
    ds.mask = mask
    ours, theirs = tmp_path / "o.vtk", tmp_path / "r.vtk"
    vtk.write_vtk(ds, ours, title="custom title")
    code, msg = ref.write_vtk(theirs, geom.size, geom.spacing, geom.origin, [("u", u), ("D", d)], mask,
                              title="custom title")
    assert code == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()


def _stepped_pack(ref, n=24, steps=5, dtype=np.float64):
    from oracle.pyoracle import make_config
    from paper_2304_11165_b200 import synthetic as sy
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = sy.SpherePacking.random((0, 0, 0), (1, 1, 1), 10, 0.1, 0.2, 7)
    sdf = pack.fluid_sdf_field(geom)
    grid = pd.build_sparse_grid(sdf, geom, pd.PhaseBand(), pd.solver_channels())
    pd.populate_diffusion_channel(grid, pd.DiffusionProfile(0.05, 1.0, 0.0, 4.0 * n))
    u = grid.channel_data("u", writable=True)
    act = grid.active_bool()
    u[act] = np.array([pd.hash_unit_value(4, int(f)) for f in grid.flat_indices()[act]])
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, pd.max_diffusivity(grid)), n_steps=steps,
                              record_every=steps)
    cfg.reaction = pd.ReactionSpec.surface_sink(3.0, 1.0)
    pd.run_simulation(grid, cfg)
    rg = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf)
    rg.populate_diffusion(0.05, 1.0, 0.0, 4.0 * n)
    rg.fill_hash("u", 4)
    code, msg, _ = rg.run(make_config(cfg.dt, steps, reaction="surface_sink", rate=3.0, band_half_width=1.0,
                                      record_every=steps))
    assert code == 0, msg
    return geom, grid, rg


@pytest.mark.gpu
def test_sparse_grid_vtk_bytes_identical(ref, cuda, tmp_path):
    from paper_2304_11165_b200 import vtk
    geom, grid, rg = _stepped_pack(ref)
    ours, theirs = tmp_path / "o.vtk", tmp_path / "r.vtk"
    vtk.write_grid_vtk(grid, ours)  # every channel, NaN blanks (odd step count: columns swapped)
    code, msg = rg.write_vtk(theirs)
    assert code == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()
    vtk.write_grid_vtk(grid, ours, ["u", "phi"], blank=-7.0)
    code, msg = rg.write_vtk(theirs, ["u", "phi"], -7.0)
    assert code == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()
    # vtk_from_sparse (device densify) + write_vtk gives the same file
    ds = vtk.vtk_from_sparse(grid, ["u", "phi"], -7.0)
    vtk.write_vtk(ds, ours)
    assert ours.read_bytes() == theirs.read_bytes()
    f = vtk.read_vtk(ours)
    m = f.array("mask").as_(np.int32)
    assert m.sum() == grid.active_node_count()


@pytest.mark.gpu
def test_multi_batch_lattice_bytes_identical(ref, cuda, tmp_path):
    """More nodes than one device batch (4 Mi): the pipelined batches join
    seamlessly."""
    from paper_2304_11165_b200 import vtk
    geom = pd.GridGeometry.make((200, 160, 140), (1e-3, 1e-3, 1e-3), (0.0, 0.0, 0.0))
    rng = np.random.default_rng(9)
    u = rng.random(geom.node_count()) * np.exp(rng.normal(0, 30, geom.node_count()))
    ds = vtk.VtkDataset(geom)
    ds.add_scalar("u", u)
    ours, theirs = tmp_path / "o.vtk", tmp_path / "r.vtk"
    vtk.write_vtk(ds, ours)
    code, msg = ref.write_vtk(theirs, geom.size, geom.spacing, geom.origin, [("u", u)])
    assert code == 0, msg
    assert ours.stat().st_size == theirs.stat().st_size
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.gpu
def test_field_vtk_bytes_identical(ref, cuda, tmp_path):
    from paper_2304_11165_b200 import levelset as ls
    from paper_2304_11165_b200 import vtk
    from paper_2304_11165_b200.synthetic import ball_sdf_field
    geom = pd.GridGeometry.make((20, 18, 16), (0.05, 0.05, 0.06), (-0.5, -0.4, -0.45))
    f = ls.DeviceField.from_host(geom, ball_sdf_field(geom, (0.0, 0.0, 0.0), 0.3))
    ls.sussman_redistance(f)
    ours, theirs = tmp_path / "o.vtk", tmp_path / "r.vtk"
    vtk.write_field_vtk(f, ours, "phi")
    code, msg = ref.write_vtk(theirs, geom.size, geom.spacing, geom.origin, [("phi", f.download())])
    assert code == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.gpu
def test_vtk_errors_match_reference(ref, cuda, tmp_path):
    from paper_2304_11165_b200 import vtk
    geom = pd.GridGeometry.make((3, 3), (1.0, 1.0))
    ds = vtk.VtkDataset(geom)
    with pytest.raises(pd.InputError, match="no arrays to write"):
        vtk.write_vtk(ds, tmp_path / "x.vtk")
    ds.add_scalar("u", np.zeros(8))
    with pytest.raises(pd.InputError, match="holds 8 values, lattice has 9 nodes"):
        vtk.write_vtk(ds, tmp_path / "x.vtk")
    ds.scalars.clear()
    ds.add_scalar("bad name", np.zeros(9))
    with pytest.raises(pd.InputError, match="contains whitespace"):
        vtk.write_vtk(ds, tmp_path / "x.vtk")
    ds.scalars.clear()
    ds.add_scalar("u", np.zeros(9))
    ds.add_scalar("u", np.zeros(9))
    with pytest.raises(pd.InputError, match="duplicate VTK array name 'u'"):
        vtk.write_vtk(ds, tmp_path / "x.vtk")
    ds.scalars.pop()
    ds.mask = np.zeros(4, np.int32)
    with pytest.raises(pd.InputError, match="mask array size mismatch"):
        vtk.write_vtk(ds, tmp_path / "x.vtk")
    ds.mask = None
    with pytest.raises(pd.IoError, match="cannot open"):
        vtk.write_vtk(ds, tmp_path / "no_such_dir" / "x.vtk")
    geom3, grid, _ = _stepped_pack(ref, n=16, steps=1)
    with pytest.raises(pd.PropertyError):
        vtk.write_grid_vtk(grid, tmp_path / "x.vtk", ["nope"])
