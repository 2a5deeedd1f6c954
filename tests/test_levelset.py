"""Level-set geometry stage (north_star subsystem 2):
mask -> indicator -> thin-feature opening -> Sussman redistancing -> band
activation into the sparse block grid, on the device, compared bit for bit
with the unmodified reference (oracle/_ref: levelset.hpp / geometry.hpp
compiled in place) on the same inputs.

CPU tests pin the oracle to the reference's own frozen regression values
(levelset_test.cpp:157-177) and check the host helpers; GPU tests are the
parity tests proper.
"""
import math

import numpy as np
import pytest

from paper_2304_11165_b200 import porediff as pd
from paper_2304_11165_b200.synthetic import ball_sdf_field


def indicator(sdf):
    # synthetic::indicator_from (synthetic.hpp:102-108): f(x) > 0 ? 1 : -1
    return np.where(np.asarray(sdf) > 0.0, 1.0, -1.0)


DEFAULT = (1000, 1e-3, 0.5, 4.0, 6.0, 1)


def unit_ball_norms(phi, geom):
    from paper_2304_11165_b200.levelset import band_error_norms

    def exact(x):
        return 1.0 - math.sqrt(sum(v * v for v in x))
    return band_error_norms(phi, geom, exact, 4.0)


def test_oracle_pinned_to_reference_frozen_ball_norms(ref):
    # levelset_test.cpp:157-177: n=16 Linf 9.412872e-02 L2 5.782716e-02 (+-15%),
    # 100..280 sweeps, converged
    geom = pd.GridGeometry.cell_centered_box(16, -1.28, 1.28, 3)
    phi0 = indicator(ball_sdf_field(geom, (0.0, 0.0, 0.0), 1.0))
    code, msg, phi, (it, res, conv) = ref.field_redistance(geom.size, geom.spacing, phi0, DEFAULT)
    assert code == 0, msg
    assert conv and 100 <= it <= 280
    n = unit_ball_norms(phi, geom)
    assert n.linf == pytest.approx(9.412872e-02, rel=0.15)
    assert n.l2 == pytest.approx(5.782716e-02, rel=0.15)


def test_host_helpers():
    from paper_2304_11165_b200.levelset import godunov_axis_sq, smoothed_sign
    assert smoothed_sign(0.0, 3.0, 0.1) == 0.0
    assert smoothed_sign(0.5, 1.0, 0.5) == 0.5 / math.sqrt(0.25 + 0.25)
    # levelset_test.cpp:58-78 kink cases: upwind picks the incoming side
    assert godunov_axis_sq(1.0, -2.0, 1) == 4.0
    assert godunov_axis_sq(-1.0, 2.0, 1) == 0.0
    assert godunov_axis_sq(-1.0, 2.0, -1) == 4.0


def _compare(ref, geom, values, opts, dtype=np.float64):
    from paper_2304_11165_b200 import levelset as ls
    f = ls.DeviceField.from_host(geom, values, dtype)
    d = ls.sussman_redistance(f, ls.LevelSetOptions(*opts[:5], bool(opts[5])))
    got = f.download()
    code, msg, want, (it, res, conv) = ref.field_redistance(geom.size, geom.spacing,
                                                            np.asarray(values, dtype), opts)
    assert code == 0, msg
    assert (d.iterations, d.final_residual, d.converged) == (it, res, conv)
    bits = np.uint64 if dtype == np.float64 else np.uint32
    bad = np.nonzero(got.view(bits) != want.view(bits))[0]
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])
    return f, d


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 33])
def test_redistance_ball_indicator_bitwise(n, ref, cuda):
    geom = pd.GridGeometry.cell_centered_box(n, -1.28, 1.28, 3)
    _compare(ref, geom, indicator(ball_sdf_field(geom, (0.05, -0.1, 0.0), 1.0)), DEFAULT)


@pytest.mark.gpu
def test_redistance_raw_sdf_no_rescale_and_iteration_cap(ref, cuda):
    geom = pd.GridGeometry.make((20, 24, 28), (0.05, 0.04, 0.035), (-0.5, -0.48, -0.5))
    sdf = ball_sdf_field(geom, (0.0, 0.0, 0.0), 0.3) * 3.0
    _compare(ref, geom, sdf, (1000, 1e-4, 0.3, 4.0, 8.0, 0))
    _, d = _compare(ref, geom, sdf, (3, 1e-3, 0.5, 4.0, 6.0, 1))
    assert d.iterations == 3 and not d.converged


@pytest.mark.gpu
def test_redistance_2d_and_fp32(ref, cuda):
    g2 = pd.GridGeometry.cell_centered_box(48, -1.28, 1.28, 2)
    _compare(ref, g2, indicator(ball_sdf_field(g2, (0.1, 0.0), 1.0)), DEFAULT)
    g3 = pd.GridGeometry.cell_centered_box(24, -1.28, 1.28, 3)
    _compare(ref, g3, indicator(ball_sdf_field(g3, (0.0, 0.0, 0.0), 1.0)), DEFAULT, np.float32)


@pytest.mark.gpu
def test_redistance_validation(cuda):
    from paper_2304_11165_b200 import levelset as ls
    geom = pd.GridGeometry.cell_centered_box(8, 0.0, 1.0, 3)
    f = ls.DeviceField.from_host(geom, np.ones(geom.node_count()))
    with pytest.raises(pd.InputError, match="no interface found"):
        ls.sussman_redistance(f)
    v = np.ones(geom.node_count())
    v[3] = np.nan
    f.upload(v)
    with pytest.raises(pd.InputError, match="non-finite"):
        ls.sussman_redistance(f)
    with pytest.raises(pd.InputError, match=r"pseudo_time_step must lie in \(0, 1\]"):
        ls.sussman_redistance(f, ls.LevelSetOptions(pseudo_time_step=1.5))


@pytest.mark.gpu
def test_image_to_grid_pipeline_bitwise(ref, cuda):
    """mask -> indicator -> opening (w=3) -> redistance -> build_sparse_grid:
    every stage equal to the reference on a porous sphere-pack image."""
    from paper_2304_11165_b200 import levelset as ls
    from paper_2304_11165_b200.synthetic import SpherePacking
    n = 40
    geom0 = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = SpherePacking.random((0, 0, 0), (1, 1, 1), 25, 0.06, 0.14, 99)
    bits = (pack.fluid_sdf_field(geom0) > 0.0).astype(np.uint8)
    mask = ls.VoxelMask((n, n, n), (1.0 / n,) * 3, bits)
    ind = ls.mask_to_indicator(mask)
    geom = ind.geom  # node 0 at the origin with the voxel spacing
    assert np.array_equal(ind.download(), np.where(bits > 0, 1.0, -1.0))
    opened = ls.filter_thin_features(ind, 3)
    code, msg, want = ref.field_filter_thin(geom.size, geom.spacing, np.where(bits > 0, 1.0, -1.0), 3)
    assert code == 0, msg
    got = opened.download()
    assert np.array_equal(got, want) and not np.array_equal(got, ind.download())
    f, _ = _compare(ref, geom, got, DEFAULT)
    phi = f.download()
    grid = ls.build_sparse_grid(f, pd.PhaseBand(), pd.solver_channels())
    rg = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, phi)
    keys, masks = rg.layout()
    assert np.array_equal(grid.keys(), keys) and np.array_equal(grid.masks(), masks)
    assert np.array_equal(grid.channel_data("phi").view(np.uint64), rg.prop("phi").view(np.uint64))
    # and the pipeline's grid steps exactly like the reference's
    grid_b = ls.build_sparse_grid(f, pd.PhaseBand(-0.05, 0.5), pd.solver_channels())
    rg_b = ref.grid_from_sdf(geom.size, geom.spacing, geom.origin, phi, -0.05, 0.5)
    kb, mb = rg_b.layout()
    assert np.array_equal(grid_b.keys(), kb) and np.array_equal(grid_b.masks(), mb)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_random_masks_through_the_level_set_stage(seed, ref, cuda):
    """Seeded random images (random-phase GRF-like masks, anisotropic voxels,
    odd box sizes, 2-D and 3-D, FP64 / FP32): opening with a random window
    and redistancing with random options, each bitwise against the
    reference (the z-march sweep for 3-D, the per-node sweep for 2-D)."""
    from paper_2304_11165_b200 import levelset as ls
    r = np.random.default_rng(500 + seed)
    dims = 3 if seed % 4 else 2
    size = tuple(int(v) for v in r.integers(9, 40, dims))
    if dims == 2:
        size = tuple(int(v) * 2 for v in size)
    vox = tuple(float(v) for v in r.uniform(0.5, 1.5, dims) / 40)
    k = r.normal(size=(6, dims)) * 6.0
    ph = r.uniform(0, 2 * np.pi, 6)
    grids = np.meshgrid(*[np.arange(s) for s in size], indexing="ij")
    field = sum(np.cos(sum(k[m, a] * grids[a] / size[a] for a in range(dims)) + ph[m]) for m in range(6))
    bits = (field > np.quantile(field, r.uniform(0.3, 0.7))).astype(np.uint8)
    bits = np.ascontiguousarray(bits.transpose(tuple(range(dims))[::-1])).reshape(-1)  # axis 0 fastest
    dtype = np.float32 if seed % 3 == 2 else np.float64
    mask = ls.VoxelMask(size, vox, bits)
    ind = ls.mask_to_indicator(mask, dtype)
    geom = ind.geom
    w = int(r.integers(1, 4))
    opened = ls.filter_thin_features(ind, w)
    code, msg, want = ref.field_filter_thin(geom.size, geom.spacing, np.where(bits > 0, 1.0, -1.0).astype(dtype), w)
    assert code == 0, msg
    got = opened.download()
    assert np.array_equal(got, want)
    if np.all(got > 0) or np.all(got < 0):
        return  # the opening removed the interface: nothing to redistance
    opts = (int(r.integers(5, 200)), float(r.choice([1e-3, 1e-5])), float(r.uniform(0.2, 0.8)),
            4.0, float(r.uniform(3.0, 8.0)), int(r.integers(0, 2)))
    _compare(ref, geom, got, opts, dtype)
