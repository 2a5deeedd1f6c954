"""Host-side pieces of the drop-in (no GPU): geometry builders, the
sphere-pack generator, hashing, pairwise sum and the stability bound match
the reference bit for bit."""
import math

import numpy as np
import pytest

from cases import CASES, host_case, sha


def test_hash_unit_value_matches_reference(ref):
    from paper_2304_11165_b200.porediff import hash_unit_value
    for seed, key in [(0, 0), (1, 12345), (5, 2**40 + 7), (2**63, 99)]:
        assert hash_unit_value(seed, key) == ref.hash_unit_value(seed, key)


def test_pairwise_sum_matches_reference(ref):
    from paper_2304_11165_b200.porediff import pairwise_sum
    rng = np.random.default_rng(3)
    for n in [0, 1, 2, 3, 7, 64, 1000, 1025, 4097]:
        v = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 5, n)
        a = pairwise_sum(v)
        b = ref.pairwise_sum(v)
        assert np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64), n


def test_sphere_packing_matches_reference(ref):
    from paper_2304_11165_b200.synthetic import SpherePacking
    for args in [(40, 0.1, 0.15, 2024), (30, 0.08, 0.16, 777), (5, 0.2, 0.2, 1)]:
        p = SpherePacking.random((0, 0, 0), (1, 1, 1), *args)
        c, r = ref.sphere_packing((0, 0, 0), (1, 1, 1), *args)
        assert np.array_equal(np.array(p.centers), c)
        assert np.array_equal(np.array(p.radii), r)


def test_sphere_pack_field_matches_reference(ref):
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import SpherePacking
    geom = pd.GridGeometry.cell_centered_box(19, 0.0, 1.0, 3)
    p = SpherePacking.random((0, 0, 0), (1, 1, 1), 25, 0.05, 0.2, 42)
    c, r = p.arrays()
    a = p.fluid_sdf_field(geom)
    b = ref.field_sphere_pack(geom.size, geom.spacing, geom.origin, c, r)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("name", [c for c in CASES if c != "c1_ball64"])
def test_host_builders_reproduce_reference_inputs(name, golden):
    g = host_case(name)
    gold = golden[name]
    assert g.chunk_count() == gold["chunks"]
    assert g.active_node_count() == gold["active"]
    assert sha(g.keys()) == gold["sha_keys"]
    assert sha(g.masks()) == gold["sha_masks"]
    for c in CASES[name]["channels"]:
        assert sha(g.channel_data(c)) == gold["sha_inputs"][c], c


def test_stability_dt_closed_forms():
    """solver_test.cpp:83-98."""
    from paper_2304_11165_b200 import porediff as pd
    g2 = pd.GridGeometry.make((4, 4), (0.1, 0.1))
    assert math.isclose(pd.stability_dt(g2, 1.0), 0.0025, rel_tol=4e-16)
    assert 0.1 * 0.1 / 8.0 < pd.stability_dt(g2, 1.0)
    h = 0.37
    g3 = pd.GridGeometry.make((4, 4, 4), (h, h, h))
    assert math.isclose(pd.stability_dt(g3, 2.0), h * h / (6.0 * 2.0), rel_tol=4e-16)
    with pytest.raises(pd.InputError):
        pd.stability_dt(g2, 0.0)


def test_grid_ordering_and_offsets():
    """grid_test.cpp:23-32,47-53,163-190: x-fastest flat index, chunk boundary
    at 8, sorted insertion-independent traversal, key/offset round trip."""
    from paper_2304_11165_b200 import porediff as pd
    geom = pd.GridGeometry.make((20, 17, 9), (1.0, 1.0, 1.0))
    assert geom.flat_index((1, 2, 3)) == 1 + 20 * (2 + 17 * 3)
    rng = np.random.default_rng(0)
    pts = [tuple(int(v) for v in (rng.integers(0, 20), rng.integers(0, 17), rng.integers(0, 9)))
           for _ in range(60)]
    a = pd.SparseBlockGrid(geom, ["u"])
    b = pd.SparseBlockGrid(geom, ["u"])
    for p in pts:
        a.insert(p)
    for p in reversed(pts):
        b.insert(p)
    assert np.array_equal(a.keys(), b.keys())
    assert np.array_equal(a.masks(), b.masks())
    lin = a._linear(a.keys())
    assert np.all(np.diff(lin) > 0)
    for p in pts:
        assert a.is_active(p)
        off = pd.SparseBlockGrid.offset_of(p)
        assert off == (p[0] & 7) | ((p[1] & 7) << 3) | ((p[2] & 7) << 6)
    c = pd.SparseBlockGrid(geom, ["u"])
    c.insert((7, 0, 0))
    c.insert((8, 0, 0))
    assert c.chunk_count() == 2
    with pytest.raises(pd.BoundsError):
        c.insert((20, 0, 0))
