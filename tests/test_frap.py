"""FRAP / effective diffusivity / tortuosity (reference
analysis.hpp:160-309).

CPU: the golden fits (tests/golden/frap.json, made by make_golden_frap.py from
the unmodified reference) are pinned to the survey's known answers, the
reference re-run reproduces them, and the host-side helpers follow the
reference's rules. GPU: run_frap on the device reproduces the reference's
recovery curves bit for bit, and fit_effective_D reproduces D_eff, tau_d and
the residual bit for bit (north_star: 1e-8 relative; we hold 0 ulp).
"""
import json
import math
from pathlib import Path

import pytest

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "frap.json").read_text())


def hx(s):
    return float.fromhex(s)


def test_golden_pinned_to_survey_kat():
    # 32^3, 40 spheres r in [0.1, 0.15], seed 2024
    g = GOLD["frap32"]
    assert hx(g["d_eff"]) == 0.83841401729453335
    assert hx(g["tau"]) == 1.1927281502602809
    # the second KAT: 64^3, same pack and schedule
    g = GOLD["frap64"]
    assert hx(g["d_eff"]) == 0.84242584501724482
    assert hx(g["tau"]) == 1.1870481015210657


def test_reference_reproduces_golden_frap16(ref):
    c = GOLD["frap16"]
    n = c["n"]
    h = 1.0 / n
    size, spacing, origin = (n, n, n), (h, h, h), (0.5 * h,) * 3
    centers, radii = ref.sphere_packing((0, 0, 0), (1, 1, 1), c["count"], c["r_min"], c["r_max"], c["seed"])
    g = ref.grid_from_sdf(size, spacing, origin, ref.field_sphere_pack(size, spacing, origin, centers, radii))
    d_eff, tau, res, ct, cr = g.frap_fit(c["bleach"], 1.0, c["t_final"], c["n_samples"], hx(c["dt"]),
                                         c["d_lo"], c["d_hi"], c["rel_tol"])
    assert (d_eff.hex(), tau.hex(), res.hex()) == (c["d_eff"], c["tau"], c["residual"])
    assert [float(x).hex() for x in cr] == c["curve_r"]


def test_host_helpers_follow_reference_rules():
    from paper_2304_11165_b200 import analysis as an
    from paper_2304_11165_b200 import porediff as pd
    geom = pd.GridGeometry.cell_centered_box(32, 0.0, 1.0, 3)
    box = an.central_bleach_box(geom, 0.25)
    assert (list(box.lo), list(box.hi)) == ([12] * 3, [20] * 3)
    # llround half away from zero: 0.5 * 5 = 2.5 -> 3
    b5 = an.central_bleach_box(pd.GridGeometry.cell_centered_box(5, 0.0, 1.0, 2), 0.5)
    assert (list(b5.lo), list(b5.hi)) == ([1, 1], [4, 4])
    with pytest.raises(pd.InputError, match=r"bleach box fraction must be in \(0, 1\]"):
        an.central_bleach_box(geom, 0.0)
    c = [an.FrapSample(0.0, 0.0), an.FrapSample(1.0, 0.5), an.FrapSample(3.0, 0.9)]
    assert an.interp_curve(c, -1.0) == 0.0 and an.interp_curve(c, 5.0) == 0.9
    assert an.interp_curve(c, 2.0) == 0.5 + 0.5 * (0.9 - 0.5)
    with pytest.raises(pd.InputError, match="empty recovery curve"):
        an.interp_curve([], 0.0)
    assert an.tortuosity_power_law(0.25, 0.5) == math.pow(0.25, -0.5)
    assert an.tortuosity_linear(0.4) == 0.4 + 1.65 * 0.6
    with pytest.raises(pd.InputError, match="power-law correlation"):
        an.tortuosity_power_law(0.0, 1.0)
    with pytest.raises(pd.InputError, match="search interval"):
        an.fit_effective_D(an.FrapExperiment(1.0, 1, 2, c), geom, box, 1.0, 0.5)
    with pytest.raises(pd.InputError, match="relative tolerance"):
        an.fit_effective_D(an.FrapExperiment(1.0, 1, 2, c), geom, box, 0.5, 1.0, an.FitOptions(rel_tol=1.0))


def _pack_grid(c):
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import SpherePacking
    geom = pd.GridGeometry.cell_centered_box(c["n"], 0.0, 1.0, 3)
    pack = SpherePacking.random((0, 0, 0), (1, 1, 1), c["count"], c["r_min"], c["r_max"], c["seed"])
    centers, radii = pack.arrays()
    dev = pd.DeviceGrid.sphere_pack(geom, centers, radii, n_props=4, prop_phi=0)
    return geom, pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["frap16", "frap32", "frap64"])
def test_frap_curve_and_fit_bitwise(name, cuda):
    from paper_2304_11165_b200 import analysis as an
    c = GOLD[name]
    geom, grid = _pack_grid(c)
    assert grid.active_node_count() == c["active"] and grid.chunk_count() == c["chunks"]
    box = an.central_bleach_box(geom, c["bleach"])
    dt = hx(c["dt"])
    exp = an.run_frap(grid, box, 1.0, an.FrapSchedule(c["t_final"], c["n_samples"], dt))
    assert [s.time.hex() for s in exp.curve] == c["curve_t"]
    assert [s.recovery.hex() for s in exp.curve] == c["curve_r"]
    fit = an.fit_effective_D(exp, geom, box, c["d_lo"], c["d_hi"], an.FitOptions(rel_tol=c["rel_tol"], dt=dt))
    assert (fit.d_eff.hex(), fit.tau_d.hex(), fit.fit_residual.hex()) == (c["d_eff"], c["tau"], c["residual"])
    assert fit.d_molecular == 1.0 and fit.tau_d * fit.d_eff == pytest.approx(1.0, rel=1e-15)


@pytest.mark.gpu
def test_run_frap_validation_and_observer(cuda):
    from paper_2304_11165_b200 import analysis as an
    from paper_2304_11165_b200 import porediff as pd
    c = GOLD["frap16"]
    geom, grid = _pack_grid(c)
    box = an.central_bleach_box(geom, c["bleach"])
    with pytest.raises(pd.InputError, match="molecular diffusivity"):
        an.run_frap(grid, box, 0.0, an.FrapSchedule(0.01))
    with pytest.raises(pd.InputError, match="t_final"):
        an.run_frap(grid, box, 1.0, an.FrapSchedule(0.0))
    with pytest.raises(pd.InputError, match="axis 1"):
        an.run_frap(grid, an.IndexBox([0, 3, 0], [4, 3, 4]), 1.0, an.FrapSchedule(0.01))
    with pytest.raises(pd.InputError, match=r"FRAP time step must lie in \(0, "):
        an.run_frap(grid, box, 1.0, an.FrapSchedule(0.01, 10, 1.0))
    # the device box sum is the reference's lexicographic host sum
    exp = an.run_frap(grid, box, 1.0, an.FrapSchedule(0.002, 4))
    u = grid.channel_data("u")
    m = 0.0
    for z in range(box.lo[2], box.hi[2]):
        for y in range(box.lo[1], box.hi[1]):
            for x in range(box.lo[0], box.hi[0]):
                v = grid.get((x, y, z), "u")
                if v is not None:
                    m += float(v)
    assert u.shape[0] == grid.chunk_count()
    assert grid.device().box_sum(grid.property_index("u"), box.lo, box.hi) == m
    denom = exp.curve[0]
    assert denom.time == 0.0 and denom.recovery == 0.0
