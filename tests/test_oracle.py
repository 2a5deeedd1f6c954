"""The CPU oracle is pinned: the plain-C restatement (oracle/ftcs_oracle.c)
reproduces the reference's golden vectors bit for bit, and (where the
reference is built here) the reference itself regenerates them."""
import numpy as np
import pytest

from cases import CASES, GOLDEN, dt_of, host_case, oracle_config, sha, time_factor

FAST = [c for c in CASES if c != "c1_ball64"]


def _row_hex(r):
    return [int(r[0])] + [float(x).hex() for x in r[1:]]


@pytest.mark.parametrize("name", FAST + [pytest.param("c1_ball64", marks=pytest.mark.slow)])
def test_port_matches_golden(name, golden, port):
    spec, gold = CASES[name], golden[name]
    grid = host_case(name)
    inputs = {c: grid.channel_data(c).copy() for c in spec["channels"]}
    # inputs from this repo's host builders are the reference's inputs
    assert sha(grid.keys()) == gold["sha_keys"]
    assert sha(grid.masks()) == gold["sha_masks"]
    for c, a in inputs.items():
        assert sha(a) == gold["sha_inputs"][c], c
    dt = float.fromhex(gold["dt"])
    assert dt == dt_of(spec, float(inputs["D"][grid.active_bool()].max()))
    cfg = oracle_config(spec, dt)
    factors = None
    tf = time_factor(spec)
    if tf:
        factors = np.array([tf(float(s) * dt) for s in range(spec["steps"])])
    src = inputs.get("f")
    code, msg, rows, u, un = port.run(grid.geom.size, grid.geom.spacing, grid.keys(), grid.masks(),
                                      inputs["phi"], inputs["u"], inputs["D"], inputs["u_next"], cfg,
                                      src=src, factors=factors)
    assert code == 0, msg
    assert [_row_hex(r) for r in rows] == gold["rows"]
    assert sha(u) == gold["sha_outputs"]["u"]
    assert sha(un) == gold["sha_outputs"]["u_next"]


@pytest.mark.parametrize("name", ["disk24_sink", "disk20_volumetric", "disk24_fp32"])
def test_full_array_fixtures_are_consistent(name, golden):
    z = np.load(GOLDEN / f"{name}.npz")
    assert sha(z["keys"]) == golden[name]["sha_keys"]
    assert sha(z["out_u"]) == golden[name]["sha_outputs"]["u"]


def test_reference_regenerates_golden(ref, golden):
    from cases import ref_case
    for name in FAST:
        spec, gold = CASES[name], golden[name]
        g = ref_case(name, ref)
        dt = dt_of(spec, g.max_diffusivity())
        code, msg, rows = g.run(oracle_config(spec, dt), time_factor(spec))
        assert code == 0, msg
        assert [_row_hex(r) for r in rows] == gold["rows"], name
        assert sha(g.prop("u")) == gold["sha_outputs"]["u"], name


def test_port_error_messages_match_reference(ref, port):
    """Non-finite node, stability gate and validation messages
    (solver.hpp:250-260, 495-503, 304-331)."""
    from cases import ref_case
    from oracle.pyoracle import make_config
    g = ref_case("disk24_sink", ref)
    keys, masks = g.layout()
    props = {c: g.prop(c) for c in ("phi", "u", "D", "u_next")}
    u = props["u"].copy()
    u[4, 9] = np.inf
    g.set_prop("u", u)
    dmax = g.max_diffusivity()
    h = 2.0 / 24
    bound = 1.0 / (2.0 * dmax) / (2.0 / (h * h))
    for cfg in (make_config(0.3 * bound, 5), make_config(10 * bound, 5), make_config(-1.0, 5),
                make_config(0.3 * bound, 0), make_config(0.3 * bound, 5, reaction="surface_sink", rate=-1.0)):
        rc, rmsg, rrows = g.run(cfg)
        pc, pmsg, prows, _, _ = port.run((24, 24), (h, h), keys, masks, props["phi"], u, props["D"],
                                         props["u_next"], cfg)
        assert (rc, rmsg) == (pc, pmsg)
        assert rc != 0
