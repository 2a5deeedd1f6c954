"""Steady-state observers (north_star (3)): the device convergence norm and
plane-flux reduction, and the steady-state D_eff / tortuosity estimator
built on them (analysis.steady_state_diffusivity).

The reference has no flux-based estimator (its only D_eff
path is the FRAP fit), so these are "parity unpinned": the device results
are checked bit for bit against the NumPy restatement below (same face
coefficient in T arithmetic, same per-chunk face order, same pairwise fold),
and the estimator against exact answers (a free box returns D)."""
import math

import numpy as np
import pytest


def pairwise(v):
    """parallel.hpp:68-84: level-by-level pairwise tree, odd tail carried."""
    v = list(v)
    if not v:
        return 0.0
    while len(v) > 1:
        nx = [v[i] + v[i + 1] for i in range(0, len(v) - 1, 2)]
        if len(v) % 2:
            nx.append(v[-1])
        v = nx
    return v[0]


def np_plane_face_sum(keys, fluid, u, d, size, axis, layer):
    """Restatement of pd_stepper_plane_flux's face sum: for each chunk whose
    key[axis] == layer // 8 (ordinal order), the faces (the other axes'
    local coordinates, lowest axis fastest) between local layer l and l+1
    (the +axis neighbour chunk when l == 7), both nodes fluid, term
    dh * (u_b - u_a) with dh = (d_a + d_b) * T(0.5) in T arithmetic, summed
    sequentially per chunk in double, chunks folded pairwise."""
    dims = keys.shape[1]
    T = u.dtype.type
    cc = [(s + 7) // 8 for s in size]
    lin = np.zeros(len(keys), np.int64)
    for a in range(dims - 1, -1, -1):
        lin = lin * cc[a] + keys[:, a]
    pos = {int(l): i for i, l in enumerate(lin)}
    local = layer & 7
    others = [a for a in range(dims) if a != axis]
    parts = []
    for c in range(len(keys)):
        if keys[c, axis] != layer >> 3:
            continue
        s = 0.0
        for t in range(8 ** (dims - 1)):
            idx = [0] * dims
            r = t
            for a in others:
                idx[a] = r & 7
                r >>= 3
            idx[axis] = local
            off = 0
            for a in range(dims - 1, -1, -1):
                off = (off << 3) | idx[a]
            c2, off2 = c, off + (1 << (3 * axis))
            if local == 7:
                k2 = keys[c].copy()
                k2[axis] += 1
                l2 = 0
                for a in range(dims - 1, -1, -1):
                    l2 = l2 * cc[a] + int(k2[a])
                c2 = pos.get(l2, -1) if k2[axis] < cc[axis] else -1
                off2 = off - 7 * (1 << (3 * axis))
            term = 0.0
            if fluid[c, off] and c2 >= 0 and fluid[c2, off2]:
                dh = (d[c, off] + d[c2, off2]) * T(0.5)
                term = float(dh * (u[c2, off2] - u[c, off]))
            s += term
        parts.append(s)
    return pairwise(parts)


def test_restatement_on_a_linear_profile():
    """Free 2-D box, D = 1, u linear in x: every face carries the same
    term, so the face sum is exact and equals faces * slope * h."""
    n = 16
    keys = np.array([[i, j] for j in range(2) for i in range(2)], np.int32)
    fluid = np.ones((4, 64), bool)
    u = np.zeros((4, 64))
    d = np.ones((4, 64))
    for c, (kx, ky) in enumerate(keys):
        for off in range(64):
            x = kx * 8 + (off & 7)
            u[c, off] = 0.25 * x
    for layer in (3, 7, 11):
        s = np_plane_face_sum(keys, fluid, u, d, (n, n), 0, layer)
        assert s == 16 * 0.25


@pytest.mark.gpu
def test_convergence_norm_and_plane_flux_bitwise(cuda):
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import SpherePacking
    n = 40
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = SpherePacking.random((0, 0, 0), (1, 1, 1), 30, 0.08, 0.16, 777)
    c, r = pack.arrays()
    dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4, prop_phi=0)
    dev.populate_diffusion(0, 2, pd.DiffusionProfile.anchored(0.05, 0.95, 4.0 * n, 0.02))
    dev.fill_hash(1, 5)
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, pd.max_diffusivity(grid)), n_steps=30, record_every=10)
    cfg.reaction = pd.ReactionSpec.surface_sink(2.0, 1.5)
    cfg.outer_bc[0] = pd.FaceBc.dirichlet(1.0)
    st = pd.FtcsStepper(grid, cfg)
    st.set_convergence(True)
    prev = grid.channel_data("u").copy()
    norms = []
    act = grid.active_bool()
    for k in range(3):
        st.run(10 * k, 10, 30)
        norms += st.convergence_norms()
        # the norm of the last step of each segment: rerun it from the host
        # state is not possible, so compare u(step) - u(step-1) via u_next
        cur = grid.channel_data("u").copy()
        old = grid.channel_data("u_next").copy()  # after the swap: u_next = u(step - 1)
        assert norms[-1] == float(np.max(np.abs(cur[act] - old[act])))
        prev = cur
    assert len(norms) == 3 and all(v > 0 for v in norms)
    keys, _ = dev.layout()
    # fluid = active and phi > wall (wall = 0 + 0): every active node here
    fluid = act & (grid.channel_data("phi") > 0.0)
    u, d = grid.channel_data("u"), grid.channel_data("D")
    for axis in range(3):
        for layer in (0, 7, 8, 19, n - 2):
            fs, fl = st.plane_flux(axis, layer)
            want = np_plane_face_sum(keys, fluid, u, d, geom.size, axis, layer)
            assert fs == want, (axis, layer, fs, want)
            area = 1.0  # face area, other axes in ascending order (pd_stepper_plane_flux)
            for a in range(3):
                if a != axis:
                    area *= geom.spacing[a]
            assert fl == -want / geom.spacing[axis] * area
    with pytest.raises(pd.InputError):
        st.plane_flux(0, n - 1)
    st.close()


@pytest.mark.gpu
def test_steady_state_free_box_returns_d_exactly(cuda):
    """All-fluid box with uniform D: the steady profile is linear between the
    Dirichlet ghost planes, so d_bulk = d_eff = D, tau = D_mol / D, and the
    flux is the same through every plane."""
    from paper_2304_11165_b200 import analysis as an
    from paper_2304_11165_b200 import porediff as pd
    n = 24
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    grid = an.build_free_box_grid(geom)
    dev = grid.device()
    dev.fill_const(grid.property_index("D"), 0.7)
    grid._mark_device_newer(["D"])
    res = an.steady_state_diffusivity(grid, axis=2, c_in=1.0, c_out=0.0, d_molecular=1.0, tol=1e-10,
                                      check_every=500)
    assert res.converged and res.porosity == 1.0
    assert res.d_bulk == pytest.approx(0.7, rel=1e-8)
    assert res.tau == pytest.approx(1.0 / 0.7, rel=1e-8)
    assert np.allclose(res.plane_fluxes, res.flux, rtol=1e-8)


@pytest.mark.gpu
def test_steady_state_sphere_pack_is_porous(cuda):
    """Sphere pack (C2-shaped, small): the pore space slows diffusion
    (d_eff < D_mol, tau > 1), flux is conserved plane to plane at steady
    state, and the convergence norms decrease."""
    from paper_2304_11165_b200 import analysis as an
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import SpherePacking
    n = 48
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = SpherePacking.random((0, 0, 0), (1, 1, 1), 40, 0.1, 0.15, 2024)
    c, r = pack.arrays()
    dev = pd.DeviceGrid.sphere_pack(geom, c, r, n_props=4, prop_phi=0)
    dev.fill_const(2, 1.0)  # molecular diffusion in the pore space
    grid = pd.SparseBlockGrid.from_device(geom, pd.solver_channels(), dev)
    res = an.steady_state_diffusivity(grid, axis=0, tol=1e-7, check_every=500)
    assert res.converged
    assert 0.0 < res.d_bulk < res.porosity < 1.0
    assert 0.0 < res.d_eff < 1.0 and res.tau > 1.0
    assert np.allclose(res.plane_fluxes, res.flux, rtol=1e-5)
    assert res.norms[-1] < res.norms[0]
