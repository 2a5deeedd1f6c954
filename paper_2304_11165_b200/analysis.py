"""FRAP experiments, effective diffusivity and tortuosity on the device —
the reference's analysis layer (analysis.hpp:19-349), SURVEY.md §8f row 3.

Same names, argument meaning, validation messages and arithmetic order as
the reference, so D_eff and tau_d come out bit-identical: every FTCS run goes
through the CUDA stepper (run_simulation), the initial condition is set by a
device kernel, and the bleached-region mass observer is evaluated on the
device at every recorded step in the reference's lexicographic order
(pd_grid_box_sum / pd_stepper_set_region). The remaining scalar work — the
recovery normalisation, the piecewise-linear interpolation, the squared-error
sum and the golden-section search — is a few hundred double operations per
fit and runs on the host in the reference's order.
"""
from __future__ import annotations

import bisect
import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import porediff as pd
from .porediff import InputError, format_scalar


@dataclass
class IndexBox:
    """analysis.hpp:36-55: lo inclusive, hi exclusive."""
    lo: Sequence[int]
    hi: Sequence[int]

    def contains(self, idx) -> bool:
        return all(self.lo[a] <= idx[a] < self.hi[a] for a in range(len(self.lo)))

    def volume(self) -> int:
        v = 1
        for a in range(len(self.lo)):
            v *= max(0, self.hi[a] - self.lo[a])
        return v


def _llround(x: float) -> int:
    # std::llround: half away from zero
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def central_bleach_box(geom: pd.GridGeometry, fraction: float = 0.1) -> IndexBox:
    """analysis.hpp:61-73."""
    if not (fraction > 0.0) or fraction > 1.0:
        raise InputError("bleach box fraction must be in (0, 1]")
    lo, hi = [], []
    for a in range(geom.dims):
        n = geom.size[a]
        w = min(max(_llround(fraction * float(n)), 1), n)
        lo.append((n - w) // 2)
        hi.append((n - w) // 2 + w)
    return IndexBox(lo, hi)


@dataclass
class FrapSample:
    time: float = 0.0
    recovery: float = 0.0


@dataclass
class FrapExperiment:
    d_molecular: float = 0.0
    region_nodes: int = 0
    phase_nodes: int = 0
    curve: List[FrapSample] = field(default_factory=list)


@dataclass
class FrapSchedule:
    t_final: float = 0.0
    n_samples: int = 200
    dt: float = 0.0


@dataclass
class TortuosityResult:
    d_molecular: float = 0.0
    d_eff: float = 0.0
    tau_d: float = 0.0
    fit_residual: float = 0.0
    edge_warning: bool = False


@dataclass
class FitOptions:
    rel_tol: float = 1e-3
    n_samples: int = 0
    dt: float = 0.0


def interp_curve(curve: Sequence[FrapSample], t: float) -> float:
    """analysis.hpp:129-141: piecewise-linear, clamped at both ends."""
    if not curve:
        raise InputError("cannot interpolate an empty recovery curve")
    if t <= curve[0].time:
        return curve[0].recovery
    if t >= curve[-1].time:
        return curve[-1].recovery
    i = bisect.bisect_left([s.time for s in curve], t)
    b, a = curve[i], curve[i - 1]
    w = (t - a.time) / (b.time - a.time)
    return a.recovery + w * (b.recovery - a.recovery)


def build_free_box_grid(geom: pd.GridGeometry, dtype=np.float64, device: int = 0) -> pd.SparseBlockGrid:
    """analysis.hpp:147-153: every node active, phi = 1, u = D = u_next = 0;
    built on the device."""
    chans = pd.solver_channels()
    dev = pd.DeviceGrid.full(geom, len(chans), prop_phi=chans.index("phi"), phi_value=1.0, dtype=dtype,
                             device=device)
    return pd.SparseBlockGrid.from_device(geom, chans, dev, dtype)


def run_frap(grid: pd.SparseBlockGrid, bleach: IndexBox, d_molecular: float,
             schedule: FrapSchedule) -> FrapExperiment:
    """analysis.hpp:160-225, on the device."""
    geom = grid.geometry()
    if not (d_molecular > 0.0) or not math.isfinite(d_molecular):
        raise InputError("molecular diffusivity must be positive and finite")
    if not (schedule.t_final > 0.0) or not math.isfinite(schedule.t_final):
        raise InputError("FRAP schedule needs t_final > 0")
    if schedule.n_samples < 1:
        raise InputError("FRAP schedule needs at least one sample")
    for a in range(geom.dims):
        lo, hi = bleach.lo[a], bleach.hi[a]
        if lo < 0 or hi > geom.size[a] or lo >= hi:
            raise InputError(f"bleach region is empty or outside the grid on axis {a}")

    # initial condition and counts in one pass (device)
    pu, pdd = grid.property_index("u"), grid.property_index("D")
    dev = grid.device()
    region, phase = dev.frap_init(pu, pdd, bleach.lo, bleach.hi, d_molecular)
    grid._mark_device_newer(["u", "D"])
    if region == 0:
        raise InputError("bleach region contains no active nodes")
    if region == phase:
        raise InputError("bleach region covers the whole phase; recovery is undefined")

    bound = pd.stability_dt(geom, d_molecular)
    dt = schedule.dt
    if dt == 0.0:
        dt = 0.4 * bound
    elif not (dt > 0.0) or not (dt < bound):
        raise InputError("FRAP time step must lie in (0, " + format_scalar(bound) + ")")
    n_steps = int(math.ceil(schedule.t_final / dt))

    cfg = pd.SimulationConfig()
    cfg.dt = dt
    cfg.n_steps = max(1, n_steps)
    cfg.record_every = max(1, cfg.n_steps // max(1, schedule.n_samples))

    exp = FrapExperiment(d_molecular, region, phase, [])
    res = pd.run_simulation(grid, cfg, region=(list(bleach.lo), list(bleach.hi)))
    cv = geom.cell_volume()
    denom = 0.0  # equilibrium mass share of the region, set at step 0
    for d, m in zip(res.diagnostics, res.region_sums):
        m *= cv
        if d.step == 0:
            denom = d.total_mass * float(region) / float(phase)
        exp.curve.append(FrapSample(d.time, m / denom))
    return exp


def frap_fit_objective(reference: FrapExperiment, box_geometry: pd.GridGeometry, box_bleach: IndexBox,
                       d_candidate: float, dt: float = 0.0, n_samples: int = 0) -> float:
    """analysis.hpp:231-250."""
    if len(reference.curve) < 2:
        raise InputError("reference FRAP curve needs at least two samples")
    grid = build_free_box_grid(box_geometry)
    try:
        schedule = FrapSchedule(reference.curve[-1].time,
                                n_samples if n_samples > 0 else len(reference.curve), dt)
        candidate = run_frap(grid, box_bleach, d_candidate, schedule)
    finally:
        grid.close(keep=False)  # a probe: its fields are not needed
    total = 0.0
    for s in reference.curve:
        diff = interp_curve(candidate.curve, s.time) - s.recovery
        total += diff * diff
    return total


def fit_effective_D(reference: FrapExperiment, box_geometry: pd.GridGeometry, box_bleach: IndexBox,
                    d_lo: float, d_hi: float, options: FitOptions = FitOptions()) -> TortuosityResult:
    """analysis.hpp:263-309: golden-section search of the free-box
    diffusivity whose FRAP curve best matches the reference."""
    if not (d_lo > 0.0) or not (d_hi > d_lo) or not math.isfinite(d_hi):
        raise InputError("search interval must satisfy 0 < d_lo < d_hi (finite)")
    if not (options.rel_tol > 0.0) or options.rel_tol >= 1.0:
        raise InputError("fit relative tolerance must be in (0, 1)")
    dt = options.dt if options.dt > 0.0 else 0.4 * pd.stability_dt(box_geometry, d_hi)

    def objective(d):
        return frap_fit_objective(reference, box_geometry, box_bleach, d, dt, options.n_samples)

    invphi = (math.sqrt(5.0) - 1.0) / 2.0
    a, b = d_lo, d_hi
    c = b - invphi * (b - a)
    d = a + invphi * (b - a)
    fc = objective(c)
    fd = objective(d)
    while b - a > options.rel_tol * 0.5 * (a + b):
        if fc < fd:
            b = d
            d = c
            fd = fc
            c = b - invphi * (b - a)
            fc = objective(c)
        else:
            a = c
            c = d
            fc = fd
            d = a + invphi * (b - a)
            fd = objective(d)
    r = TortuosityResult()
    r.d_molecular = reference.d_molecular
    r.d_eff = c if fc < fd else d
    r.fit_residual = min(fc, fd)
    r.tau_d = reference.d_molecular / r.d_eff
    margin = 4.0 * options.rel_tol
    r.edge_warning = r.d_eff <= d_lo * (1.0 + margin) or r.d_eff >= d_hi * (1.0 - margin)
    return r


def tortuosity_power_law(psi: float, exponent: float) -> float:
    """analysis.hpp:312-316."""
    if not (psi > 0.0) or psi > 1.0:
        raise InputError("power-law correlation needs porosity in (0, 1]")
    return math.pow(psi, -exponent)


def tortuosity_linear(psi: float, beta: float = 1.65) -> float:
    """analysis.hpp:319-321."""
    return psi + beta * (1.0 - psi)


def write_frap_csv(path: str, exp: FrapExperiment) -> None:
    """analysis.hpp:325-333: "time,recovery_fraction", round-trip scalars."""
    try:
        with open(path, "w", newline="\n") as f:
            f.write("time,recovery_fraction\n")
            for s in exp.curve:
                f.write(f"{format_scalar(s.time)},{format_scalar(s.recovery)}\n")
    except OSError:
        raise pd.IoError(f"cannot open '{path}' for writing") from None


# ---------------------------------------------------------------------------
# Steady-state flux estimator of D_eff and tortuosity (north_star (3)).
# The reference has no flux-based estimator (its only D_eff path is the FRAP
# fit above), so this has no reference counterpart: "parity unpinned". It is
# checked against a NumPy restatement (tests/test_observe.py) and, on a free
# box, against the exact answer D_eff = D.
# ---------------------------------------------------------------------------

@dataclass
class SteadyStateResult:
    steps: int                 # FTCS steps taken
    converged: bool            # rate criterion met before max_steps
    rate: float                # last normalised rate max|du| L^2 / (dt D_mol |dc|)
    flux: float                # total diffusive flux through the measuring plane (+axis direction)
    plane_fluxes: List[float]  # flux through every interior plane (conservation check)
    d_bulk: float              # F L / (A dc): bulk effective diffusivity
    porosity: float            # fluid nodes / box nodes
    d_eff: float               # d_bulk / porosity: pore-scale effective diffusivity
    tau: float                 # D_mol / d_eff (the FRAP fit's tau_d convention)
    norms: List[float] = field(default_factory=list)


def steady_state_diffusivity(grid: pd.SparseBlockGrid, axis: int = 0, c_in: float = 1.0, c_out: float = 0.0,
                             d_molecular: float = 1.0, dt: float = 0.0, tol: float = 1e-8,
                             check_every: int = 200, max_steps: int = 10 ** 7,
                             plane: int = -1) -> SteadyStateResult:
    """Drives the grid's u to the steady state of a through-diffusion
    experiment -- Dirichlet c_in on the low face of `axis`, c_out on the high
    face, no flux elsewhere and at the pore walls -- with the device FTCS
    stepper, stopping when the normalised rate max|u^{n+1}-u^n| L^2 /
    (dt D_mol |c_in - c_out|) of a recorded step drops below `tol` (device
    convergence observer). Then the flux F through the plane between node
    layers `plane` and `plane`+1 (default: the middle) gives
    d_bulk = F L / (A |dc|), with A the box cross-section and L =
    (size[axis] + 1) h the distance between the two Dirichlet ghost planes
    (so a free box with uniform D returns D exactly), d_eff = d_bulk /
    porosity and tau = D_mol / d_eff. The grid's D channel is used as is
    (populate it with D_mol in the pore space for a molecular-diffusion
    experiment); u starts from its current values."""
    geom = grid.geometry()
    if not (0 <= axis < geom.dims):
        raise InputError("flux axis out of range")
    dc = c_in - c_out
    if not (dc != 0.0) or not math.isfinite(dc):
        raise InputError("steady state needs c_in != c_out")
    if not (d_molecular > 0.0):
        raise InputError("molecular diffusivity must be positive and finite")
    if check_every < 1 or max_steps < 1:
        raise InputError("check_every and max_steps must be at least 1")
    n_ax = geom.size[axis]
    if plane < 0:
        plane = (n_ax - 1) // 2
    if not (0 <= plane < n_ax - 1):
        raise InputError("flux plane outside the box interior")
    dmax = pd.max_diffusivity(grid)
    bound = pd.stability_dt(geom, dmax) if dmax > 0 else math.inf
    if dt == 0.0:
        dt = 0.4 * bound
    elif not (0.0 < dt < bound):
        raise InputError("time step must lie in (0, " + format_scalar(bound) + ")")
    cfg = pd.SimulationConfig(dt=dt, n_steps=max_steps, record_every=check_every)
    cfg.outer_bc[2 * axis] = pd.FaceBc.dirichlet(c_in)
    cfg.outer_bc[2 * axis + 1] = pd.FaceBc.dirichlet(c_out)
    h = geom.spacing[axis]
    length = (n_ax + 1) * h
    scale = length * length / (dt * d_molecular * abs(dc))
    st = pd.FtcsStepper(grid, cfg)
    try:
        st.set_convergence(True)
        steps, rate, norms, converged = 0, math.inf, [], False
        while steps < max_steps:
            n = min(check_every * 16, max_steps - steps)
            st.run(steps, n, steps + n)
            got = st.convergence_norms()
            norms.extend(got)
            steps += n
            if got:
                rate = got[-1] * scale
                if rate < tol:
                    converged = True
                    break
        fluxes = [st.plane_flux(axis, L)[1] for L in range(n_ax - 1)]
        flux = fluxes[plane]
    finally:
        st.close()
    area = 1.0
    for a in range(geom.dims):
        if a != axis:
            area *= geom.size[a] * geom.spacing[a]
    d_bulk = flux * length / (area * dc)
    porosity = grid.active_node_count() / geom.node_count()
    d_eff = d_bulk / porosity
    return SteadyStateResult(steps, converged, rate, flux, fluxes, d_bulk, porosity, d_eff,
                             d_molecular / d_eff if d_eff > 0 else math.inf, norms)
