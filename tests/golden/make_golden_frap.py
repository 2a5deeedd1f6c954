"""Generates tests/golden/frap.json: FRAP recovery curves and effective
diffusivity / tortuosity fits computed by the UNMODIFIED reference
(run_frap + fit_effective_D, analysis.hpp:160-309, through
oracle/_ref/libporediff_ref.so built in place by oracle/Makefile).

    python tests/golden/make_golden_frap.py

Geometry (D_eff/tau KAT): a cell-centred n^3 box on
[0,1]^3, pore space = complement of SpherePacking::random({0,0,0},{1,1,1},
count, r_min, r_max, seed) (synthetic.hpp:25-56), band PhaseBand{0, inf}.
All values are float.hex strings (bitwise comparisons).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "frap.json"

# name: n, spheres (count, r_min, r_max, seed), bleach fraction, t_final,
# n_samples, dt = dt_frac * stability_dt(D = dt_dmax), fit interval, rel_tol
CASES = {
    "frap16": dict(n=16, count=12, r_min=0.1, r_max=0.2, seed=7, bleach=0.3, t_final=0.02, n_samples=20,
                   dt_frac=0.4, dt_dmax=1.2, d_lo=0.2, d_hi=1.2, rel_tol=1e-2),
    "frap32": dict(n=32, count=40, r_min=0.1, r_max=0.15, seed=2024, bleach=0.25, t_final=0.05, n_samples=100,
                   dt_frac=0.4, dt_dmax=1.2, d_lo=0.2, d_hi=1.2, rel_tol=1e-3),
    # SURVEY.md §8d second D_eff/tau KAT (64^3: 0.84242584501724482 / 1.1870481015210657)
    "frap64": dict(n=64, count=40, r_min=0.1, r_max=0.15, seed=2024, bleach=0.25, t_final=0.05, n_samples=100,
                   dt_frac=0.4, dt_dmax=1.2, d_lo=0.2, d_hi=1.2, rel_tol=1e-3),
}


def stability_dt(h, dmax):
    inv = 0.0
    for _ in range(3):
        inv += 1.0 / (h * h)
    return 1.0 / (2.0 * dmax) / inv


def main():
    R = Ref()
    out = {}
    for name, c in CASES.items():
        n = c["n"]
        h = 1.0 / n
        size, spacing, origin = (n, n, n), (h, h, h), (0.5 * h, 0.5 * h, 0.5 * h)
        centers, radii = R.sphere_packing((0, 0, 0), (1, 1, 1), c["count"], c["r_min"], c["r_max"], c["seed"])
        sdf = R.field_sphere_pack(size, spacing, origin, centers, radii)
        g = R.grid_from_sdf(size, spacing, origin, sdf)
        dt = c["dt_frac"] * stability_dt(h, c["dt_dmax"])
        d_eff, tau, res, ct, cr = g.frap_fit(c["bleach"], 1.0, c["t_final"], c["n_samples"], dt, c["d_lo"],
                                             c["d_hi"], c["rel_tol"])
        out[name] = dict(c, dt=dt.hex(), active=int(g.active_count()), chunks=int(g.chunk_count()),
                         d_eff=d_eff.hex(), tau=tau.hex(), residual=res.hex(),
                         curve_t=[float(x).hex() for x in ct], curve_r=[float(x).hex() for x in cr])
        print(name, "D_eff", repr(d_eff), "tau", repr(tau), "samples", len(ct))
    OUT.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
