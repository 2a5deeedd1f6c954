"""Generates tests/golden/golden.json (+ small .npz inputs/outputs) by running
the UNMODIFIED reference (oracle/_ref/libporediff_ref.so, compiled in place
from /root/reference by oracle/Makefile) on every case of tests/cases.py.

    python tests/golden/make_golden.py

Rows are stored as float.hex strings so comparisons are bitwise. The GPU box
has no /root/reference: tests there compare against these committed values
(and against oracle/_ref, which travels as a prebuilt .so).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from cases import CASES, GOLDEN, dt_of, oracle_config, ref_case, sha, time_factor  # noqa: E402
from oracle.pyoracle import Ref  # noqa: E402

FULL_ARRAYS = {"disk24_sink", "disk20_volumetric", "disk24_fp32"}


def hexrow(r):
    return [int(r[0])] + [float(x).hex() for x in r[1:]]


def main():
    R = Ref()
    out = {}
    for name, spec in CASES.items():
        g = ref_case(name, R)
        keys, masks = g.layout()
        inputs = {c: g.prop(c) for c in spec["channels"]}
        dmax = g.max_diffusivity()
        dt = dt_of(spec, dmax)
        cfg = oracle_config(spec, dt)
        code, msg, rows = g.run(cfg, time_factor(spec))
        assert code == 0, (name, code, msg)
        outputs = {c: g.prop(c) for c in ("u", "u_next")}
        entry = {
            "chunks": int(len(keys)),
            "active": int(g.active_count()),
            "dmax": float(dmax).hex(),
            "dt": float(dt).hex(),
            "sha_keys": sha(keys),
            "sha_masks": sha(masks),
            "sha_inputs": {c: sha(a) for c, a in inputs.items()},
            "sha_outputs": {c: sha(a) for c, a in outputs.items()},
            "rows": [hexrow(r) for r in rows],
        }
        if name in FULL_ARRAYS:
            np.savez_compressed(GOLDEN / f"{name}.npz", keys=keys, masks=masks,
                                **{f"in_{c}": a for c, a in inputs.items()},
                                **{f"out_{c}": a for c, a in outputs.items()})
        out[name] = entry
        print(name, entry["chunks"], entry["active"], rows[-1])
    # SURVEY.md §8d / Appendix A C1 values (recorded there from the same
    # reference run): pinned here so a drifted reference build is caught.
    c1 = out["c1_ball64"]
    assert float.fromhex(c1["rows"][-1][2]) == 0.4449934885835134
    assert float.fromhex(c1["rows"][-1][3]) == 0.49553969128943648
    assert float.fromhex(c1["rows"][-1][4]) == 0.50652925641333113
    assert float.fromhex(c1["dt"]) == 2.564311247270007e-05
    (GOLDEN / "golden.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
