"""Size-independent properties at the bench's full size (C5, 2048^3, 1.98 G
active nodes), where no CPU oracle can follow: with the sink off and the box
sealed, total mass is conserved to the reference acceptance bound
(acceptance_test.cpp:259-312: relative drift <= 1e-12 per step) and the
maximum principle holds (min / max of u never leave their initial range);
with the sink on, mass is non-increasing. Exact cross-chunk diagnostics come
from the per-chunk partials + pairwise tree."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c5_fullsize_conservation_and_maximum_principle(cuda):
    import torch
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200 import synthetic as sy
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")
    n = 2048
    pack = sy.pack_for_porosity(0.2, 128.0 / 2048, 12345)
    dom = shard.Domain(n, pack, 0, 1, 0)
    st = dom.stepper(dt_frac=0.4, sink_rate=0.0)  # sink rate 0: pure diffusion, sealed box
    m0, lo0, hi0 = dom.diagnostics(st)
    steps = 10
    dom.run(st, 0, steps)
    m1, lo1, hi1 = dom.diagnostics(st)
    assert abs(m1 - m0) <= 1e-12 * steps * abs(m0), (m0, m1)
    assert lo1 >= lo0 and hi1 <= hi0, (lo0, lo1, hi0, hi1)
    torch.cuda.synchronize()
    from paper_2304_11165_b200._lib import lib
    lib.pd_stepper_destroy(st)
    st2 = dom.stepper(dt_frac=0.4, sink_rate=2.0)
    dom.run(st2, steps, steps)
    m2, lo2, hi2 = dom.diagnostics(st2)
    assert m2 < m1 and lo2 >= 0.0
    lib.pd_stepper_destroy(st2)
    dom.dev.close()
