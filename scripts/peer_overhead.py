"""Cost of the fused halo exchange on one GPU: the bench domain split into
`world` z-slab shards that all live on cuda:0 (raw-pointer peers, one stream
per shard, every step enqueued without a host sync: wait -> march with the
boundary-plane push -> signal), against the unsharded run of the same domain.
On one GPU the shards share the SMs, so the sharded step time is the sum of
the shard kernels plus the exchange overhead; the difference to the
unsharded step is what the exchange costs. Results are also checked bit for
bit against the unsharded run (owned u of every shard).

Slab balance: before the exchange is wired up, every shard is stepped alone
(pd_stepper_run over its owned range) and the per-shard kernel times give
the load imbalance max/mean - 1 of the cuts (--balance layers | chunks |
cost, the per-layer cost model of shard.layer_cost; --balance all measures
the three and runs the exchange with "cost"; the bench default is "chunks").

    python scripts/peer_overhead.py [--n 1024] [--world 2] [--steps 20] [--balance cost]
"""
import argparse
import ctypes as C
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2304_11165_b200 import porediff as pd
from paper_2304_11165_b200 import shard
from paper_2304_11165_b200._lib import lib
from paper_2304_11165_b200 import synthetic as sy


def build(geom, centers, radii, lo, hi):
    h = C.c_void_p()
    pd._check(lib.pd_build_sphere_pack_region(
        8, (C.c_int64 * 3)(*geom.size), (C.c_double * 3)(*geom.spacing), (C.c_double * 3)(*geom.origin),
        len(radii), centers.ctypes.data_as(C.POINTER(C.c_double)), radii.ctypes.data_as(C.POINTER(C.c_double)),
        0.0, math.inf, (C.c_int64 * 3)(*lo), (C.c_int64 * 3)(*hi), 4, 0, 0, C.byref(h)))
    n = C.c_int64()
    lib.pd_grid_info(h, C.byref(n), None)
    dev = pd.DeviceGrid(h, geom, np.float64, int(n.value), 4)
    dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * geom.size[0]))
    dev.fill_hash(1, 1)
    return dev


def stepper(dev, dt, rng=None):
    cfg = pd.SimulationConfig(dt=dt, n_steps=1 << 40, record_every=1 << 40)
    cfg.reaction = pd.ReactionSpec.surface_sink(1.0, 1.0)
    cc = pd._to_c_config(cfg, -1)
    h = C.c_void_p()
    pd._check(lib.pd_stepper_create(dev.h, C.byref(cc), 0, 1, 2, 3, C.byref(h)))
    if rng is not None:
        pd._check(lib.pd_stepper_set_range(h, *rng))
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--balance", default="cost", choices=["layers", "chunks", "cost", "all"])
    a = ap.parse_args()
    n, world, steps = a.n, a.world, a.steps
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    r = 128.0 * n / 2048 / n
    pack = sy.pack_for_porosity(0.2, r, 2048)
    centers, radii = pack.arrays()
    cc = (n + 7) // 8
    full = build(geom, centers, radii, (0, 0, 0), (cc, cc, cc))
    dt = 0.4 * pd.stability_dt(geom, full.max_active(2))
    s_full = stepper(full, dt)
    rows = (pd._lib.pd_diag * 1)()
    nr = C.c_int64()
    pd._check(lib.pd_stepper_run(s_full, 0, 3, 1 << 40, None, rows, C.byref(nr)))  # warm
    torch.cuda.synchronize()
    ms = C.c_double()
    pd._check(lib.pd_stepper_run(s_full, 3, steps, 1 << 40, None, rows, C.byref(nr)))
    lib.pd_stepper_last_ms(s_full, C.byref(ms))
    t_full = ms.value / steps
    u_full = full.download(1)
    keys_full, _ = full.layout()
    lib.pd_stepper_destroy(s_full)
    full.close()

    ch, ac, fu = shard.layer_work(geom, pack)
    weights = {"layers": None, "chunks": ch, "cost": shard.layer_cost(ch, fu)}

    def make_shards(mode):
        out = []
        for rk in range(world):
            z0, z1 = shard.slab_bounds(cc, world, rk, weights[mode])
            dev = build(geom, centers, radii, (0, 0, max(0, z0 - 1)), (cc, cc, min(cc, z1 + 1)))
            keys, _ = dev.layout()
            plan = shard.exchange_plan(keys, z0, z1, rk, world)
            s = stepper(dev, dt, (plan.begin, plan.end))
            cols = (C.c_void_p * 4)()
            pd._check(lib.pd_grid_column_ptrs(dev.h, cols))
            sync = C.c_void_p()
            pd._check(lib.pd_stepper_sync_words(s, C.byref(sync)))
            out.append((dev, plan, s, keys, cols, sync))
        return out

    def shard_times(shs):
        """Each shard stepped alone (no exchange): its kernel ms per step."""
        ts = []
        for dev, plan, s, *_ in shs:
            pd._check(lib.pd_stepper_run(s, 0, 2, 1 << 40, None, rows, C.byref(nr)))
            pd._check(lib.pd_stepper_run(s, 2, steps, 1 << 40, None, rows, C.byref(nr)))
            lib.pd_stepper_last_ms(s, C.byref(ms))
            ts.append(ms.value / steps)
            pd._check(lib.pd_stepper_run(s, 2 + steps, steps + 2, 1 << 40, None, rows, C.byref(nr)))  # even count
        return ts

    modes = ["layers", "chunks", "cost"] if a.balance == "all" else [a.balance]
    for mode in modes:
        shs = make_shards(mode)
        ts = shard_times(shs)
        print(f"{n}^3, {world} shards, balance={mode}: shard kernel ms/step {[round(t, 3) for t in ts]}, "
              f"sum {sum(ts):.3f} (unsharded {t_full:.3f}), imbalance max/mean-1 = "
              f"{max(ts) / (sum(ts) / len(ts)) - 1:+.2%}", flush=True)
        if mode != modes[-1]:
            for dev, plan, s, *_ in shs:
                lib.pd_stepper_destroy(s)
                dev.close()
    shards = shs
    # the timing runs above advanced every shard an even number of steps from
    # the same state; restart all of them from u0 for the exchange check
    for dev, *_ in shards:
        dev.fill_hash(1, 1)
        dev.fill_const(3, 0.0)
    for rk, (dev, plan, s, keys, cols, sync) in enumerate(shards):
        for side, nb, src in ((0, rk - 1, plan.send_down), (1, rk + 1, plan.send_up)):
            if 0 <= nb < world:
                o = shards[nb]
                dst = np.ascontiguousarray(o[1].recv_up if side == 0 else o[1].recv_down, np.int32)
                src = np.ascontiguousarray(src, np.int32)
                pd._check(lib.pd_stepper_set_peer(s, side, o[4], 4, o[5], src.ctypes.data, dst.ctypes.data,
                                                  len(src)))
    for sh in shards:
        pd._check(lib.pd_stepper_peer_reset(sh[2]))

    def run(k0, k):
        for st in range(k0, k0 + k):
            for dev, plan, s, *_ in shards:
                pd._check(lib.pd_stepper_enqueue(s, st, plan.begin, plan.end, 1.0))
            for sh in shards:
                pd._check(lib.pd_stepper_swap(sh[2]))

    run(0, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    run(3, steps)
    torch.cuda.synchronize()
    t_sh = (time.perf_counter() - t0) * 1e3 / steps
    for dev, plan, s, *_ in shards:
        pd._check(lib.pd_stepper_status(s, 3 + steps))
    lin_full = (keys_full[:, 2].astype(np.int64) * cc + keys_full[:, 1]) * cc + keys_full[:, 0]
    pos = {int(l): i for i, l in enumerate(lin_full)}
    same = True
    for dev, plan, s, keys, *_ in shards:
        u = dev.download(1)
        kk = keys[plan.begin:plan.end]
        idx = np.array([pos[int(l)] for l in (kk[:, 2].astype(np.int64) * cc + kk[:, 1]) * cc + kk[:, 0]])
        same &= np.array_equal(u[plan.begin:plan.end].view(np.uint64), u_full[idx].view(np.uint64))
    ghosts = sum(len(sh[1].recv_down) + len(sh[1].recv_up) for sh in shards)
    print(f"{n}^3, {world} shards on one GPU, {steps} steps: unsharded {t_full:.3f} ms/step (device), "
          f"sharded with fused push {t_sh:.3f} ms/step (wall, all shards) -> exchange overhead "
          f"{(t_sh - t_full) / t_full * 100:+.1f} %; pushed chunk planes/step {ghosts}; bit-identical: {same}")
    for dev, plan, s, *_ in shards:
        lib.pd_stepper_destroy(s)
        dev.close()


if __name__ == "__main__":
    main()
