#!/usr/bin/env python
"""Benchmark of the fused FTCS sparse-block step (BASELINE.json metric:
active-point updates/s and % of the HBM roofline, vs the host CPU).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[4], the configuration the metric is quoted
on; it fits one B200): a 2048^3 cell-centred box on [0,1]^3, pore space =
complement of a random overlapping-sphere pack (radius 128 voxels, count for
~20% porosity, seed 12345), FP64 (the parity mode), sigmoid D(phi), surface
sink on the interface band, u0 = hash_unit_value(1, flat). Built on the
device (pd_build_sphere_pack_grid), so nothing but the stepper is timed.

A "step" is one FTCS time step over every active node. value = active
nodes x K / (max-over-ranks device time of the K steps). The grid (~3 x 25 GB
of u/u_next/D) is far larger than L2, so no L2 flush is needed between steps.

Multi-GPU (torchrun, one rank per GPU): z-slab decomposition by chunk
layers; each rank builds its slab plus one ghost chunk layer per side and
exchanges boundary u planes with NCCL every step. Strong scaling: the same
2048^3 domain is split over N GPUs. See DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "active-point updates/s (GPts/s) & % HBM roofline"
BYTES_PER_UPDATE = 24  # FP64: u_n read + D read + u_{n+1} write


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", "--box", dest="n", type=int, default=2048, help="box edge in nodes")
    ap.add_argument("--psi", type=float, default=0.2, help="target porosity")
    ap.add_argument("--radius-vox", type=float, default=128.0)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--cpu-sample", type=int, default=192, help="edge of the CPU sample crop")
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU sample duration")
    ap.add_argument("--e2e-n", type=int, default=512, help="box edge of the end-to-end host-buffer run")
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload(args):
    from paper_2304_11165_b200 import synthetic as sy
    r = args.radius_vox / args.n
    pack = sy.pack_for_porosity(args.psi, r, args.seed)
    return pack


def config_dict(args, n_gpus):
    return {"workload": f"C5 sparse {args.n}^3 random overlapping-sphere pore space, ~{int(args.psi*100)}% "
                        f"porosity, r={int(args.radius_vox)} vox, surface sink, FP64",
            "box": args.n, "porosity_target": args.psi, "sphere_radius_vox": args.radius_vox,
            "seed": args.seed, "precision": "fp64", "parallelism": f"zslab{n_gpus}",
            "l2": "inputs larger than L2 (no flush needed)"}


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md)
# ---------------------------------------------------------------------------


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    (pynvml) every 20 ms, falling back to nvidia-smi every 200 ms."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self.stop = threading.Event()
        self.index = index
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(mx), {k for k, b in self.REASONS.items() if r & b}))
            self.stop.wait(0.02)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) == 6 and f[0].replace(".", "").isdigit():
                    self.samples.append((float(f[0]), float(f[1]),
                                         {names[i] for i in range(4) if "Active" in f[2 + i] and not f[2 + i].startswith("Not")}))
            except Exception:
                pass
            self.stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self._run_smi()

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(n):
    """dram bytes per launch of the step kernel from the committed ncu
    capture summary (profiles/ftcs_step_traffic.json; captured at 2048^3),
    or None for other box sizes."""
    f = ROOT / "profiles" / "ftcs_step_traffic.json"
    if f.exists() and n == 2048:
        d = json.loads(f.read_text())
        return d.get("dram_bytes_per_launch"), d
    return None, None


# ---------------------------------------------------------------------------
# CPU baselines (reference compiled in place; test infrastructure)
# ---------------------------------------------------------------------------


_REF_GRID_CACHE = {}


def cpu_sample(args, pack, edge, steps, threads=None, target_s=None):
    """Times the reference's own run_simulation on a crop [0,edge)^3 of the
    same pore geometry (same spheres and spacing); geometry build untimed.
    With target_s, a short calibration run sizes the step count so the timed
    run takes about target_s seconds of CPU wall time."""
    import ctypes as C

    from oracle.pyoracle import Ref, make_config
    from paper_2304_11165_b200 import porediff as pd

    R = Ref()
    if threads:
        R.L.ref_set_worker_count(threads)
    h = 1.0 / args.n
    geom = pd.GridGeometry.make((edge,) * 3, (h,) * 3, (0.5 * h,) * 3)
    centers, radii = pack.arrays()
    # spheres that can touch the crop (exact: the others are never the min)
    lo, hi = 0.0, edge * h
    near = np.all((centers > lo - radii[:, None] - 2 * h) & (centers < hi + radii[:, None] + 2 * h), axis=1)
    if not near.any():  # crop inside the pore space (small custom boxes): the nearest spheres keep the SDF
        # finite (a timing sample; the default configuration always has spheres in the crop)
        mid = 0.5 * (lo + hi)
        near[np.argsort(np.linalg.norm(centers - mid, axis=1))[:8]] = True
    sub = type(pack)(list(map(tuple, centers[near])), list(radii[near]))
    sdf = sub.fluid_sdf_field(geom)
    g = R.grid_from_sdf(geom.size, geom.spacing, geom.origin, sdf)
    g.populate_diffusion(0.0, 1.0, 0.0, 4.0 * args.n)
    g.fill_hash("u", 1)
    dmax = g.max_diffusivity()
    dt = 0.4 * pd.stability_dt(geom, dmax)
    if target_s:
        cal = make_config(dt, 5, reaction="surface_sink", rate=1.0, band_half_width=1.0, record_every=5)
        t0 = time.perf_counter()
        g.run(cal)
        per_step = (time.perf_counter() - t0) / 5
        steps = max(5, int(target_s / max(per_step, 1e-6)))
    cfg = make_config(dt, steps, reaction="surface_sink", rate=1.0, band_half_width=1.0, record_every=steps)
    t0 = time.perf_counter()
    code, msg, rows = g.run(cfg)
    secs = time.perf_counter() - t0
    assert code == 0, msg
    active = g.active_count()
    cores = R.L.ref_worker_count()
    if threads:
        R.L.ref_set_worker_count(0)
    return active * steps / secs, active, secs, cores, steps


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks for exercising the N > 1 path on a one-GPU box: every rank on
    # cuda:0 (PD_BENCH_SAME_GPU=1) with a gloo control plane
    # (PD_DIST_BACKEND=gloo); the peer exchange itself is CUDA IPC either way
    if os.environ.get("PD_BENCH_SAME_GPU") == "1":
        local = 0
    backend = os.environ.get("PD_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    pack = workload(args)
    dom = shard.build_domain(args.n, pack, rank, world, device=local)
    stepper = dom.stepper(dt_frac=0.4, sink_rate=1.0)

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # warm-up
    dom.run(stepper, 0, args.warmup)
    sync()
    launches0 = dom.launches(stepper)
    with Clocks(local) as clk:
        sync()
        t0 = time.perf_counter()
        ms = dom.run(stepper, args.warmup, args.steps)
        sync()
        wall = time.perf_counter() - t0
    # step kernels + (N>1) the exchange's own kernels: peer wait + signal per
    # step (fused push), or two face packs and two unpacks (NCCL transport)
    launches = dom.launches(stepper) - launches0
    launches += dom.extra_launches_per_step * args.steps
    # exact global diagnostics of the final state (all ranks take part)
    diag = dom.diagnostics(stepper)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    act_t = torch.tensor([dom.owned_active], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(act_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    active = float(act_t.item())
    step_ms = ms_max / args.steps
    value = active * args.steps / (ms_max / 1e3)
    peak, peak_src = measured_peak()
    # dominant kernel: the step kernel alone (CUDA events on its stream),
    # timed region only
    kern_ms = dom.last_kernel_ms / args.steps
    achieved = dom.owned_active * BYTES_PER_UPDATE / (kern_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(args.n)

    chunks_total = int(dom.total_chunks(world))  # a collective: every rank takes part
    e2e = None
    if not args.no_e2e and rank == 0:
        e2e = run_e2e(args, pack)
    cpu = None
    if not args.no_cpu and rank == 0:
        try:
            v, a, secs, cores, st = cpu_sample(args, pack, args.cpu_sample, args.cpu_steps,
                                               target_s=args.cpu_seconds)
            cpu = {"value": v / 1e9, "unit": "GPts/s", "cores": cores, "kind": "reference",
                   "sample": f"reference run_simulation (oracle/_ref, -O3 -ffp-contract=off, "
                             f"{cores} std::thread workers) on the [0,{args.cpu_sample})^3 crop of the same "
                             f"geometry: {a} active nodes x {st} steps in {secs:.2f} s"}
            # SURVEY §8d also asks for the single-thread figure (RD_THREADS=1)
            v1, a1, secs1, _, st1 = cpu_sample(args, pack, args.cpu_sample, args.cpu_steps, threads=1,
                                               target_s=max(2.0, args.cpu_seconds / 4))
            cpu["single_thread"] = {"value": v1 / 1e9, "unit": "GPts/s", "cores": 1,
                                    "sample": f"same crop, 1 worker: {a1} active nodes x {st1} steps in {secs1:.2f} s"}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "GPts/s", "cores": None, "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value / 1e9, "unit": "GPts/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-built sphere pack)",
            "config": config_dict(args, world),
            "active_nodes": int(active), "chunks": chunks_total,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
                         "algorithmic_bytes_per_launch": dom.owned_active * BYTES_PER_UPDATE,
                         "peak_source": peak_src, "bytes_per_update": BYTES_PER_UPDATE,
                         "kernel_ms_per_step": kern_ms, "traffic_source": traffic_src and "profiles/ftcs_step_traffic.json"},
            "roofline_frac_of_step": dom.owned_active * BYTES_PER_UPDATE / (step_ms / 1e3) / 1e9 / peak,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "wall_s_timed_region": wall,
            "final_diagnostics": {"total_mass": diag[0], "min_u": diag[1], "max_u": diag[2],
                                  "note": "exact across ranks: rank-ordered per-chunk partials + pairwise_sum"},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, pack):
    """Same metric through the reference-facing API with HOST buffers: one
    run_simulation call on a host SparseBlockGrid (pinned upload of every
    channel, the FTCS steps, diagnostics rows, download of u and u_next), on a
    --e2e-n^3 crop of the same geometry."""
    import ctypes as C

    import torch

    from paper_2304_11165_b200 import porediff as pd

    n = args.e2e_n
    h = 1.0 / args.n
    geom = pd.GridGeometry.make((n,) * 3, (h,) * 3, (0.5 * h,) * 3)
    centers, radii = pack.arrays()
    dev = pd.DeviceGrid.sphere_pack(geom, centers, radii, n_props=4, prop_phi=0)
    dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * args.n))
    dev.fill_hash(1, 1)
    keys, masks = dev.layout()
    nch = len(keys)
    # pinned host slabs (the caller's grid)
    host = {}
    for p, name in enumerate(pd.solver_channels()):
        t = torch.empty((nch, 512), dtype=torch.float64, pin_memory=True)
        arr = t.numpy()
        arr[:] = dev.download(p)
        host[name] = (t, arr)
    dev.close()
    dmax = float(host["D"][1].max())
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, dmax), n_steps=args.e2e_steps,
                              record_every=args.e2e_steps)
    cfg.reaction = pd.ReactionSpec.surface_sink(1.0, 1.0)

    def once():
        g = pd.SparseBlockGrid.from_layout(geom, pd.solver_channels(), keys, masks, None)
        for name in pd.solver_channels():
            g._data[name] = host[name][1]  # zero-copy: the pinned host buffers
        t0 = time.perf_counter()
        res = pd.run_simulation(g, cfg)
        out_u = g.channel_data("u")
        out_un = g.channel_data("u_next")
        secs = time.perf_counter() - t0
        g.close()
        return secs, res

    once()  # warm-up (context, allocator)
    secs, res = once()
    active = int(host["phi"][1].size and sum(bin(int(w)).count("1") for w in masks.ravel()))
    slab = nch * 512 * 8
    return {"value": active * args.e2e_steps / secs / 1e9, "unit": "GPts/s", "h2d_bytes_per_step": 4 * slab,
            # run_simulation leaves u and u_next device-newer; the reads of
            # both pull exactly those two slabs (phi and D never change)
            "d2h_bytes_per_step": 2 * slab + 40 * len(res.diagnostics),
            "workload": f"run_simulation on a host grid, [0,{n})^3 crop of the same geometry, "
                        f"{args.e2e_steps} steps per call (one call = one e2e step)",
            "active_nodes": active, "seconds": secs}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pack = workload(args)
    edge = args.cpu_sample
    vals = []
    for _ in range(min(args.warmup, 1)):
        cpu_sample(args, pack, edge, 3)
    # each timed step is a bounded sample: ~cpu_seconds / steps of CPU work
    per = max(1.0, args.cpu_seconds / max(1, args.steps))
    total_pts, total_s, cores, active, st = 0.0, 0.0, None, 0, 0
    for _ in range(args.steps):
        v, active, secs, cores, st = cpu_sample(args, pack, edge, args.cpu_steps, target_s=per)
        total_pts += active * st
        total_s += secs
        vals.append(v)
    value = total_pts / total_s / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GPts/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, world),
        "cpu_baseline": {"value": value, "unit": "GPts/s", "cores": cores, "kind": "reference",
                         "sample": f"each step = reference run_simulation (oracle/_ref, {cores} std::thread "
                                   f"workers) of ~{st} FTCS steps on the [0,{edge})^3 crop ({active} active "
                                   f"nodes) of the same geometry"},
        "e2e": {"value": value, "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
