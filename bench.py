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

Multi-GPU (one rank per GPU): `bench.py --gpus N` re-launches itself under
torch.distributed.run with N ranks when it is not already inside one (the
driver's torchrun launch works the same). z-slab decomposition by chunk
layers, cut at equal prefix sums of per-layer cost; each rank builds its slab
plus one ghost chunk layer per side, and the step kernel pushes its boundary
planes into the neighbours' ghost layers over NVLink peer memory. Strong
scaling: the same 2048^3 domain is split over N GPUs.

The reference arm (--impl reference) and the cpu_baseline leg run the
UNMODIFIED reference (oracle/_ref, compiled in place) through one shared
sampling protocol (reference_rate below); the reference arm imports nothing
from the product package.
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
    ap.add_argument("--e2e-n", type=int, default=0,
                    help="box edge of the end-to-end host-buffer run (0: the bench box when host RAM allows)")
    ap.add_argument("--e2e-steps", type=int, default=1000)
    ap.add_argument("--cpu-calls", type=int, default=3, help="timed reference calls of the cpu_baseline leg")
    ap.add_argument("--ref-threads", type=int, default=0, help="reference arm worker threads (0: all host cores)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def pack_count(psi, radius):
    """Sphere count of pack_for_porosity (Boolean model, unit box):
    psi = exp(-count * 4/3 pi r^3)."""
    return int(round(math.log(1.0 / psi) / (4.0 / 3.0 * math.pi * radius ** 3)))


def workload(args):
    """The bench's sphere pack, drawn by the product's SpherePacking.random
    (bit-identical to the reference's SpherePacking::random,
    synthetic.hpp:42-55)."""
    from paper_2304_11165_b200 import synthetic as sy
    r = args.radius_vox / args.n
    return sy.SpherePacking.random((0, 0, 0), (1, 1, 1), pack_count(args.psi, r), r, r, args.seed)


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


def ref_spheres(R, args):
    """The same pack drawn by the reference itself (synthetic.hpp:42-55)."""
    r = args.radius_vox / args.n
    return R.sphere_packing((0, 0, 0), (1, 1, 1), pack_count(args.psi, r), r, r, args.seed)


def crop_spheres(R, centers, radii, size, h, origin):
    """Spheres that can be the minimum of fluid_sdf somewhere in the crop
    (exact, see tests/test_headline_parity.py): M = max over the crop of the
    field of the spheres meeting the crop box bounds the true field, and a
    sphere whose box distance minus radius exceeds M is never the minimum."""
    lo = np.asarray(origin, float)
    hi = lo + (np.asarray(size) - 1) * h
    d = np.linalg.norm(np.maximum(0.0, np.maximum(lo - centers, centers - hi)), axis=1) - radii
    first = d <= 0.0
    if not first.any():
        return centers, radii
    f0 = R.field_sphere_pack(size, (h,) * 3, origin, centers[first], radii[first])
    keep = d <= float(np.max(f0))
    return centers[keep], radii[keep]


def reference_rate(args, edge, calls, per_call_s, threads=None, warm=True):
    """THE CPU sampling protocol of both the reference arm and the
    cpu_baseline leg: the reference's own pipeline (field_from over the pack,
    build_sparse_grid, populate_diffusion_channel, u = hash_unit_value(1, .),
    surface sink 1/1, dt = 0.4 * stability_dt(max D)) on the [0, edge)^3 crop
    of the bench geometry (same spheres, spacing and origin), built once
    (untimed); a calibration call sizes S steps per call to ~per_call_s; then
    `calls` run_simulation calls of S steps each are timed back to back on the
    same grid. Returns (G pts/s, per-call seconds, S, active nodes, worker
    threads). Only oracle/ is touched (test infrastructure)."""
    from oracle.pyoracle import Ref, make_config
    import ctypes as C
    R = Ref()
    R.L.ref_set_worker_count(threads or 0)
    try:
        h = 1.0 / args.n
        size, origin = (edge,) * 3, (0.5 * h,) * 3
        centers, radii = ref_spheres(R, args)
        sc, sr = crop_spheres(R, centers, radii, size, h, origin)
        g = R.grid_from_sdf(size, (h,) * 3, origin, R.field_sphere_pack(size, (h,) * 3, origin, sc, sr))
        g.populate_diffusion(0.0, 1.0, 0.0, 4.0 * args.n)
        g.fill_hash("u", 1)
        code = C.c_int()
        bound = R.L.ref_stability_dt(3, (C.c_double * 3)(h, h, h), g.max_diffusivity(), C.byref(code))
        dt = 0.4 * bound

        def call(steps):
            cfg = make_config(dt, steps, reaction="surface_sink", rate=1.0, band_half_width=1.0, record_every=steps)
            t0 = time.perf_counter()
            rc, msg, _ = g.run(cfg)
            secs = time.perf_counter() - t0
            assert rc == 0, msg
            return secs

        cal = 4
        per_step = call(cal) / cal
        if warm:
            call(cal)
            per_step = min(per_step, call(cal) / cal)
        steps = max(2, int(per_call_s / max(per_step, 1e-9)))
        secs = [call(steps) for _ in range(calls)]
        active = g.active_count()
        return active * steps * calls / sum(secs) / 1e9, secs, steps, active, R.L.ref_worker_count()
    finally:
        R.L.ref_set_worker_count(0)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2304_11165_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
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
    t_build = time.perf_counter()
    dom = shard.build_domain(args.n, pack, rank, world, device=local)
    stepper = dom.stepper(dt_frac=0.4, sink_rate=1.0)
    t_build = time.perf_counter() - t_build

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # warm-up
    dom.run(stepper, 0, args.warmup)
    sync()
    launches0 = dom.launches(stepper)
    wait0 = dom.peer_wait_ns(stepper)
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
    kern_ms = dom.last_kernel_ms / args.steps
    wait_ms = (dom.peer_wait_ns(stepper) - wait0) / 1e6 / args.steps
    mine = torch.tensor([ms, kern_ms, float(dom.owned_active), float(dom.owned_chunks), wait_ms],
                        dtype=torch.float64, device=red_dev)
    if world > 1:
        allv = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine)
        per_rank = torch.stack(allv).cpu().numpy()
    else:
        per_rank = mine.cpu().numpy()[None, :]
    ms_max = float(per_rank[:, 0].max())
    active = float(per_rank[:, 2].sum())
    step_ms = ms_max / args.steps
    value = active * args.steps / (ms_max / 1e3)
    peak, peak_src = measured_peak()
    # dominant kernel: the step kernel alone (CUDA events on its stream),
    # timed region only, on the slowest rank
    kmax = int(per_rank[:, 1].argmax())
    kern_ms_max = float(per_rank[kmax, 1])
    achieved = float(per_rank[kmax, 2]) * BYTES_PER_UPDATE / (kern_ms_max / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(args.n)
    chunks_total = int(per_rank[:, 3].sum())
    ranks = [{"rank": r, "step_ms": float(per_rank[r, 0]) / args.steps, "kernel_ms": float(per_rank[r, 1]),
              "active_nodes": int(per_rank[r, 2]), "chunks": int(per_rank[r, 3]),
              "halo_wait_ms_per_step": float(per_rank[r, 4])} for r in range(world)]
    # work imbalance: per-rank step-kernel time minus the time spent blocked
    # on the neighbours (the fused exchange's per-step wait)
    work = per_rank[:, 1] - per_rank[:, 4]
    imbalance = float(work.max() / work.mean() - 1.0) if work.mean() > 0 else 0.0
    # the bench domain leaves the device before the end-to-end run needs it
    dom.close(stepper)
    del dom
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    e2e = None
    if not args.no_e2e and rank == 0:
        try:
            e2e = run_e2e(args, pack)
        except Exception as e:  # reported, not fatal
            e2e = {"value": None, "unit": "GPts/s", "error": f"{type(e).__name__}: {e}"}
    cpu = None
    if not args.no_cpu and rank == 0:
        cpu = cpu_baseline_leg(args)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value / 1e9, "unit": "GPts/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-built sphere pack)",
            "config": config_dict(args, world),
            "active_nodes": int(active), "chunks": chunks_total,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
                         "algorithmic_bytes_per_launch": float(per_rank[kmax, 2]) * BYTES_PER_UPDATE,
                         "peak_source": peak_src, "bytes_per_update": BYTES_PER_UPDATE,
                         "kernel_ms_per_step": kern_ms_max, "traffic_source": traffic_src and "profiles/ftcs_step_traffic.json"},
            "roofline_frac_of_step": active * BYTES_PER_UPDATE / (step_ms / 1e3) / 1e9 / peak / world,
            "per_rank": ranks, "load_imbalance": imbalance,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "wall_s_timed_region": wall, "build_s": t_build,
            "final_diagnostics": {"total_mass": diag[0], "min_u": diag[1], "max_u": diag[2],
                                  "note": "exact across ranks: rank-ordered per-chunk partials + pairwise_sum"},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_leg(args):
    """The cpu_baseline object: the reference arm itself (`bench.py --impl
    reference`, a fresh process that loads only oracle/_ref) on this box's
    host cores, all threads and then one thread -- the same protocol and the
    same process state as the driver's reference arm."""
    common = ["--box", str(args.n), "--psi", str(args.psi), "--radius-vox", str(args.radius_vox),
              "--seed", str(args.seed), "--cpu-sample", str(args.cpu_sample)]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = {}
    for key, threads, steps, secs in (("all", 0, args.cpu_calls, args.cpu_seconds),
                                      ("one", 1, 1, max(2.0, args.cpu_seconds / 4))):
        cmd = [sys.executable, str(Path(__file__).resolve()), "--impl", "reference", "--steps", str(steps),
               "--warmup", "1", "--cpu-seconds", str(secs), "--ref-threads", str(threads)] + common
        try:
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
            line = [l for l in p.stdout.splitlines() if l.startswith("{")]
            out[key] = json.loads(line[-1])["cpu_baseline"] if line else {"value": None, "sample": p.stderr[-400:]}
        except Exception as e:  # reported, not fatal
            out[key] = {"value": None, "sample": f"failed: {e}"}
    cpu = dict(out["all"])
    cpu["single_thread"] = out["one"]
    return cpu


def host_ram_bytes():
    try:
        import psutil
        return psutil.virtual_memory().available
    except Exception:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")


def run_e2e(args, pack):
    """The same metric through the reference-facing API with HOST buffers:
    one run_simulation call (args.e2e_steps steps) on a host SparseBlockGrid
    whose four channel slabs live in pinned host memory. Timed: creation of
    the device mirror and the upload of every channel (H2D), the stepper
    build, the steps, the diagnostics rows, and the download of u and u_next
    (D2H, what the steps changed). Default box: the bench box itself, when
    the host has the RAM for its pinned slabs; else the largest power-of-two
    crop of the same geometry that fits (stated in `workload`)."""
    import torch

    from paper_2304_11165_b200 import porediff as pd

    n = args.e2e_n
    h = 1.0 / args.n
    centers, radii = pack.arrays()
    if n <= 0:
        n = args.n
        while n > 256:
            geom = pd.GridGeometry.make((n,) * 3, (h,) * 3, (0.5 * h,) * 3)
            _, act_chunks = _layer_chunks(pd, geom, centers, radii)
            need = act_chunks * 512 * 8 * 4
            if need * 1.3 < host_ram_bytes():
                break
            n //= 2
    geom = pd.GridGeometry.make((n,) * 3, (h,) * 3, (0.5 * h,) * 3)
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
        dev.download_into(p, arr)
        host[name] = (t, arr)
    dmax = dev.max_active(2)
    dev.close()
    cfg = pd.SimulationConfig(dt=0.4 * pd.stability_dt(geom, dmax), n_steps=args.e2e_steps,
                              record_every=args.e2e_steps)
    cfg.reaction = pd.ReactionSpec.surface_sink(1.0, 1.0)
    keep = {name: host[name][1].copy() if n <= 512 else None for name in ("u", "u_next")}

    def once():
        g = pd.SparseBlockGrid.from_layout(geom, pd.solver_channels(), keys, masks, None)
        for name in pd.solver_channels():
            g._data[name] = host[name][1]  # zero-copy: the pinned host buffers
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pd.run_simulation(g, cfg)
        out_u = g.channel_data("u")
        out_un = g.channel_data("u_next")
        secs = time.perf_counter() - t0
        g.close()
        return secs, res

    if n <= 512:  # small boxes: one untimed warm-up call (context, allocator), state restored
        once()
        for name in ("u", "u_next"):
            host[name][1][:] = keep[name]
    secs, res = once()
    active = int(np.bitwise_count(masks).sum())
    slab = nch * 512 * 8
    return {"value": active * args.e2e_steps / secs / 1e9, "unit": "GPts/s", "h2d_bytes_per_step": 4 * slab,
            # run_simulation leaves u and u_next device-newer; the reads of
            # both pull exactly those two slabs (phi and D never change)
            "d2h_bytes_per_step": 2 * slab + 40 * len(res.diagnostics),
            "workload": f"one run_simulation call on a host grid (pinned slabs): the [0,{n})^3 box of the bench "
                        f"geometry{' (the whole bench box)' if n == args.n else ' (crop: host RAM)'}, "
                        f"{args.e2e_steps} steps per call (one call = one e2e step); device mirror build, "
                        f"uploads, stepper build, steps and downloads all timed",
            "active_nodes": active, "seconds": secs, "box": n}


def _layer_chunks(pd, geom, centers, radii):
    from paper_2304_11165_b200 import shard

    class _P:
        def arrays(self):
            return centers, radii
    chunks, active, _ = shard.layer_work(geom, _P())
    return int(active.sum()), int(chunks.sum())


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    headers compiled in place) through reference_rate(), the same protocol as
    the cpu_baseline leg. Imports nothing from paper_2304_11165_b200."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per = max(0.5, args.cpu_seconds / max(1, args.steps))
    edge = args.cpu_sample
    thr = args.ref_threads or None
    if args.warmup > 0:
        reference_rate(args, edge, 1, 0.2, threads=thr, warm=False)
    value, secs, st, active, cores = reference_rate(args, edge, args.steps, per, threads=thr)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GPts/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(secs) / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, world),
        "cpu_baseline": {"value": value, "unit": "GPts/s", "cores": cores, "kind": "reference",
                         "sample": f"reference_rate(): each step = one reference run_simulation call (oracle/_ref, "
                                   f"{cores} std::thread workers of {host_cores()} host cores) of {st} FTCS steps "
                                   f"on the [0,{edge})^3 crop ({active} active nodes) of the same geometry"},
        "e2e": {"value": value, "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: re-execute this command under
    torch.distributed.run with N ranks on 127.0.0.1 and pass its output and
    exit code through."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
