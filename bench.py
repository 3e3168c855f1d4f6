#!/usr/bin/env python
"""Throughput of the B200-native LOD diffusion step (arxiv 2110.13368 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]

One "step" = one [diffuse_decay_step; cell_sources_sinks_step] pass over the
whole grid. Metric: voxel-substrate updates per second
(vsu/s, FP64) and the fraction of the measured HBM roofline.

Default workload at N=1 is BASELINE.json configs[2] (C3: 256^3 x 4 substrates,
100k cells), the single-GPU LOD roofline benchmark the north_star targets;
configs[1] (C2, 16 MB) fits in L2 and is a parity case, not a bench line.
For N>1 (torchrun, one rank per GPU) each rank advances its own C3 replica
(ensemble sharding, no data-path collective; "scaling": "weak").

`--impl reference` times the reference's own CPU implementation (the
unmodified sources compiled into oracle/_ref by oracle/Makefile) on this
host's cores for the same workload; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel-substrate diffusion updates/sec (FP64) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "vsu/s"
BYTES_PER_VSU_STEP = 48  # 3 sweeps x (8 B read + 8 B write), SURVEY.md §8 d2
BYTES_PER_VSU_STEP_FUSED = 32  # DRAM bytes when x+y run fused through L2 (one read + one write) + z
BYTES_PER_VSU_STEP_XYZ = 16  # ensembles: x, y, z of a replica fused through L2 (one read + one write)
BYTES_PER_VSU_SWEEP = 16  # per value per sweep (a fused x+y launch performs two, x+y+z three)
SWEEPS_PER_LAUNCH = {"sweep_xyz": 3, "sweep_xy": 2, "sweep_x": 1, "sweep_y": 1, "sweep_z": 1}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload, kernel_class):
    """DRAM bytes per launch of `kernel_class` on `workload` from the committed
    ncu --set full summaries (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(workload, {}).get(kernel_class)


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference_timing(w, sample_budget_s=20.0, max_steps=None):
    """Times the reference CPU path (oracle/_ref) on this host: all cores and one core."""
    import oracle
    cores = oracle.nproc()
    out = {"kind": "reference" if oracle.reference_available() else "port", "cores": cores}
    if not oracle.reference_available():
        return None
    ref = oracle.Reference(w, workers=cores)
    t1 = ref.run(1)  # warm-up step (also sizes the sample)
    n = max(1, min(int(sample_budget_s * 0.6 / max(t1, 1e-6)), 50 if max_steps is None else max_steps))
    t = ref.run(n)
    out["value"] = w.voxels * w.S * n / t  # one microenvironment (replica 0 for C5)
    out["sample"] = f"{n} full steps of {w.name.split(':')[0]} on {cores} threads (reference WorkerPool parallel({cores}))"
    ref.close()
    ser = oracle.Reference(w, workers=0)
    t1s = ser.run(1)
    ns = max(1, min(int(sample_budget_s * 0.4 / max(t1s, 1e-6)), 10))
    ts = ser.run(ns)
    out["single_core"] = {"value": w.voxels * w.S * ns / ts, "cores": 1,
                          "sample": f"{ns} full steps, BackendKind::serial()"}
    ser.close()
    return out


def run_reference_arm(args, w):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    cfg = config_for(args, w, world)
    if not oracle.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbiodiff_ref.so not built"}))
        return
    cores = oracle.nproc()
    ref = oracle.Reference(w, workers=cores)
    t_w = ref.run(max(1, min(args.warmup, 3)))
    per = t_w / max(1, min(args.warmup, 3))
    budget = 120.0
    n = max(1, min(args.steps, int(budget / max(per, 1e-9))))
    t = ref.run(n)
    # One microenvironment per reference run: for the C5 ensemble that is
    # replica 0 (the replicas are independent; the reference runs them one by one).
    value = w.voxels * w.S * n / t
    what = "replica 0 of C5" if w.replicas > 1 else w.name.split(':')[0]
    sample = (f"{n} of {args.steps} requested full steps of {what} on {cores} threads "
              f"(reference WorkerPool parallel({cores}), steady_clock around the step loop)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / n, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded (paper_2110_13368_b200/workloads.py)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    ref.close()
    print(json.dumps(line), flush=True)


def config_for(args, w, world):
    return {"workload": w.name, "grid": list(w.n), "substrates": w.S, "cells": w.n_agents,
            "dt_min": w.dt, "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "l2": f"field {w.voxels * w.S * 8 / 1e6:.0f} MB per replica vs 126 MB L2"
                  + (" (inputs larger than L2)" if w.voxels * w.S * 8 > 126e6 else " (fits in L2)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 1000 for C1-C3, 20 for C4)")
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["c1", "c2", "c3", "c4", "c5"],
                    help="default: c3 at N=1, c4 (z-slab decomposition) at N>1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.workload is None:
        args.workload = "c3" if world == 1 else "c4"
    big = args.workload == "c4"
    if args.steps is None:
        args.steps = 20 if big else (200 if args.workload == "c5" else 1000)
    if args.warmup is None:
        args.warmup = 3 if big else 20
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.e2e_steps is None:
        args.e2e_steps = 1 if big else 5

    from paper_2110_13368_b200 import workloads as W
    w = W.CONFIGS[args.workload](args.steps)

    if args.impl == "reference":
        run_reference_arm(args, w)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2110_13368_b200 as B

    def barrier():
        if dist is not None:
            dist.barrier()

    device = local if world > 1 else 0
    ensemble = args.workload == "c5"
    zslab = (big or world > 1) and not ensemble
    if ensemble:
        # C5: this rank's share of the 512 replicas in one stacked session; no communication.
        from paper_2110_13368_b200.ensemble import ensemble_session, shard
        lo, hi = shard(W.C5_REPLICAS, world, rank)
        s = ensemble_session([W.c5_replica(r, args.steps) for r in range(lo, hi)], device=device)
        local_values = w.voxels * w.S * (hi - lo)
    elif zslab:
        # C4: one z-slab per rank, interface planes over NCCL (csrc/slab.cu).
        from paper_2110_13368_b200.zslab import ZSlabRank
        uid = [B.Session.nccl_unique_id() if (rank == 0 and world > 1) else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        zr = ZSlabRank(w, rank, world, device, uid[0])
        s = zr.session
        local_values = w.n[0] * w.n[1] * (zr.z1 - zr.z0) * w.S
    else:
        s = W.session_for(w, device=device)
        local_values = w.voxels * w.S
    field_bytes = local_values * 8
    vsu_total = w.vsu_per_step if (zslab or ensemble) else w.vsu_per_step * world

    # Warm-up (also instantiates graphs / loads modules).
    s.advance(args.warmup, w.dt)
    s.synchronize()
    barrier()

    # Timed region: exactly K steps of the production path (advance = CUDA-graph
    # replay), CUDA events on the session stream around it.
    l0 = s.launch_count()
    with ClockSampler(device) as clk:
        s.synchronize()
        barrier()
        s.event_record(0)
        s.advance(args.steps, w.dt)
        s.event_record(1)
        ms = s.event_elapsed(0, 1)
        s.synchronize()
        barrier()
    launches = s.launch_count() - l0
    # Per-kernel pass for the roofline: the same K steps again with a CUDA
    # event pair around every kernel (graphs off: events between kernels),
    # so the launch durations are measured, not inferred. For launch-bound
    # configs (C1, C2) this pass is slower than the graph-replayed region.
    s.set_kernel_timing(True)
    s.synchronize()
    barrier()
    s.event_record(6)
    s.advance(args.steps, w.dt)
    s.event_record(7)
    ms_kernel_pass = s.event_elapsed(6, 7)
    s.synchronize()
    barrier()
    ktimes = s.kernel_times()
    s.set_kernel_timing(False)
    if dist is not None:
        import torch
        t = torch.tensor([ms], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = vsu_total * args.steps / (ms / 1e3)

    # Roofline of the dominant kernel (largest share of the timed region).
    peak, peak_src = peaks()
    sweep_classes = [c for c in ("sweep_xyz", "sweep_xy", "sweep_x", "sweep_y", "sweep_z") if ktimes[c][0]]
    fused = ktimes["sweep_xy"][0] > 0
    fused3 = ktimes["sweep_xyz"][0] > 0
    # 16 B per value per sweep, 48 B/vsu per step. A fused
    # x+y launch performs two sweeps (32 B/value algorithmic); its DRAM
    # traffic (ncu, "traffic") is one read + one write — the fusion's gain.
    bytes_per_vsu_step = BYTES_PER_VSU_STEP
    dom = max(sweep_classes, key=lambda c: ktimes[c][1])
    n_l, t_l = ktimes[dom]
    avg_ms = t_l / n_l
    alg_bytes = BYTES_PER_VSU_SWEEP * local_values * SWEEPS_PER_LAUNCH[dom]
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    kernel_total = sum(v[1] for v in ktimes.values())
    step_achieved = bytes_per_vsu_step * vsu_total * args.steps / (ms / 1e3) / 1e9 / world

    # Host-buffer e2e legs need pinned copies of the field: skipped (null) above
    # 8 GB per rank (C4 on one GPU is 34 GB).
    e2e_ms = res_ms = None
    E = max(1, args.e2e_steps)
    if field_bytes <= 8e9:
        # End to end through the C ABI with host buffers (pinned), strict drop-in
        # semantics: every step uploads the field, steps once, reads it back.
        import torch
        host_in = torch.from_numpy(np.tile(w.initial, local_values // w.S)).pin_memory()
        host_out = torch.empty(local_values, dtype=torch.float64).pin_memory()
        hin = host_in.numpy()
        hout = host_out.numpy()
        E = max(1, args.e2e_steps)
        barrier()
        s.event_record(2)
        for _ in range(E):
            s.upload_field(hin)
            s.diffuse_decay_step()
            s.cell_sources_sinks_step(w.dt)
            s.download_field(hout)
        s.event_record(3)
        e2e_ms = s.event_elapsed(2, 3)
        # Resident run through the same API: upload once, K steps, read back once.
        barrier()
        s.event_record(4)
        s.upload_field(hin)
        s.advance(args.steps, w.dt)
        s.download_field(hout)
        s.event_record(5)
        res_ms = s.event_elapsed(4, 5)
        if dist is not None:
            t = torch.tensor([e2e_ms, res_ms], device=f"cuda:{device}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms, res_ms = (float(x) for x in t.tolist())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not big:
        try:
            cpu = cpu_reference_timing(w)
            if cpu is not None:
                cpu["unit"] = UNIT
        except Exception as e:  # the baseline is reported, never required
            cpu = {"error": str(e)}

    if rank == 0:
        cfg = config_for(args, w, world)
        if zslab:
            cfg["parallelism"] = f"z-slab x{world} (partitioned z-solve, NCCL plane exchange)" if world > 1 \
                else "single GPU (one z-slab)"
        if ensemble:
            cfg["parallelism"] = f"{W.C5_REPLICAS} replicas sharded over {world} GPU(s), no communication, " \
                                 f"one stacked session per GPU"
            cfg["l2"] = f"{W.C5_REPLICAS // world} replicas x {w.voxels * w.S * 8 / 1e6:.1f} MB per GPU"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (zslab or ensemble) else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded spherical-tumour layout (paper_2110_13368_b200/workloads.py, SURVEY.md §8 d3)",
            "config": cfg,
            "roofline": {
                "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(args.workload, dom) if not zslab else None,
                "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms, "peak_source": peak_src,
                "kernel_share_of_step": t_l / kernel_total if kernel_total else None,
                "kernel_pass_ms_per_step": ms_kernel_pass / args.steps,
                "step": {"achieved": step_achieved, "frac": step_achieved / peak,
                         "bytes_per_vsu": bytes_per_vsu_step, "note": "per GPU",
                         "xy_fused": fused, "xyz_fused": fused3,
                         "dram_bytes_per_vsu": (BYTES_PER_VSU_STEP_XYZ if fused3 else
                                                BYTES_PER_VSU_STEP_FUSED if fused else BYTES_PER_VSU_STEP)},
                "per_kernel_ms": {k: {"launches": v[0], "avg_ms": (v[1] / v[0]) if v[0] else None}
                                  for k, v in ktimes.items()},
            },
            "cpu_baseline": cpu,
            "e2e": {"value": vsu_total * E / (e2e_ms / 1e3) if e2e_ms else None, "unit": UNIT,
                    "h2d_bytes_per_step": field_bytes * world, "d2h_bytes_per_step": field_bytes * world,
                    "steps": E, "semantics": "per step: upload field (pinned host) + step + download field"},
            "e2e_resident": {"value": vsu_total * args.steps / (res_ms / 1e3) if res_ms else None, "unit": UNIT,
                             "h2d_bytes_per_step": field_bytes * world / args.steps,
                             "d2h_bytes_per_step": field_bytes * world / args.steps,
                             "semantics": "upload once, advance(K), download once"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    s.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
