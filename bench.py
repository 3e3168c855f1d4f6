#!/usr/bin/env python
"""Throughput of the B200-native LOD diffusion step (arxiv 2110.13368 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cN]

One "step" = one [diffuse_decay_step; cell_sources_sinks_step] pass over the
whole grid. Metric: voxel-substrate updates per second
(vsu/s, FP64) and the fraction of the measured HBM roofline.

N=1 default: BASELINE.json configs[2] (C3: 256^3 x 4 substrates, 100k
cells), the single-GPU LOD roofline benchmark the north_star targets;
configs[1] (C2, 16 MB) fits in L2 and is a parity case, not the bench line.
N>1 default (torchrun, one rank per GPU): C4 (1024^3 x 4, 1M cells), strong
scaling, in a substrate x z-slab layout (paper_2110_13368_b200/shards.py:
k substrate shards with no communication x P z-slabs exchanging interface
planes over NCCL; 8 GPUs = 4 x 2). Rank 0 also times C4 on one GPU
("scaling_vs_1gpu") and the reference on a bounded C4 sample, so a scaling
run carries its own evidence.

Timed region: W warm-up steps, the graphs of the timed call instantiated
(prepare_advance), then 3 repetitions of exactly K steps, each bracketed by
barrier + synchronize, CUDA events on the session stream, max over ranks;
the line reports the median repetition. Inputs are larger than L2 (C3/C4).

`--impl reference` times the reference's own CPU implementation (the
unmodified sources compiled into oracle/_ref by oracle/Makefile) on this
host's cores for the same workload (C4: the bounded sample above); under
torchrun only rank 0 runs it.
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
    """(DRAM bytes per launch, capture id) of `kernel_class` on `workload` from
    the committed ncu --set full capture summaries (profiles/ncu_traffic.json):
    a cached ncu figure, not measured by this run (ncu cannot run inside a
    timed bench)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    v = d.get(workload, {}).get(kernel_class)
    return v, d.get("_captures", {}).get(workload)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


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
    """Times the reference CPU path (oracle/_ref) on this host: all cores and one core.
    C4 is timed on its bounded sample (workloads.c4_sample)."""
    import oracle
    if not oracle.reference_available():
        return None
    from paper_2110_13368_b200 import workloads as W
    ws = W.c4_sample(w) if w.voxels > 2e8 else w
    cores = oracle.nproc()
    out = {"kind": "reference", "cores": cores, "cpu_model": cpu_model()}
    ref = oracle.Reference(ws, workers=cores)
    t1 = ref.run(1)  # warm-up step (also sizes the sample)
    n = max(1, min(int(sample_budget_s * 0.6 / max(t1, 1e-6)), 50 if max_steps is None else max_steps))
    t = ref.run(n)
    out["value"] = ws.voxels * ws.S * n / t  # one microenvironment (replica 0 for C5)
    out["sample"] = (f"{n} full steps of {ws.name.split(':')[0] if ws is w else ws.name} on {cores} threads "
                     f"(reference WorkerPool parallel({cores}))")
    ref.close()
    ser = oracle.Reference(ws, workers=0)
    t1s = ser.run(1)
    ns = max(1, min(int(sample_budget_s * 0.4 / max(t1s, 1e-6)), 10))
    ts = ser.run(ns)
    out["single_core"] = {"value": ws.voxels * ws.S * ns / ts, "cores": 1,
                          "sample": f"{ns} full steps, BackendKind::serial()"}
    ser.close()
    return out


def run_reference_arm(args, w):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from paper_2110_13368_b200 import workloads as W
    cfg = config_for(args, w, world)
    if not oracle.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbiodiff_ref.so not built"}))
        return
    # C4 (34 GB field, ~4 s per reference step on 16 threads) is timed on its
    # bounded sample; the per-vsu rate is the metric.
    ws = W.c4_sample(w) if w.voxels > 2e8 else w
    cores = oracle.nproc()
    ref = oracle.Reference(ws, workers=cores)
    t_w = ref.run(max(1, min(args.warmup, 3)))
    per = t_w / max(1, min(args.warmup, 3))
    budget = 120.0
    n = max(1, min(args.steps, int(budget / max(per, 1e-9))))
    t = ref.run(n)
    # One microenvironment per reference run: for the C5 ensemble that is
    # replica 0 (the replicas are independent; the reference runs them one by one).
    value = ws.voxels * ws.S * n / t
    what = "replica 0 of C5" if w.replicas > 1 else (ws.name if ws is not w else w.name.split(':')[0])
    sample = (f"{n} of {args.steps} requested full steps of {what} on {cores} threads "
              f"(reference WorkerPool parallel({cores}), steady_clock around the step loop)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / n, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded (paper_2110_13368_b200/workloads.py)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    ref.close()
    print(json.dumps(line), flush=True)


def config_for(args, w, world):
    return {"workload": w.name, "grid": list(w.n), "substrates": w.S, "cells": w.n_agents,
            "dt_min": w.dt, "parallelism": f"x{world}" if world > 1 else "single GPU",
            "l2": f"field {w.voxels * w.S * 8 / 1e6:.0f} MB per replica vs 126 MB L2"
                  + (" (inputs larger than L2)" if w.voxels * w.S * 8 > 126e6 else " (fits in L2)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps per repetition (default 1000 for C1-C3, 200 for C5, 20 for C4)")
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3, help="timed repetitions (the median is reported)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["c1", "c2", "c3", "c4", "c5"],
                    help="default: c3 at N=1, c4 (substrate x z-slab layout) at N>1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single-gpu-reference", action="store_true",
                    help="N>1: skip rank 0's one-GPU C4 timing (scaling_vs_1gpu)")
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
    args.reps = max(1, args.reps)
    if args.e2e_steps is None:
        args.e2e_steps = 5 if big else 20

    from paper_2110_13368_b200 import workloads as W
    w = W.CONFIGS[args.workload](args.steps)

    if args.impl == "reference":
        run_reference_arm(args, w)
        return

    dist = None
    # BIODIFF_BENCH_GLOO=1 (validation of the N>1 code path on a 1-GPU box):
    # a gloo process group, every rank on GPU local % device_count, and the
    # z-slab planes crossing through host buffers instead of NCCL (which
    # refuses two ranks on one device). Driver runs use NCCL, one GPU per rank.
    gloo = world > 1 and os.environ.get("BIODIFF_BENCH_GLOO") == "1"
    if world > 1:
        import torch
        import torch.distributed as dist
        if gloo:
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2110_13368_b200 as B

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(vals):
        if dist is None:
            return vals
        import torch
        t = torch.tensor(vals, device="cpu" if gloo else f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    device = local if world > 1 else 0
    ensemble = args.workload == "c5"
    layout = None
    if ensemble:
        # C5: this rank's share of the 512 replicas in one stacked session; no communication.
        from paper_2110_13368_b200.ensemble import ensemble_session, shard
        lo, hi = shard(W.C5_REPLICAS, world, rank)
        s = ensemble_session([W.c5_replica(r, args.steps) for r in range(lo, hi)], device=device)
        local_values = w.voxels * w.S * (hi - lo)
    elif world > 1 or big:
        # k substrate shards x P z-slabs (shards.py); slabs of a shard exchange planes over NCCL.
        from paper_2110_13368_b200.shards import ShardRank, layout_for
        k, P = layout_for(world, w.S, w.n[2])
        if gloo:
            sr = ShardRank(w, rank, world, device, transport="host")
        else:
            uids = [B.Session.nccl_unique_id() if (rank == 0 and P > 1) else None for _ in range(k)]
            if dist is not None:
                dist.broadcast_object_list(uids, src=0)
            sr = ShardRank(w, rank, world, device, uids)
        s = sr.session
        local_values = sr.values
        layout = (k, P)
    else:
        s = W.session_for(w, device=device)
        local_values = w.voxels * w.S
    field_bytes = local_values * 8
    vsu_total = w.vsu_per_step if (layout or ensemble) else w.vsu_per_step * world

    # Warm-up (also loads modules), then the timed call's graphs are instantiated.
    s.advance(args.warmup, w.dt)
    s.prepare_advance(args.steps, w.dt)
    s.synchronize()
    barrier()

    # Timed region: `reps` x exactly K steps of the production path (advance =
    # CUDA-graph replay), CUDA events on the session stream around each.
    l0 = s.launch_count()
    rep_ms = []
    with ClockSampler(device) as clk:
        for _ in range(args.reps):
            s.synchronize()
            barrier()
            s.event_record(0)
            s.advance(args.steps, w.dt)
            s.event_record(1)
            s.synchronize()
            barrier()
            rep_ms.append(s.event_elapsed(0, 1))
    launches = s.launch_count() - l0  # all reps
    rep_ms = max_over_ranks(rep_ms)
    ms = statistics.median(rep_ms)
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
    value = vsu_total * args.steps / (ms / 1e3)

    # Roofline of the dominant kernel (largest share of the timed region).
    peak, peak_src = peaks()
    sweep_classes = [c for c in ("resident", "sweep_xyz", "sweep_xy", "sweep_x", "sweep_y", "sweep_z")
                     if ktimes[c][0]]
    fused = ktimes["sweep_xy"][0] > 0
    fused3 = ktimes["sweep_xyz"][0] > 0
    # 16 B per value per sweep, 48 B/vsu per step. A fused
    # x+y launch performs two sweeps (32 B/value algorithmic); its DRAM
    # traffic (ncu, "traffic") is one read + one write — the fusion's gain.
    bytes_per_vsu_step = BYTES_PER_VSU_STEP
    dom = max(sweep_classes, key=lambda c: ktimes[c][1])
    n_l, t_l = ktimes[dom]
    avg_ms = t_l / n_l
    if dom == "resident":  # one cooperative launch runs every step of the advance() call
        alg_bytes = BYTES_PER_VSU_STEP * local_values * args.steps
    else:
        alg_bytes = BYTES_PER_VSU_SWEEP * local_values * SWEEPS_PER_LAUNCH[dom]
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    kernel_total = sum(v[1] for v in ktimes.values())
    step_achieved = bytes_per_vsu_step * vsu_total * args.steps / (ms / 1e3) / 1e9 / world

    # End to end through the public API with host buffers, every step (the
    # coupled cell/diffusion loop of PhysiCell): the step's
    # inputs — every agent's position, from pinned host memory — go up, the
    # grouping is rebuilt on the device, the step runs, and its result for the
    # cells — the densities each agent senses (sample_agent_densities) — comes
    # back to pinned host memory. The field is the simulation STATE and stays
    # resident (the paper's managed-memory point).
    import torch
    E = max(1, args.e2e_steps)
    n_ag = s.agent_count()
    e2e_ms = None
    if n_ag:
        pos_host = torch.from_numpy(np.ascontiguousarray(
            np.concatenate([W.c5_replica(r, 1).agent_pos for r in range(lo, hi)]) if ensemble else w.agent_pos
        ).reshape(-1)).pin_memory()
        sense_host = torch.empty(n_ag * s.S, dtype=torch.float64).pin_memory()
        pin_pos, pin_sense = pos_host.numpy(), sense_host.numpy()
        s.prepare_advance(1, w.dt)
        s.synchronize()
        barrier()
        s.event_record(2)
        for _ in range(E):
            s.set_agent_positions(pin_pos)
            s.rebuild_voxel_grouping()
            s.advance(1, w.dt)
            s.sample_agent_densities(pin_sense)
        s.event_record(3)
        e2e_ms = s.event_elapsed(2, 3)
    # The strict drop-in variant of the same API (the reference's in-place
    # diffuse_decay_step on a HOST field): upload the whole field, step, read
    # it all back, every step — PCIe-bound by construction. Skipped above 8 GB.
    rt_ms = None
    E2 = min(E, 5)
    if field_bytes <= 8e9:
        host_in = torch.from_numpy(np.tile(w.initial if not layout else w.initial[sr.s_range[0]:sr.s_range[1]],
                                           local_values // s.S)).pin_memory()
        host_out = torch.empty(local_values, dtype=torch.float64).pin_memory()
        hin, hout = host_in.numpy(), host_out.numpy()
        s.synchronize()
        barrier()
        s.event_record(4)
        for _ in range(E2):
            s.upload_field(hin)
            s.advance(1, w.dt)
            s.download_field(hout)
        s.event_record(5)
        rt_ms = s.event_elapsed(4, 5)
    e2e_ms, rt_ms = max_over_ranks([e2e_ms or 0.0, rt_ms or 0.0])

    # N>1: rank 0 times the same workload on ONE GPU (scaling evidence in the line).
    single = None
    if world > 1 and rank == 0 and not args.no_single_gpu_reference and not ensemble:
        try:
            one = W.session_for(w, device=device)
            one.advance(args.warmup, w.dt)
            one.prepare_advance(args.steps, w.dt)
            one.synchronize()
            one.event_record(0)
            one.advance(args.steps, w.dt)
            one.event_record(1)
            one_ms = one.event_elapsed(0, 1)
            one.close()
            single = {"value": w.vsu_per_step * args.steps / (one_ms / 1e3), "ms_per_step": one_ms / args.steps,
                      "scaling_vs_1gpu": value / (w.vsu_per_step * args.steps / (one_ms / 1e3)),
                      "note": "rank 0, same workload, one session on one GPU, same K"}
        except Exception as e:  # reported, never required
            single = {"error": str(e)}
    barrier()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_timing(w)
            if cpu is not None:
                cpu["unit"] = UNIT
        except Exception as e:  # the baseline is reported, never required
            cpu = {"error": str(e)}

    if rank == 0:
        cfg = config_for(args, w, world)
        if layout:
            k, P = layout
            cfg["parallelism"] = (f"{k} substrate shard(s) x {P} z-slab(s) = {world} GPU(s): shards need no "
                                  f"communication, slabs exchange interface planes over "
                                  f"{'host buffers (gloo validation mode)' if gloo else 'NCCL'}")
        if ensemble:
            cfg["parallelism"] = f"{W.C5_REPLICAS} replicas sharded over {world} GPU(s), no communication, " \
                                 f"one stacked session per GPU"
            cfg["l2"] = f"{W.C5_REPLICAS // world} replicas x {w.voxels * w.S * 8 / 1e6:.1f} MB per GPU"
        traffic, capture = ncu_traffic(args.workload, dom) if world == 1 else (None, None)
        h2d = (n_ag * 24) * world if n_ag else 0
        d2h = (n_ag * s.S * 8) * world if n_ag else 0
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (layout and world > 1) or (ensemble and world > 1) else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded spherical-tumour layout (paper_2110_13368_b200/workloads.py, SURVEY.md §8 d3)",
            "config": cfg,
            "timing": {"reps": args.reps, "rep_ms": rep_ms, "statistic": "median of reps (max over ranks each)",
                       "graphs": "instantiated before the timed region (prepare_advance)"},
            "roofline": {
                "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": (f"cached ncu --set full capture ({capture}), profiles/ncu_traffic.json"
                                   if traffic else None),
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
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": E,
                    "semantics": "per step through the C ABI: agent positions H2D (pinned) + device regrouping "
                                 "+ one step + densities at every agent's voxel D2H (pinned); the field "
                                 "(state) stays resident"},
            "e2e_field_roundtrip": {"value": vsu_total * E2 / (rt_ms / 1e3) if rt_ms else None, "unit": UNIT,
                                    "h2d_bytes_per_step": field_bytes * world,
                                    "d2h_bytes_per_step": field_bytes * world, "steps": E2,
                                    "semantics": "per step: upload the whole field (pinned) + one step + "
                                                 "download the whole field (PCIe-bound)"},
            "gpu_launches": launches,
            "gpu_launches_per_rep": launches // args.reps,
            "clocks": clk.summary(),
        }
        if single is not None:
            line["single_gpu"] = single
        if gloo:
            line["validation_mode"] = ("BIODIFF_BENCH_GLOO=1: gloo process group, ranks sharing GPU(s), z-slab planes "
                                       "through host buffers (not a scaling measurement)")
        print(json.dumps(line), flush=True)
    s.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
