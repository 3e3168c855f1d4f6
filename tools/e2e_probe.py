"""Where the coupled-loop e2e step spends its time (design tool).

    python tools/e2e_probe.py [--workload c3] [--steps 20]

Host wall time of each call of the bench's e2e loop (set_agent_positions,
rebuild_voxel_grouping, advance(1), sample_agent_densities), averaged.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2110_13368_b200 import workloads as W
    w = W.CONFIGS[args.workload](args.steps)
    s = W.session_for(w)
    pos = torch.from_numpy(np.ascontiguousarray(w.agent_pos).reshape(-1)).pin_memory().numpy()
    sense = torch.empty(s.agent_count() * s.S, dtype=torch.float64).pin_memory().numpy()
    s.advance(3, w.dt)
    s.prepare_advance(1, w.dt)
    s.synchronize()
    t = {"set_positions": 0.0, "rebuild": 0.0, "advance": 0.0, "sample": 0.0}
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a = time.perf_counter()
        s.set_agent_positions(pos)
        b = time.perf_counter()
        s.rebuild_voxel_grouping()
        c = time.perf_counter()
        s.advance(1, w.dt)
        d = time.perf_counter()
        s.sample_agent_densities(sense)
        e = time.perf_counter()
        t["set_positions"] += b - a
        t["rebuild"] += c - b
        t["advance"] += d - c
        t["sample"] += e - d
    total = time.perf_counter() - t0
    out = {k: round(1e6 * v / args.steps, 1) for k, v in t.items()}
    out["total_us_per_step"] = round(1e6 * total / args.steps, 1)
    out["workload"] = args.workload
    print(json.dumps(out))


if __name__ == "__main__":
    main()
