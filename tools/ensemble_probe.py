"""Per-sweep kernel timing of a stacked ensemble (design tool, not the bench).

    python tools/ensemble_probe.py [--R 512] [--n 64] [--S 2] [--steps 50] [--env K=V ...]

C5-shaped: R replicas of n^3 x S with the boundary clamp and per-replica
coefficients, no agents. Prints achieved GB/s per kernel class at 16 B per
value per sweep (32 B for the fused x+y class).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=512)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--S", type=int, default=2)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--env", nargs="*", default=[])
    args = ap.parse_args()
    for kv in args.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    import numpy as np
    from paper_2110_13368_b200 import workloads as W
    from paper_2110_13368_b200.ensemble import ensemble_session
    ws = []
    for r in range(args.R):
        w = W.make(f"r{r}", args.n, args.S, 0, args.steps, seed=1000 + r)
        f = 0.5 + np.random.default_rng(5000 + r).random(2)
        w.substrates = [(nm, D * f[0], lam * f[1], ic, dv) for (nm, D, lam, ic, dv) in w.substrates]
        ws.append(w)
    s = ensemble_session(ws)
    w = ws[0]
    s.advance(3, w.dt, with_sources=False)
    s.synchronize()
    s.set_kernel_timing(True)
    s.event_record(0)
    s.advance(args.steps, w.dt, with_sources=False)
    s.event_record(1)
    total = s.event_elapsed(0, 1)
    t = s.kernel_times()
    values = w.voxels * w.S * args.R
    out = {"env": args.env, "R": args.R, "n": args.n, "S": args.S, "ms_per_step": total / args.steps,
           "step_GBps_48B": 48.0 * values / (total / args.steps / 1e3) / 1e9}
    for k, (cnt, ms) in t.items():
        if cnt:
            b = (16.0 if k != "sweep_xy" else 16.0) * values
            out[k] = {"us": 1e3 * ms / cnt, "GBps": b / (ms / cnt / 1e3) / 1e9 if k.startswith("sweep") else None}
    print(json.dumps(out))
    s.close()


if __name__ == "__main__":
    main()
