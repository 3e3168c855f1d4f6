"""Per-sweep kernel timing probe (design tool, not the bench).

    python tools/sweep_probe.py [--n 256] [--S 4] [--steps 50] [--env BIODIFF_RMAX=64 ...]

Times each kernel class over `steps` diffuse_decay_steps on an n^3 x S grid
with the boundary clamp (C3-shaped, no agents) and prints achieved GB/s at
16 B per value per sweep. Variants are selected through the environment
(BIODIFF_SWEEP_PATH, BIODIFF_RMAX, BIODIFF_NO_SETTLE) before the session
is created.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs=3, default=[256, 256, 256])
    ap.add_argument("--S", type=int, default=4)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--env", nargs="*", default=[])
    args = ap.parse_args()
    for kv in args.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    from paper_2110_13368_b200 import workloads as W
    w = W.make("probe", tuple(args.n), args.S, 0, args.steps)
    s = W.session_for(w)
    s.advance(3, w.dt, with_sources=False)
    s.synchronize()
    s.set_kernel_timing(True)
    s.event_record(0)
    s.advance(args.steps, w.dt, with_sources=False)
    s.event_record(1)
    total = s.event_elapsed(0, 1)
    t = s.kernel_times()
    bytes_ = 16.0 * w.voxels * w.S
    out = {"env": args.env, "n": args.n, "S": args.S, "ms_per_step": total / args.steps}
    for k, (cnt, ms) in t.items():
        if cnt:
            out[k] = {"us": 1e3 * ms / cnt, "GBps": bytes_ / (ms / cnt / 1e3) / 1e9 if k.startswith("sweep") else None}
    print(json.dumps(out))
    s.close()


if __name__ == "__main__":
    main()
