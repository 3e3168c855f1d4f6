"""Per-GPU work of a substrate-shard layout (design tool, not the bench).

    python tools/shard_probe.py [--workload c4] [--steps 5]

Times one substrate shard (substrates [0, 1) of the workload, the whole
domain: what one GPU of a k = S shard layout runs) against the unsharded
session on the same GPU: ratio = shard ms x S / full ms. 1.0 means the
shard layout scales perfectly (no communication at all).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(s, w, steps):
    s.advance(3, w.dt)
    s.prepare_advance(steps, w.dt)
    s.synchronize()
    s.event_record(0)
    s.advance(steps, w.dt)
    s.event_record(1)
    s.synchronize()
    return s.event_elapsed(0, 1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--parts", type=int, default=0, help="substrate shards (default: S)")
    args = ap.parse_args()
    from paper_2110_13368_b200 import workloads as W
    from paper_2110_13368_b200.shards import shard_session, split_substrates
    w = W.CONFIGS[args.workload](args.steps)
    parts = args.parts or w.S
    out = {"workload": args.workload, "parts": parts}
    sh = shard_session(w, split_substrates(w.S, parts)[0])
    out["shard_ms"] = timed(sh, w, args.steps)
    sh.close()
    full = W.session_for(w)
    out["full_ms"] = timed(full, w, args.steps)
    full.close()
    out["per_gpu_work_ratio"] = out["shard_ms"] * parts / out["full_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
