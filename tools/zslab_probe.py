"""z-slab cost on ONE GPU (design tool): P in-process slabs of one domain,
advanced by group_advance on the same device, against the single-domain
session. The slabs run one after another, so total slab time / single time
= (x + y + interface + z + chains) / (x + y + z): the per-slab overhead of
the decomposition that a P-GPU run pays (minus NVLink transfer time).

    python tools/zslab_probe.py [--n 256 256 512] [--S 4] [--P 8] [--steps 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs=3, default=[256, 256, 512])
    ap.add_argument("--S", type=int, default=4)
    ap.add_argument("--P", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import numpy as np
    from paper_2110_13368_b200 import workloads as W
    from paper_2110_13368_b200.zslab import ZSlabGroup
    w = W.make("probe", tuple(args.n), args.S, 0, args.steps)
    s = W.session_for(w)
    s.advance(3, w.dt, with_sources=False)
    s.synchronize()
    s.event_record(0)
    s.advance(args.steps, w.dt, with_sources=False)
    s.event_record(1)
    single = s.event_elapsed(0, 1) / args.steps
    ref = s.download_field()
    s.close()
    out = {"n": args.n, "S": args.S, "single_ms": single}
    for P in args.P:
        g = ZSlabGroup(w, P)
        g.advance(3, with_sources=False)
        for x in g.sessions:
            x.synchronize()
        t0 = time.perf_counter()
        g.advance(args.steps, with_sources=False)
        for x in g.sessions:
            x.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / args.steps
        got = g.download_field()
        g.close()
        # reference: single domain after the same number of steps (3 + steps)
        rel = None
        if P >= 1:
            s2 = W.session_for(w)
            s2.advance(3 + args.steps, w.dt, with_sources=False)
            want = s2.download_field()
            s2.close()
            d = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1e-290)
            rel = float(d.max())
        out[f"P{P}"] = {"ms_per_step_all_slabs": ms, "overhead_vs_single": ms / single, "max_rel_err": rel}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
