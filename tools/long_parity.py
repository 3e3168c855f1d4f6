"""Full-length parity against the REFERENCE ITSELF (oracle/_ref, all host
threads) on BASELINE.json's configs: C1 and C2 for their full 360 simulated
minutes (36,000 steps), C3 for 1000 steps. The GPU runs through the C ABI
(graph-replayed advance), the reference through its own WorkerPool step loop
(SPEC.md:297); the fields are compared bit for bit and at north_star's
relative 1e-10. Test/verification tool (runs the reference): not the product
path.

    python tools/long_parity.py [--configs c1 c2 c3] [--out profiles/r01_long_parity.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

STEPS = {"c1": 36000, "c2": 36000, "c3": 1000}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["c1", "c2", "c3"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import numpy as np
    import oracle
    from paper_2110_13368_b200 import workloads as W
    results = {}
    for cfg in args.configs:
        steps = STEPS[cfg]
        w = W.CONFIGS[cfg](steps)
        s = W.session_for(w)
        t0 = time.perf_counter()
        s.advance(steps, w.dt, with_sources=True)
        got = s.download_field()
        gpu_s = time.perf_counter() - t0
        s.close()
        ref = oracle.Reference(w, workers=oracle.nproc())
        ref_s = ref.run(steps)
        want = ref.field()
        ref.close()
        same = int(np.count_nonzero(got.view(np.int64) != want.view(np.int64)))
        mag = np.maximum(np.abs(got), np.abs(want))
        rel = float(np.max(np.where(mag > 0, np.abs(got - want) / np.where(mag > 0, mag, 1), 0)))
        results[cfg] = {"workload": w.name, "steps": steps, "sim_minutes": steps * w.dt, "values": int(got.size),
                        "differing_values": same, "bitwise_equal": same == 0, "max_rel_diff": rel,
                        "north_star_1e-10": rel <= 1e-10, "gpu_wall_s": gpu_s, "reference_wall_s": ref_s,
                        "reference_threads": oracle.nproc(), "field_sum": float(got.sum())}
        print(json.dumps({cfg: results[cfg]}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
