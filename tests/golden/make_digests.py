"""Generates tests/golden/digests.json from the REFERENCE ITSELF.

The full-length and full-size parity cases are too large to commit as
fields, so this stores the SHA-256 of the reference's final field
(little-endian float64 bytes, oracle.field_sha256) plus a few summary numbers
for diagnostics. tests/test_long_parity_gpu.py runs the same workloads
through the CUDA library and compares digests (bit equality):

* c1 / c2: BASELINE.json configs[0] / [1] for their whole 360 simulated
  minutes (36,000 steps);
* c3: configs[2] for 1000 steps;
* c4: configs[3] (1024^3 x 4, 1M cells) for 2 steps on one domain — the
  north_star's "same grid, cells and step count" at C4's size (the reference
  field is built directly, ref_shim.cpp ref_create, not staged);
* c5_rNNN: 8 replicas of configs[4]'s 512-replica stack (each run alone by
  the reference; the GPU runs the whole stack);
* spec511: SPEC.md acceptance criterion 2 (64^3, 2 substrates, 25 agents,
  1000 steps).

Run where /root/reference exists (oracle/_ref is built from it):

    python tests/golden/make_digests.py [--only c1 c4 ...] [--workers N]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2110_13368_b200 import workloads as W  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "digests.json")

C5_SAMPLE = [0, 73, 146, 219, 292, 365, 438, 511]
C5_STEPS = 50


def spec511():
    return W.make("spec511: 64^3 x 2 substrates, 25 agents (SPEC.md acceptance 2)", 64, 2, 25, 1000, seed=511)


def cases():
    """name -> (workload factory, steps). Factories keep big workloads lazy."""
    c = {
        "c1": (lambda: W.c1(36000), 36000),
        "c2": (lambda: W.c2(36000), 36000),
        "c3": (lambda: W.c3(1000), 1000),
        "c4": (lambda: W.c4(2), 2),
        "spec511": (spec511, 1000),
    }
    for r in C5_SAMPLE:
        c[f"c5_r{r:03d}"] = ((lambda r=r: W.c5_replica(r, C5_STEPS)), C5_STEPS)
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    ap.add_argument("--workers", type=int, default=oracle.nproc())
    args = ap.parse_args()
    oracle.build(quiet=True)
    table = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            table = json.load(f)
    for name, (make, steps) in cases().items():
        if args.only and name not in args.only:
            continue
        w = make()
        t0 = time.perf_counter()
        ref = oracle.Reference(w, workers=args.workers)
        secs = ref.run(steps)
        digest = ref.field_digest()
        # a few values for diagnostics when a digest differs
        import numpy as np
        probe = np.empty(4)
        idx = [0, ref.count // 3, ref.count // 2, ref.count - 1]
        vals = []
        for i in idx:
            ref.field_range(i, 1, probe)
            vals.append(float(probe[0]))
        ref.close()
        table[name] = {"workload": w.name, "shape": list(w.n), "S": w.S, "agents": int(w.n_agents),
                       "steps": steps, "sha256": digest, "probe_index": idx, "probe_values": vals,
                       "reference_threads": args.workers, "reference_step_loop_s": round(secs, 3)}
        print(f"{name}: {digest} ({time.perf_counter() - t0:.1f} s)", flush=True)
        with open(OUT, "w") as f:
            json.dump(table, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
