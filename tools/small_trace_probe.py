"""Per-phase times of the small-field kernel (design tool).

    BIODIFF_RES_TRACE=/tmp/t.bin python tools/small_trace_probe.py c2

Runs 8 steps in one launch with per-CTA globaltimer stamps and prints, for
steps 2-7, each phase's mean and max over CTAs (µs): x, y, slab store,
barrier 1, z, barrier 2, events (+ barrier 3), slab refill."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2110_13368_b200 import workloads as W
    path = os.environ["BIODIFF_RES_TRACE"]
    w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"](8)
    s = W.session_for(w)
    s.advance(8, w.dt)
    s.synchronize()
    s.close()
    raw = np.fromfile(path, dtype=np.int64)
    hdr, t = raw[:4], raw[4:].view(np.uint64).astype(np.float64)
    C = int(hdr[1])
    t = t.reshape(8, C, 12)
    seq = [("x", 0, 1), ("y", 1, 2), ("store", 2, 8), ("barrier1", 8, 3), ("z", 3, 4), ("barrier2", 4, 5),
           ("events+barrier3", 5, 6), ("refill", 6, 7)]
    out = []
    for name, a, b in seq:
        d = (t[2:, :, b] - t[2:, :, a]) / 1e3
        out.append(f"{name} {d.mean():.2f}/{d.max():.2f}")
    step = (t[3:, :, 0] - t[2:-1, :, 0]) / 1e3
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'c2'} CTAs={C} step {step.mean():.2f} us | " + " | ".join(out))


if __name__ == "__main__":
    main()
