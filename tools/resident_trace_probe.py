"""Phase trace of the resident small-grid kernel (design tool, not the bench).

    python tools/resident_trace_probe.py [--workload c1|c2] [--steps 20]

Runs one advance() with BIODIFF_RES_TRACE set: lane 0 of every tile stamps
the global timer when the tile starts, when its dependency wait ends and when
its chain / stores are done (steps 0-7). Prints, per step and axis, the
phase span, the mean wait and the mean work time of a tile.
"""
import argparse
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c1")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    path = os.path.join(tempfile.gettempdir(), "res_trace.bin")
    os.environ["BIODIFF_RES_TRACE"] = path
    from paper_2110_13368_b200 import workloads as W
    w = W.CONFIGS[args.workload](args.steps)
    s = W.session_for(w)
    s.advance(args.steps, w.dt)
    s.synchronize()
    s.close()
    raw = np.fromfile(path, dtype=np.int64)
    max_tiles, grid, block, smem = raw[:4]
    if max_tiles == -1:  # one-cluster kernel: [step][cta][8 phase stamps]
        tr = raw[4:].view(np.uint64).reshape(8, grid, 12).astype(np.float64)
        t0 = tr[tr > 0].min()
        names = ["x", "y", "store+sync", "z", "sync", "load", "events"]
        print(f"one-cluster kernel: {grid} CTAs x {block} threads, {smem} B smem")
        for st in range(min(8, args.steps)):
            v = tr[st]
            spans = [(v[:, i + 1] - v[:, i]) / 1e3 for i in range(7)]
            print(f"step {st}: start {(v[:, 0].min() - t0) / 1e3:8.2f} us, " + ", ".join(
                f"{n} {sp.mean():5.2f}/{sp.max():5.2f}" for n, sp in zip(names, spans)) + "  (mean/max over CTAs, us)")
            sub = [("store", 2, 8), ("sync1", 8, 3)]
            print("        " + ", ".join(f"{n} {((v[:, b] - v[:, a]) / 1e3).mean():5.2f}/{((v[:, b] - v[:, a]) / 1e3).max():5.2f}"
                                    for n, a, b in sub))
        return
    tr = raw[4:].view(np.uint64).reshape(8, 4, max_tiles, 6).astype(np.float64)
    print(f"grid {grid} x {block} threads, {smem} B smem, {max_tiles} tiles max")
    t0 = tr[tr > 0].min()
    for st in range(min(8, args.steps)):
        for ax in range(4):
            v = tr[st, ax]
            v = v[v[:, 0] > 0]
            if not len(v):
                continue
            wait = (v[:, 1] - v[:, 0]) / 1e3
            work = (v[:, 2] - v[:, 1]) / 1e3
            print(f"step {st} phase {'xyzs'[ax]}: {len(v):4d} tiles, start {(v[:, 0].min() - t0) / 1e3:8.2f}"
                  f"..{(v[:, 0].max() - t0) / 1e3:8.2f} us, end {(v[:, 2].max() - t0) / 1e3:8.2f} us, "
                  f"wait mean {wait.mean():6.2f} max {wait.max():6.2f}, work mean {work.mean():6.2f} "
                  f"max {work.max():6.2f} us")
            ok = v[:, 3] > 0
            if ok.any():
                u = v[ok]
                print(f"      issue {((u[:, 3] - u[:, 1]) / 1e3).mean():6.2f}  fwd {((u[:, 4] - u[:, 3]) / 1e3).mean():6.2f}"
                      f"  bwd {((u[:, 5] - u[:, 4]) / 1e3).mean():6.2f}  tail {((u[:, 2] - u[:, 5]) / 1e3).mean():6.2f} us")


if __name__ == "__main__":
    main()
