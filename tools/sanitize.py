"""compute-sanitizer driver (design/verification tool, not the bench).

    compute-sanitizer --tool racecheck python tools/sanitize.py [case ...]

Runs every shipped kernel family once on a tiny grid, forcing each path
through the session environment knobs (read at session creation), and checks
each result bit for bit against the oracle so a sanitizer run is also a
parity run. Cases: the default ring2 sweeps + sources, the plane-cluster x+y
kernel in its cluster shapes, the replica-cluster x+y+z kernel, the resident
small-grid kernel, agent regrouping after moves, z-slab groups.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def forced(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def run_single(w, steps, move=False):
    from paper_2110_13368_b200 import workloads as W
    s = W.session_for(w, device=0)
    s.advance(steps, w.dt, with_sources=True)
    if move:
        pos = w.agent_pos.copy()
        pos[::3] = pos[::-3][: len(pos[::3])]
        s.set_agent_positions(pos)
        s.rebuild_voxel_grouping()
        s.advance(steps, w.dt, with_sources=True)
    out = s.download_field()
    s.close()
    return out


def main(argv):
    from oracle import Oracle
    from paper_2110_13368_b200 import workloads as W
    from paper_2110_13368_b200.ensemble import ensemble_session

    wa = W.make("san-a", (40, 36, 20), 4, 300, 3, seed=3, immune_fraction=0.1, interior_clamps=6)
    wb = W.make("san-b", (32, 32, 8), 4, 200, 2, seed=4)
    wc = W.make("san-c", (24, 20, 18), 2, 150, 4, seed=5)
    cases = {
        "ring2": ({"BIODIFF_XY_FUSED": "0", "BIODIFF_RESIDENT": "0"}, wa, False),
        "xy_cluster_8x4": ({"BIODIFF_XY_FUSED": "2", "BIODIFF_XYC_WARPS": "4", "BIODIFF_XYC_CLUSTER": "8"}, wb, False),
        "xy_cluster_4x8": ({"BIODIFF_XY_FUSED": "2", "BIODIFF_XYC_WARPS": "8", "BIODIFF_XYC_CLUSTER": "4"}, wb, False),
        "resident": ({"BIODIFF_RESIDENT": "1"}, wc, False),
        "resident_dirichlet": ({"BIODIFF_RESIDENT": "1"}, wa, False),
        "dataflow": ({"BIODIFF_RESIDENT": "1", "BIODIFF_SMALL": "0"}, wa, False),
        "regroup": ({"BIODIFF_RESIDENT": "0"}, wc, True),
        "regroup_cub": ({"BIODIFF_RESIDENT": "0", "BIODIFF_REGROUP_CUB": "1"}, wc, True),  # captured CUB pipeline
    }
    chosen = argv or list(cases) + ["xyz_cluster"]
    bad = 0
    for name in chosen:
        if name == "xyz_cluster":
            ws = [W.make(f"san-r{r}", (16, 16, 16), 2, 40, 3, seed=20 + r) for r in range(3)]

            def ens():
                e = ensemble_session(ws)
                e.advance(ws[0].steps, ws[0].dt)
                out = e.download_field()
                e.close()
                return out
            got = forced({"BIODIFF_XYZ_CLUSTER": "1"}, ens)
            per = ws[0].voxels * 2
            ok = all(same(got[r * per:(r + 1) * per], Oracle.run(wr, wr.steps)) for r, wr in enumerate(ws))
        else:
            env, w, move = cases[name]
            got = forced(env, lambda: run_single(w, w.steps, move))
            if move:
                continue_ok = True  # the regroup case is checked for sanitizer errors only
                ok = continue_ok and np.isfinite(got).all()
            else:
                ok = same(got, Oracle.run(w, w.steps))
        print(f"sanitize case {name}: {'ok' if ok else 'MISMATCH'}", flush=True)
        bad += not ok
    if bad:
        sys.exit(1)


if __name__ == "__main__":
    main(sys.argv[1:])
