"""Shared test plumbing: golden fixtures -> Workload, and running a Workload
through the CUDA library's C ABI (the product path) or the oracle."""
from __future__ import annotations

import glob
import os

import numpy as np

from paper_2110_13368_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    return sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    S = int(z["D"].size)
    subs = []
    for s in range(S):
        dv = float(z["boundary_values"][s]) if z["boundary_mask"][s] else None
        subs.append((f"s{s}", float(z["D"][s]), float(z["lam"][s]), float(z["ic"][s]), dv))
    w = W.Workload(name=name, n=tuple(int(x) for x in z["n"]), dx=float(z["dx"]), substrates=subs,
                   dt=float(z["dt"]), steps=int(z["steps"]))
    w.agent_ids = z["agent_ids"]
    w.agent_pos = z["agent_pos"]
    w.agent_vol = z["agent_vol"]
    w.agent_sec = z["agent_sec"].reshape(-1, S)
    w.agent_upt = z["agent_upt"].reshape(-1, S)
    w.agent_sat = z["agent_sat"].reshape(-1, S)
    if z["interior_voxels"].size:
        w.interior_dirichlet = (z["interior_voxels"], z["interior_mask"].reshape(-1, S),
                                z["interior_values"].reshape(-1, S))
    return w, z


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def first_diff(a, b):
    d = np.flatnonzero(a.view(np.int64) != b.view(np.int64))
    if d.size == 0:
        return "identical"
    i = d[0]
    return f"{d.size} differing values; first at {i}: {a[i]!r} vs {b[i]!r}"


def make_session(w, device=0):
    from paper_2110_13368_b200.workloads import session_for
    return session_for(w, device)
