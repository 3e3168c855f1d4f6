"""Ensembles of independent replicas (C5: parameter sweeps / ABC).

All replicas of a batch share the mesh, substrate count and dt; each has its
own diffusion/decay coefficients, Dirichlet entries and agents. They live in
one session, stacked replica-major, so each sweep is ONE kernel launch over
every replica. Across GPUs the replicas are sharded with no communication.
"""
from __future__ import annotations

import numpy as np

import paper_2110_13368_b200 as B


def ensemble_session(ws, device: int = 0) -> B.Session:
    """One session holding every Workload of `ws` (same mesh, S and dt)."""
    w0 = ws[0]
    for w in ws:
        if w.n != w0.n or w.S != w0.S or w.dt != w0.dt or w.dx != w0.dx:
            raise ValueError("ensemble replicas must share mesh, substrate count and dt")
    R = len(ws)
    mesh = B.mesh_from_bounds(*w0.bounds(), w0.dx, w0.dx, w0.dx)
    s = B.Session(mesh, w0.S, device, replicas=R)
    s.ensemble_set_substrates(np.stack([w.diffusion for w in ws]), np.stack([w.decay for w in ws]), w0.dt)
    nvox = w0.voxels
    vs, ms, xs = [], [], []
    for r, w in enumerate(ws):
        if w.boundary_clamp()[0].any() or w.interior_dirichlet is not None:
            v, m, x = w.dirichlet_entries()
            vs.append(v + r * nvox)
            ms.append(m)
            xs.append(x)
    if vs:
        s.set_dirichlet(np.concatenate(vs), np.concatenate(ms), np.concatenate(xs))
    if any(w.n_agents for w in ws):
        rep = np.concatenate([np.full(w.n_agents, r, np.int32) for r, w in enumerate(ws)])
        cat = lambda f: np.concatenate([getattr(w, f).reshape(w.n_agents, -1) for w in ws])  # noqa: E731
        s.ensemble_set_agents(rep, np.concatenate([w.agent_ids for w in ws]), cat("agent_pos"),
                              np.concatenate([w.agent_vol for w in ws]), cat("agent_sec"), cat("agent_upt"),
                              cat("agent_sat"))
    s.upload_field(np.concatenate([w.initial_field() for w in ws]))
    return s


def shard(total: int, nranks: int, rank: int):
    """Contiguous replica range of this rank."""
    lo = total * rank // nranks
    hi = total * (rank + 1) // nranks
    return lo, hi
