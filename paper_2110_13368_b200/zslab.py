"""z-slab domain decomposition of the LOD step.

Each slab session owns global planes [z0, z1) and takes the GLOBAL inputs
(mesh, substrates, Dirichlet entries with global voxel indices, all agents),
keeping its share. The z-sweep is a partitioned solve (see csrc/slab.cu).

* ``ZSlabGroup`` — several slabs driven by one process (one GPU or several);
  the boundary planes move by device / peer copies. Used to check the
  partitioned solve against the single-domain solve on one GPU.
* ``ZSlabRank`` — one slab per process (torchrun rank = slab index); the
  planes move with NCCL send/recv on the session stream. The NCCL unique id
  is broadcast by the caller (``bench.py`` uses torch.distributed).
"""
from __future__ import annotations

import numpy as np

import paper_2110_13368_b200 as B


def split_planes(nz: int, parts: int):
    """Contiguous, as-even-as-possible z ranges [(z0, z1), ...]."""
    if parts < 1 or parts > nz:
        raise ValueError(f"cannot split {nz} planes into {parts} slabs")
    edges = [round(p * nz / parts) for p in range(parts + 1)]
    return [(edges[p], edges[p + 1]) for p in range(parts)]


def slab_dirichlet(w, z0: int, z1: int):
    """The workload's Dirichlet entries restricted to planes [z0, z1), in global
    voxel indices, generated plane by plane (no global arrays at 1024^3)."""
    nx, ny, nz = w.n
    mask, vals = w.boundary_clamp()
    S = w.S
    keys = []
    if mask.any():
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        ring = np.flatnonzero(((i == 0) | (i == nx - 1) | (j == 0) | (j == ny - 1)).ravel()).astype(np.int64)
        full = np.arange(nx * ny, dtype=np.int64)
        for k in range(z0, z1):
            keys.append((full if k in (0, nz - 1) else ring) + k * nx * ny)
    keys = np.concatenate(keys) if keys else np.zeros(0, np.int64)
    m = np.tile(mask, (keys.size, 1))
    x = np.tile(vals, (keys.size, 1))
    if w.interior_dirichlet is not None:
        iv, im, ival = w.interior_dirichlet
        sel = (iv >= z0 * nx * ny) & (iv < z1 * nx * ny)
        if sel.any():
            # merge through the full entry list restricted to the slab
            gk, gm, gx = w.dirichlet_entries()
            s2 = (gk >= z0 * nx * ny) & (gk < z1 * nx * ny)
            return gk[s2], gm[s2], gx[s2]
    return keys, m.reshape(-1, S), x.reshape(-1, S)


def slab_session(w, z0: int, z1: int, device: int = 0) -> B.Session:
    mesh = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    s = B.Session(mesh, w.S, device, zslab=(z0, z1))
    s.set_substrates(w.diffusion, w.decay, w.dt)
    v, m, x = slab_dirichlet(w, z0, z1)
    if v.size:
        s.set_dirichlet(v, m, x)
    if w.n_agents:
        s.set_agents(w.agent_ids, w.agent_pos, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat)
    s.fill_field(w.initial)
    return s


class ZSlabGroup:
    """P slabs in this process; `devices` maps slab -> CUDA device (default all on 0)."""

    def __init__(self, w, parts: int, devices=None):
        self.w = w
        self.ranges = split_planes(w.n[2], parts)
        devices = devices or [0] * parts
        self.sessions = [slab_session(w, z0, z1, devices[p]) for p, (z0, z1) in enumerate(self.ranges)]
        B.Session.link_local(self.sessions)

    def advance(self, steps: int, with_sources: bool = True):
        B.Session.group_advance(self.sessions, steps, self.w.dt, with_sources)

    def upload_field(self, field: np.ndarray):
        nx, ny, _ = self.w.n
        per = nx * ny * self.w.S
        for s, (z0, z1) in zip(self.sessions, self.ranges):
            s.upload_field(field[z0 * per:z1 * per])

    def download_field(self) -> np.ndarray:
        return np.concatenate([s.download_field() for s in self.sessions])

    def close(self):
        for s in self.sessions:
            s.close()


class ZSlabRank:
    """This process's slab of a `nranks`-way z decomposition over NCCL."""

    def __init__(self, w, rank: int, nranks: int, device: int, unique_id: bytes):
        self.w = w
        self.rank, self.nranks = rank, nranks
        self.z0, self.z1 = split_planes(w.n[2], nranks)[rank]
        self.session = slab_session(w, self.z0, self.z1, device)
        if nranks > 1:
            self.session.connect_nccl(unique_id, nranks, rank)

    def advance(self, steps: int, with_sources: bool = True):
        self.session.advance(steps, self.w.dt, with_sources)
