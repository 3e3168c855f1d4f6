"""Substrate shards and substrate x z-slab layouts.

Every part of the step is independent per substrate — the Thomas
coefficients (solver.cpp:72-95), the Dirichlet mask (solver.cpp:273) and the
reaction update (agents.cpp:103-108) — so an S-substrate problem splits into
substrate shards with no communication at all, each bit-identical to its
columns of the unsharded run. A shard can also be a z-slab, which gives a
2-D layout: ``k`` substrate shards x ``P`` z-slabs on k*P GPUs. Only the
slabs of one substrate shard exchange interface planes (csrc/slab.cu), so at
8 GPUs a 4 x 2 layout has one slab interface per chain instead of seven.

* ``shard_session`` — one shard (GLOBAL inputs, see include/biodiff_b200.h).
* ``ShardGroup``  — a whole layout in this process (one or several GPUs),
  used to check the layouts against the single-domain solve on one GPU.
* ``ShardRank``   — this process's shard of a layout over torchrun ranks;
  the slabs of a substrate shard share one NCCL communicator.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import numpy as np

import paper_2110_13368_b200 as B
from paper_2110_13368_b200.zslab import slab_dirichlet, split_planes


def split_substrates(S: int, parts: int) -> List[Tuple[int, int]]:
    """Contiguous, as-even-as-possible substrate ranges [(s0, s1), ...]."""
    if parts < 1 or parts > S:
        raise ValueError(f"cannot split {S} substrates into {parts} shards")
    edges = [round(p * S / parts) for p in range(parts + 1)]
    return [(edges[p], edges[p + 1]) for p in range(parts)]


def layout_for(world: int, S: int, nz: int, substrate_parts: Optional[int] = None) -> Tuple[int, int]:
    """(substrate shards k, z-slabs P) with k * P == world. Default: as many
    substrate shards as divide both S and world (no communication), the rest
    as z-slabs; BIODIFF_SUBSTRATE_SHARDS (or substrate_parts) overrides."""
    import os
    if substrate_parts is None and os.environ.get("BIODIFF_SUBSTRATE_SHARDS"):
        substrate_parts = int(os.environ["BIODIFF_SUBSTRATE_SHARDS"])
    if substrate_parts is None:
        substrate_parts = max(k for k in range(1, min(S, world) + 1) if S % k == 0 and world % k == 0)
    if world % substrate_parts or substrate_parts > S:
        raise ValueError(f"{substrate_parts} substrate shards do not divide {world} ranks / {S} substrates")
    P = world // substrate_parts
    if P > nz:
        raise ValueError(f"{P} z-slabs for {nz} planes")
    return substrate_parts, P


def rank_piece(rank: int, world: int, S: int, nz: int, substrate_parts: Optional[int] = None):
    """This rank's (substrate range, z range, slab index, slab count, shard index)."""
    k, P = layout_for(world, S, nz, substrate_parts)
    shard, slab = divmod(rank, P)
    return split_substrates(S, k)[shard], split_planes(nz, P)[slab], slab, P, shard


def shard_session(w, s_range, z_range=None, device: int = 0) -> B.Session:
    """A session for substrates s_range (and planes z_range) of workload `w`,
    set up from the GLOBAL inputs exactly as an unsharded caller would."""
    mesh = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    z0, z1 = z_range if z_range is not None else (0, w.n[2])
    s = B.Session(mesh, w.S, device, zslab=(z0, z1), shard=tuple(s_range))
    s.set_substrates(w.diffusion, w.decay, w.dt)
    v, m, x = slab_dirichlet(w, z0, z1)  # the global entries of these planes, built plane by plane
    if v.size:
        s.set_dirichlet(v, m, x)
    if w.n_agents:
        s.set_agents(w.agent_ids, w.agent_pos, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat)
    s.fill_field(w.initial)
    return s


class ShardGroup:
    """A k x P layout in this process; `devices` maps piece index
    (shard * P + slab) -> CUDA device (default all on 0)."""

    def __init__(self, w, substrate_parts: int, z_parts: int = 1, devices=None):
        self.w = w
        self.s_ranges = split_substrates(w.S, substrate_parts)
        self.z_ranges = split_planes(w.n[2], z_parts)
        n = substrate_parts * z_parts
        devices = devices or [0] * n
        self.pieces = []  # [shard][slab] sessions
        for a, sr in enumerate(self.s_ranges):
            row = []
            for b, zr in enumerate(self.z_ranges):
                zr_arg = zr if z_parts > 1 else None
                row.append(shard_session(w, sr, zr_arg, devices[a * z_parts + b]))
            if z_parts > 1:
                B.Session.link_local(row)
            self.pieces.append(row)

    @property
    def sessions(self):
        return [s for row in self.pieces for s in row]

    def advance(self, steps: int, with_sources: bool = True):
        for row in self.pieces:  # the substrate shards never communicate
            if len(row) > 1:
                B.Session.group_advance(row, steps, self.w.dt, with_sources)
            else:
                row[0].advance(steps, self.w.dt, with_sources)
        for s in self.sessions:
            s.synchronize()

    def upload_field(self, field: np.ndarray):
        for s in self.sessions:
            s.upload_field_global(field)

    def download_field(self) -> np.ndarray:
        out = np.empty(self.w.voxels * self.w.S)
        for s in self.sessions:
            s.download_field_global(out)
        return out

    def close(self):
        for s in self.sessions:
            s.close()


def process_group_exchange(slab_to_rank, group=None):
    """A host-transport exchange (Session.connect_host_transport) over a
    torch.distributed process group (gloo): slab peer p is global rank
    slab_to_rank(p). Sends and receives of one call are posted together."""
    import torch
    import torch.distributed as dist

    def exchange(send, send_peer, recv, recv_peer):
        reqs = []
        if send is not None:
            reqs.append(dist.isend(torch.from_numpy(send), slab_to_rank(send_peer), group=group))
        if recv is not None:
            reqs.append(dist.irecv(torch.from_numpy(recv), slab_to_rank(recv_peer), group=group))
        for r in reqs:
            r.wait()
    return exchange


class ShardRank:
    """This process's piece of a k x P layout over `world` ranks. The P slabs
    of a substrate shard exchange interface planes: over NCCL
    (`unique_ids[shard]` is the NCCL unique id of that shard's slabs,
    broadcast by the caller, e.g. bench.py over torch.distributed), or over
    the default torch.distributed process group through host buffers
    (transport="host", e.g. gloo; several ranks may share one GPU)."""

    def __init__(self, w, rank: int, world: int, device: int, unique_ids=None, substrate_parts: Optional[int] = None,
                 transport: str = "nccl"):
        self.w = w
        (self.s_range, self.z_range, self.slab, self.P,
         self.shard) = rank_piece(rank, world, w.S, w.n[2], substrate_parts)
        self.session = shard_session(w, self.s_range, self.z_range if self.P > 1 else None, device)
        if self.P > 1:
            if transport == "nccl":
                self.session.connect_nccl(unique_ids[self.shard], self.P, self.slab)
            elif transport == "host":
                base = self.shard * self.P
                self.session.connect_host_transport(self.P, self.slab, process_group_exchange(lambda p: base + p))
            else:
                raise ValueError(f"unknown transport {transport!r}")

    @property
    def values(self) -> int:
        nx, ny, _ = self.w.n
        return nx * ny * (self.z_range[1] - self.z_range[0]) * (self.s_range[1] - self.s_range[0])

    def advance(self, steps: int, with_sources: bool = True):
        self.session.advance(steps, self.w.dt, with_sources)
