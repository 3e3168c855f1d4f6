"""Synthetic inputs for the BASELINE.json configurations.

Everything is seeded and built programmatically, mirroring the reference's
own builders: boundary Dirichlet clamps as build_microenvironment does
(config.cpp:506-525: every boundary voxel, masked substrates) and agents as
build_agents does (config.cpp:529-566: ids 0..N-1, volume 2494 um^3 by
default, config.hpp:32). Positions come from numpy's PCG64 (not mt19937_64):
both the GPU arm and the CPU reference receive the same arrays, so parity
does not depend on the generator.

Substrates: s0 oxygen D=1e5 um^2/min, lambda=0.1/min, IC 38,
Dirichlet 38 on the boundary; s1 immunostimulatory factor D=1e3,
lambda=0.016, IC 0; s2 D=1e4, lambda=0.01; s3 D=1e2, lambda=1e-3 (s2/s3 are
builder choices recorded here). dx=dy=dz=20 um, domain [-10n, 10n]^3,
dt=0.01 min.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

SUBSTRATES = [
    # name, D, lambda, initial condition, boundary Dirichlet value (None = free)
    ("oxygen", 1.0e5, 0.1, 38.0, 38.0),
    ("immunostimulatory_factor", 1.0e3, 0.016, 0.0, None),
    ("s2_factor", 1.0e4, 0.01, 0.0, None),
    ("s3_factor", 1.0e2, 1.0e-3, 0.0, None),
]

CELL_VOLUME = 2494.0  # config.hpp:32


@dataclass
class Workload:
    name: str
    n: tuple                      # (nx, ny, nz)
    dx: float
    substrates: List[tuple]       # (name, D, lambda, ic, dirichlet|None)
    dt: float
    steps: int
    agent_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    agent_pos: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    agent_vol: np.ndarray = field(default_factory=lambda: np.zeros(0))
    agent_sec: np.ndarray = field(default_factory=lambda: np.zeros((0, 1)))
    agent_upt: np.ndarray = field(default_factory=lambda: np.zeros((0, 1)))
    agent_sat: np.ndarray = field(default_factory=lambda: np.zeros((0, 1)))
    interior_dirichlet: Optional[tuple] = None  # (voxels, mask[E,S], values[E,S])
    seed: int = 42
    replicas: int = 1

    @property
    def S(self) -> int:
        return len(self.substrates)

    @property
    def voxels(self) -> int:
        return int(self.n[0]) * int(self.n[1]) * int(self.n[2])

    @property
    def vsu_per_step(self) -> int:
        return self.voxels * self.S * self.replicas

    def bounds(self):
        nx, ny, nz = self.n
        h = self.dx
        return (-h * nx / 2, h * nx / 2, -h * ny / 2, h * ny / 2, -h * nz / 2, h * nz / 2)

    @property
    def diffusion(self):
        return np.array([s[1] for s in self.substrates])

    @property
    def decay(self):
        return np.array([s[2] for s in self.substrates])

    @property
    def initial(self):
        return np.array([s[3] for s in self.substrates])

    def initial_field(self) -> np.ndarray:
        return np.tile(self.initial, self.voxels)

    def boundary_clamp(self):
        mask = np.array([1 if s[4] is not None else 0 for s in self.substrates], np.uint8)
        vals = np.array([s[4] if s[4] is not None else 0.0 for s in self.substrates])
        return mask, vals

    def boundary_voxels(self) -> np.ndarray:
        nx, ny, nz = self.n
        k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        b = (i == 0) | (i == nx - 1) | (j == 0) | (j == ny - 1) | (k == 0) | (k == nz - 1)
        return np.flatnonzero(b.ravel()).astype(np.int64)

    def dirichlet_entries(self):
        """All entries in voxel order: boundary clamp (config.cpp:518-525) plus
        optional interior clamps, merged as DirichletMap::add would."""
        mask, vals = self.boundary_clamp()
        S = self.S
        if mask.any():
            keys = self.boundary_voxels()
            m = np.tile(mask, (keys.size, 1))
            x = np.tile(vals, (keys.size, 1))
        else:
            keys = np.zeros(0, np.int64)
            m = np.zeros((0, S), np.uint8)
            x = np.zeros((0, S))
        if self.interior_dirichlet is not None:
            iv, im, ival = self.interior_dirichlet
            allk = np.union1d(keys, iv)
            M = np.zeros((allk.size, S), np.uint8)
            X = np.zeros((allk.size, S))
            pos = np.searchsorted(allk, keys)
            M[pos] = m
            X[pos] = x
            present = np.zeros(allk.size, bool)
            present[pos] = True
            for e, v in enumerate(iv):
                p = np.searchsorted(allk, v)
                if not present[p]:  # new entry: stored as given (mesh.cpp:158)
                    M[p] = im[e]
                    X[p] = ival[e]
                    present[p] = True
                else:  # merge: later adds win per masked substrate (mesh.cpp:149-156)
                    sel = im[e].astype(bool)
                    M[p, sel] = 1
                    X[p, sel] = ival[e, sel]
            keys, m, x = allk, M, X
        return keys, m, x

    @property
    def n_agents(self) -> int:
        return int(self.agent_ids.size)


def _tumour_agents(rng, n_agents, n, dx, S, immune_fraction=0.0, dense_core_fraction=0.2):
    """Spherical tumour: uniform in a ball of radius 0.3*width plus a dense
    core (several cells per voxel, exercising the ascending-id collision
    order, agents.cpp:62-65). Tumour cells take up oxygen (U=10/min) and
    secrete the factor (S=1/min toward 1); immune cells sit in a shell and
    secrete s2/s3. Per-cell multipliers in [0.5, 1.5]."""
    width = dx * min(n)
    R = 0.3 * width
    n_immune = int(round(immune_fraction * n_agents))
    n_tumour = n_agents - n_immune
    n_core = int(dense_core_fraction * n_tumour)

    def in_ball(count, radius):
        d = rng.normal(size=(count, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True) + 1e-300
        r = radius * rng.random(count) ** (1.0 / 3.0)
        return d * r[:, None]

    pos_t = in_ball(n_tumour - n_core, R)
    core_r = max(dx * 1.5, R * 0.08)
    pos_c = in_ball(n_core, core_r)
    d = rng.normal(size=(n_immune, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True) + 1e-300
    pos_i = d * (R * (1.05 + 0.25 * rng.random(n_immune)))[:, None]
    pos = np.concatenate([pos_t, pos_c, pos_i]).reshape(-1, 3)
    half = np.array([dx * n[0] / 2, dx * n[1] / 2, dx * n[2] / 2])
    pos = np.clip(pos, -half, half)

    sec = np.zeros((n_agents, S))
    upt = np.zeros((n_agents, S))
    sat = np.zeros((n_agents, S))
    mult = 0.5 + rng.random((n_agents, S))
    nt = n_tumour
    upt[:nt, 0] = 10.0 * mult[:nt, 0]
    if S > 1:
        sec[:nt, 1] = 1.0 * mult[:nt, 1]
        sat[:nt, 1] = 1.0
    if n_immune:
        upt[nt:, 0] = 2.0 * mult[nt:, 0]
        for s in range(2, S):
            sec[nt:, s] = 0.5 * mult[nt:, s]
            sat[nt:, s] = 2.0
        if S > 1:
            upt[nt:, 1] = 0.1 * mult[nt:, 1]
    # Shuffle ids so that colliding agents are not id-sorted by construction.
    ids = rng.permutation(n_agents).astype(np.int64)
    vol = CELL_VOLUME * (0.8 + 0.4 * rng.random(n_agents))
    return ids, pos, vol, sec, upt, sat


def make(name: str, n, S: int, n_agents: int, steps: int, seed: int = 42, immune_fraction: float = 0.0,
         dx: float = 20.0, dt: float = 0.01, interior_clamps: int = 0) -> Workload:
    if isinstance(n, int):
        n = (n, n, n)
    rng = np.random.default_rng(seed)
    w = Workload(name=name, n=tuple(n), dx=dx, substrates=SUBSTRATES[:S] if S <= 4 else
                 SUBSTRATES + [(f"s{s}", 1e3 * (1 + s), 0.01 * s, 0.0, None) for s in range(4, S)],
                 dt=dt, steps=steps, seed=seed)
    if n_agents:
        (w.agent_ids, w.agent_pos, w.agent_vol, w.agent_sec, w.agent_upt,
         w.agent_sat) = _tumour_agents(rng, n_agents, w.n, dx, S, immune_fraction)
    else:
        w.agent_sec = np.zeros((0, S))
        w.agent_upt = np.zeros((0, S))
        w.agent_sat = np.zeros((0, S))
    if interior_clamps:
        vox = rng.choice(w.voxels, size=interior_clamps, replace=False).astype(np.int64)
        m = (rng.random((interior_clamps, S)) < 0.6).astype(np.uint8)
        m[:, 0] |= 1
        vals = 50.0 * rng.random((interior_clamps, S))
        w.interior_dirichlet = (vox, m, vals)
    return w


# BASELINE.json configs (SURVEY.md §8 "Sizes").
def c1(steps=36000):
    return make("C1: 50^3 x 1 substrate (oxygen), 1k cells", 50, 1, 1000, steps)


def c2(steps=36000):
    return make("C2: 100^3 x 2 substrates, 10k cells, cancer-immune layout", 100, 2, 10000, steps,
                immune_fraction=0.1)


def c3(steps=200):
    return make("C3: 256^3 x 4 substrates, 100k cells, spherical tumour", 256, 4, 100000, steps,
                immune_fraction=0.1)


def c4(steps=20):
    return make("C4: 1024^3 x 4 substrates, 1M cells", 1024, 4, 1000000, steps, immune_fraction=0.1)


def c4_sample(w: Workload, planes: int = 64) -> Workload:
    """A bounded CPU sample of C4 (the reference cannot time 1024^3 x 4 in a
    few minutes): the central `planes` z-planes of the same grid — 1024-point
    x and y lines, the same substrates — with C4's cells in those planes.
    Bounds stay centred, so the planes and cell positions are C4's own."""
    nx, ny, nz = w.n
    smp = Workload(name=f"C4 sample: central {planes} of {nz} planes ({nx}x{ny}x{planes} x {w.S}), "
                        f"C4's cells in them", n=(nx, ny, planes), dx=w.dx, substrates=list(w.substrates),
                   dt=w.dt, steps=w.steps, seed=w.seed)
    half = w.dx * planes / 2
    sel = np.abs(w.agent_pos[:, 2]) < half
    smp.agent_ids, smp.agent_pos, smp.agent_vol = w.agent_ids[sel], w.agent_pos[sel], w.agent_vol[sel]
    smp.agent_sec, smp.agent_upt, smp.agent_sat = w.agent_sec[sel], w.agent_upt[sel], w.agent_sat[sel]
    return smp


def c5_replica(r: int, steps=100):
    """One replica of C5 (512 x 64^3 x 2): seeded per-replica D/lambda (+-50%) and layout."""
    w = make(f"C5 replica {r}: 64^3 x 2, 1k cells", 64, 2, 1000, steps, seed=1000 + r)
    rng = np.random.default_rng(5000 + r)
    f = 0.5 + rng.random((2, 2))
    w.substrates = [(nm, D * f[0, i], lam * f[1, i], ic, dv) for i, (nm, D, lam, ic, dv) in enumerate(w.substrates)]
    return w


C5_REPLICAS = 512


def c5(steps=200):
    """C5 as a whole: replica 0 stands for the batch (vsu counts all 512)."""
    w = c5_replica(0, steps)
    w.name = f"C5: ensemble of {C5_REPLICAS} x (64^3 x 2 substrates, 1k cells), per-replica D/lambda and layouts"
    w.replicas = C5_REPLICAS
    return w


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def session_for(w: Workload, device: int = 0):
    """Sets a Workload up through the C ABI exactly as a reference caller
    would: mesh (from_bounds), SolverWorkspaces::build, DirichletMap,
    AgentPopulation, initial field."""
    import paper_2110_13368_b200 as B
    mesh = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    s = B.Session(mesh, w.S, device)
    s.set_substrates(w.diffusion, w.decay, w.dt)
    big = w.voxels * w.S > (1 << 27)  # C4: no whole-grid host arrays (34 GB field, 8 GB index grids)
    if w.boundary_clamp()[0].any() or w.interior_dirichlet is not None:
        if big:
            from paper_2110_13368_b200.zslab import slab_dirichlet
            v, m, x = slab_dirichlet(w, 0, w.n[2])  # the same entries, generated plane by plane
        else:
            v, m, x = w.dirichlet_entries()
        s.set_dirichlet(v, m, x)
    if w.n_agents:
        s.set_agents(w.agent_ids, w.agent_pos, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat)
    if big:
        s.fill_field(w.initial)  # the uniform initial condition, set on the device
    else:
        s.upload_field(w.initial_field())
    return s
