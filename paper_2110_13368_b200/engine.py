"""The engine loop around the hot path (the reference's
core/engine.cpp is absent from the snapshot, CMakeLists.txt:11).

Three-tier clock: dt_diff < dt_mech < dt_cell with integral ratios
(config.cpp:237-244; default 10 diffusion steps per mechanics step and 60
mechanics steps per cell step). Time is counted in integer diffusion steps
(t_now = steps * dt_diff). Each mechanics interval is ONE
device call — ``Session.advance(per_mech, dt)``, CUDA-graph replayed — so
the field stays in HBM for the whole run and the host only wakes up for the
hooks (no-ops by default) and for snapshots.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Callable, Optional

import paper_2110_13368_b200 as B


def _ratio(a: float, b: float, what: str) -> int:
    """Positive integral a/b (config.cpp:237-244) or ConfigError."""
    if not (a > 0 and b > 0):
        raise B.ConfigError(f"{what}: step sizes must be positive")
    r = a / b
    n = int(round(r))
    if n < 1 or abs(r - n) > 1e-9 * max(1.0, r):
        raise B.ConfigError(f"{what}: ratio {r} is not a positive integer")
    return n


@dataclass
class SimulationClock:
    dt_diff: float = 0.01
    dt_mech: float = 0.1
    dt_cell: float = 6.0
    t_max: float = 60.0
    diffusion_steps: int = 0
    mechanics_steps: int = 0
    cell_steps: int = 0

    def __post_init__(self):
        self.per_mech = _ratio(self.dt_mech, self.dt_diff, "dt_mech / dt_diff")
        self.per_cell = _ratio(self.dt_cell, self.dt_mech, "dt_cell / dt_mech")
        if self.t_max < 0:
            raise B.ConfigError("max_time must be non-negative")
        x = self.t_max / self.dt_diff
        self.total_steps = int(round(x)) if abs(x - round(x)) <= 1e-9 * max(1.0, x) else int(math.ceil(x))

    @property
    def t_now(self) -> float:
        return self.diffusion_steps * self.dt_diff  # integer step counting


@dataclass
class RunMetrics:
    wall_seconds: float = 0.0
    diffusion_seconds: float = 0.0  # device time of [diffuse_decay_step; cell_sources_sinks_step] steps
    hook_seconds: float = 0.0
    snapshot_seconds: float = 0.0
    diffusion_steps: int = 0
    mechanics_steps: int = 0
    cell_steps: int = 0
    snapshots: int = 0

    def as_lines(self):
        """key=value metric lines."""
        return [f"{k}={v}" for k, v in self.__dict__.items()]


def run_simulation(session: B.Session, clock: SimulationClock, with_sources: bool = True,
                   mech_hook: Optional[Callable] = None, cell_hook: Optional[Callable] = None,
                   snapshot_interval: float = 0.0, snapshot_hook: Optional[Callable] = None) -> RunMetrics:
    """for each mechanics step: per_mech x [diffuse_decay_step; cell_sources_sinks_step];
    every per_cell mechanics steps: cell hook; stop at t_max."""
    m = RunMetrics()
    t0 = time.perf_counter()
    snap_every = int(round(snapshot_interval / clock.dt_diff)) if snapshot_interval and snapshot_interval > 0 else 0
    next_snap = snap_every if snap_every else None
    while clock.diffusion_steps < clock.total_steps:
        n = min(clock.per_mech, clock.total_steps - clock.diffusion_steps)
        if next_snap is not None:
            n = min(n, next_snap - clock.diffusion_steps)
        session.event_record(14)
        session.advance(n, clock.dt_diff, with_sources)
        session.event_record(15)
        m.diffusion_seconds += session.event_elapsed(14, 15) / 1e3
        clock.diffusion_steps += n
        if next_snap is not None and clock.diffusion_steps == next_snap:
            ts = time.perf_counter()
            if snapshot_hook:
                snapshot_hook(clock.t_now, session.download_field())
            m.snapshots += 1
            m.snapshot_seconds += time.perf_counter() - ts
            next_snap += snap_every
        if clock.diffusion_steps % clock.per_mech == 0:
            clock.mechanics_steps += 1
            th = time.perf_counter()
            if mech_hook:
                mech_hook(clock)
            if clock.mechanics_steps % clock.per_cell == 0:
                clock.cell_steps += 1
                if cell_hook:
                    cell_hook(clock)
            m.hook_seconds += time.perf_counter() - th
    session.synchronize()
    m.wall_seconds = time.perf_counter() - t0
    m.diffusion_steps, m.mechanics_steps, m.cell_steps = clock.diffusion_steps, clock.mechanics_steps, clock.cell_steps
    return m
