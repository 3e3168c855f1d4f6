"""The engine loop around the hot path (the reference's
core/engine.cpp is absent from the snapshot, CMakeLists.txt:11).

Python view of the native engine (csrc/engine.cpp, C ABI
``biodiff_clock_make`` / ``biodiff_run_simulation``). Three-tier clock:
dt_diff < dt_mech < dt_cell with integral ratios (config.cpp:237-244; default
10 diffusion steps per mechanics step and 60 mechanics steps per cell step).
Time is counted in integer diffusion steps (t_now = steps * dt_diff,
SPEC.md:320). Each mechanics interval is ONE device call — a CUDA-graph
replay — so the field stays in HBM for the whole run and the host only wakes
up for the hooks (no-ops by default) and for snapshots.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields
from typing import Callable, Optional

import paper_2110_13368_b200 as B

_i64, _d = ctypes.c_int64, ctypes.c_double


class CClock(ctypes.Structure):  # include/biodiff_b200.h biodiff_clock
    _fields_ = [("dt_diff", _d), ("dt_mech", _d), ("dt_cell", _d), ("t_max", _d), ("per_mech", _i64),
                ("per_cell", _i64), ("total_steps", _i64), ("diffusion_steps", _i64), ("mechanics_steps", _i64),
                ("cell_steps", _i64), ("t_now", _d), ("pending", _i64)]


class CMetrics(ctypes.Structure):  # biodiff_run_metrics
    _fields_ = [("wall_seconds", _d), ("diffusion_seconds", _d), ("hook_seconds", _d), ("snapshot_seconds", _d),
                ("diffusion_steps", _i64), ("mechanics_steps", _i64), ("cell_steps", _i64), ("snapshots", _i64)]


HOOK = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(CClock))
_bound = False


def _lib():
    global _bound
    L = B.lib()
    if not _bound:
        L.biodiff_clock_make.restype = ctypes.c_int
        L.biodiff_clock_make.argtypes = [_d, _d, _d, _d, ctypes.POINTER(CClock)]
        L.biodiff_run_simulation.restype = ctypes.c_int
        L.biodiff_run_simulation.argtypes = [ctypes.c_void_p, ctypes.POINTER(CClock), ctypes.c_int32, _d, HOOK, HOOK,
                                             HOOK, ctypes.c_void_p, ctypes.POINTER(CMetrics)]
        _bound = True
    return L


@dataclass
class SimulationClock:  # SPEC.md:275-281 (validated by the native SimulationClock::make)
    dt_diff: float = 0.01
    dt_mech: float = 0.1
    dt_cell: float = 6.0
    t_max: float = 60.0
    diffusion_steps: int = 0
    mechanics_steps: int = 0
    cell_steps: int = 0
    pending: int = 0  # boundary hooks still to run on resume (1 snapshot, 2 mechanics, 4 cell)

    def __post_init__(self):
        c = CClock()
        B._check(_lib().biodiff_clock_make(self.dt_diff, self.dt_mech, self.dt_cell, self.t_max, ctypes.byref(c)))
        self.per_mech, self.per_cell, self.total_steps = int(c.per_mech), int(c.per_cell), int(c.total_steps)

    @property
    def t_now(self) -> float:
        return self.diffusion_steps * self.dt_diff  # integer step counting

    def _c(self) -> CClock:
        c = CClock()
        for f in ("dt_diff", "dt_mech", "dt_cell", "t_max", "diffusion_steps", "mechanics_steps", "cell_steps",
                  "pending"):
            setattr(c, f, getattr(self, f))
        return c

    def _sync(self, c: CClock):
        self.diffusion_steps, self.mechanics_steps, self.cell_steps = (int(c.diffusion_steps),
                                                                       int(c.mechanics_steps), int(c.cell_steps))
        self.pending = int(c.pending)


@dataclass
class RunMetrics:
    wall_seconds: float = 0.0
    diffusion_seconds: float = 0.0  # device time of the [diffuse_decay_step; cell_sources_sinks_step] replays
    hook_seconds: float = 0.0
    snapshot_seconds: float = 0.0
    diffusion_steps: int = 0
    mechanics_steps: int = 0
    cell_steps: int = 0
    snapshots: int = 0

    def as_lines(self):
        """key=value metric lines."""
        return [f"{f.name}={getattr(self, f.name)}" for f in fields(self)]


def run_simulation(session: B.Session, clock: SimulationClock, with_sources: bool = True,
                   mech_hook: Optional[Callable] = None, cell_hook: Optional[Callable] = None,
                   snapshot_interval: float = 0.0, snapshot_hook: Optional[Callable] = None) -> RunMetrics:
    """for each mechanics step: per_mech x [diffuse_decay_step; cell_sources_sinks_step];
    every per_cell mechanics steps: cell hook; snapshots every `snapshot_interval`
    simulated minutes (``snapshot_hook(t_now, field)``); stop at t_max.
    Runs in the native engine; Python hooks are called back between device calls."""
    errors = []

    def wrap(fn, snap=False):
        if fn is None:
            return HOOK()  # null: no-op in the engine

        def cb(_user, cp):
            try:
                clock._sync(cp.contents)
                if snap:
                    fn(clock.t_now, session.download_field())
                else:
                    fn(clock)
                return 0
            except BaseException as e:  # surfaced after the native call returns
                errors.append(e)
                return 1
        return HOOK(cb)

    hooks = (wrap(mech_hook), wrap(cell_hook), wrap(snapshot_hook, snap=True))
    c = clock._c()
    m = CMetrics()
    rc = _lib().biodiff_run_simulation(session._h, ctypes.byref(c), 1 if with_sources else 0,
                                       float(snapshot_interval or 0.0), hooks[0], hooks[1], hooks[2], None,
                                       ctypes.byref(m))
    clock._sync(c)
    if errors:
        raise errors[0]
    B._check(rc)
    return RunMetrics(**{f.name: getattr(m, f.name) for f in fields(RunMetrics)})
