"""Engine loop: clock accounting on CPU, the run on GPU."""
import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.engine import SimulationClock, run_simulation
from tests.helpers import bits_equal, make_session


def test_clock_defaults_and_ratio_validation():
    c = SimulationClock(t_max=60.0)
    assert (c.total_steps, c.per_mech, c.per_cell) == (6000, 10, 60)
    assert SimulationClock(t_max=0.0).total_steps == 0
    with pytest.raises(B.ConfigError):
        SimulationClock(dt_diff=0.1, dt_mech=0.25)  # ratio 2.5
    with pytest.raises(B.ConfigError):
        SimulationClock(dt_diff=0.0)


@pytest.mark.gpu
def test_engine_step_accounting_and_result():
    """60 sim-min at the defaults: exactly 6000 / 600 / 10 steps (SPEC.md:515 criterion 7);
    the field equals 6000 plain steps."""
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("engine", (20, 18, 16), 2, 200, 6000, seed=4)
    s = make_session(w)
    mech, cell, snaps = [], [], []
    m = run_simulation(s, SimulationClock(t_max=60.0), mech_hook=lambda c: mech.append(c.diffusion_steps),
                       cell_hook=lambda c: cell.append(c.mechanics_steps), snapshot_interval=15.0,
                       snapshot_hook=lambda t, f: snaps.append(t))
    assert (m.diffusion_steps, m.mechanics_steps, m.cell_steps) == (6000, 600, 10)
    assert len(mech) == 600 and mech[0] == 10 and cell == [60 * k for k in range(1, 11)]
    assert snaps == [15.0, 30.0, 45.0, 60.0] and m.snapshots == 4
    got = s.download_field()
    ref = make_session(w)
    ref.advance(6000, w.dt)
    assert bits_equal(got, ref.download_field())
    assert m.diffusion_seconds > 0 and all(line.count("=") == 1 for line in m.as_lines())


@pytest.mark.gpu
def test_engine_zero_time_keeps_initial_condition():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("engine0", (10, 10, 10), 1, 0, 1)
    s = make_session(w)
    m = run_simulation(s, SimulationClock(t_max=0.0))
    assert m.diffusion_steps == 0
    assert np.array_equal(s.download_field(), w.initial_field())


@pytest.mark.gpu
def test_engine_snapshots_off_the_mechanics_grid_keep_the_cadence():
    """A snapshot interval that is not a multiple of dt_mech splits device
    calls but never shifts the 10:60 cadence (hooks at every 10th step)."""
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("engine2", (12, 12, 12), 1, 50, 1, seed=7)
    s = make_session(w)
    mech, snaps = [], []
    c = SimulationClock(t_max=1.2, dt_cell=0.6)
    m = run_simulation(s, c, mech_hook=lambda k: mech.append(k.diffusion_steps), snapshot_interval=0.15,
                       snapshot_hook=lambda t, f: snaps.append((round(t, 9), f.size)))
    assert mech == list(range(10, 121, 10)) and m.cell_steps == 2
    assert [t for t, _ in snaps] == [0.15, 0.3, 0.45, 0.6, 0.75, 0.9, 1.05, 1.2]
    assert all(n == w.voxels * w.S for _, n in snaps)
    ref = make_session(w)
    ref.advance(120, w.dt)
    assert bits_equal(s.download_field(), ref.download_field())


@pytest.mark.gpu
def test_engine_hook_error_stops_the_run_and_resumes():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("engine3", (10, 10, 10), 1, 0, 1)
    s = make_session(w)
    c = SimulationClock(t_max=1.0)

    def boom(k):
        if k.mechanics_steps == 4:
            raise RuntimeError("stop here")

    with pytest.raises(RuntimeError, match="stop here"):
        run_simulation(s, c, mech_hook=boom)
    assert (c.diffusion_steps, c.mechanics_steps) == (40, 4)
    m = run_simulation(s, c)  # continues from the clock's counters
    assert c.diffusion_steps == 100 and m.diffusion_steps == 100
    ref = make_session(w)
    ref.advance(100, w.dt)
    assert bits_equal(s.download_field(), ref.download_field())


@pytest.mark.gpu
def test_engine_resume_with_snapshots_keeps_the_snapshot_grid():
    """a run resumed with snapshots on continues the snapshot grid
    from the clock's position (no negative advance, no repeated snapshot)."""
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("engine4", (10, 10, 10), 1, 20, 1, seed=3)
    s = make_session(w)
    c = SimulationClock(t_max=1.0)
    snaps, mech = [], []

    def boom(k):
        mech.append(k.mechanics_steps)
        if k.mechanics_steps == 4:
            raise RuntimeError("stop here")

    with pytest.raises(RuntimeError, match="stop here"):
        run_simulation(s, c, mech_hook=boom, snapshot_interval=0.15,
                       snapshot_hook=lambda t, f: snaps.append(round(t, 9)))
    assert (c.diffusion_steps, c.mechanics_steps) == (40, 4) and snaps == [0.15, 0.3]
    m = run_simulation(s, c, mech_hook=lambda k: mech.append(k.mechanics_steps), snapshot_interval=0.15,
                       snapshot_hook=lambda t, f: snaps.append(round(t, 9)))
    # the aborted mechanics hook (step 4) is re-run first, then the grid continues
    assert mech == [1, 2, 3, 4, 4, 5, 6, 7, 8, 9, 10]
    assert snaps == [0.15, 0.3, 0.45, 0.6, 0.75, 0.9] and m.snapshots == 4
    assert (c.diffusion_steps, c.mechanics_steps, c.pending) == (100, 10, 0)
    ref = make_session(w)
    ref.advance(100, w.dt)
    assert bits_equal(s.download_field(), ref.download_field())


@pytest.mark.gpu
def test_engine_aborted_boundary_hooks_are_pending_and_rerun():
    """a snapshot hook that aborts at a mechanics boundary must not
    lose that mechanics step (or its cell step) on resume."""
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("engine5", (10, 10, 10), 1, 0, 1)
    s = make_session(w)
    c = SimulationClock(t_max=1.2, dt_cell=0.3)  # per_cell = 3
    snaps, mech, cell = [], [], []
    state = {"fail": True}

    def snap(t, f):
        if round(t, 9) == 0.3 and state["fail"]:
            state["fail"] = False
            raise RuntimeError("disk full")
        snaps.append(round(t, 9))

    hooks = dict(mech_hook=lambda k: mech.append(k.mechanics_steps),
                 cell_hook=lambda k: cell.append(k.mechanics_steps), snapshot_interval=0.3, snapshot_hook=snap)
    with pytest.raises(RuntimeError, match="disk full"):
        run_simulation(s, c, **hooks)
    assert (c.diffusion_steps, c.mechanics_steps, c.cell_steps) == (30, 3, 1)
    assert c.pending == 1 | 2 | 4 and mech == [1, 2] and cell == []
    run_simulation(s, c, **hooks)
    assert snaps == [0.3, 0.6, 0.9, 1.2]
    assert mech == list(range(1, 13)) and cell == [3, 6, 9, 12]
    assert (c.diffusion_steps, c.mechanics_steps, c.cell_steps, c.pending) == (120, 12, 4, 0)
