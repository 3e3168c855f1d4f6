"""GPU parity: the CUDA library, called through its C ABI, against the
oracle and the reference-generated golden fixtures. The bar is bit
equality (integer/index work exact; FP64 kernels use explicitly rounded
operations in the reference's order — SURVEY.md Appendix A). Where a test
compares at a tolerance it says so: north_star's relative 1e-10 per voxel."""
import os

import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from tests.helpers import bits_equal, first_diff, golden_names, load_golden, make_session

pytestmark = pytest.mark.gpu

NORTH_STAR_REL_TOL = 1e-10  # BASELINE.json north_star: relative L-inf per voxel


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200 (no CPU fallback)")


def _skip_experimental(path=None, env=None):
    """Variants measured slower and compiled only by EXPERIMENTAL=1 builds:
    ring2 with 4 slots, the lagged-ticket x+y kernel (BIODIFF_XY_FUSED=1)."""
    if B.experimental_build():
        return
    if path == "r2s4" or (env or {}).get("BIODIFF_XY_FUSED") == "1":
        pytest.skip("variant built only with EXPERIMENTAL=1")


def _paths(monkeypatch, path):
    """Selects a sweep kernel family (read at session creation): auto = ring2
    (register-chunk ring, x 4 slots, y/z 3), r2sN = ring2 with N slots,
    ringN = the r01 ring kernels with N slots, resident = whole line in
    shared memory, smem_plain, global."""
    monkeypatch.delenv("BIODIFF_RING_SLOTS", raising=False)
    monkeypatch.delenv("BIODIFF_RING_PERSIST", raising=False)
    if path.startswith("r2s"):
        monkeypatch.setenv("BIODIFF_SWEEP_PATH", "ring2")
        monkeypatch.setenv("BIODIFF_RING_SLOTS", path[3:])
    elif path in ("ringnp", "ringall"):  # ring with no / every axis persistent
        monkeypatch.setenv("BIODIFF_RING_PERSIST", "0" if path == "ringnp" else "all")
        monkeypatch.delenv("BIODIFF_SWEEP_PATH", raising=False)
    elif path == "auto":
        monkeypatch.delenv("BIODIFF_SWEEP_PATH", raising=False)
    elif path.startswith("ring"):
        monkeypatch.setenv("BIODIFF_SWEEP_PATH", "ring")
        monkeypatch.setenv("BIODIFF_RING_SLOTS", path[4:])
    else:
        monkeypatch.setenv("BIODIFF_SWEEP_PATH", path)


SWEEP_SHAPES = [
    ((16, 16, 16), 1), ((20, 18, 16), 2), ((24, 20, 18), 4), ((17, 9, 11), 1), ((33, 7, 5), 3),
    ((64, 64, 64), 4), ((100, 30, 20), 2), ((300, 6, 5), 2), ((8, 8, 500), 1), ((50, 50, 50), 1),
    ((1, 12, 9), 2), ((7, 1, 40), 1), ((5, 3, 2), 8), ((40, 3, 3), 40),
]


@pytest.mark.parametrize("path", ["auto", "ringnp", "ringall", "r2s2", "r2s4", "ring2", "ring3", "resident", "global",
                                  "smem_plain"])
@pytest.mark.parametrize("shape,S", SWEEP_SHAPES)
def test_single_sweep_bitwise(shape, S, path, monkeypatch):
    """diffusion_sweep (solver.cpp:248-265) along every active axis, every kernel path."""
    _skip_experimental(path=path)
    _paths(monkeypatch, path)
    w = W.make("t", shape, S, 0, 1, seed=2)
    rng = np.random.default_rng(hash((shape, S)) & 0xffff)
    f0 = rng.random(w.voxels * S) * 50.0
    s = make_session(w)
    ws = Oracle.workspaces(shape, (w.dx,) * 3, w.diffusion, w.decay, w.dt)
    for ax in ws:
        s.upload_field(f0)
        s.diffusion_sweep(ax)
        got = s.download_field()
        want = f0.copy()
        Oracle.sweep(want, shape, S, ax, ws[ax])
        assert bits_equal(got, want), f"axis {ax}: {first_diff(got, want)}"
    s.close()


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("path", ["auto", "r2s2", "ring3", "resident", "global"])
def test_golden_fixture_bitwise(name, path, monkeypatch):
    """Full runs vs the reference's own outputs (tests/golden, made by oracle/_ref)."""
    _paths(monkeypatch, path)
    w, z = load_golden(name)
    m = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    s = B.Session(m, w.S)
    s.set_substrates(w.diffusion, w.decay, w.dt)
    s.set_dirichlet(z["dir_voxels"], z["dir_mask"], z["dir_values"])  # the reference's canonical map
    if w.n_agents:
        s.set_agents(w.agent_ids, w.agent_pos, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat)
        gv, go, order = s.agent_grouping()
        assert np.array_equal(gv, z["group_voxel"]) and np.array_equal(go, z["group_offsets"])
        assert np.array_equal(order, z["group_order"])
    s.upload_field(w.initial_field())
    if bool(z["initial_clamp"]):
        s.apply_dirichlet_conditions()
    with_sources = bool(z["with_sources"])
    for _ in range(w.steps):
        s.diffuse_decay_step()
        if with_sources and w.n_agents:
            s.cell_sources_sinks_step(w.dt)
    got = s.download_field()
    assert bits_equal(got, z["field"]), first_diff(got, z["field"])
    s.close()


@pytest.mark.parametrize("resident", ["0", "1"])
@pytest.mark.parametrize("name", golden_names())
def test_golden_fixture_advance_graph(name, resident, monkeypatch):
    """Same runs through advance(): CUDA-graph replay of the SPEC.md:297 loop,
    or the resident multi-step kernel."""
    monkeypatch.setenv("BIODIFF_RESIDENT", resident)
    w, z = load_golden(name)
    if bool(z["initial_clamp"]) or not bool(z["with_sources"]):
        pytest.skip("advance() runs the plain engine loop")
    s = make_session(w)
    # prepare_advance instantiates the graphs and runs nothing
    s.prepare_advance(w.steps, w.dt, with_sources=True)
    assert bits_equal(s.download_field(), w.initial_field())
    l0 = s.launch_count()
    s.advance(w.steps, w.dt, with_sources=True)
    assert s.launch_count() > l0
    got = s.download_field()
    assert bits_equal(got, z["field"]), first_diff(got, z["field"])
    s.close()


@pytest.mark.parametrize("cfg,steps", [("c1", 300), ("c2", 40)])
def test_config_runs_bitwise_vs_oracle(cfg, steps):
    """C1 (50^3 x 1, 1k cells) and C2 (100^3 x 2, 10k cells) at full grid size."""
    w = W.CONFIGS[cfg](steps)
    s = make_session(w)
    s.advance(steps, w.dt, with_sources=True)
    got = s.download_field()
    want = Oracle.run(w, steps)
    assert bits_equal(got, want), first_diff(got, want)
    rep = s.cross_check(want, 0.0, 0.0)
    assert rep.passed and rep.max_abs == 0.0 and rep.worst_value_index == -1
    s.close()


def test_c3_full_size_bitwise_two_steps():
    """C3 (256^3 x 4, 100k cells): two full steps bit-identical to the oracle."""
    w = W.c3(2)
    s = make_session(w)
    s.advance(2, w.dt, with_sources=True)
    got = s.download_field()
    want = Oracle.run(w, 2)
    assert bits_equal(got, want), first_diff(got, want)
    s.close()


def test_interior_dirichlet_and_partial_masks():
    w = W.make("t", (40, 36, 30), 3, 500, 1, seed=31, interior_clamps=200, immune_fraction=0.3)
    s = make_session(w)
    s.advance(20, w.dt)
    got = s.download_field()
    want = Oracle.run(w, 20)
    assert bits_equal(got, want), first_diff(got, want)
    # Clamp semantic: every clamped (voxel, s) holds its value exactly after a diffusion step.
    s.diffuse_decay_step()
    got = s.download_field()
    v, m, x = w.dirichlet_entries()
    S = w.S
    for e in range(0, v.size, 37):
        for k in range(S):
            if m[e, k]:
                assert got[v[e] * S + k] == x[e, k]
    s.close()


def test_standalone_dirichlet_and_sources_match_oracle():
    w = W.make("t", (30, 20, 10), 2, 2000, 1, seed=41, interior_clamps=30)
    rng = np.random.default_rng(3)
    f0 = rng.random(w.voxels * w.S) * 40
    s = make_session(w)
    s.upload_field(f0)
    s.apply_dirichlet_conditions()
    want = f0.copy()
    v, m, x = w.dirichlet_entries()
    Oracle.dirichlet(want, w.S, v, m, x)
    got = s.download_field()
    assert bits_equal(got, want)
    s.apply_dirichlet_conditions()  # idempotent
    assert bits_equal(s.download_field(), want)
    s.cell_sources_sinks_step(w.dt)
    g = Oracle.group(w.agent_ids, w.agent_pos, w.bounds(), (w.dx,) * 3, w.n)
    Oracle.sources(want, w.S, g, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat, w.dt, 1.0 / w.dx ** 3)
    got = s.download_field()
    assert bits_equal(got, want), first_diff(got, want)
    s.close()


def test_no_agents_no_dirichlet_and_empty_inputs():
    w = W.make("t", (12, 12, 12), 1, 0, 1)
    w.substrates = [("a", 1000.0, 0.0, 0.0, None)]
    rng = np.random.default_rng(8)
    f0 = rng.random(w.voxels)
    s = make_session(w)
    s.set_dirichlet(np.zeros(0, np.int64), np.zeros((0, 1), np.uint8), np.zeros((0, 1)))
    s.set_agents(np.zeros(0, np.int64), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 1)), np.zeros((0, 1)),
                 np.zeros((0, 1)))
    s.upload_field(f0)
    s.advance(100, w.dt, with_sources=True)
    got = s.download_field()
    assert abs(got.sum() - f0.sum()) <= 1e-12 * f0.sum()  # mass conservation
    want = Oracle.run(w, 100, field=f0)
    assert bits_equal(got, want)
    s.close()


@pytest.mark.parametrize("resident", ["0", "1"])
def test_advance_equals_stepwise_and_counts_launches(resident, monkeypatch):
    """advance(57) == 57 x [diffuse_decay_step; cell_sources_sinks_step]: graph
    replay launches the same kernels; the resident kernel runs the steps of an
    advance in one cooperative launch (the source factors and per-tile lists
    are built once, by the first advance)."""
    monkeypatch.setenv("BIODIFF_RESIDENT", resident)
    w = W.make("t", (32, 24, 20), 2, 300, 1, seed=5)
    a = make_session(w)
    b = make_session(w)
    a.advance(50, w.dt)
    a0 = a.launch_count()  # grouping, source factors, per-tile lists: once
    a.advance(7, w.dt)
    for _ in range(57):
        b.diffuse_decay_step()
        b.cell_sources_sinks_step(w.dt)
    assert bits_equal(a.download_field(), b.download_field())
    if resident == "0":
        assert a.launch_count() == b.launch_count() > 0
    else:
        assert a.launch_count() - a0 == 1 and b.launch_count() > 57
    a.close()
    b.close()


@pytest.mark.parametrize("kernel", ["dataflow", "cluster"])
@pytest.mark.parametrize("shape,S", SWEEP_SHAPES)
def test_resident_kernel_full_steps_bitwise(shape, S, kernel, monkeypatch):
    """The single-launch multi-step kernels — the L2 dataflow kernel
    (resident.cuh) and the one-cluster kernel (small.cuh, field in the
    cluster's shared memory) — over every sweep shape: 1-D / 2-D / n=1 axes,
    odd rows, S up to 40 (falls back where a tile does not fit), agents with
    collisions and interior clamps: bit-identical to the oracle."""
    monkeypatch.setenv("BIODIFF_RESIDENT", "1")
    monkeypatch.setenv("BIODIFF_SMALL", "1" if kernel == "cluster" else "0")
    w = W.make("t", shape, S, 120, 7, seed=sum(shape) + S, interior_clamps=3, immune_fraction=0.3)
    s = make_session(w)
    s.set_kernel_timing(True)
    s.advance(7, w.dt)
    got = s.download_field()
    t = s.kernel_times()
    want = Oracle.run(w, 7)
    assert bits_equal(got, want), first_diff(got, want)
    if S <= 32 and min(shape) >= 2:  # 3-D fields only (resident_path)
        assert t["resident"][0] == 1 and t["sweep_x"][0] == 0
    s.close()


@pytest.mark.parametrize("cfg,steps,small", [("c1", 2000, "auto"), ("c1", 500, "0"), ("c2", 300, "auto"),
                                             ("c2", 300, "0")])
def test_resident_kernel_configs_bitwise(cfg, steps, small, monkeypatch):
    """C1 / C2 at full size take a single-launch kernel by default (C1: the
    one-cluster kernel; C2: its slab-grid mode); both also through the L2
    dataflow kernel."""
    if small != "auto":
        monkeypatch.setenv("BIODIFF_SMALL", small)
    w = W.CONFIGS[cfg](steps)
    s = make_session(w)
    s.set_kernel_timing(True)
    s.advance(steps, w.dt)
    assert s.kernel_times()["resident"][0] == 1
    got = s.download_field()
    want = Oracle.run(w, steps)
    assert bits_equal(got, want), first_diff(got, want)
    s.close()


@pytest.mark.parametrize("fused", ["1", "0"])
def test_kernel_timing_reports_every_class(fused, monkeypatch):
    _skip_experimental(env={"BIODIFF_XY_FUSED": fused})
    monkeypatch.setenv("BIODIFF_XY_FUSED", fused)
    w = W.make("t", (64, 64, 64), 2, 1000, 1, seed=6, interior_clamps=10)
    s = make_session(w)
    s.set_kernel_timing(True)
    s.advance(3, w.dt)
    t = s.kernel_times()
    if fused == "1":  # x and y run as one fused launch per 3-D step (xy.cuh)
        assert t["sweep_xy"][0] == t["sweep_z"][0] == 3 and t["sweep_x"][0] == t["sweep_y"][0] == 0
    else:
        assert t["sweep_x"][0] == t["sweep_y"][0] == t["sweep_z"][0] == 3 and t["sweep_xy"][0] == 0
    assert t["sources"][0] == 3 and t["dirichlet"][0] == 3
    assert all(ms > 0 for n, ms in t.values() if n)
    s.close()


def test_errors_map_to_reference_categories():
    w = W.make("t", (10, 10, 10), 1, 0, 1)
    s = make_session(w)
    with pytest.raises(B.StateError):
        s.advance(3, w.dt * 2)  # dt must match the workspace (solver.hpp:57-68)
    one = np.ones(11)
    p = one.ctypes.data_as(B._P(B._d))
    with pytest.raises(B.StateError):  # workspace line length != mesh axis (solver.cpp:251-253)
        B._check(B.lib().biodiff_set_workspace(s._h, 0, 11, 3, 0.01, p, p, p))
    with pytest.raises(B.StateError):
        s.cell_sources_sinks_step(0.0)  # agents.cpp:78
    with pytest.raises(B.StateError):
        s.set_agents([1, 1], np.zeros((2, 3)), [1, 1], np.zeros(2), np.zeros(2), np.zeros(2))  # duplicate id
    with pytest.raises(B.StateError):
        s.set_agents([1], [[1e9, 0, 0]], [1], [0.0], [0.0], [0.0])  # outside the domain
    with pytest.raises(B.StateError):
        s.set_dirichlet([5000], [[1]], [[1.0]])  # voxel outside mesh
    with pytest.raises(B.ConfigError):
        B.Session(s.mesh, 0)
    s.close()


def test_cross_check_semantics():
    w = W.make("t", (10, 10, 10), 2, 0, 1)
    s = make_session(w)
    f = w.initial_field() + 1.0
    s.upload_field(f)
    g = f.copy()
    g[123] += 1e-3
    rep = s.cross_check(g, 1e-9, 1e-9)
    assert not rep.passed and rep.worst_value_index == 123 and rep.worst_voxel == 61 and rep.worst_substrate == 1
    assert s.cross_check(f, 0.0, 0.0).passed
    s.close()


def test_cross_check_nan_inf_matches_reference_device():
    """the device cross_check gives the reference's verdict on
    NaN / Inf entries (comparisons with NaN are false), not a stricter one."""
    import oracle
    from tests.test_validation import _nan_inf_cases
    if not oracle.reference_available():
        pytest.skip("reference build absent")
    w = W.make("t", (2, 2, 1), 3, 0, 1)
    s = make_session(w)
    for a, b in _nan_inf_cases():
        s.upload_field(a)
        for tol in [(1e-9, 1e-9), (0.0, 0.0)]:
            rep = s.cross_check(b, *tol)
            ma, mr, wi, ok = oracle.ref_cross_check(a, b, 3, *tol)
            assert (rep.max_abs, rep.max_rel, rep.worst_value_index, rep.passed) == (ma, mr, wi, ok), (a, b, tol)
    s.close()


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_long_run_within_north_star_tolerance(cfg):
    """3000 steps (30 sim-min) at the C1/C2 grids: bitwise in practice; the
    north_star bar (relative 1e-10 per voxel) is asserted explicitly."""
    steps = 3000 if cfg == "c1" else 600
    w = W.CONFIGS[cfg](steps)
    s = make_session(w)
    s.advance(steps, w.dt)
    got = s.download_field()
    want = Oracle.run(w, steps)
    rep = s.cross_check(want, 0.0, NORTH_STAR_REL_TOL)
    assert rep.passed, rep
    assert bits_equal(got, want), first_diff(got, want)
    s.close()


FUSED_ENVS = [
    {"BIODIFF_XY_FUSED": "0"},                                                  # separate x and y ring sweeps
    {"BIODIFF_XY_FUSED": "1"},                                                  # default lag
    {"BIODIFF_XY_FUSED": "1", "BIODIFF_XY_LAG": "1"},                           # y items wait on counters
    {"BIODIFF_XY_FUSED": "1", "BIODIFF_XY_LAG": "1000000"},                     # all x items, then all y items
    {"BIODIFF_XY_FUSED": "1", "BIODIFF_XY_CTAS_PER_SM": "1", "BIODIFF_XY_LAG": "2"},  # few CTAs, many items each
    {"BIODIFF_XY_FUSED": "1", "BIODIFF_XY_SLOTS": "2"},                         # two-slot ring
    {"BIODIFF_XY_FUSED": "2"},                                                  # plane clusters (xyc.cuh)
    {"BIODIFF_XY_FUSED": "2", "BIODIFF_XYC_CLUSTER": "2", "BIODIFF_XYC_WARPS": "3", "BIODIFF_XYC_SLOTS": "2"},
    {"BIODIFF_XY_FUSED": "2", "BIODIFF_XYC_CLUSTER": "4", "BIODIFF_XYC_WARPS": "8"},   # one CTA per SM
    {"BIODIFF_XY_FUSED": "2", "BIODIFF_XYC_CLUSTER": "16", "BIODIFF_XYC_WARPS": "1"},  # non-portable cluster size
    {"BIODIFF_XY_FUSED": "2", "BIODIFF_XYC_REVERSE": "0", "BIODIFF_XYC_DYNAMIC": "0",  # static planes, bottom up
     "BIODIFF_XYC_STAGGER_NS": "0"},
]


@pytest.mark.parametrize("env", FUSED_ENVS, ids=["unfused", "fused", "lag1", "lagmax", "1cta", "slots2", "cluster",
                                                 "cluster2x3", "cluster4x8", "cluster16x1", "cluster_static"])
@pytest.mark.parametrize("shape,S", SWEEP_SHAPES + [((36, 200, 5), 4), ((130, 160, 3), 2)])
def test_fused_xy_step_bitwise(shape, S, env, monkeypatch):
    """The fused x+y kernel (ticketed items, per-plane release/acquire
    counters) gives the oracle's bits for full steps at every lag setting."""
    _skip_experimental(env=env)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = W.make("t", shape, S, 150, 1, seed=9, interior_clamps=4)
    s = make_session(w)
    s.advance(6, w.dt, with_sources=True)
    got = s.download_field()
    want = Oracle.run(w, 6)
    assert bits_equal(got, want), first_diff(got, want)
    s.set_kernel_timing(True)
    s.diffuse_decay_step()
    t = s.kernel_times()
    assert t["sweep_xy"][0] + t["sweep_x"][0] == 1
    if env.get("BIODIFF_XY_FUSED") not in ("1", "2"):
        assert t["sweep_xy"][0] == 0
    s.close()


def _random_cases(n, seed=2024):
    rng = np.random.default_rng(seed)
    cases = []
    for k in range(n):
        shape = tuple(int(x) for x in rng.choice([1, 2, 3, 5, 16, 31, 32, 33, 63, 64, 65, 96, 97, 130], size=3))
        if max(shape) == 1:
            shape = (33, 2, 1)
        S = int(rng.choice([1, 2, 3, 4, 5, 8]))
        cases.append((shape, S, int(rng.integers(0, 400)), int(rng.integers(1, 9)), int(rng.integers(0, 6)), k))
    return cases


@pytest.mark.parametrize("shape,S,agents,steps,clamps,k", _random_cases(48))
def test_random_shapes_bitwise(shape, S, agents, steps, clamps, k):
    """Randomised shapes around the chunk (32) and tile boundaries, 1-D / 2-D /
    3-D, substrate counts with and without the swizzled x path, agents and
    interior clamps: full steps bit-identical to the oracle."""
    w = W.make("rand", shape, S, agents, steps, seed=100 + k, interior_clamps=clamps, immune_fraction=0.3)
    s = make_session(w)
    s.advance(steps, w.dt, with_sources=True)
    got = s.download_field()
    want = Oracle.run(w, steps)
    assert bits_equal(got, want), first_diff(got, want)
    s.close()
