"""GPU: moving agents and the on-device voxel grouping.

AgentPopulation::set_position + rebuild_voxel_grouping (agents.cpp:45-73)
run on the device (csrc/agents.cu: voxel keys, stable radix sort by (voxel,
id), CSR). Checked against the oracle's grouping (oracle/biodiff_oracle.c,
pinned to the reference) and full runs bit for bit; errors as the reference
raises them (mesh.cpp:74-76, agents.cpp:53)."""
import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.ensemble import ensemble_session
from paper_2110_13368_b200.zslab import ZSlabGroup
from tests.helpers import bits_equal, first_diff, make_session

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200 (no CPU fallback)")


def _oracle_grouping(w):
    return Oracle.group(w.agent_ids, w.agent_pos, w.bounds(), (w.dx,) * 3, w.n)


def _move(rng, w, frac=0.5, scale=2.5):
    """Random walk of a fraction of the agents (several voxels), clipped to the domain;
    some agents pile onto one voxel (collisions) and some land exactly on faces."""
    lo, hi = np.array(w.bounds()[0::2]), np.array(w.bounds()[1::2])
    pos = w.agent_pos.copy()
    sel = rng.random(w.n_agents) < frac
    pos[sel] += rng.normal(0, scale * w.dx, (sel.sum(), 3))
    pos = np.clip(pos, lo, hi)
    k = max(1, w.n_agents // 20)
    pos[:k] = pos[k]           # a dense pile-up in one voxel
    pos[k:2 * k, 0] = hi[0]    # upper faces clamp to the last voxel
    return pos


@pytest.mark.parametrize("shape,S,n", [((24, 20, 18), 2, 800), ((50, 50, 50), 1, 1000), ((17, 9, 11), 3, 300),
                                       ((64, 64, 64), 4, 5000)])
def test_grouping_matches_oracle_after_moves(shape, S, n):
    w = W.make("t", shape, S, n, 1, seed=sum(shape) + S, immune_fraction=0.2)
    s = make_session(w)
    gv, go, order = s.agent_grouping()
    wv, wo, word = _oracle_grouping(w)
    assert np.array_equal(gv, wv) and np.array_equal(go, wo) and np.array_equal(order, word)
    rng = np.random.default_rng(n)
    for _ in range(3):
        w.agent_pos = _move(rng, w)
        s.set_agent_positions(w.agent_pos)
        s.rebuild_voxel_grouping()
        gv, go, order = s.agent_grouping()
        wv, wo, word = _oracle_grouping(w)
        assert np.array_equal(gv, wv) and np.array_equal(go, wo) and np.array_equal(order, word)
    s.close()


def test_moving_agents_full_run_bitwise():
    """Steps, move + rebuild, more steps (graphs captured before the rebuild
    are replayed after it), against the oracle with the same moves."""
    w = W.make("t", (40, 36, 30), 2, 2000, 1, seed=77, immune_fraction=0.3, interior_clamps=20)
    s = make_session(w)
    rng = np.random.default_rng(5)
    want = w.initial_field()
    for epoch in range(4):
        s.advance(60, w.dt, with_sources=True)
        want = Oracle.run(w, 60, field=want)
        got = s.download_field()
        assert bits_equal(got, want), f"epoch {epoch}: {first_diff(got, want)}"
        w.agent_pos = _move(rng, w)
        s.set_agent_positions(w.agent_pos)
        s.rebuild_voxel_grouping()
    s.close()


@pytest.mark.parametrize("path", ["one_cta", "cub_graph", "cub_eager"])
def test_set_position_by_id_and_errors(path, monkeypatch):
    """Every regrouping path (one-CTA sort; the CUB pipeline replayed as a
    graph, or eagerly): a failed rebuild keeps the previous grouping, and a
    later good one (same captured graph) replaces it."""
    if path != "one_cta":
        monkeypatch.setenv("BIODIFF_REGROUP_CUB", "1")
    if path == "cub_eager":
        monkeypatch.setenv("BIODIFF_REGROUP_GRAPH", "0")
    w = W.make("t", (20, 20, 20), 1, 100, 1, seed=3)
    s = make_session(w)
    aid = int(w.agent_ids[17])
    p = np.array(w.bounds()[1::2]) - 1e-9  # near the upper corner
    s.set_agent_position(aid, p)
    w.agent_pos[17] = p
    s.rebuild_voxel_grouping()
    assert all(np.array_equal(a, b) for a, b in zip(s.agent_grouping(), _oracle_grouping(w)))
    with pytest.raises(B.StateError, match="no agent with id"):  # agents.cpp:53 (std::invalid_argument)
        s.set_agent_position(10 ** 12, p)
    # A position outside the domain: nearest_voxel's domain_error (mesh.cpp:74-76).
    bad = p + np.array([0.0, 0.0, 1.0])
    before = s.agent_grouping()
    s.set_agent_position(aid, bad)
    with pytest.raises(B.StateError, match=r"outside the simulation domain"):
        s.rebuild_voxel_grouping()
    # the failed rebuild keeps the previous grouping (the
    # reference throws before reassigning groups_), and steps still use it.
    assert all(np.array_equal(a, b) for a, b in zip(s.agent_grouping(), before))
    s.advance(3, w.dt, with_sources=True)
    assert bits_equal(s.download_field(), Oracle.run(w, 3))
    s.upload_field(w.initial_field())
    s.set_agent_position(aid, p)
    s.rebuild_voxel_grouping()
    assert all(np.array_equal(a, b) for a, b in zip(s.agent_grouping(), _oracle_grouping(w)))
    for k in range(3):  # alternate sort buffers, failures in between
        w.agent_pos = _move(np.random.default_rng(k), w)
        w.agent_pos[17] = p
        s.set_agent_positions(w.agent_pos)
        s.rebuild_voxel_grouping()
        assert all(np.array_equal(a, b) for a, b in zip(s.agent_grouping(), _oracle_grouping(w)))
        s.set_agent_position(aid, bad)
        with pytest.raises(B.StateError, match=r"outside the simulation domain"):
            s.rebuild_voxel_grouping()
        assert all(np.array_equal(a, b) for a, b in zip(s.agent_grouping(), _oracle_grouping(w)))
        s.set_agent_position(aid, p)
    s.close()


def test_agent_csv_through_the_session(tmp_path):
    """load_agents_csv == set_agents; save_agents_csv writes the device's moved agents."""
    w = W.make("t", (30, 20, 10), 2, 700, 1, seed=9, immune_fraction=0.5)
    names = ["oxygen", "factor"]
    path = tmp_path / "agents.csv"
    B.write_agents_csv(path, names, w.agent_ids, w.agent_pos, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat)
    a = make_session(w)
    b = make_session(w)
    b.load_agents_csv(path, names)
    a.advance(25, w.dt)
    b.advance(25, w.dt)
    assert bits_equal(a.download_field(), b.download_field())
    rng = np.random.default_rng(1)
    moved = _move(rng, w)
    b.set_agent_positions(moved)
    out = tmp_path / "moved.csv"
    b.save_agents_csv(out, names)
    ids, xyz, vol, sec, upt, sat = B.parse_agents_csv(B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx), out, names)
    assert np.array_equal(ids, w.agent_ids) and bits_equal(xyz, moved) and bits_equal(sec, w.agent_sec)
    d = b.download_agents()
    assert bits_equal(d[1], moved) and bits_equal(d[2], w.agent_vol)
    a.close()
    b.close()


def test_ensemble_agents_move_per_replica():
    """Ensembles: positions in replica-major agent order; each replica regroups in its own mesh copy."""
    ws = [W.make(f"r{r}", (24, 20, 16), 2, 300, 1, seed=100 + r) for r in range(5)]
    s = ensemble_session(ws)
    rng = np.random.default_rng(4)
    for w in ws:
        w.agent_pos = _move(rng, w)
    s.set_agent_positions(np.concatenate([w.agent_pos for w in ws]))
    s.rebuild_voxel_grouping()
    s.advance(30, ws[0].dt, with_sources=True)
    got = s.download_field()
    per = ws[0].voxels * ws[0].S
    for r, w in enumerate(ws):
        want = Oracle.run(w, 30)
        assert bits_equal(got[r * per:(r + 1) * per], want), f"replica {r}"
    s.close()


def test_zslab_agents_cross_slabs():
    """z-slabs: every slab holds every agent and groups the ones inside it;
    agents that move across a slab boundary change owner at the rebuild."""
    w = W.make("t", (20, 18, 64), 2, 600, 1, seed=21, immune_fraction=0.2)
    g = ZSlabGroup(w, 3)
    single = make_session(w)
    rng = np.random.default_rng(8)
    for epoch in range(3):
        g.advance(15)
        single.advance(15, w.dt)
        a, b = g.download_field(), single.download_field()
        d = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-290)
        assert d.max() <= 1e-13, (epoch, d.max())
        pos = _move(rng, w, scale=12.0)  # large moves: many cross a slab boundary
        for s in g.sessions + [single]:
            s.set_agent_positions(pos)
            s.rebuild_voxel_grouping()
        w.agent_pos = pos
    total = sum(s.agent_grouping()[1][-1] for s in g.sessions)
    assert total == w.n_agents  # each agent grouped by exactly one slab
    # what each slab's agents sense: their voxel's values; the others NaN —
    # together exactly the single domain's samples
    want = single.sample_agent_densities()
    merged = np.full_like(want, np.nan)
    for sl in g.sessions:
        got = sl.sample_agent_densities()
        own = ~np.isnan(got)
        assert not np.any(own & ~np.isnan(merged))  # no agent sampled by two slabs
        merged[own] = got[own]
    d = np.abs(merged - want) / np.maximum(np.abs(want), 1e-290)
    assert d.max() <= 1e-13
    g.close()
    single.close()


@pytest.mark.parametrize("n,buf,zc", [(400, "pageable", "1"), (400, "pinned", "1"), (3000, "pinned", "1"),
                                       (3000, "pinned", "0"), (3000, "pageable", "1")])
def test_sample_agent_densities_reads_each_agents_voxel(n, buf, zc, monkeypatch):
    """What each agent senses: field.values[agent.voxel * S + s] (agents.hpp:22,
    mesh.hpp:62-90), in agent-index order, after steps and after a move; the
    one-CTA and CUB regroupings (n), into pageable or page-locked mapped
    buffers (written by the gather kernel directly unless
    BIODIFF_ZC_POSITIONS=0)."""
    import torch
    monkeypatch.setenv("BIODIFF_ZC_POSITIONS", zc)
    w = W.make("t", (20, 18, 16), 2, n, 1, seed=4, immune_fraction=0.3)
    s = make_session(w)
    out = torch.empty((n, w.S), dtype=torch.float64).pin_memory().numpy() if buf == "pinned" else None
    rng = np.random.default_rng(2)
    for _ in range(2):
        s.advance(5, w.dt)
        f = s.download_field().reshape(-1, w.S)
        gv, go, order = _oracle_grouping(w)
        vox = np.empty(w.n_agents, np.int64)
        for g in range(gv.size):
            vox[order[go[g]:go[g + 1]]] = gv[g]
        got = s.sample_agent_densities(out)
        assert bits_equal(got, f[vox])
        w.agent_pos = _move(rng, w)
        s.set_agent_positions(w.agent_pos)
        s.rebuild_voxel_grouping()
    with pytest.raises(B.StateError):
        B._check(B.lib().biodiff_sample_agent_densities(s._h, B._dptr(np.zeros(3)), 3))
    s.close()


@pytest.mark.parametrize("zero_copy", ["1", "0"])
@pytest.mark.parametrize("n", [301, 2000])
def test_positions_from_page_locked_buffers(zero_copy, n, monkeypatch):
    """set_agent_positions from a page-locked, device-mapped caller buffer
    (torch pin_memory = cudaHostAlloc) goes through the zero-copy kernel
    (BIODIFF_ZC_POSITIONS=1, default) or the DMA copy; both give the
    oracle's grouping, also from an 8-byte-offset view (DMA fallback) and for
    odd value counts."""
    import torch
    monkeypatch.setenv("BIODIFF_ZC_POSITIONS", zero_copy)
    w = W.make("t", (24, 20, 18), 2, n, 1, seed=n, immune_fraction=0.2)
    s = make_session(w)
    rng = np.random.default_rng(n)
    for offset in (0, 1):
        w.agent_pos = _move(rng, w)
        buf = torch.empty(3 * n + 1, dtype=torch.float64).pin_memory()
        view = buf.numpy()[offset:offset + 3 * n]
        view[:] = w.agent_pos.reshape(-1)
        s.set_agent_positions(view.reshape(n, 3))
        s.rebuild_voxel_grouping()
        gv, go, order = s.agent_grouping()
        wv, wo, word = _oracle_grouping(w)
        assert np.array_equal(gv, wv) and np.array_equal(go, wo) and np.array_equal(order, word)
    s.close()


def test_regroup_graph_across_populations_and_timing(monkeypatch):
    """The captured CUB regrouping pipeline is per population: a new
    set_agents (another size) re-captures it, and kernel timing (eager
    pipeline) in between gives the same grouping."""
    monkeypatch.setenv("BIODIFF_REGROUP_CUB", "1")
    w = W.make("t", (24, 20, 18), 2, 900, 1, seed=21, immune_fraction=0.2)
    s = make_session(w)
    rng = np.random.default_rng(21)
    for n, timing in ((900, False), (1500, True), (700, False)):
        w2 = W.make("t", (24, 20, 18), 2, n, 1, seed=n, immune_fraction=0.3)
        s.set_agents(w2.agent_ids, w2.agent_pos, w2.agent_vol, w2.agent_sec, w2.agent_upt, w2.agent_sat)
        s.set_kernel_timing(timing)
        for _ in range(3):
            w2.agent_pos = _move(rng, w2)
            s.set_agent_positions(w2.agent_pos)
            s.rebuild_voxel_grouping()
            gv, go, order = s.agent_grouping()
            wv, wo, word = _oracle_grouping(w2)
            assert np.array_equal(gv, wv) and np.array_equal(go, wo) and np.array_equal(order, word)
    s.close()
