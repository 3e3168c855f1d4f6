"""GPU: batched ensembles (C5-style) — every replica of one stacked session must
be bit-identical to the same replica run alone (and to the oracle)."""
import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.ensemble import ensemble_session, shard
from tests.helpers import bits_equal, first_diff, make_session

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")


def replicas(n, shape, S, agents, steps, clamps=0):
    out = []
    for r in range(n):
        w = W.make(f"rep{r}", shape, S, agents, steps, seed=100 + r, interior_clamps=clamps, immune_fraction=0.2)
        rng = np.random.default_rng(7000 + r)
        f = 0.5 + rng.random((2, S))
        w.substrates = [(nm, D * f[0, i], lam * f[1, i], ic, dv) for i, (nm, D, lam, ic, dv) in enumerate(w.substrates)]
        out.append(w)
    return out


# L2 replica batches (DeviceSession::step_body_batches): "0" = off; small
# budgets force 1-2 replicas per batch and batch visits shorter than the run.
# BIODIFF_XYZ_CLUSTER=1: one thread-block cluster per replica for x, y and z
# (xyc.cuh sweep_xyz_cluster; S in {1, 2, 4}, else the separate sweeps).
BATCHING = [{"BIODIFF_L2_BATCH_MB": "0", "BIODIFF_XYZ_CLUSTER": "0"},
            {"BIODIFF_L2_BATCH_MB": "0.2", "BIODIFF_BATCH_STEPS": "3"},
            {"BIODIFF_L2_BATCH_MB": "2.5", "BIODIFF_BATCH_STEPS": "4"},
            {"BIODIFF_XYZ_CLUSTER": "1"},
            {"BIODIFF_XYZ_CLUSTER": "1", "BIODIFF_XYC_SLOTS": "2", "BIODIFF_XYC_DYNAMIC": "0"},
            {"BIODIFF_XYZ_CLUSTER": "1", "BIODIFF_XYC_WARPS": "3", "BIODIFF_XYC_CLUSTER": "2"}]


@pytest.mark.parametrize("batching", BATCHING, ids=["off", "tiny", "small", "xyz", "xyz_ns2_static", "xyz_2x3"])
@pytest.mark.parametrize("n,shape,S,agents,steps,clamps", [
    (4, (24, 20, 18), 2, 200, 10, 3),
    (7, (32, 32, 32), 2, 300, 6, 0),
    (3, (64, 64, 64), 2, 1000, 4, 5),
    (5, (16, 12, 40), 3, 80, 8, 2),
])
def test_ensemble_replicas_bitwise_equal_single_runs(n, shape, S, agents, steps, clamps, batching, monkeypatch):
    for k, v in batching.items():
        monkeypatch.setenv(k, v)
    ws = replicas(n, shape, S, agents, steps, clamps)
    e = ensemble_session(ws)
    e.advance(steps, ws[0].dt)
    got = e.download_field()
    e.close()
    per = ws[0].voxels * S
    for r, w in enumerate(ws):
        s = make_session(w)
        s.advance(steps, w.dt)
        want = s.download_field()
        s.close()
        part = got[r * per:(r + 1) * per]
        assert bits_equal(part, want), f"replica {r}: {first_diff(part, want)}"
    want0 = Oracle.run(ws[0], steps)
    assert bits_equal(got[:per], want0)


def test_ensemble_batches_with_moving_agents(monkeypatch):
    """Batched advance after an on-device regroup: per-replica group ranges follow the rebuild."""
    monkeypatch.setenv("BIODIFF_L2_BATCH_MB", "0.2")
    monkeypatch.setenv("BIODIFF_BATCH_STEPS", "2")
    ws = replicas(6, (20, 16, 12), 2, 150, 1)
    e = ensemble_session(ws)
    e.advance(5, ws[0].dt)
    rng = np.random.default_rng(3)
    lo, hi = np.array(ws[0].bounds()[0::2]), np.array(ws[0].bounds()[1::2])
    for w in ws:
        w.agent_pos = np.clip(w.agent_pos + rng.normal(0, 40.0, w.agent_pos.shape), lo, hi)
    e.set_agent_positions(np.concatenate([w.agent_pos for w in ws]))
    e.rebuild_voxel_grouping()
    e.advance(7, ws[0].dt)
    got = e.download_field()
    per = ws[0].voxels * ws[0].S
    for r, w in enumerate(ws):
        # replay: 5 steps at the old positions, then 7 at the new ones
        old = w.agent_pos
        w.agent_pos = replicas(6, (20, 16, 12), 2, 150, 1)[r].agent_pos
        first = Oracle.run(w, 5)
        w.agent_pos = old
        want = Oracle.run(w, 7, field=first)
        assert bits_equal(got[r * per:(r + 1) * per], want), f"replica {r}"


def test_ensemble_c5_replicas_and_sharding():
    assert [shard(512, 8, r) for r in (0, 7)] == [(0, 64), (448, 512)]
    ws = [W.c5_replica(r, steps=3) for r in range(6)]
    e = ensemble_session(ws)
    e.advance(3, ws[0].dt)
    got = e.download_field()
    per = ws[0].voxels * ws[0].S
    for r in (0, 5):
        want = Oracle.run(ws[r], 3)
        assert bits_equal(got[r * per:(r + 1) * per], want)
