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


@pytest.mark.parametrize("n,shape,S,agents,steps,clamps", [
    (4, (24, 20, 18), 2, 200, 10, 3),
    (7, (32, 32, 32), 2, 300, 6, 0),
    (3, (64, 64, 64), 2, 1000, 4, 5),
    (5, (16, 12, 40), 3, 80, 8, 2),
])
def test_ensemble_replicas_bitwise_equal_single_runs(n, shape, S, agents, steps, clamps):
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
