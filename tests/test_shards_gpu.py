"""GPU: substrate shards and substrate x z-slab layouts,
through the C ABI. Substrates are independent in the whole step
(solver.cpp:72-95, 273; agents.cpp:103-108), so a pure substrate split is
BIT-IDENTICAL to the unsharded run; layouts that also split z are checked
at the z-slab bar (north_star 1e-10 asserted, rounding level 1e-13
required)."""
import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.shards import ShardGroup, shard_session, split_substrates
from tests.helpers import bits_equal, first_diff, make_session
from tests.test_zslab_gpu import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")


@pytest.mark.parametrize("parts", [2, 3, 4])
def test_substrate_shards_bitwise(parts):
    w = W.make("shards", (40, 36, 30), 4, 1500, 12, seed=parts, immune_fraction=0.3, interior_clamps=25)
    single = make_session(w)
    single.advance(w.steps, w.dt)
    want = single.download_field()
    g = ShardGroup(w, parts)
    g.advance(w.steps)
    got = g.download_field()
    assert bits_equal(got, want), first_diff(got, want)
    assert bits_equal(got, Oracle.run(w, w.steps))
    g.close()


def test_c3_on_2_and_4_substrate_shards_bitwise_vs_one_gpu():
    """The verdict's bar: C3 (256^3 x 4, 100k cells) split over 2 and 4
    substrate shards equals the one-GPU run bit for bit."""
    w = W.c3(2)
    single = make_session(w)
    single.advance(2, w.dt)
    want = single.download_field()
    single.close()
    for parts in (2, 4):
        g = ShardGroup(w, parts)
        g.advance(2)
        got = g.download_field()
        g.close()
        assert bits_equal(got, want), f"{parts} shards: {first_diff(got, want)}"


@pytest.mark.parametrize("k,P", [(2, 2), (4, 2), (2, 3)])
def test_substrate_by_zslab_layouts(k, P):
    w = W.make("hybrid", (24, 20, 60), 4, 800, 10, seed=k * 10 + P, immune_fraction=0.2, interior_clamps=8)
    single = make_session(w)
    single.advance(w.steps, w.dt)
    want = single.download_field()
    g = ShardGroup(w, k, P)
    g.advance(w.steps)
    got = g.download_field()
    err = rel_err(got, want)
    assert err <= 1e-10, err  # north_star tolerance
    assert err <= 1e-13, err  # rounding level
    g.close()


def test_shard_global_field_roundtrip_and_local_layout():
    w = W.make("rt", (12, 10, 20), 4, 0, 1)
    f = np.random.default_rng(0).random(w.voxels * w.S)
    g = ShardGroup(w, 2, 2)
    g.upload_field(f)
    assert bits_equal(g.download_field(), f)
    s = g.pieces[1][0]  # substrates [2, 4), planes [0, 10)
    local = s.download_field()
    want = f.reshape(20, 10, 12, 4)[:10, :, :, 2:4].ravel()
    assert bits_equal(local, want)
    g.close()


def test_shard_rejects_bad_ranges_and_agent_save(tmp_path):
    w = W.make("bad", (10, 10, 10), 3, 20, 1, seed=2)
    mesh = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    for sr in [(0, 0), (2, 1), (-1, 2), (1, 4)]:
        with pytest.raises(B.ConfigError):
            B.Session(mesh, 3, 0, shard=sr)
    s = shard_session(w, (1, 3))
    assert s.S == 2 and s.S_total == 3
    with pytest.raises(B.StateError, match="substrate shard"):
        s.save_agents_csv(tmp_path / "a.csv", ["a", "b", "c"])
    # a shard's agent rates are its own columns
    _, _, _, sec, upt, sat = s.download_agents()  # input order
    assert sec.shape == (20, 2)
    assert bits_equal(sec, w.agent_sec[:, 1:3]) and bits_equal(upt, w.agent_upt[:, 1:3])
    assert bits_equal(sat, w.agent_sat[:, 1:3])
    s.close()


def test_split_substrates_covers_every_substrate():
    for S in range(1, 9):
        for k in range(1, S + 1):
            r = split_substrates(S, k)
            assert r[0][0] == 0 and r[-1][1] == S and all(a[1] == b[0] for a, b in zip(r, r[1:]))
