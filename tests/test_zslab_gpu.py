"""GPU: the z-slab partitioned solve against the single-domain
solve and the oracle. In-process slabs on one GPU exercise the same kernels,
plane exports, inflow corrections and exchange order as the NCCL path (which
needs one GPU per rank). Tolerance: north_star's relative 1e-10 per voxel is
asserted, and the observed error is additionally required to stay at the
rounding level (1e-13 relative) — the partitioned solve is not bit-identical
(different summation order at the slab interfaces)."""
import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.zslab import ZSlabGroup, split_planes
from tests.helpers import make_session

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")


FLOOR = 1e-290  # values this small are at the edge of FP64 underflow: compare absolutely


def rel_err(a, b):
    """max |a-b| / max(|a|,|b|) over voxels, with an absolute floor near underflow."""
    d = np.abs(a - b)
    m = np.maximum(np.maximum(np.abs(a), np.abs(b)), FLOOR)
    r = d / m
    i = int(np.argmax(r))
    if r[i] > 1e-13:
        print(f"worst value index {i}: {a[i]!r} vs {b[i]!r}")
    return float(r[i])


CASES = [
    # shape, S, agents, steps, parts, interior clamps
    ((20, 18, 64), 2, 300, 20, 2, 5),
    ((24, 20, 96), 3, 500, 15, 2, 0),
    ((16, 16, 200), 1, 200, 10, 2, 3),
    ((32, 24, 270), 4, 800, 8, 3, 6),
    ((16, 12, 400), 2, 300, 6, 4, 4),
]


@pytest.mark.parametrize("shape,S,agents,steps,parts,clamps", CASES)
def test_zslab_group_matches_single_domain(shape, S, agents, steps, parts, clamps):
    w = W.make("zslab", shape, S, agents, steps, seed=sum(shape) + S, immune_fraction=0.2, interior_clamps=clamps)
    single = make_session(w)
    single.advance(steps, w.dt)
    want = single.download_field()
    single.close()
    g = ZSlabGroup(w, parts)
    g.advance(steps)
    got = g.download_field()
    g.close()
    err = rel_err(got, want)
    assert err <= 1e-10, err  # north_star tolerance
    assert err <= 1e-13, err  # rounding level
    oracle = Oracle.run(w, steps)
    assert rel_err(got, oracle) <= 1e-13


def test_zslab_single_slab_is_bitwise():
    w = W.make("zslab1", (20, 16, 40), 2, 100, 10, seed=3)
    a = make_session(w)
    a.advance(10, w.dt)
    g = ZSlabGroup(w, 1)
    g.advance(10)
    assert np.array_equal(a.download_field().view(np.int64), g.download_field().view(np.int64))


@pytest.mark.parametrize("parts", [3, 8, 16])
def test_zslab_thin_slabs_exact_interface(parts):
    """The interface recurrences keep every cross-slab coupling, so even
    4-plane slabs (D = 1e5 couples ~0.54^m across a slab) stay at rounding
    level — no minimum thickness."""
    w = W.make("thin", (16, 16, 64), 2, 200, 12, seed=parts, interior_clamps=3)
    single = make_session(w)
    single.advance(12, w.dt)
    want = single.download_field()
    g = ZSlabGroup(w, parts)
    g.advance(12)
    assert rel_err(g.download_field(), want) <= 1e-13


def test_zslab_upload_download_roundtrip_and_split():
    w = W.make("rt", (12, 10, 50), 2, 0, 1)
    assert split_planes(50, 3) == [(0, 17), (17, 33), (33, 50)]
    g = ZSlabGroup(w, 2)
    f = np.random.default_rng(0).random(w.voxels * w.S)
    g.upload_field(f)
    assert np.array_equal(g.download_field(), f)
    g.close()


def test_zslab_group_advance_checks_like_advance():
    """the group advance makes advance()'s checks for every slab."""
    w = W.make("chk", (12, 10, 40), 2, 50, 1, seed=5)
    g = ZSlabGroup(w, 2)
    with pytest.raises(B.StateError, match="does not match the solver workspace dt"):
        B.Session.group_advance(g.sessions, 2, w.dt * 2)
    with pytest.raises(B.StateError, match="positive"):
        B.Session.group_advance(g.sessions, 2, 0.0)
    with pytest.raises(B.StateError, match="non-negative"):
        B.Session.group_advance(g.sessions, -1, w.dt)
    g.advance(3)  # still usable after the rejected calls
    single = make_session(w)
    single.advance(3, w.dt)
    assert rel_err(g.download_field(), single.download_field()) <= 1e-13
    g.close()
