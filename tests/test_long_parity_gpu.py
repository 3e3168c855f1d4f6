"""GPU: every BASELINE.json configuration at its own size and step count
against the REFERENCE ITSELF (north_star: "the same grid, cells and step
count"), through the C ABI's graph-replayed advance.

The reference's final fields are pinned as SHA-256 digests in
tests/golden/digests.json (made by tests/golden/make_digests.py from
oracle/_ref, the unmodified reference sources): equal digests = bit-identical
fields. The z-slab and substrate-shard layouts of C4 are checked against the
single-domain C4 solve, which the c4 digest ties to the reference:
substrate shards bitwise, z-slabs within 1e-13 relative (the partitioned
z solve re-associates at the slab interfaces; north_star's bar is 1e-10).
"""
import json
import os

import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import field_sha256
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.ensemble import ensemble_session
from paper_2110_13368_b200.shards import ShardGroup
from paper_2110_13368_b200.zslab import ZSlabGroup
from tests.golden.make_digests import C5_SAMPLE, C5_STEPS, spec511
from tests.helpers import make_session

pytestmark = pytest.mark.gpu

DIGESTS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "digests.json")
FLOOR = 1e-290


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")


def digests():
    with open(DIGESTS) as f:
        return json.load(f)


def session_digest(s, offset=0, count=None):
    count = s.value_count - offset if count is None else count
    return field_sha256(lambda off, n, out: s.download_field_range(offset + off, n, out), count)


def check_digest(name, s, offset=0, count=None):
    want = digests()[name]
    got = session_digest(s, offset, count)
    if got != want["sha256"]:
        probe = np.empty(1)
        vals = [float(s.download_field_range(offset + i, 1, probe)[0]) for i in want["probe_index"]]
        pytest.fail(f"{name}: field differs from the reference after {want['steps']} steps; "
                    f"probes GPU {vals} vs reference {want['probe_values']}")


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_full_length_run_bitwise_vs_reference(cfg):
    """C1 and C2 for their whole 360 simulated minutes (36,000 steps), C3 for 1000 steps."""
    steps = digests()[cfg]["steps"]
    w = W.CONFIGS[cfg](steps)
    s = make_session(w)
    s.advance(steps, w.dt)
    check_digest(cfg, s)
    s.close()


def test_c4_full_size_bitwise_vs_reference():
    """1024^3 x 4 substrates, 1M cells, one GPU, 2 steps (34.4 GB field)."""
    steps = digests()["c4"]["steps"]
    w = W.c4(steps)
    s = make_session(w)
    s.advance(steps, w.dt)
    check_digest("c4", s)
    s.close()


def test_c5_full_stack_sampled_replicas_bitwise_vs_reference():
    """All 512 replicas in one stacked session; 8 sampled replicas pinned to the reference."""
    ws = [W.c5_replica(r, C5_STEPS) for r in range(W.C5_REPLICAS)]
    e = ensemble_session(ws)
    e.advance(C5_STEPS, ws[0].dt)
    per = ws[0].voxels * ws[0].S
    for r in C5_SAMPLE:
        check_digest(f"c5_r{r:03d}", e, r * per, per)
    e.close()


def test_spec_acceptance_2_backend_equivalence_size():
    """SPEC.md acceptance 2 at its size: 64^3 x 2, 25 agents, 1000 steps, bitwise."""
    w = spec511()
    s = make_session(w)
    s.advance(1000, w.dt)
    check_digest("spec511", s)
    s.close()


def max_rel_err(read_a, read_b, count, chunk=1 << 25):
    worst = 0.0
    a = np.empty(min(chunk, count))
    b = np.empty(min(chunk, count))
    for off in range(0, count, chunk):
        n = min(chunk, count - off)
        read_a(off, n, a)
        read_b(off, n, b)
        d = np.abs(a[:n] - b[:n]) / np.maximum(np.maximum(np.abs(a[:n]), np.abs(b[:n])), FLOOR)
        worst = max(worst, float(d.max()))
    return worst


@pytest.fixture(scope="module")
def c4_single():
    """The single-domain C4 solve after 3 steps (bitwise == the reference per the c4 digest test)."""
    w = W.c4(3)
    s = make_session(w)
    s.advance(3, w.dt)
    s.synchronize()
    yield w, s
    s.close()


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_c4_zslabs_match_single_domain(parts, c4_single):
    """C4 split into P in-process z-slabs on one GPU (the multi-GPU data path
    with peer copies for NCCL), 3 steps, vs the single domain: <= 1e-13."""
    w, single = c4_single
    g = ZSlabGroup(w, parts)
    g.advance(3)
    nx, ny, _ = w.n
    per_plane = nx * ny * w.S
    worst = 0.0
    for s, (z0, z1) in zip(g.sessions, g.ranges):
        cnt = (z1 - z0) * per_plane
        worst = max(worst, max_rel_err(lambda o, n, out: s.download_field_range(o, n, out),
                                       lambda o, n, out: single.download_field_range(z0 * per_plane + o, n, out),
                                       cnt))
    g.close()
    assert worst <= 1e-10, worst  # north_star
    assert worst <= 1e-13, worst  # rounding level


def test_c4_substrate_by_zslab_layout_4x2(c4_single):
    """The 8-GPU C4 layout (4 substrate shards x 2 z-slabs) in-process: every
    shard's columns within 1e-13 of the single domain (bitwise per shard
    would need the single-domain z solve; the 2 slabs re-associate)."""
    w, single = c4_single
    g = ShardGroup(w, 4, 2)
    g.advance(3)
    nx, ny, _ = w.n
    S = w.S
    worst = 0.0
    planes = 16
    for a, (s0, s1) in enumerate(g.s_ranges):
        for b, (z0, z1) in enumerate(g.z_ranges):
            sess = g.pieces[a][b]
            SL = s1 - s0
            for k in range(z0, z1, planes):
                k1 = min(k + planes, z1)
                nv = (k1 - k) * nx * ny
                loc = sess.download_field_range((k - z0) * nx * ny * SL, nv * SL).reshape(nv, SL)
                ref = single.download_field_range(k * nx * ny * S, nv * S).reshape(nv, S)[:, s0:s1]
                d = np.abs(loc - ref) / np.maximum(np.maximum(np.abs(loc), np.abs(ref)), FLOOR)
                worst = max(worst, float(d.max()))
    g.close()
    assert worst <= 1e-13, worst
