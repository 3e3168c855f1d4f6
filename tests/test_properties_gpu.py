"""SPEC.md invariants and examples checked on the GPU path (through the C
ABI): the maximum principle, decay-only exactness, the pure-diffusion steady
state, line mass conservation and symmetry, and the source
step's locality, boundedness, determinism and commutation.
The bitwise comparisons against the reference live in test_gpu_parity.py /
test_long_parity_gpu.py; these are the properties the reference documents
for its own operators."""
import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from tests.helpers import bits_equal, make_session

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")


def workload(n, subs, dt=0.01, dx=20.0):
    w = W.Workload(name="prop", n=tuple(n), dx=dx, substrates=subs, dt=dt, steps=1)
    S = len(subs)
    w.agent_ids = np.zeros(0, np.int64)
    w.agent_pos = np.zeros((0, 3))
    w.agent_vol = np.zeros(0)
    w.agent_sec = np.zeros((0, S))
    w.agent_upt = np.zeros((0, S))
    w.agent_sat = np.zeros((0, S))
    return w


@pytest.mark.parametrize("path", ["auto", "graphless"])
def test_maximum_principle(path, monkeypatch):
    """lambda >= 0, no sources, no Dirichlet: max(field) never
    increases and min(field) stays >= 0 across steps."""
    if path == "graphless":
        monkeypatch.setenv("BIODIFF_NO_GRAPH", "1")
    w = workload((28, 24, 20), [("a", 1e5, 0.1, 0.0, None), ("b", 3e2, 0.0, 0.0, None), ("c", 0.0, 2.0, 0.0, None)])
    rng = np.random.default_rng(7)
    f = rng.random(w.voxels * w.S) * 50.0
    s = make_session(w)
    s.upload_field(f)
    prev = f.reshape(-1, w.S)
    for _ in range(25):
        s.diffuse_decay_step()
        cur = s.download_field().reshape(-1, w.S)
        assert np.all(cur.max(axis=0) <= prev.max(axis=0))
        assert cur.min() >= 0.0
        prev = cur
    s.close()


def test_decay_only_is_the_product_of_the_split_factors():
    """D = 0, lambda > 0: every value is multiplied by the x, y and
    z pivots (1 / (1 + dt*lambda/dims)) in that order — bit for bit."""
    w = workload((12, 10, 9), [("a", 0.0, 3.0, 0.0, None), ("b", 0.0, 0.25, 0.0, None)])
    ws = Oracle.workspaces(w.n, (w.dx,) * 3, w.diffusion, w.decay, w.dt)
    rng = np.random.default_rng(8)
    f = rng.random(w.voxels * w.S) * 10.0
    s = make_session(w)
    s.upload_field(f)
    s.diffuse_decay_step()
    got = s.download_field()
    s.close()
    want = f.reshape(-1, w.S).copy()
    for ax in range(3):
        dinv = np.asarray(ws[ax][1]).reshape(-1, w.S)[0]  # row 0 pivot (every row equal when D = 0)
        want = want * dinv
    assert bits_equal(got, want.reshape(-1))


def test_uniform_field_is_a_steady_state_of_pure_diffusion_and_zero_stays_zero():
    """SPEC.md:150-152 / 162: uniform field, lambda = 0, zero-flux boundaries:
    unchanged (to rounding); the zero field stays exactly zero."""
    w = workload((20, 18, 16), [("a", 1e5, 0.0, 0.0, None), ("b", 1e3, 0.0, 0.0, None)])
    s = make_session(w)
    s.upload_field(np.full(w.voxels * w.S, 38.0))
    for _ in range(10):
        s.diffuse_decay_step()
    got = s.download_field()
    assert np.max(np.abs(got - 38.0)) <= 1e-12 * 38.0
    s.upload_field(np.zeros(w.voxels * w.S))
    s.diffuse_decay_step()
    assert not np.any(s.download_field())
    s.close()


def test_spike_line_mass_conserved_and_symmetric_line_stays_symmetric():
    """a single-voxel spike on a 16-point line conserves the
    line mass (lambda = 0) to 1e-13; a symmetric line stays symmetric."""
    w = workload((16, 1, 1), [("a", 1e5, 0.0, 0.0, None)])
    s = make_session(w)
    f = np.zeros(16)
    f[5] = 100.0
    s.upload_field(f)
    s.diffusion_sweep(0)
    got = s.download_field()
    assert abs(got.sum() - 100.0) <= 1e-13 * 100.0
    pal = np.array([1.0, 4.0, 9.0, 2.0, 7.0, 3.0, 8.0, 5.0])
    f = np.concatenate([pal, pal[::-1]])
    s.upload_field(f)
    s.diffusion_sweep(0)
    got = s.download_field()
    assert np.max(np.abs(got - got[::-1])) <= 1e-13 * np.max(np.abs(got))
    s.close()


def _agents(rng, w, n, S, collide=True):
    lo = np.array(w.bounds()[0::2])
    hi = np.array(w.bounds()[1::2])
    pos = lo + rng.random((n, 3)) * (hi - lo)
    if collide:  # several agents in a few voxels
        pos[: n // 4] = pos[0] + rng.random((n // 4, 3)) * 0.5
    ids = rng.permutation(n).astype(np.int64) * 3 + 1
    vol = 2494.0 * (0.5 + rng.random(n))
    sec = rng.random((n, S)) * 5.0
    upt = rng.random((n, S)) * 2.0
    sat = rng.random((n, S)) * 30.0
    upt[::7] = 0.0
    return ids, pos, vol, sec, upt, sat


def test_sources_locality_boundedness_and_commutation():
    """SPEC.md:249-252 for cell_sources_sinks_step on the GPU: voxels without
    agents are bitwise unchanged; every updated value lies within
    [min(rho_old, min S*rho*/(S+U)), max(rho_old, max rho*)]; the result does
    not depend on the order agents are handed over (per-voxel order is by id,
    distinct voxels commute) and is identical run to run."""
    rng = np.random.default_rng(11)
    w = workload((16, 14, 12), [("a", 1e5, 0.1, 0.0, None), ("b", 1e3, 0.01, 0.0, None)])
    S = w.S
    ids, pos, vol, sec, upt, sat = _agents(rng, w, 400, S)
    f = rng.random(w.voxels * S) * 40.0

    def run(perm):
        s = make_session(w)
        s.set_agents(ids[perm], pos[perm], vol[perm], sec[perm], upt[perm], sat[perm])
        s.upload_field(f)
        s.cell_sources_sinks_step(w.dt)
        out = s.download_field()
        s.close()
        return out

    base = run(np.arange(len(ids)))
    assert bits_equal(base, run(np.arange(len(ids))))          # determinism
    assert bits_equal(base, run(rng.permutation(len(ids))))    # input order / commutation
    mesh = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    vox = np.array([B.nearest_voxel(mesh, p) for p in pos]) if hasattr(B, "nearest_voxel") else None
    if vox is None:
        lo = np.array(w.bounds()[0::2])
        ijk = np.clip(np.floor((pos - lo) / w.dx).astype(int), 0, np.array(w.n) - 1)
        vox = ijk[:, 0] + w.n[0] * (ijk[:, 1] + w.n[1] * ijk[:, 2])
    occupied = np.zeros(w.voxels, bool)
    occupied[vox] = True
    old = f.reshape(-1, S)
    new = base.reshape(-1, S)
    assert bits_equal(new[~occupied], old[~occupied])               # locality
    for v in np.flatnonzero(occupied):
        members = vox == v
        for s_ in range(S):
            su = sec[members, s_] + upt[members, s_]
            fixed = np.where(su > 0, sec[members, s_] * sat[members, s_] / np.where(su > 0, su, 1.0), np.inf)
            lo_b = min(old[v, s_], fixed.min()) if np.isfinite(fixed.min()) else old[v, s_]
            hi_b = max(old[v, s_], sat[members, s_].max())
            assert lo_b - 1e-12 * abs(lo_b) <= new[v, s_] <= hi_b + 1e-12 * abs(hi_b)   # boundedness
