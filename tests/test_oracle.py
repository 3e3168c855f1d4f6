"""CPU: pins the C restatement (oracle/biodiff_oracle.c) against the
reference itself (oracle/_ref, compiled from /root/reference) and against the
committed golden fixtures generated from the reference
(tests/golden/make_golden.py). Bit equality throughout."""
import numpy as np
import pytest

import oracle
from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from tests.helpers import bits_equal, first_diff, golden_names, load_golden

needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="reference build absent")


@pytest.mark.parametrize("name", golden_names())
def test_oracle_reproduces_golden(name):
    w, z = load_golden(name)
    rho = Oracle.run(w, w.steps, with_sources=bool(z["with_sources"]), initial_clamp=bool(z["initial_clamp"]))
    assert bits_equal(rho, z["field"]), first_diff(rho, z["field"])


@pytest.mark.parametrize("name", golden_names())
def test_oracle_coefficients_and_grouping_match_golden(name):
    w, z = load_golden(name)
    ws = Oracle.workspaces(w.n, (w.dx,) * 3, w.diffusion, w.decay, w.dt)
    for ax in range(3):
        if f"ws{ax}_q" in z:
            q, d, c = ws[ax]
            assert bits_equal(q, z[f"ws{ax}_q"]) and bits_equal(d, z[f"ws{ax}_dinv"]) and bits_equal(c, z[f"ws{ax}_cb"])
        else:
            assert ax not in ws
    dv, dm, dx_ = w.dirichlet_entries()
    assert np.array_equal(dv, z["dir_voxels"]) and np.array_equal(dm, z["dir_mask"])
    assert bits_equal(dx_, z["dir_values"])
    if w.n_agents:
        gv, go, order = Oracle.group(w.agent_ids, w.agent_pos, w.bounds(), (w.dx,) * 3, w.n)
        assert np.array_equal(gv, z["group_voxel"])
        assert np.array_equal(go, z["group_offsets"])
        assert np.array_equal(order, z["group_order"])


SHAPES = [((9, 7, 5), 1), ((12, 10, 9), 3), ((16, 1, 1), 2), ((10, 8, 1), 2), ((1, 6, 7), 1), ((5, 1, 9), 4),
          ((1, 1, 1), 2), ((2, 2, 2), 1)]


@needs_ref
@pytest.mark.parametrize("shape,S", SHAPES)
def test_oracle_sweeps_match_reference(shape, S):
    w = W.make("t", shape, S, 0, 1, seed=3)
    ref = oracle.Reference(w, dirichlet=False, agents=False)
    rng = np.random.default_rng(5)
    f0 = rng.random(ref.count) * 10
    ws = Oracle.workspaces(shape, (w.dx,) * 3, w.diffusion, w.decay, w.dt)
    for ax in ws:
        ref.set_field(f0)
        ref.sweep(ax)
        mine = f0.copy()
        Oracle.sweep(mine, shape, S, ax, ws[ax])
        assert bits_equal(mine, ref.field()), first_diff(mine, ref.field())


@needs_ref
@pytest.mark.parametrize("workers", [0, 1, 3, 8])
def test_oracle_full_steps_match_reference_any_worker_count(workers):
    w = W.make("t", (14, 11, 9), 3, 150, 1, seed=9, immune_fraction=0.2, interior_clamps=7)
    ref = oracle.Reference(w, workers=workers)
    ref.run(15)
    mine = Oracle.run(w, 15)
    assert bits_equal(mine, ref.field()), first_diff(mine, ref.field())


@needs_ref
def test_oracle_grouping_matches_reference_with_collisions():
    w = W.make("t", (8, 8, 8), 2, 400, 1, seed=21)  # dense core -> many agents per voxel
    ref = oracle.Reference(w)
    gv, go, order = ref.grouping()
    mine = Oracle.group(w.agent_ids, w.agent_pos, w.bounds(), (w.dx,) * 3, w.n)
    assert np.array_equal(gv, mine[0]) and np.array_equal(go, mine[1]) and np.array_equal(order, mine[2])
    assert (np.diff(go) > 1).any(), "workload must exercise voxel collisions"


@needs_ref
def test_reference_validation_methods_pass():
    """Method 1 and the Method 3 mutant check of the reference itself
    (validation.cpp:65-110, 274-287) — pins the build of oracle/_ref."""
    order_t, _, errs_t, pass_t = oracle.ref_convergence(0, 4)
    order_s, _, errs_s, pass_s = oracle.ref_convergence(1, 4)
    assert pass_t and 0.8 <= order_t <= 1.2
    assert pass_s and 1.7 <= order_s <= 2.3
    assert oracle.ref_mutant_check() == (True, True, True)


# ---- SPEC known-answer examples, on the oracle -----------------------------

def test_spec_decay_only_product_exact():
    """D=0, lambda=3, dt=0.01, dims=3 -> 1/(1.01)^3 as three rounded multiplies."""
    q, dinv, cb = Oracle.precompute(4, [0.0], [3.0], 20.0, 0.01, 3)
    assert q[0] == 0.0 and np.all(cb == 0.0)
    assert np.all(dinv == 1.0 / 1.01)
    w = W.make("t", (4, 4, 4), 1, 0, 1)
    w.substrates = [("x", 0.0, 3.0, 1.0, None)]
    rho = Oracle.run(w, 1)
    assert np.all(rho == 0.97059014792764442)


def test_spec_uniform_steady_state_and_zero_field():
    w = W.make("t", (6, 5, 4), 2, 0, 1)
    w.substrates = [("a", 1e5, 0.0, 7.0, None), ("b", 10.0, 0.0, 0.0, None)]
    rho = Oracle.run(w, 5)
    assert np.allclose(rho[0::2], 7.0, rtol=0, atol=1e-12)
    assert np.all(rho[1::2] == 0.0)


def test_spec_mass_conservation_32cubed():
    """SPEC.md:184 (lambda=0, no Dirichlet, no agents): relative mass drift <= 1e-12 (1000 steps)."""
    w = W.make("t", 32, 1, 0, 1)
    w.substrates = [("a", 1000.0, 0.0, 0.0, None)]
    rng = np.random.default_rng(1)
    f0 = rng.random(w.voxels)
    rho = Oracle.run(w, 1000, field=f0)
    assert abs(rho.sum() - f0.sum()) <= 1e-12 * f0.sum()


def test_spec_reaction_fixed_point_19():
    """one agent S=1, U=1, rho*=38 -> 19 within 1e-9 by t=60 min (D=0, lambda=0)."""
    w = W.make("t", (3, 3, 3), 1, 0, 1)
    w.substrates = [("a", 0.0, 0.0, 0.0, None)]
    w.agent_ids = np.array([0])
    w.agent_pos = np.zeros((1, 3))
    w.agent_vol = np.array([w.dx ** 3])
    w.agent_sec = np.array([[1.0]])
    w.agent_upt = np.array([[1.0]])
    w.agent_sat = np.array([[38.0]])
    rho = Oracle.run(w, 6000)
    assert abs(rho[13] - 19.0) <= 1e-9
    assert np.all(np.delete(rho, 13) == 0.0)


def test_spec_dirichlet_mask_semantics():
    """mask [1,0], values [5,9] -> s0 = 5, s1 untouched."""
    rho = np.array([1.0, 2.0, 3.0, 4.0])
    Oracle.dirichlet(rho, 2, np.array([1]), np.array([[1, 0]], np.uint8), np.array([[5.0, 9.0]]))
    assert rho.tolist() == [1.0, 2.0, 5.0, 4.0]
