"""The paper's validation methods (validation.cpp) in this repo: the host-side
writers must be byte-identical to the reference's (CPU tests), and Method 1
and the Method 3 mutant check must reproduce the reference's numbers when
the solves run on the B200 path (GPU tests)."""
import math

import numpy as np
import pytest

import oracle
import paper_2110_13368_b200 as B
from paper_2110_13368_b200 import validation as V
from paper_2110_13368_b200 import workloads as W

needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="reference build absent")


@needs_ref
def test_format_double_matches_std_to_chars():
    rng = np.random.default_rng(3)
    vals = [0.0, -0.0, 1.0, 38.0, 0.5, 1e-5, 1e-4, 123456.0, 1e21, 1e22, 1.5e-300, 5e-324, 2.2250738585072014e-308,
            123456789012345680000.0, 0.1, 1.0 / 3.0, 2.0 ** 60, 9007199254740993.0, 1e16, 1e15, 12345e-10,
            -7.25, 19.000000000000004]
    vals += list(rng.random(200) * 10.0 ** rng.integers(-320, 300, 200))
    vals += list(-rng.random(50) * 100)
    for v in vals:
        assert V.format_double(v) == oracle.ref_format_double(v), v


@needs_ref
@pytest.mark.parametrize("table", [True, False])
def test_snapshot_writers_byte_identical(table):
    w = W.make("snap", (13, 9, 7), 3, 0, 1)
    ref = oracle.Reference(w, dirichlet=False, agents=False)
    rng = np.random.default_rng(11)
    f = rng.random(ref.count) * 10.0 ** rng.integers(-5, 5, ref.count)
    ref.set_field(f)
    mesh = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    for s in range(3):
        for z in (0, 3, 6):
            mine = (V.write_snapshot_table if table else V.write_snapshot_pgm)(f, mesh, 3, s, z)
            assert mine == ref.snapshot(table, s, z)
    const = np.full(ref.count, 2.5)  # constant slice renders mid-gray 128
    ref.set_field(const)
    assert V.write_snapshot_pgm(const, mesh, 3, 1, 2) == ref.snapshot(False, 1, 2)


def test_cross_check_semantics_host():
    a = np.arange(12, dtype=float)
    b = a.copy()
    b[7] += 1e-3
    r = V.cross_check(a, b, 3, 1e-9, 1e-9)
    assert not r.passed and r.worst_value_index == 7 and r.worst_voxel == 2 and r.worst_substrate == 1
    assert V.cross_check(a, a, 3, 0.0, 0.0).passed


def _nan_inf_cases():
    """(a, b) pairs with NaN / Inf entries: ADVICE r01 — the reference's loop
    compares with NaN as false, so NaN differences neither fail nor count."""
    base = np.linspace(0.5, 3.0, 12)
    cases = []
    for ai, bi in [(np.nan, 1.0), (1.0, np.nan), (np.nan, np.nan), (np.inf, np.inf), (np.inf, 1.0),
                   (-np.inf, np.inf), (np.inf, np.nan)]:
        a, b = base.copy(), base.copy()
        a[4], b[4] = ai, bi
        cases.append((a, b))
        a2, b2 = a.copy(), b.copy()
        b2[9] += 1e-3  # plus one ordinary failing difference
        cases.append((a2, b2))
    return cases


@needs_ref
@pytest.mark.parametrize("tol", [(1e-9, 1e-9), (0.0, 0.0), (1e-2, 0.0)])
def test_cross_check_nan_inf_matches_reference_host(tol):
    for a, b in _nan_inf_cases():
        r = V.cross_check(a, b, 3, *tol)
        ma, mr, wi, ok = oracle.ref_cross_check(a, b, 3, *tol)
        assert (r.max_abs, r.max_rel, r.worst_value_index, r.passed) == (ma, mr, wi, ok), (a, b)


def test_analytic_solution_values():
    assert V.analytic_solution_1d(0.0, 0.0, 1000.0, 2000.0, 1) == 2.0
    assert abs(V.analytic_solution_1d(500.0, 1e6, 1000.0, 2000.0, 4) - 1.0) < 1e-12


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("kind,code", [("temporal", 0), ("spatial", 1)])
def test_method1_convergence_on_gpu_matches_reference(kind, code):
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    rep = V.run_convergence_test(kind, 4)
    order, steps, errors, passed = oracle.ref_convergence(code, 4)
    assert rep.passed and passed
    assert np.array_equal(np.array(rep.steps), steps)
    assert np.array_equal(np.array(rep.errors), errors), (rep.errors, errors)  # bit-identical solves
    assert rep.fitted_order == order


@pytest.mark.gpu
@needs_ref
def test_method3_mutant_check_on_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    r = V.run_dirichlet_mutant_check()
    assert r.passed, r
    assert oracle.ref_mutant_check() == (True, True, True)
    # The clean GPU field equals the reference's own clean run, bit for bit.
    mesh, f = V.mutant_scenario_run(False)
    w = W.make("mutant", 16, 1, 0, 100)
    w.substrates = [("factor", 1000.0, 0.1, 1.0, None)]
    ref = oracle.Reference(w, dirichlet=False, agents=False)
    centre = B.nearest_voxel(mesh, [0.0, 0.0, 0.0])
    oracle._rchk(oracle.ref_lib().ref_add_dirichlet(
        ref.h, 1, np.array([centre], np.int64).ctypes.data_as(oracle._P(oracle._i64)),
        np.array([1], np.uint8).ctypes.data_as(oracle._P(oracle._u8)),
        np.array([38.0]).ctypes.data_as(oracle._P(oracle._d))))
    ref.apply_dirichlet()
    ref.run(100, with_sources=False)
    want = ref.field()
    assert np.array_equal(f.view(np.int64), want.view(np.int64))
    assert V.write_snapshot_table(f, mesh, 1, 0, 8) == ref.snapshot(True, 0, 8)
