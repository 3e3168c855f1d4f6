"""CPU: the C-ABI library loads, exports every entry point include/biodiff_b200.h
declares, and its host-side helpers (no device work) reproduce the
reference's bits; sessions refuse to run without an sm_100 device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2110_13368_b200 as B
from paper_2110_13368_b200 import workloads as W
from tests.helpers import bits_equal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "biodiff_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int32_t|const char\*)\s+(biodiff_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = B.lib()
    for n in names:
        assert getattr(lib, n) is not None
    assert set(B.EXPORTED_SYMBOLS) == set(names)


def test_library_is_sm100a_cuda_code():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", B.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass, "bulk async copies (cp.async.bulk) expected in the sweep kernels"


def test_version():
    assert B.lib().biodiff_version() == 10000


def test_mesh_from_bounds_matches_reference_rules():
    m = B.mesh_from_bounds(-1000, 1000, -1000, 1000, -1000, 1000, 20, 20, 20)
    assert m.shape == (100, 100, 100)
    m = B.mesh_from_bounds(0, 105, 0, 10, 0, 10, 10, 10, 10)  # llround(10.5) = 11, upper bound snapped
    assert m.nx == 11 and m.x_max == 110.0
    with pytest.raises(B.ConfigError):
        B.mesh_from_bounds(0, 1, 0, 1, 0, 1, 0, 1, 1)
    with pytest.raises(B.ConfigError):
        B.mesh_from_bounds(0, 1, 0, 100, 0, 100, 20, 20, 20)


def test_nearest_voxel_rules():
    m = B.mesh_from_bounds(-160, 160, -160, 160, -160, 160, 20, 20, 20)
    assert B.nearest_voxel(m, [0, 0, 0]) == 8 + 8 * 16 + 8 * 256
    assert B.nearest_voxel(m, [-160, -160, -160]) == 0
    assert B.nearest_voxel(m, [160, 160, 160]) == 16 ** 3 - 1  # upper boundary clamps
    with pytest.raises(B.StateError):
        B.nearest_voxel(m, [161, 0, 0])
    rng = np.random.default_rng(0)
    h = (20.0, 20.0, 20.0)
    for p in rng.uniform(-160, 160, size=(200, 3)):
        assert B.nearest_voxel(m, p) == oracle.oracle_lib().orc_nearest_voxel(
            np.array(m.bounds()).ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            np.array(h).ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            np.array([16, 16, 16], np.int32).ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
            np.ascontiguousarray(p).ctypes.data_as(ctypes.POINTER(ctypes.c_double)))


@pytest.mark.parametrize("shape,S", [((50, 50, 50), 1), ((100, 100, 100), 2), ((256, 256, 256), 4),
                                     ((13, 1, 1), 3), ((10, 8, 1), 2)])
def test_precompute_matches_oracle_bits(shape, S):
    w = W.make("t", shape, S, 0, 1)
    m = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    dims = 1 + (shape[1] > 1) + (shape[2] > 1)
    for ax in range(3):
        q, d, c = B.precompute_thomas_coefficients(m, w.diffusion, w.decay, w.dt, ax, dims)
        oq, od, oc = oracle.Oracle.precompute(shape[ax], w.diffusion, w.decay, w.dx, w.dt, dims)
        assert bits_equal(q, oq) and bits_equal(d.ravel(), od) and bits_equal(c.ravel(), oc)


@pytest.mark.skipif(not oracle.reference_available(), reason="reference build absent")
def test_precompute_matches_reference_bits():
    w = W.make("t", (37, 23, 11), 4, 0, 1)
    ref = oracle.Reference(w, dirichlet=False, agents=False)
    m = B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)
    for ax in range(3):
        rq, rd, rc, dims = ref.workspace(ax)
        q, d, c = B.precompute_thomas_coefficients(m, w.diffusion, w.decay, w.dt, ax, dims)
        assert bits_equal(q, rq) and bits_equal(d.ravel(), rd) and bits_equal(c.ravel(), rc)


def test_precompute_argument_errors():
    m = B.mesh_from_bounds(0, 100, 0, 100, 0, 100, 20, 20, 20)
    with pytest.raises(B.StateError):  # std::invalid_argument -> status 2 (errors.hpp:19-22)
        B.precompute_thomas_coefficients(m, [1.0], [0.1], 0.0, 0, 3)
    with pytest.raises(B.StateError):
        B.precompute_thomas_coefficients(m, [1.0], [0.1], 0.01, 0, 4)


def test_session_needs_a_b200(gpu_available):
    if gpu_available:
        pytest.skip("GPU present; covered by the gpu suite")
    m = B.mesh_from_bounds(0, 100, 0, 100, 0, 100, 20, 20, 20)
    with pytest.raises(B.StateError, match="no CUDA device|sm_100|CUDA"):
        B.Session(m, 1)


def test_device_count_is_queryable():
    assert B.device_count() >= 0
