"""The C++ host mirror (csrc/host.hpp) used the way the reference's own C++
callers use its API, compiled with g++ against libbiodiff_b200.so, checked
against the reference build (set-up artefacts, CPU) and the oracle (device
steps, GPU)."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_2110_13368_b200 as B
from oracle import Oracle
from tests.helpers import first_diff

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "host_api_driver.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "host_api_driver")


@pytest.fixture(scope="module")
def driver():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(os.path.getmtime(SRC), os.path.getmtime(B.LIB_PATH)):
        libdir = os.path.dirname(B.LIB_PATH)
        subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "paper_2110_13368_b200", "csrc"),
                        SRC, "-o", EXE, f"-L{libdir}", "-lbiodiff_b200", f"-Wl,-rpath,{libdir}"], check=True)
    return EXE


def _mesh_workload():
    """The same microenvironment in the oracle's terms."""
    from paper_2110_13368_b200 import workloads as W
    w = W.make("cpp", (20, 18, 16), 2, 0, 25)
    w.substrates = [("oxygen", 1e5, 0.1, 38.0, 38.0), ("factor", 1e3, 0.016, 0.0, None)]
    return w


def test_host_setup_matches_reference(driver, tmp_path):
    out = tmp_path / "cpu.bin"
    r = subprocess.run([driver, "cpu", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "dirichlet=" in r.stdout
    raw = np.fromfile(out, dtype=np.uint8)
    w = _mesh_workload()
    ws = Oracle.workspaces(w.n, (w.dx,) * 3, w.diffusion, w.decay, w.dt)
    off = 0
    for ax in range(3):
        for arr in ws[ax]:
            nbytes = arr.size * 8
            got = raw[off:off + nbytes].view(np.float64)
            assert np.array_equal(got.view(np.int64), np.ascontiguousarray(arr).view(np.int64))
            off += nbytes
    assert off < raw.size  # grouping follows


@pytest.mark.gpu
def test_host_api_device_run_matches_oracle(driver, tmp_path):
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    out = tmp_path / "gpu.bin"
    r = subprocess.run([driver, "gpu", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(out, dtype=np.float64)
    # The driver places agents with std::mt19937_64; the oracle replays the run
    # from the driver's own grouping dump (cpu mode) and the same parameters.
    cpu = tmp_path / "cpu.bin"
    subprocess.run([driver, "cpu", str(cpu)], check=True, capture_output=True)
    w = _mesh_workload()
    rho = w.initial_field()
    h = (w.dx,) * 3
    ws = Oracle.workspaces(w.n, h, w.diffusion, w.decay, w.dt)
    # Dirichlet: boundary oxygen 38 + one interior clamp of the factor.
    dv, dm, dx_ = w.dirichlet_entries()
    nx, ny, nz = w.n
    extra = 7 + 5 * nx + 4 * nx * ny
    dv = np.append(dv, extra)
    dm = np.vstack([dm, [[0, 1]]]).astype(np.uint8)
    dx_ = np.vstack([dx_, [[0.0, 2.5]]])
    order = np.argsort(dv, kind="stable")
    dv, dm, dx_ = dv[order], dm[order], dx_[order]
    raw = np.fromfile(cpu, dtype=np.uint8)
    off = sum(a.size * 8 for ax in range(3) for a in ws[ax])
    ints = raw[off:].view(np.int64)
    gv, go, ordr = [], [0], []
    p = 0
    while p < ints.size:
        v, n = ints[p], ints[p + 1]
        gv.append(v)
        ordr.extend(ints[p + 2:p + 2 + n])
        go.append(go[-1] + n)
        p += 2 + n
    grouping = (np.array(gv, np.int64), np.array(go, np.int64), np.array(ordr, np.int64))
    N = 150
    vol = np.full(N, 2494.0)
    sec = np.tile([0.0, 1.0], N)
    upt = np.tile([10.0, 0.1], N)
    sat = np.tile([0.0, 1.0], N)
    for _ in range(25):
        for ax in range(3):
            Oracle.sweep(rho, w.n, 2, ax, ws[ax])
        Oracle.dirichlet(rho, 2, dv, dm, dx_)
        Oracle.sources(rho, 2, grouping, vol, sec, upt, sat, w.dt, 1.0 / w.dx ** 3)
    assert np.array_equal(got.view(np.int64), rho.view(np.int64)), first_diff(got, rho)
