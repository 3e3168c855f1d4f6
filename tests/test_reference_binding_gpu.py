"""INTEGRATION.md §1 compiled and run: the reference's own Microenvironment,
SolverWorkspaces and AgentPopulation (its headers and objects, oracle/_ref)
bound to libbiodiff_b200.so through include/biodiff_b200.h; 200 steps on the
GPU through the binding vs the reference's own diffuse_decay_step /
cell_sources_sinks_step loop on its WorkerPool, bit for bit
(tests/cpp/reference_binding.cpp, built by oracle/Makefile `binding`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "reference_binding")


@pytest.mark.gpu
def test_reference_types_bound_to_b200_match_reference_loop():
    if not os.path.exists(EXE):
        if os.path.isdir("/root/reference/proj/src"):
            import oracle
            oracle.build()
        else:
            pytest.skip("oracle/_ref/reference_binding not built (needs /root/reference where it is built)")
    r = subprocess.run([EXE, "200", "16"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 differ from the reference" in r.stdout
