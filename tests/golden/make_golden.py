"""Generates tests/golden/*.npz from the REFERENCE ITSELF.

Run in a container where /root/reference exists (the reference is compiled
from its own sources by oracle/Makefile into oracle/_ref/libbiodiff_ref.so):

    python tests/golden/make_golden.py

Each fixture stores the complete inputs (mesh, substrate parameters, dt,
steps, Dirichlet entries, agent arrays) and the reference's outputs (final
field after `steps` x [diffuse_decay_step; cell_sources_sinks_step],
SPEC.md:297; the x/y/z workspaces; the Dirichlet map and agent grouping as
the reference canonicalised them). The tests replay the inputs through the
C restatement (CPU) and the CUDA library (GPU) and require bit equality.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2110_13368_b200 import workloads as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cases():
    # The reference's built-in mutant scenario (validation.cpp:244-262):
    # 16^3, D=1000, lambda=0.1, IC 1, centre clamp 38, dt 0.01, initial clamp, 100 steps.
    w = W.make("mutant16", 16, 1, 0, 100)
    w.substrates = [("factor", 1000.0, 0.1, 1.0, None)]
    centre = 8 + 8 * 16 + 8 * 256  # nearest_voxel((0,0,0)) on [-160,160]^3, h=20
    w.interior_dirichlet = (np.array([centre], np.int64), np.array([[1]], np.uint8), np.array([[38.0]]))
    yield "mutant16", w, True, False
    yield "c1_mini", W.make("c1_mini", 16, 1, 60, 30, seed=7), False, True
    yield "c2_mini", W.make("c2_mini", (20, 18, 16), 2, 300, 20, seed=11, immune_fraction=0.1,
                            interior_clamps=6), False, True
    yield "c3_mini", W.make("c3_mini", (24, 20, 18), 4, 800, 10, seed=13, immune_fraction=0.1,
                            interior_clamps=10), False, True
    yield "flat2d", W.make("flat2d", (24, 20, 1), 3, 100, 40, seed=17, interior_clamps=4), False, True
    yield "line1d", W.make("line1d", (64, 1, 1), 2, 20, 50, seed=19), False, True
    yield "odd_rowlen", W.make("odd_rowlen", (17, 9, 11), 1, 40, 25, seed=23, interior_clamps=3), False, True
    yield "long_x", W.make("long_x", (300, 6, 5), 2, 50, 8, seed=29), False, True


def main():
    oracle.build(quiet=True)
    for name, w, initial_clamp, with_sources in cases():
        ref = oracle.Reference(w)
        if initial_clamp:
            ref.apply_dirichlet()
        ref.run(w.steps, with_sources=with_sources)
        field = ref.field()
        dv, dm, dx_ = ref.dirichlet()
        gv, go, order = ref.grouping() if w.n_agents else (np.zeros(0, np.int64),) * 3
        wsd = {}
        for ax in range(3):
            r = ref.workspace(ax)
            if r is not None:
                wsd[f"ws{ax}_q"], wsd[f"ws{ax}_dinv"], wsd[f"ws{ax}_cb"], wsd[f"ws{ax}_dims"] = r
        iv, im, ival = w.interior_dirichlet if w.interior_dirichlet is not None else (
            np.zeros(0, np.int64), np.zeros((0, w.S), np.uint8), np.zeros((0, w.S)))
        bm, bv = w.boundary_clamp()
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"),
            n=np.array(w.n), dx=w.dx, dt=w.dt, steps=w.steps,
            D=w.diffusion, lam=w.decay, ic=w.initial, boundary_mask=bm, boundary_values=bv,
            interior_voxels=iv, interior_mask=im, interior_values=ival,
            agent_ids=w.agent_ids, agent_pos=w.agent_pos, agent_vol=w.agent_vol,
            agent_sec=w.agent_sec, agent_upt=w.agent_upt, agent_sat=w.agent_sat,
            initial_clamp=initial_clamp, with_sources=with_sources,
            field=field, dir_voxels=dv, dir_mask=dm, dir_values=dx_,
            group_voxel=gv, group_offsets=go, group_order=order, **wsd)
        ref.close()
        print(f"{name}: {w.n} S={w.S} steps={w.steps} agents={w.n_agents} dirichlet={dv.size} "
              f"range=[{field.min():.6g}, {field.max():.6g}]")


if __name__ == "__main__":
    main()
