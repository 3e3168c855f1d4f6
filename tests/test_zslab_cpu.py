"""CPU, multi-process: the z-slab decomposition protocol of csrc/slab.cu,
restated with the oracle's line solver, run by world_size-2 (and 3) gloo
process groups that exchange the interface planes with torch.distributed
send/recv exactly in the order the NCCL path does (pieces of the planes):
    x, y sweeps ; interface pre-pass: dhat, xhat_0 with zero inflow (one read)
    recv D_{p-1} <- p-1 ; D_p = dhat_p + phi_last * D_{p-1} ; send D_p -> p+1
    recv X_{p+1} <- p+1 ; X_p = xhat_0 + Phi_0 D_{p-1} + Psi_0 X_{p+1} ; send X_p -> p-1
    z solve with inflows D_{p-1} (row 0) and X_{p+1} (last row) ; Dirichlet ; sources
The gathered result must match the single-domain oracle run to rounding."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import Oracle
from paper_2110_13368_b200 import workloads as W
from paper_2110_13368_b200.zslab import split_planes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spikes(q, dinv, cb, n, S):
    phi = np.zeros((n, S))
    Phi = np.zeros((n, S))
    psi = np.zeros((n, S))
    for s in range(S):
        f = 1.0
        for m in range(n):
            f = (0.0 + q[s] * f) * dinv[m, s]
            phi[m, s] = f
        Phi[n - 1, s] = phi[n - 1, s]
        for m in range(n - 2, -1, -1):
            Phi[m, s] = phi[m, s] + cb[m, s] * Phi[m + 1, s]
        g = cb[n - 1, s] * 1.0
        psi[n - 1, s] = g
        for m in range(n - 2, -1, -1):
            g = cb[m, s] * g
            psi[m, s] = g
    return Phi, psi, phi[n - 1].copy()


def interface(r3, q, d, c, S):
    """zslab_interface: dhat (last-row forward) and xhat_0 = sum_m prod_{k<m} cb_k f_m, zero inflow."""
    n, plane = r3.shape
    s = np.arange(plane) % S
    f = np.zeros(plane)
    acc = np.zeros(plane)
    prod = np.ones(plane)
    for m in range(n):
        f = r3[m] * d[m, s] if m == 0 else (r3[m] + q[s] * f) * d[m, s]
        acc = acc + prod * f
        prod = prod * c[m, s]
    return f, acc


def z_solve_inflow(r3, q, d, c, S, d_in, x_in):
    """The global z recurrence on the slab: row 0 continues from d_in, the last row takes x_in."""
    n, plane = r3.shape
    s = np.arange(plane) % S
    f = np.empty_like(r3)
    for m in range(n):
        prev = (d_in if d_in is not None else None) if m == 0 else f[m - 1]
        f[m] = r3[m] * d[m, s] if (m == 0 and d_in is None) else (r3[m] + q[s] * prev) * d[m, s]
    x = f[n - 1] + c[n - 1, s] * x_in if x_in is not None else f[n - 1]
    r3[n - 1] = x
    for m in range(n - 2, -1, -1):
        x = f[m] + c[m, s] * x
        r3[m] = x


def _rank_main(rank, world, port, w, steps, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    nx, ny, nz = w.n
    S = w.S
    z0, z1 = split_planes(nz, world)[rank]
    n = z1 - z0
    plane = nx * ny * S
    h = (w.dx,) * 3
    ws = Oracle.workspaces(w.n, h, w.diffusion, w.decay, w.dt)
    qz, dz, cz = ws[2]
    dz = dz.reshape(nz, S)[z0:z1].copy()
    cz = cz.reshape(nz, S)[z0:z1].copy()
    Phi, psi, phi_last = spikes(qz, dz, cz, n, S)
    dv, dm, dx_ = w.dirichlet_entries()
    sel = (dv >= z0 * nx * ny) & (dv < z1 * nx * ny)
    dv, dm, dx_ = dv[sel] - z0 * nx * ny, dm[sel], dx_[sel]
    gv, go, order = Oracle.group(w.agent_ids, w.agent_pos, w.bounds(), h, w.n)
    keep = (gv >= z0 * nx * ny) & (gv < z1 * nx * ny)
    idx = np.flatnonzero(keep)
    lgv = gv[idx] - z0 * nx * ny
    lgo = np.zeros(idx.size + 1, np.int64)
    lorder = []
    for t, g in enumerate(idx):
        members = order[go[g]:go[g + 1]]
        lorder.extend(members)
        lgo[t + 1] = lgo[t] + members.size
    lorder = np.array(lorder, np.int64)
    rho = np.tile(w.initial, nx * ny * n)
    inv_vox = 1.0 / (w.dx ** 3)
    shape = (nx, ny, n)
    for _ in range(steps):
        Oracle.sweep(rho, shape, S, 0, ws[0])
        Oracle.sweep(rho, shape, S, 1, ws[1])
        r3 = rho.reshape(n, plane)
        dhat, xhat0 = interface(r3, qz, dz, cz, S)
        d_in = torch.zeros(plane, dtype=torch.float64)
        x_in = torch.zeros(plane, dtype=torch.float64)
        pieces = np.array_split(np.arange(plane // S), 3)  # whole columns, as DeviceSession::plane_pieces
        for pc in pieces:  # forward chain, piece by piece
            sl = slice(pc[0] * S, (pc[-1] + 1) * S)
            if rank > 0:
                buf = torch.zeros(sl.stop - sl.start, dtype=torch.float64)
                dist.recv(buf, src=rank - 1)
                d_in[sl] = buf
            if rank < world - 1:
                dout = dhat[sl] + np.tile(phi_last, pc.size) * d_in[sl].numpy()
                dist.send(torch.from_numpy(dout), dst=rank + 1)
        for pc in pieces:  # backward chain
            sl = slice(pc[0] * S, (pc[-1] + 1) * S)
            if rank < world - 1:
                buf = torch.zeros(sl.stop - sl.start, dtype=torch.float64)
                dist.recv(buf, src=rank + 1)
                x_in[sl] = buf
            if rank > 0:
                xout = (xhat0[sl] + np.tile(Phi[0], pc.size) * d_in[sl].numpy()
                        + np.tile(psi[0], pc.size) * x_in[sl].numpy())
                dist.send(torch.from_numpy(xout), dst=rank - 1)
        z_solve_inflow(r3, qz, dz, cz, S, d_in.numpy() if rank > 0 else None,
                       x_in.numpy() if rank < world - 1 else None)
        Oracle.dirichlet(rho, S, dv, dm, dx_)
        if lgv.size:
            Oracle.sources(rho, S, (lgv, lgo, lorder), w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat,
                           w.dt, inv_vox)
    sizes = [split_planes(nz, world)[r][1] - split_planes(nz, world)[r][0] for r in range(world)]
    if rank == 0:
        parts = [torch.from_numpy(rho)]
        for r in range(1, world):
            buf = torch.zeros(nx * ny * sizes[r] * S, dtype=torch.float64)
            dist.recv(buf, src=r)
            parts.append(buf)
        np.save(out_path, torch.cat(parts).numpy())
    else:
        dist.send(torch.from_numpy(rho), dst=0)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,S,agents,steps", [(2, (10, 8, 24), 2, 120, 6), (3, (8, 8, 30), 3, 150, 5)])
def test_zslab_protocol_gloo_matches_single_domain(world, shape, S, agents, steps):
    w = W.make("zslab-cpu", shape, S, agents, steps, seed=world, immune_fraction=0.2, interior_clamps=4)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "field.npy")
        mp.spawn(_rank_main, args=(world, _free_port(), w, steps, out), nprocs=world, join=True)
        got = np.load(out)
    want = Oracle.run(w, steps)
    diff = np.abs(got - want)
    mag = np.maximum(np.abs(got), np.abs(want))
    rel = np.where(mag > 0, diff / np.where(mag > 0, mag, 1), 0)
    assert rel.max() <= 1e-13, rel.max()
