"""GPU, several processes: the one-slab-per-rank step (DeviceSession::
slab_step_nccl — the phases, plane pieces and send/receive order the NCCL
path runs) with the planes moved by the host transport over a gloo process
group. 2-4 processes share the one GPU; rank 0 gathers the pieces and
compares with a single-domain session (north_star 1e-10 asserted, rounding
level 1e-13 required; the substrate-only split must be bitwise)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import paper_2110_13368_b200 as B

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, k, shape, S, steps, pieces, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BIODIFF_ZSLAB_MIN_PIECE=str(pieces))
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2110_13368_b200 import workloads as W
        from paper_2110_13368_b200.shards import ShardRank
        w = W.make("xport", shape, S, 600, steps, seed=11 + world, immune_fraction=0.2, interior_clamps=6)
        r = ShardRank(w, rank, world, 0, substrate_parts=k, transport="host")
        r.advance(steps)
        out = np.zeros(w.voxels * w.S)
        r.session.download_field_global(out)
        # gather: every piece writes its planes / columns; a NaN-free sum works
        # because the pieces are disjoint and the rest is zero
        t = torch.from_numpy(out)
        dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)
        if rank == 0:
            from tests.helpers import make_session
            single = make_session(w)
            single.advance(steps, w.dt)
            want = single.download_field()
            got = t.numpy()
            d = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1e-290)
            q.put(("ok", float(d.max()), bool(np.array_equal(got.view(np.int64), want.view(np.int64))),
                   r.P, r.session.launch_count()))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # reported to the parent
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}", False, 0, 0))
        raise


@pytest.mark.parametrize("world,k,shape,S,pieces", [
    (2, 1, (20, 16, 48), 2, 64),   # 2 z-slabs, several plane pieces per exchange
    (3, 1, (16, 12, 45), 3, 1 << 20),
    (4, 2, (16, 16, 40), 4, 128),  # 2 substrate shards x 2 z-slabs
    (2, 2, (16, 16, 24), 4, 1 << 20),  # substrate shards only: no exchange, bitwise
])
def test_host_transport_ranks_match_single_domain(world, k, shape, S, pieces):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, shape, S, 6, pieces, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        status, err, bitwise, P, launches = q.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert status == "ok", err
    assert launches > 0
    if P == 1:
        assert bitwise
    else:
        assert err <= 1e-10, err
        assert err <= 1e-13, err
    assert all(p.exitcode == 0 for p in procs)
