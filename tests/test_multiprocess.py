"""Multi-rank host logic on CPU (gloo, world_size 2): slot partitioning with global slot keys.

Each rank steps its slice [r*B, (r+1)*B) of one logical batch through the CPU oracle with
slot0 = r*B (exactly what bench.py does per GPU); the gathered per-rank fingerprints must equal
the single-process batch, and the NCCL-style scalar reductions (episode count SUM, time MAX) are
exercised with gloo.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, game, B, steps, out):
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sess = oracle.Session(game, B, 4, slot0=rank * B)
    eps = 0
    for _ in range(steps):
        cols = sess.b.columns(with_obs=False)
        assert sess.step(sess.sample_random_actions(cols)) == -1
        c = sess.b.columns(with_obs=False)
        eps += int((c["terminated"] | c["truncated"]).sum())
    fps = b"".join(sess.b.fingerprints())
    t = torch.tensor([eps], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    mx = torch.tensor([float(rank + 1)])
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, fps)
    if rank == 0:
        out.put((int(t.item()), float(mx.item()), b"".join(gathered)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("game", ["go_9x9", "backgammon"])
def test_two_rank_slices_equal_one_batch(oracle, game):
    world, B, steps = 2, 6, 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, game, B, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    eps, mx, fps = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = oracle.Session(game, world * B, 4)
    total = 0
    for _ in range(steps):
        cols = full.b.columns(with_obs=False)
        full.step(full.sample_random_actions(cols))
        c = full.b.columns(with_obs=False)
        total += int((c["terminated"] | c["truncated"]).sum())
    assert fps == b"".join(full.b.fingerprints())
    assert eps == total
    assert mx == float(world)
