"""bench.py's rank bookkeeping dry-run on CPU (gloo, world_size 2): the shard plan (weak and strong
scaling, global slot offsets) and the only collectives of the benchmark (MAX of the timed region,
SUM of the episode counters), exercised through bench.py's own functions."""

import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import bench as bm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    weak = bm.shard_plan("go_19x19", 0, 0, rank, world)
    strong = bm.shard_plan("backgammon", 0, 1 << 17, rank, world)
    ms, eps = bm.reduce_over_ranks(10.0 + rank, torch.tensor([100 + rank], dtype=torch.int64), world,
                                   torch.device("cpu"))
    if rank == 0:
        out.put((weak, strong, ms, eps))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_plan_and_reductions_over_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    weak, strong, ms, eps = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert weak == {"B": 1 << 17, "slot0": 0, "scaling": "weak", "global_batch": 1 << 18}
    assert strong == {"B": 1 << 16, "slot0": 0, "scaling": "strong", "global_batch": 1 << 17}
    assert ms == 11.0 and eps == 201


def test_shard_plan_slot_offsets():
    assert bench.shard_plan("backgammon", 0, 1 << 17, 3, 8) == {"B": 1 << 14, "slot0": 3 << 14, "scaling": "strong",
                                                                  "global_batch": 1 << 17}
    assert bench.shard_plan("chess", 0, 0, 5, 8)["slot0"] == 5 << 17
    with pytest.raises(SystemExit):
        bench.shard_plan("backgammon", 0, 1000, 0, 3)


def test_host_random_actions_matches_the_oracle_sampler(oracle):
    import numpy as np

    rng = np.random.default_rng(0)
    mask = rng.random((257, 82)) < 0.3
    mask[5] = False
    for ks, s0 in ((0x1234, 0), (0xDEADBEEF, 1000)):
        assert np.array_equal(bench.host_random_actions(mask, ks, s0), oracle.random_actions(mask, ks, s0))
