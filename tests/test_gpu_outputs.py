"""Zero-copy / binary batch_outputs agree with the host contract (bench.py:86-97)."""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("game", ["go_9x9", "go_19x19", "backgammon", "chess", "shogi"])
def test_outputs_device_dlpack_and_wire(game):
    import torch

    sess = bb.BatchSession(game, 37, 3)
    for _ in range(9):
        sess.step(sess.sample_random_actions())
    b = sess.batch
    host = bb.batch_outputs(b)
    dev = bb.batch_outputs(b, device=True)
    caps = bb.batch_outputs_dlpack(b)
    wire = bb.unpack_outputs(bb.pack_outputs(b))
    assert set(host) == set(dev) == set(caps) == set(wire)
    for k, h in host.items():
        d = dev[k]
        assert d.is_cuda
        assert np.array_equal(d.cpu().numpy(), h), k
        t = torch.from_dlpack(caps[k])
        assert t.data_ptr() == d.data_ptr()      # zero copy
        assert wire[k].dtype == h.dtype and wire[k].shape == h.shape
        assert np.array_equal(wire[k], h), k


@pytest.mark.parametrize("game", ["go_9x9", "go_19x19", "backgammon", "chess", "shogi", "othello"])
def test_pinned_host_actions_zero_copy(game):
    """batch_step on pinned host action buffers (read / written in place by the kernel, bench e2e)
    gives the same trajectory as device actions, and recycled buffers never leak state."""
    import torch

    from paper_2303_17503_b200.agents import random_actions_device

    n, root = 53, bb.RngKey(11)
    from paper_2303_17503_b200.core import resolve

    gdef = resolve(game)
    ref = bb.batch_init(gdef, root.child(0), n)
    zc = bb.batch_init(gdef, root.child(0), n)
    acts = [torch.empty(n, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    acts[0].copy_(random_actions_device(zc, root.child(1)))
    for t in range(40):
        a = random_actions_device(ref, root.child(2 * t + 1))
        ref = bb.batch_step(ref, a, root.child(2 * (t + 1)))
        zc = bb.batch_step(zc, acts[t % 2], root.child(2 * (t + 1)), next_key=root.child(2 * t + 3),
                           next_actions=acts[(t + 1) % 2])
        torch.cuda.synchronize()
        assert np.array_equal(acts[t % 2].numpy(), a.cpu().numpy()), t
        assert np.array_equal(acts[(t + 1) % 2].numpy(), random_actions_device(ref, root.child(2 * t + 3)).cpu().numpy())
        for k in ("legal_action_mask", "rewards", "terminated", "truncated", "current_player", "observation"):
            assert np.array_equal(getattr(zc, k), getattr(ref, k)), (t, k)


@pytest.mark.parametrize("game", ["go_19x19", "backgammon", "chess", "tic_tac_toe"])
def test_result_fetcher_one_step_behind(game):
    """session.ResultFetcher (bbk_fetch_async): fetch(batch_t) returns batch_{t-1}'s rewards / flags /
    current player, drain() the last batch's -- equal to the batches' own columns."""
    import torch

    B = 64
    sess = bb.BatchSession(game, B, 7, validate=False)
    spec = bb.core.resolve(game).spec
    f = bb.ResultFetcher(B, spec.num_players, torch.device("cuda", 0))
    prev = None
    assert f.fetch(sess.batch) is None
    prev = sess.batch
    for t in range(12):
        sess.step(sess.sample_random_actions())
        got = f.fetch(sess.batch)
        for name in bb.ResultFetcher.FIELDS:
            np.testing.assert_array_equal(got[name], np.asarray(getattr(prev, name)), err_msg=f"{game} {name} t={t}")
        prev = sess.batch
    last = f.drain()
    for name in bb.ResultFetcher.FIELDS:
        np.testing.assert_array_equal(last[name], np.asarray(getattr(prev, name)))
    assert f.drain() is None
