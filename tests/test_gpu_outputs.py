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
