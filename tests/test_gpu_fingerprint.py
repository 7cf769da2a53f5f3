"""Device-side state fingerprints (csrc/fingerprint.cu) equal the host state_fingerprint
(reference core.py:417-441) slot by slot, and the oracle's fingerprints at scale."""

import hashlib

import numpy as np
import pytest

import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu

GAMES = ["go_9x9", "go_19x19", "backgammon", "chess", "shogi"]
SMALL = ["tic_tac_toe", "connect_four", "othello", "hex", "2048", "kuhn_poker", "leduc_holdem"]


@pytest.mark.parametrize("game", GAMES + SMALL)
def test_device_fingerprints_equal_host(game):
    # short episodes so that finished / reset slots and long Go histories all occur
    max_steps = {"go_9x9": 40, "go_19x19": 12, "backgammon": 60, "chess": 30, "shogi": 30}.get(game, 20)
    sess = bb.BatchSession(game, 96, 5, max_steps=max_steps)
    for t in range(max_steps + 7):
        sess.step(sess.sample_random_actions())
        if t % 6 == 5 or t == max_steps:
            b = sess.batch
            dev = bb.device_fingerprints(b)
            host = np.stack([np.frombuffer(bb.state_fingerprint(s), np.uint8) for s in b.states])
            assert np.array_equal(dev, host), (game, t)
            h = hashlib.blake2b(digest_size=16)
            for s in b.states:
                h.update(bb.state_fingerprint(s))
            assert bb.batch_fingerprint(b) == h.digest()


@pytest.mark.parametrize("game", GAMES)
def test_device_fingerprints_equal_oracle_at_scale(oracle, game):
    n = 4096 if game in ("go_9x9", "backgammon") else 1024
    steps = 40
    sess = bb.BatchSession(game, n, 11)
    orc = oracle.Session(game, n, 11)
    for _ in range(steps):
        a = sess.sample_random_actions().cpu().numpy()
        sess.step(a)
        assert orc.step(a) < 0
    dev = bb.device_fingerprints(sess.batch)
    ref = np.stack([np.frombuffer(f, np.uint8) for f in orc.b.fingerprints()])
    assert np.array_equal(dev, ref)
