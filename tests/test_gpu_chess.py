"""Chess device kernel vs the perft-pinned CPU oracle (bit-exact), plus rule scenarios."""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu


def test_opening_and_knight_shuffle_repetition():
    batch = bb.batch_init("chess", bb.RngKey(0), 2)
    assert (batch.legal_action_mask.sum(axis=1) == 20).all()
    back = 21 * 73 + 59
    cycle = [6 * 73 + 63, 6 * 73 + 63, back, back]
    for i, a in enumerate(cycle * 2):
        assert not batch.terminated.any(), i
        batch = bb.batch_step(batch, [a, a], bb.RngKey(100 + i))
    assert batch.terminated.all() and (batch.rewards == 0).all()
    obs = batch.observation
    assert obs[:, :, :, 12].all() and obs[:, :, :, 13].all()


def test_many_seeds_vs_oracle(oracle):
    from test_gpu_parity import run_pair

    for seed in (1, 2, 99):
        run_pair(oracle, "chess", 64, 260, seed=seed, obs_every=5, enc_every=20)


def test_observe_other_player_matches_oracle(oracle):
    sess = bb.BatchSession("chess", 4, 7)
    orc = oracle.Session("chess", 4, 7)
    for t in range(25):
        a = sess.sample_random_actions().cpu().numpy()
        sess.step(a)
        orc.step(a)
    for i, st in enumerate(sess.batch.states):
        for p in range(2):
            role = st.player_to_role[p]
            assert np.array_equal(bb.observe(st, p), orc.b.observe(i, role)), (i, p)
