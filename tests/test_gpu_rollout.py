"""Batched random rollouts (agents.rollout) vs the CPU oracle and the
reference's BASELINE config-0 golden (go_9x9, 1024 envs to termination)."""

import numpy as np
import pytest

import goldens
import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("game,n,max_steps", [("go_9x9", 256, None), ("go_19x19", 64, 60), ("backgammon", 256, None),
                                              ("chess", 128, None), ("shogi", 64, 80)])
def test_rollout_matches_oracle(oracle, game, n, max_steps):
    res = bb.rollout(game, n, 4, max_steps=max_steps, check_every=1)
    orc = oracle.Session(game, n, 4, max_steps=max_steps)
    done = np.zeros(n, bool)
    ret = np.zeros((n, 2), np.float32)
    length = np.zeros(n, np.int32)
    t = 0
    while not done.all():
        assert orc.step(orc.sample_random_actions()) < 0
        t += 1
        c = orc.b.columns(with_obs=False)
        fresh = (c["terminated"] | c["truncated"]) & ~done
        ret[fresh] = c["rewards"][fresh]
        length[fresh] = c["step_count"][fresh]
        done |= fresh
    assert res.steps == t
    assert np.array_equal(res.returns, ret) and np.array_equal(res.lengths, length)


def test_rollout_config0_go9_b1024_step_count():
    rec = goldens.load("go9_config1_b1024")
    res = bb.rollout("go_9x9", 1024, 0, check_every=1)
    assert res.steps == rec["steps"]
    assert np.all(res.lengths > 0) and np.all(np.abs(res.returns).sum(axis=1) == 2.0)


def test_rollout_one_player_and_small_games():
    res = bb.rollout("2048", 64, 1, max_steps=50, check_every=4)
    assert res.returns.shape == (64, 1) and np.all(res.lengths <= 50) and np.all(res.returns >= 0)
    res = bb.rollout("tic_tac_toe", 512, 2)
    assert np.all((res.lengths >= 5) & (res.lengths <= 9))
    assert set(np.unique(res.returns.sum(axis=1))) == {0.0}


def test_bench_run_counts_episodes_like_the_session_loop():
    """bench_run(BenchConfig) (bench.py:63-97) on the device."""
    res = bb.bench_run(bb.BenchConfig("go_9x9", 256, 150, seed=3))
    sess = bb.BatchSession("go_9x9", 256, 3)
    eps = 0
    for _ in range(150):
        b = sess.step(sess.sample_random_actions())
        eps += int((b.terminated | b.truncated).sum())
    assert res.episodes_completed == eps and res.samples_per_second > 0 and res.threads == 1
