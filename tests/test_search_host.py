"""Host side of the batched UCT search (no GPU): the Twister the device uses equals Python's
random.Random stream that reference mcts_agent draws from (agents.py:85), the search fixtures
are well formed, and the match runner's argument checks mirror agents.run_matches."""

import ctypes
import random

import numpy as np
import pytest

import goldens
import paper_2303_17503_b200 as bb
from paper_2303_17503_b200 import _native
from paper_2303_17503_b200.agents import _random_choice


@pytest.mark.parametrize("seed", [0, 1, 7, 2**31 - 1, 2**32 - 1, 2**32, 0x9E3779B97F4A7C15, 2**64 - 1])
def test_twister_matches_python_random(seed):
    below = np.array([0] * 700 + [1, 2, 3, 7, 9, 82, 122, 362, 4672, 2187] * 150, dtype=np.uint32)
    out = np.zeros(len(below), dtype=np.uint32)
    _native.lib().bbk_mt19937_host(seed, below.ctypes.data_as(ctypes.c_void_p), len(below),
                                   out.ctypes.data_as(ctypes.c_void_p))
    r = random.Random(seed)
    exp = [r.getrandbits(32) if b == 0 else r.randrange(int(b)) for b in below]
    assert out.tolist() == exp


def test_twister_for_reference_key_states():
    # the seeds mcts_agent actually sees: RngKey(...).child(i).state
    for i in range(20):
        ks = bb.RngKey(i).child(3 * i).state
        below = np.array([9, 8, 7, 6, 5, 4, 3, 2, 1] * 100, dtype=np.uint32)
        out = np.zeros(len(below), dtype=np.uint32)
        _native.lib().bbk_mt19937_host(ks, below.ctypes.data_as(ctypes.c_void_p), len(below),
                                       out.ctypes.data_as(ctypes.c_void_p))
        r = random.Random(ks)
        assert out.tolist() == [r.randrange(int(b)) for b in below]


def test_search_fixtures_well_formed():
    names = goldens.search_names()
    assert len(names) >= 10
    for name in names:
        rec = goldens.load(name)
        assert "generator" in rec and "reference boardbatch" in rec["generator"]
        if name.startswith("mcts_matches_"):
            assert len(rec["games"]) == len(rec["results"])
            for res, games in zip(rec["results"], rec["games"]):
                r0 = [g[0] for g in games]
                assert res[3:] == [sum(x > 0 for x in r0), sum(x < 0 for x in r0), sum(x == 0 for x in r0)]
        else:
            assert len(rec["actions"]) == rec["batch"]
            assert len(rec["roots_fp"]) == 32


def test_random_choice_is_reference_random_agent():
    # random_agent: legal[key.randint(len(legal))] with randint = state % bound (rng.py:97-101)
    rng = np.random.default_rng(0)
    mask = rng.random((64, 37)) < 0.3
    mask[5] = False
    keys = rng.integers(0, 2**63, size=64, dtype=np.int64).astype(np.uint64) * np.uint64(2) + np.uint64(1)
    got = _random_choice(mask, keys)
    for i in range(64):
        legal = np.flatnonzero(mask[i])
        assert got[i] == (0 if legal.size == 0 else legal[int(keys[i]) % legal.size])


def test_run_matches_argument_checks():
    with pytest.raises(ValueError):
        bb.run_matches("tic_tac_toe", [bb.random_policy()], 2, bb.RngKey(0))
    for game in ("backgammon", "kuhn_poker"):
        with pytest.raises(bb.UnsupportedGame):
            bb.run_matches(game, [bb.mcts_policy(4), bb.random_policy()], 2, bb.RngKey(0))
    with pytest.raises(bb.UnsupportedGame):
        bb.run_matches("2048", [bb.random_policy(), bb.random_policy()], 2, bb.RngKey(0))
    assert bb.run_matches("tic_tac_toe", [bb.random_policy(), bb.mcts_policy(8)], 0, bb.RngKey(0)) == []
    assert bb.mcts_policy(16).name == "mcts16"
