"""Batched UCT search on the device vs the reference's own mcts_agent decisions.

The fixtures (tests/golden/mcts_*.json, made by make_golden_mcts.py from the reference) hold,
for a batch of roots reached by random play, the action reference ``mcts_agent`` chose in every
slot. Bit-exact bar: the same action in every slot (the search consumes the same Twister
stream in the same order and evaluates UCB in the same double-precision order).
"""

import numpy as np
import pytest

import goldens
import paper_2303_17503_b200 as bb
from paper_2303_17503_b200 import search

pytestmark = pytest.mark.gpu


def _game(game):
    from paper_2303_17503_b200.games import go

    if game.startswith("go_") and game not in bb.available_games():
        return go.make_game(int(game[3:].split("x")[0]))
    return game


def _roots(rec):
    sess = bb.BatchSession(_game(rec["game"]), rec["batch"], rec["seed"], max_steps=rec["max_steps"])
    for _ in range(rec["t"]):
        sess.step(sess.sample_random_actions())
    return sess.batch


@pytest.mark.parametrize("name", [n for n in goldens.search_names() if not n.startswith("mcts_matches_")])
def test_search_matches_reference_mcts_agent(name):
    rec = goldens.load(name)
    batch = _roots(rec)
    assert bb.batch_fingerprint(batch).hex() == rec["roots_fp"]
    got = bb.mcts_actions(batch, bb.RngKey(rec["key_seed"]), rec["sims"], exploration=rec["exploration"],
                          value_transform=tuple(rec["value_transform"]))
    assert got.tolist() == rec["actions"]


@pytest.mark.parametrize("name", ["mcts_connect_four_s0_b16_t4", "mcts_go_9x9_s0_b4_t20"])
def test_scalar_mcts_agent_matches_batched(name):
    rec = goldens.load(name)
    batch = _roots(rec)
    key = bb.RngKey(rec["key_seed"])
    for i, st in enumerate(batch.states[:4]):
        if st.terminated or st.truncated:
            continue
        assert bb.mcts_agent(st, key.child(i), rec["sims"]) == rec["actions"][i]


def test_mcts_finds_immediate_win():
    # reference test_agents.py:45-61: X on 0,1 with O on 3,4, X to move wins at 2 only
    state = bb.init("tic_tac_toe", bb.RngKey(0))
    for a in [0, 3, 1, 4]:
        state = bb.step(state, a)
    for seed in range(5):
        assert bb.mcts_agent(state, bb.RngKey(seed), 256) == 2


def test_mcts_deterministic_and_legal():
    state = bb.init("connect_four", bb.RngKey(4))
    a = bb.mcts_agent(state, bb.RngKey(11), 64)
    assert a == bb.mcts_agent(state, bb.RngKey(11), 64)
    assert state.legal_action_mask[a]
    hx = bb.init("hex", bb.RngKey(5))
    assert hx.legal_action_mask[bb.mcts_agent(hx, bb.RngKey(6), 1)]


def test_mcts_rejects_chance_and_hidden_info_games():
    for game_id in ("2048", "backgammon", "kuhn_poker", "leduc_holdem"):
        state = bb.init(game_id, bb.RngKey(0))
        with pytest.raises(bb.UnsupportedGame):
            bb.mcts_agent(state, bb.RngKey(1), 4)


def test_mcts_rejects_finished_state():
    state = bb.init("tic_tac_toe", bb.RngKey(0))
    for a in [0, 3, 1, 4, 2]:
        state = bb.step(state, a)
    assert state.terminated
    with pytest.raises(bb.TerminalStep):
        bb.mcts_agent(state, bb.RngKey(0), 4)


def test_mcts_affine_invariance_of_choice():
    # reference test_agents.py:79-86
    for seed in range(6):
        state = bb.init("connect_four", bb.RngKey(seed))
        state = bb.step(state, seed % 7)
        base = bb.mcts_agent(state, bb.RngKey(100 + seed), 48)
        doubled = bb.mcts_agent(state, bb.RngKey(100 + seed), 48, value_transform=(2.0, 0.0))
        shifted = bb.mcts_agent(state, bb.RngKey(100 + seed), 48, value_transform=(2.0, 0.3))
        assert base == doubled == shifted


def test_search_pool_reuse_and_chess_shogi():
    # the pool is an ordinary batch of the game's state, so chess and shogi (no reference
    # search to compare with) search too: legal, deterministic, pool reusable
    for game in ("chess", "shogi"):
        sess = bb.BatchSession(game, 4, 0)
        for _ in range(3):
            sess.step(sess.sample_random_actions())
        b = sess.batch
        pool = search.SearchPool(b.game.batch_kernel, b._v, 4, 3)
        a1 = bb.mcts_actions(b, bb.RngKey(1), 3, pool=pool)
        a2 = bb.mcts_actions(b, bb.RngKey(1), 3, pool=pool)
        assert np.array_equal(a1, a2)
        mask = b.legal_action_mask
        assert all(mask[i, a1[i]] for i in range(4))


MATCH_NAMES = [n for n in goldens.search_names() if n.startswith("mcts_matches_")]


def _policy(a):
    return bb.random_policy() if a == "random" else bb.mcts_policy(a)


@pytest.mark.parametrize("name", MATCH_NAMES)
def test_run_matches_matches_reference(name):
    rec = goldens.load(name)
    pol = [_policy(a) for a in rec["agents"]]
    game = _game(rec["game"])
    res = bb.run_matches(game, pol, rec["games_per_pair"], bb.RngKey(rec["key_seed"]))
    assert [[r.game_id, r.agent_a, r.agent_b, r.wins_a, r.wins_b, r.draws] for r in res] == rec["results"]
    # every game's final rewards and length
    k = 0
    for i in range(len(pol)):
        for j in range(i + 1, len(pol)):
            pair_key = bb.RngKey(rec["key_seed"]).child(k)
            final, length = bb.play_games(game, (pol[i], pol[j]),
                                          [pair_key.child(g) for g in range(rec["games_per_pair"])])
            got = [[float(final[g, 0]), float(final[g, 1]), int(length[g])] for g in range(len(length))]
            assert got == rec["games"][k]
            k += 1


def test_graph_and_eager_paths_agree():
    rec = goldens.load("mcts_go_9x9_s0_b8_t20_sims16")
    batch = _roots(rec)
    v = batch._v
    rows = list(range(rec["batch"]))
    keys = [bb.RngKey(rec["key_seed"]).child(i).state for i in rows]
    eager = search.search(v, rows, keys, rec["sims"], graphs=False).cpu().numpy().tolist()
    graphed = search.search(v, rows, keys, rec["sims"], graphs=True).cpu().numpy().tolist()
    assert eager == graphed == rec["actions"]
