"""The reference's own Go / backgammon / env-core unit scenarios, run through the device API.

Ports of reference pkg/tests/test_go.py, test_backgammon.py and test_core.py
scenarios: same keys, same action sequences, same assertions -- only the
package under test differs (scalar init/step run a batch of one on the B200).
"""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu

PASS = 81


def test_go_opening_mask_has_82_actions():            # test_go.py:23-26
    state = bb.init("go_9x9", bb.RngKey(0))
    assert int(state.legal_action_mask.sum()) == 82
    assert state.legal_action_mask[PASS]


def test_go_double_pass_white_wins_by_komi():          # test_go.py:29-37
    state = bb.init("go_9x9", bb.RngKey(1))
    state = bb.step(state, PASS)
    assert not state.terminated
    state = bb.step(state, PASS)
    assert state.terminated
    white_player = [p for p in range(2) if state.player_to_role[p] == 1][0]
    assert state.rewards[white_player] == 1.0
    assert state.rewards[1 - white_player] == -1.0


def test_go_capture_before_suicide_in_corner():        # test_go.py:40-50
    state = bb.init("go_9x9", bb.RngKey(2))
    for a in (1, 0, 9):
        state = bb.step(state, a)
    board = state.core.board
    assert board[0] == 0 and board[1] == 1 and board[9] == 1


def test_go_single_stone_suicide_masked():             # test_go.py:53-62
    state = bb.init("go_9x9", bb.RngKey(3))
    for a in (1, 20, 9):
        state = bb.step(state, a)
    assert not state.legal_action_mask[0]
    with pytest.raises(bb.IllegalAction):
        bb.step(state, 0)


def test_go_ko_retake_masked():                        # test_go.py:72-86
    state = bb.init("go_9x9", bb.RngKey(6))
    for a in (1, 2, 9, 12, 19, 20, 60, 10, 11):
        state = bb.step(state, a)
    board = state.core.board
    assert board[10] == 0 and board[11] == 1
    assert not state.legal_action_mask[10]
    with pytest.raises(bb.IllegalAction):
        bb.step(state, 10)
    assert len(np.flatnonzero(state.legal_action_mask)) > 1


def test_go_history_planes_and_colour_plane():         # test_go.py:121-152
    state = bb.init("go_9x9", bb.RngKey(8))
    first = bb.step(state, 40)
    obs = bb.observe(first, first.current_player)
    assert obs[:, :, 1].sum() == 1.0 and obs[:, :, 0].sum() == 0.0
    assert obs[:, :, 4:16].sum() == 0.0
    state = bb.init("go_9x9", bb.RngKey(9))
    white = [p for p in range(2) if state.player_to_role[p] == 1][0]
    assert np.all(bb.observe(state, white)[:, :, 16] == 1.0)
    assert np.all(bb.observe(state, 1 - white)[:, :, 16] == 0.0)
    s2 = bb.step(bb.step(bb.init("go_9x9", bb.RngKey(10)), 0), 80)
    obs = bb.observe(s2, s2.current_player)
    assert obs[:, :, 0].sum() + obs[:, :, 1].sum() == 2.0
    assert obs[:, :, 2].sum() + obs[:, :, 3].sum() == 1.0
    assert obs[:, :, 4].sum() + obs[:, :, 5].sum() == 0.0


def test_go_pass_always_legal_and_no_repeats():        # test_go.py:178-206
    key = bb.RngKey(12)
    state = bb.init("go_9x9", key.child(0))
    seen = {state.core.hash}
    for t in range(1, 120):
        if state.terminated or state.truncated:
            break
        assert state.legal_action_mask[PASS]
        legal = np.flatnonzero(state.legal_action_mask)
        a = int(legal[key.child(t).randint(len(legal))])
        state = bb.step(state, a)
        if a != PASS:
            assert state.core.hash not in seen
            seen.add(state.core.hash)


def test_go19_truncation_zero_rewards():               # test_core.py:135-148 on go_19x19
    key = bb.RngKey(5)
    state = bb.init("go_19x19", key.child(0), max_steps=3)
    t = 0
    while not (state.terminated or state.truncated):
        t += 1
        legal = np.flatnonzero(state.legal_action_mask)
        state = bb.step(state, int(legal[key.child(2 * t - 1).randint(len(legal))]), key.child(2 * t))
    assert state.truncated and not state.terminated and state.step_count == 3
    assert np.all(state.rewards == 0)
    with pytest.raises(bb.TerminalStep):
        bb.step(state, 361)


def _conserved(core):
    for role, sign in ((0, 1), (1, -1)):
        on_board = sum(v for v in core.points if v * sign > 0) * sign
        if on_board + core.bar[role] + core.off[role] != 15:
            return False
    return True


def test_backgammon_initial_position_and_conservation():   # test_backgammon.py:21-46
    start = (2, 0, 0, 0, 0, -5, 0, -3, 0, 0, 0, 5, -5, 0, 0, 0, 3, 0, 5, 0, 0, 0, 0, -2)
    state = bb.init("backgammon", bb.RngKey(0))
    assert state.core.points == start and state.core.role_to_move == 0
    assert len(state.core.remaining) in (2, 4) and state.legal_action_mask.any()
    key = bb.RngKey(1)
    for g in range(6):
        gkey = key.child(g)
        state = bb.init("backgammon", gkey.child(0))
        t = 0
        while not (state.terminated or state.truncated):
            assert _conserved(state.core)
            t += 1
            legal = np.flatnonzero(state.legal_action_mask)
            state = bb.step(state, int(legal[gkey.child(2 * t).randint(len(legal))]), gkey.child(2 * t + 1))
        assert _conserved(state.core)
        if state.terminated:
            assert abs(float(state.rewards[0])) in (1.0, 2.0, 3.0)
            assert float(state.rewards.sum()) == 0.0


def test_backgammon_blocked_destination_masked():      # test_backgammon.py:49-60
    state = bb.init("backgammon", bb.RngKey(2))
    if 5 in state.core.remaining:
        assert not state.legal_action_mask[25 * 6 + 4]


def test_env_core_contract_all_games():                # test_core.py:52-84
    for game in bb.available_games():
        spec = bb.game_spec(game)
        state = bb.init(game, bb.RngKey(17))
        assert not state.terminated and not state.truncated and state.step_count == 0
        assert state.legal_action_mask.shape == (spec.num_actions,) and state.legal_action_mask.any()
        assert np.all(state.rewards == 0)
        assert sorted(state.player_to_role) == list(range(spec.num_players))
        assert state.player_to_role[state.current_player] == state.core.role_to_move
        for p in range(spec.num_players):
            obs = bb.observe(state, p)
            assert obs.shape == spec.observation_shape and obs.dtype == np.float32
        with pytest.raises(bb.InvalidPlayer):
            bb.observe(state, spec.num_players)


def test_pgx_style_facade():
    """make(env_id) / init / step with the north-star State fields, vs BatchSession."""
    import torch

    env = bb.make("go_19x19", batch_size=64)
    state = env.init(7)
    sess = bb.BatchSession("go_19x19", 64, 7)
    for t in range(20):
        a = env.random_action(state)
        assert torch.equal(a, sess.sample_random_actions())
        state = env.step(state, a)
        sess.step(a)
        for f in ("current_player", "observation", "legal_action_mask", "rewards", "terminated", "truncated"):
            assert torch.equal(getattr(state, f), getattr(sess.batch.device, f)), f
    assert state.observation.shape == (64, 19, 19, 17) and state.legal_action_mask.dtype == torch.bool
