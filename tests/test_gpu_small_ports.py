"""The reference's own unit scenarios for its small engines, run on the device.

Ports of reference pkg/tests/test_tictactoe.py, test_connect_four.py,
test_hexgame.py, test_othello.py, test_2048.py, test_kuhn.py and
test_leduc.py: the public-API scenarios use the same keys and action
sequences; the scenarios that build a Core by hand in the reference write the
same Core into a device slot (layouts in csrc/small.cuh) and step it there.
The independent checkers below (line winner, Othello flips, Hex connection)
restate the reference's tests/oracles.py helpers.
"""

import itertools

import numpy as np
import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.core import resolve

pytestmark = pytest.mark.gpu


def _play(game, actions, key=0, keys=None):
    state = bb.init(game, bb.RngKey(key))
    for i, a in enumerate(actions):
        state = bb.step(state, a, None if keys is None else bb.RngKey(keys + i))
    return state


def _inject(game, blob: bytes):
    """A device slot holding the given Core blob (stepped with validate=False)."""
    import torch

    gdef = resolve(game)
    kern = gdef.batch_kernel
    v = kern.init(gdef, bb.RngKey(1), 1, 256)
    v.priv.blob[0].copy_(torch.tensor(list(blob.ljust(48, b"\0")), dtype=torch.uint8).to(v.device))
    v._host = {}
    return gdef, kern, v


def _apply(game, v, action, key=2):
    gdef = resolve(game)
    kern = gdef.batch_kernel
    nv = kern.step(gdef, v, np.array([action]), bb.RngKey(key), 256, validate=False)
    return nv, kern.state_at(gdef, nv, 0, 256)


def _winner_player(state, role):
    return [p for p in range(2) if state.player_to_role[p] == role][0]


# ------------------------------------------------------------------ tic-tac-toe
LINES = ((0, 1, 2), (3, 4, 5), (6, 7, 8), (0, 3, 6), (1, 4, 7), (2, 5, 8), (0, 4, 8), (2, 4, 6))


def _ttt_winner(board):
    for i, j, k in LINES:
        if board[i] and board[i] == board[j] == board[k]:
            return board[i]
    return 0


def test_ttt_opening_and_one_mark():                 # test_tictactoe.py:18-27
    assert int(bb.init("tic_tac_toe", bb.RngKey(4)).legal_action_mask.sum()) == 9
    state = _play("tic_tac_toe", [4])
    assert int(state.legal_action_mask.sum()) == 8
    assert state.current_player != _play("tic_tac_toe", []).current_player


def test_ttt_top_row_win_and_draw():                  # test_tictactoe.py:30-46
    state = _play("tic_tac_toe", [0, 3, 1, 4, 2])
    assert state.terminated
    w = _winner_player(state, 0)
    assert state.rewards[w] == 1.0 and state.rewards[1 - w] == -1.0
    state = _play("tic_tac_toe", [0, 2, 1, 3, 5, 4, 6, 8, 7])
    assert state.terminated and np.all(state.rewards == 0.0)


def test_ttt_occupied_cell_illegal_and_planes():      # test_tictactoe.py:49-66
    with pytest.raises(bb.IllegalAction):
        bb.step(_play("tic_tac_toe", [4]), 4)
    init_state = bb.init("tic_tac_toe", bb.RngKey(9))
    for p in range(2):
        assert bb.observe(init_state, p).sum() == 0.0
    state = bb.step(init_state, 4)
    mover = init_state.current_player
    om, oo = bb.observe(state, mover), bb.observe(state, 1 - mover)
    assert om[1, 1, 0] == 1.0 and om[1, 1, 1] == 0.0
    assert oo[1, 1, 0] == 0.0 and oo[1, 1, 1] == 1.0


def test_ttt_winner_agrees_with_line_oracle():        # test_tictactoe.py:96-117
    key = bb.RngKey(77)
    for g in range(60):
        gkey = key.child(g)
        state = bb.init("tic_tac_toe", gkey.child(0))
        board, t = [0] * 9, 0
        while not state.terminated:
            t += 1
            legal = np.flatnonzero(state.legal_action_mask)
            a = int(legal[gkey.child(t).randint(len(legal))])
            board[a] = state.core.role_to_move + 1
            state = bb.step(state, a)
        w = _ttt_winner(board)
        rr = state.core.rewards
        assert rr == ((0.0, 0.0) if w == 0 else ((1.0, -1.0) if w == 1 else (-1.0, 1.0)))


def test_ttt_batch_equals_scalar_replay():            # test_tictactoe.py:120-136
    root = bb.RngKey(42)
    n = 16
    batch = bb.batch_init("tic_tac_toe", root.child(0), n)
    solo = [bb.init("tic_tac_toe", root.child(0).child(i)) for i in range(n)]
    for t in range(1, 30):
        actions = bb.random_actions(batch, root.child(2 * t - 1))
        skey = root.child(2 * t)
        batch = bb.batch_step(batch, actions, skey)
        for i in range(n):
            if solo[i].terminated or solo[i].truncated:
                solo[i] = bb.init("tic_tac_toe", skey.child(i))
            else:
                solo[i] = bb.step(solo[i], int(actions[i]), skey.child(i))
            assert bb.state_fingerprint(solo[i]) == bb.state_fingerprint(batch.states[i]), (t, i)


# ------------------------------------------------------------------ Connect Four
def test_c4_vertical_and_diagonal_wins():             # test_connect_four.py:17-38
    state = _play("connect_four", [0, 1, 0, 1, 0, 1, 0], key=1)
    w = _winner_player(state, 0)
    assert state.terminated and state.rewards[w] == 1.0 and state.rewards[1 - w] == -1.0
    state = _play("connect_four", [0, 1, 1, 2, 2, 3, 2, 3, 3, 6, 3], key=1)
    assert state.terminated and state.rewards[_winner_player(state, 0)] == 1.0


def test_c4_full_column_masked_and_illegal():         # test_connect_four.py:25-30
    state = _play("connect_four", [3, 3, 3, 3, 3, 3], key=1)
    assert not state.legal_action_mask[3] and int(state.legal_action_mask.sum()) == 6
    with pytest.raises(bb.IllegalAction):
        bb.step(state, 3)


def test_c4_draw_on_full_board():                     # test_connect_four.py:41-52
    moves = [6, 6, 5, 5, 1, 4, 1, 5, 5, 1, 2, 5, 5, 0, 1, 6, 6, 0, 0, 1, 4,
             0, 4, 0, 3, 3, 1, 4, 0, 4, 2, 4, 6, 3, 6, 3, 3, 3, 2, 2, 2, 2]
    state = bb.init("connect_four", bb.RngKey(3))
    for a in moves[:-1]:
        state = bb.step(state, a)
        assert not state.terminated
    state = bb.step(state, moves[-1])
    assert state.terminated and sum(state.core.heights) == 42 and np.all(state.rewards == 0.0)


def test_c4_heights_monotone_and_gravity_plane():     # test_connect_four.py:55-105
    key = bb.RngKey(5)
    for seed in range(10):
        gkey = key.child(seed)
        state = bb.init("connect_four", gkey.child(0))
        prev, t = (0,) * 7, 0
        while not state.terminated:
            t += 1
            legal = np.flatnonzero(state.legal_action_mask)
            state = bb.step(state, int(legal[gkey.child(t).randint(len(legal))]))
            h = state.core.heights
            assert all(a >= b for a, b in zip(h, prev)) and max(h) <= 6 and sum(h) == sum(prev) + 1
            prev = h
    init_state = bb.init("connect_four", bb.RngKey(0))
    obs = bb.observe(bb.step(init_state, 3), init_state.current_player)
    assert obs[5, 3, 0] == 1.0 and obs[:5, 3, 0].sum() == 0.0


# ------------------------------------------------------------------ Hex
SWAP = 121


def _hex_lists(core):
    out = [[0] * 11 for _ in range(11)]
    for r in range(11):
        for c in range(11):
            bit = 1 << (r * 11 + c)
            out[r][c] = 1 if core.bb0 & bit else 2 if core.bb1 & bit else 0
    return out


def _hex_connected(board, mark):
    """Flood from the start edge (role 0 top->bottom, role 1 left->right)."""
    from collections import deque

    starts = [(0, c) for c in range(11)] if mark == 1 else [(r, 0) for r in range(11)]
    seen = {p for p in starts if board[p[0]][p[1]] == mark}
    dq = deque(seen)
    while dq:
        r, c = dq.popleft()
        if (mark == 1 and r == 10) or (mark == 2 and c == 10):
            return True
        for dr, dc in ((-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0)):
            q = (r + dr, c + dc)
            if 0 <= q[0] < 11 and 0 <= q[1] < 11 and q not in seen and board[q[0]][q[1]] == mark:
                seen.add(q)
                dq.append(q)
    return False


def test_hex_swap_rules():                            # test_hexgame.py:24-57
    state = bb.init("hex", bb.RngKey(0))
    assert int(state.legal_action_mask.sum()) == 121 and not state.legal_action_mask[SWAP]
    state = bb.step(state, 5)
    assert int(state.legal_action_mask.sum()) == 121 and state.legal_action_mask[SWAP]
    state = bb.step(state, 6)
    assert not state.legal_action_mask[SWAP] and int(state.legal_action_mask.sum()) == 119
    state = bb.step(bb.init("hex", bb.RngKey(1)), 2 * 11 + 7)
    swapped = bb.step(state, SWAP)
    board = _hex_lists(swapped.core)
    assert board[2][7] == 0 and board[7][2] == 2 and swapped.core.swapped and swapped.core.role_to_move == 0
    state = bb.init("hex", bb.RngKey(2))
    with pytest.raises(bb.IllegalAction):
        bb.step(state, SWAP)
    state = bb.step(bb.step(state, 0), 1)
    with pytest.raises(bb.IllegalAction):
        bb.step(state, SWAP)


def test_hex_full_column_wins_for_role0():            # test_hexgame.py:60-73
    state = bb.init("hex", bb.RngKey(3))
    for r in range(11):
        state = bb.step(state, r * 11 + 4)
        if state.terminated:
            break
        state = bb.step(state, r * 11 + 9)
        assert not state.terminated
    w = _winner_player(state, 0)
    assert state.terminated and state.rewards[w] == 1.0 and state.rewards[1 - w] == -1.0


def test_hex_terminal_agrees_with_flood_oracle_and_no_draws():   # test_hexgame.py:76-113
    sess = bb.BatchSession("hex", 256, 9)
    for _ in range(140):
        b = sess.step(sess.sample_random_actions())
        term = b.terminated
        for i in np.flatnonzero(term)[:24]:
            s = b.states[i]
            board = _hex_lists(s.core)
            mover = 1 - s.core.role_to_move
            assert _hex_connected(board, mover + 1)
            assert s.core.rewards == ((1.0, -1.0) if mover == 0 else (-1.0, 1.0))
        assert not np.any(b.truncated)


def test_hex_planes():                                # test_hexgame.py:116-131
    state = bb.init("hex", bb.RngKey(4))
    for p in range(2):
        assert bb.observe(state, p)[:, :, 3].sum() == 0.0
    state = bb.step(state, 60)
    for p in range(2):
        obs = bb.observe(state, p)
        assert np.all(obs[:, :, 3] == 1.0)
        assert np.all(obs[:, :, 2] == float(state.player_to_role[p]))
    state = bb.step(state, 61)
    assert bb.observe(state, 0)[:, :, 3].sum() == 0.0


# ------------------------------------------------------------------ Othello
PASS = 64


def _oth_blob(board, role, pass_count=0):
    b0 = b1 = 0
    for r in range(8):
        for c in range(8):
            if board[r][c] == 1:
                b0 |= 1 << (r * 8 + c)
            elif board[r][c] == 2:
                b1 |= 1 << (r * 8 + c)
    return b0.to_bytes(8, "little") + b1.to_bytes(8, "little") + bytes([role, pass_count])


def _oth_moves(mine, theirs):
    moves = 0
    for r in range(8):
        for c in range(8):
            i = r * 8 + c
            if (mine | theirs) >> i & 1:
                continue
            for dr, dc in ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)):
                rr, cc, seen = r + dr, c + dc, 0
                while 0 <= rr < 8 and 0 <= cc < 8 and theirs >> (rr * 8 + cc) & 1:
                    rr, cc, seen = rr + dr, cc + dc, seen + 1
                if seen and 0 <= rr < 8 and 0 <= cc < 8 and mine >> (rr * 8 + cc) & 1:
                    moves |= 1 << i
                    break
    return moves


def test_othello_opening_and_masks_along_random_games():   # test_othello.py:37-66, 113-126
    state = bb.init("othello", bb.RngKey(0))
    exp = _oth_moves((1 << 28) | (1 << 35), (1 << 27) | (1 << 36))
    assert [int(a) for a in np.flatnonzero(state.legal_action_mask)] == [i for i in range(64) if exp >> i & 1]
    assert int(state.legal_action_mask.sum()) == 4
    key = bb.RngKey(41)
    for g in range(8):
        gkey = key.child(g)
        state = bb.init("othello", gkey.child(0))
        t = 0
        while not state.terminated:
            core = state.core
            r = core.role_to_move
            mine, theirs = (core.bb0, core.bb1) if r == 0 else (core.bb1, core.bb0)
            exp = _oth_moves(mine, theirs)
            mask = state.legal_action_mask
            got = sum(1 << int(a) for a in np.flatnonzero(mask[:64]))
            assert got == exp
            assert mask[PASS] == (exp == 0)
            if mask[PASS]:
                assert int(mask.sum()) == 1
            t += 1
            legal = np.flatnonzero(mask)
            state = bb.step(state, int(legal[gkey.child(t).randint(len(legal))]))
    with pytest.raises(bb.IllegalAction):
        bb.step(bb.init("othello", bb.RngKey(2)), PASS)


def test_othello_double_pass_majority_and_draw():     # test_othello.py:129-150
    board = [[1] * 8 for _ in range(8)]
    board[7][7] = 0
    _, _, v = _inject("othello", _oth_blob(board, 0))
    v, s1 = _apply("othello", v, PASS)
    assert not s1.terminated and s1.legal_action_mask[PASS] and int(s1.legal_action_mask.sum()) == 1
    v, s2 = _apply("othello", v, PASS)
    assert s2.terminated and s2.core.rewards == (1.0, -1.0)
    board = [[1] * 8 for _ in range(4)] + [[2] * 8 for _ in range(4)]
    _, _, v = _inject("othello", _oth_blob(board, 0))
    v, _ = _apply("othello", v, PASS)
    v, s = _apply("othello", v, PASS)
    assert s.terminated and s.core.rewards == (0.0, 0.0)


# ------------------------------------------------------------------ 2048
def _g2048_blob(grid, score=0):
    ex = [0 if v == 0 else int(v).bit_length() - 1 for row in grid for v in row]
    return bytes(ex) + int(score).to_bytes(8, "little")


def test_2048_init_two_tiles_and_nonnegative_rewards():   # test_2048.py:97-102, 129-139
    for seed in range(30):
        tiles = [v for v in bb.init("2048", bb.RngKey(seed)).core.board if v]
        assert len(tiles) == 2 and all(v in (1, 2) for v in tiles)
    key = bb.RngKey(77)
    state = bb.init("2048", key.child(0))
    t = 0
    while not (state.terminated or state.truncated) and t < 300:
        t += 1
        legal = np.flatnonzero(state.legal_action_mask)
        state = bb.step(state, int(legal[key.child(2 * t).randint(len(legal))]), key.child(2 * t + 1))
        assert state.rewards.shape == (1,) and float(state.rewards[0]) >= 0.0


def _slide_line(vals):
    out, reward, open_slot = [], 0, -1
    for v in vals:
        if v == 0:
            continue
        if open_slot >= 0 and out[open_slot] == v:
            out[open_slot] = v + 1
            reward += 1 << (v + 1)
            open_slot = -1
        else:
            out.append(v)
            open_slot = len(out) - 1
    return out + [0] * (4 - len(out)), reward


def _slide(board, d):
    rows = [[4 * r + c for c in range(4)] for r in range(4)]
    cols = [[4 * r + c for r in range(4)] for c in range(4)]
    lines = {0: rows, 1: cols, 2: [l[::-1] for l in rows], 3: [l[::-1] for l in cols]}[d]
    out, reward = [0] * 16, 0
    for line in lines:
        vals, r = _slide_line([board[i] for i in line])
        reward += r
        for i, v in zip(line, vals):
            out[i] = v
    return tuple(out), reward


def test_2048_moves_rewards_and_spawns_follow_the_slide_rules():   # test_2048.py:24-94
    _, kern, v = _inject("2048", _g2048_blob([[2, 2, 2, 2], [0] * 4, [0] * 4, [0] * 4]))
    v, s = _apply("2048", v, 0)
    assert float(s.rewards[0]) == 8.0 and s.core.score == 8
    assert s.core.board[:2] == (2, 2) and sum(1 for x in s.core.board if x) == 3
    key = bb.RngKey(31)
    for g in range(6):
        gkey = key.child(g)
        state = bb.init("2048", gkey.child(0))
        t = 0
        while not (state.terminated or state.truncated):
            board = state.core.board
            legal = [d for d in range(4) if _slide(board, d)[0] != board]
            assert list(np.flatnonzero(state.legal_action_mask)) == legal
            t += 1
            a = legal[gkey.child(2 * t).randint(len(legal))]
            slid, reward = _slide(board, a)
            state = bb.step(state, a, gkey.child(2 * t + 1))
            new = state.core.board
            diff = [i for i in range(16) if new[i] != slid[i]]
            assert len(diff) == 1 and slid[diff[0]] == 0 and new[diff[0]] in (1, 2)
            assert float(state.rewards[0]) == float(reward)
        if state.terminated:
            assert not any(_slide(state.core.board, d)[0] != state.core.board for d in range(4))


def test_2048_one_hot_observation():                  # test_2048.py:119-126
    _, kern, v = _inject("2048", _g2048_blob([[2, 0, 0, 0], [0] * 4, [0] * 4, [0, 0, 0, 2048]]))
    obs = kern.observe_at(resolve("2048"), v, 0, 0)
    assert obs.shape == (4, 4, 31) and obs[0, 0, 0] == 1.0 and obs[3, 3, 10] == 1.0 and obs.sum() == 2.0


# ------------------------------------------------------------------ Kuhn poker
CALL, BET, FOLD, CHECK = 0, 1, 2, 3


def _kuhn_blob(hands):
    return bytes([hands[0], hands[1], 0, 0, 0, 0, 0, 0, 0, 0])


def test_kuhn_deals_and_masks():                      # test_kuhn.py:19-40
    a, b = bb.init("kuhn_poker", bb.RngKey(123)), bb.init("kuhn_poker", bb.RngKey(123))
    assert a.core.hands == b.core.hands and a.core.hands[0] != a.core.hands[1]
    seen = {bb.init("kuhn_poker", bb.RngKey(s)).core.hands for s in range(300)}
    assert seen == set(itertools.permutations(range(3), 2))
    state = bb.init("kuhn_poker", bb.RngKey(1))
    assert set(np.flatnonzero(state.legal_action_mask)) == {BET, CHECK}
    assert set(np.flatnonzero(bb.step(state, BET).legal_action_mask)) == {CALL, FOLD}
    assert set(np.flatnonzero(bb.step(state, CHECK).legal_action_mask)) == {BET, CHECK}


def test_kuhn_payoffs():                              # test_kuhn.py:42-56
    _, _, v = _inject("kuhn_poker", _kuhn_blob((2, 1)))
    v, _ = _apply("kuhn_poker", v, BET)
    v, s = _apply("kuhn_poker", v, CALL)
    assert s.terminated and s.core.rewards == (2.0, -2.0)
    _, _, v = _inject("kuhn_poker", _kuhn_blob((2, 1)))
    for a in (CHECK, BET, FOLD):
        v, s = _apply("kuhn_poker", v, a)
    assert s.terminated and s.core.rewards == (-1.0, 1.0)


def test_kuhn_observation_bits():                     # test_kuhn.py:89-105
    state = bb.init("kuhn_poker", bb.RngKey(5))
    for p in range(2):
        obs = bb.observe(state, p)
        hand = state.core.hands[state.player_to_role[p]]
        assert obs[hand] == 1.0 and obs[:3].sum() == 1.0
        assert obs[3] == 1.0 and obs[4] == 0.0 and obs[5] == 1.0 and obs[6] == 0.0
    after = bb.step(state, BET)
    bettor = state.current_player
    ob, oo = bb.observe(after, bettor), bb.observe(after, 1 - bettor)
    assert ob[3] == 0.0 and ob[4] == 1.0 and oo[5] == 0.0 and oo[6] == 1.0


# ------------------------------------------------------------------ Leduc hold'em
RAISE = 1


def _leduc_blob(hands, public=-1, round_=1, raises=0, committed=(1, 1), acted=0, to_move=0):
    return bytes([hands[0], hands[1], public + 1, round_, raises, committed[0], committed[1], acted, to_move])


def test_leduc_deck_fold_and_raise_sizes():           # test_leduc.py:16-40
    hands = [bb.init("leduc_holdem", bb.RngKey(s)).core.hands for s in range(300)]
    assert any(h[0] == h[1] for h in hands) and {c for h in hands for c in h} == {0, 1, 2}
    _, _, v = _inject("leduc_holdem", _leduc_blob((2, 0)))
    v, s = _apply("leduc_holdem", v, RAISE)
    assert s.core.committed == (3, 1)
    v, s = _apply("leduc_holdem", v, FOLD)
    assert s.terminated and s.core.rewards == (1.0, -1.0)
    _, _, v = _inject("leduc_holdem", _leduc_blob((2, 0)))
    v, _ = _apply("leduc_holdem", v, CALL)
    v, s = _apply("leduc_holdem", v, CALL, key=3)
    assert s.core.round == 2 and s.core.public >= 0 and s.core.role_to_move == 0
    v, s = _apply("leduc_holdem", v, RAISE)
    assert s.core.committed == (5, 1)


def test_leduc_max_commitment_and_third_raise():      # test_leduc.py:42-67
    _, _, v = _inject("leduc_holdem", _leduc_blob((2, 2)))
    for a in (RAISE, RAISE, CALL, RAISE, RAISE):
        v, s = _apply("leduc_holdem", v, a, key=1)
    assert s.core.committed == (9, 13)
    v, s = _apply("leduc_holdem", v, CALL, key=1)
    assert s.terminated and max(s.core.committed) == 13
    state = bb.init("leduc_holdem", bb.RngKey(17))
    state = bb.step(state, RAISE, bb.RngKey(100))
    state = bb.step(state, RAISE, bb.RngKey(101))
    with pytest.raises(bb.IllegalAction):
        bb.step(state, RAISE, bb.RngKey(102))


def test_leduc_showdowns():                           # test_leduc.py:70-111
    _, _, v = _inject("leduc_holdem", _leduc_blob((0, 2), public=0, round_=2))
    v, _ = _apply("leduc_holdem", v, CALL)
    v, s = _apply("leduc_holdem", v, CALL)
    assert s.terminated and s.core.rewards[0] > 0          # J pairs the public J
    _, _, v = _inject("leduc_holdem", _leduc_blob((1, 1)))
    v, _ = _apply("leduc_holdem", v, CALL, key=6)
    v, s = _apply("leduc_holdem", v, CALL, key=6)
    assert s.core.round == 2 and s.core.public != 1
    v, _ = _apply("leduc_holdem", v, CALL, key=6)
    v, s = _apply("leduc_holdem", v, CALL, key=6)
    assert s.terminated and s.core.rewards == (0.0, 0.0)


def test_leduc_public_card_and_observation():         # test_leduc.py:114-142
    for seed in range(100):
        key = bb.RngKey(seed)
        state = bb.init("leduc_holdem", key.child(0))
        hands = state.core.hands
        state = bb.step(bb.step(state, CALL, key.child(1)), CALL, key.child(2))
        deck = [0, 0, 1, 1, 2, 2]
        deck.remove(hands[0])
        deck.remove(hands[1])
        assert state.core.public in deck
    state = bb.init("leduc_holdem", bb.RngKey(11))
    for p in range(2):
        obs = bb.observe(state, p)
        assert obs.shape == (34,) and obs[state.core.hands[state.player_to_role[p]]] == 1.0
        assert obs[3:6].sum() == 0.0 and obs[7] == 1.0 and obs[21] == 1.0
