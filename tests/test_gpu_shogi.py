"""Shogi device kernel vs the perft-pinned CPU oracle (bit-exact), plus injected rule positions."""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.core import resolve

pytestmark = pytest.mark.gpu

OU, KI, KE, FU = 8, 5, 3, 1


def _inject_and_step(board_abs, hands, stm, action):
    """Overwrite slot 0 of a fresh device batch with a position, then play `action` on the device."""
    import torch

    gdef = resolve("shogi")
    kern = gdef.batch_kernel
    v = kern.init(gdef, bb.RngKey(1), 1, 256)
    b = torch.zeros(96, dtype=torch.uint8)
    for sq, code in board_abs.items():
        b[sq] = code
    v.priv.board[0].copy_(b.to(v.device))
    m = torch.zeros(16, dtype=torch.uint8)
    m[:14] = torch.tensor(hands, dtype=torch.uint8)
    m[14] = stm
    v.priv.misc[0].copy_(m.to(v.device))
    v._host = {}
    return kern.step(gdef, v, np.array([action]), bb.RngKey(2), 256, validate=False)


def test_uchifuzume_on_device(oracle):
    # white king (0,7) -> (0,8) (white's frame: square 73 -> 72, direction LEFT) gives
    # "8k/9/7GN/9/9/9/9/9/K8 b P": black's pawn drop in front of the king would mate.
    board = {7: 16 | OU, 25: KI, 26: KE, 72: OU}
    hands = [1, 0, 0, 0, 0, 0, 0] + [0] * 7
    v = _inject_and_step(board, hands, 1, 3 * 81 + 72)
    mask = v.legal_action_mask[0]
    ob = oracle.ShogiBatch(1).init(5)
    ob.set_sfen(0, "8k/9/7GN/9/9/9/9/9/K8 b P 1")
    exp = ob.columns()["legal_action_mask"][0]
    assert not mask[20 * 81 + 17]
    assert np.array_equal(mask, exp)
    board[26] = 0   # without the knight the king escapes: the drop is legal
    v = _inject_and_step(board, hands, 1, 3 * 81 + 72)
    assert v.legal_action_mask[0][20 * 81 + 17]


def test_many_seeds_vs_oracle(oracle):
    from test_gpu_parity import run_pair

    for seed in (1, 2, 99):
        run_pair(oracle, "shogi", 48, 260, seed=seed, obs_every=5, enc_every=20)


def test_observe_other_player_matches_oracle(oracle):
    sess = bb.BatchSession("shogi", 4, 7)
    orc = oracle.Session("shogi", 4, 7)
    for t in range(30):
        a = sess.sample_random_actions().cpu().numpy()
        sess.step(a)
        orc.step(a)
    for i, st in enumerate(sess.batch.states):
        for p in range(2):
            role = st.player_to_role[p]
            assert np.array_equal(bb.observe(st, p), orc.b.observe(i, role)), (i, p)
