"""Shogi oracle pinning: perft known-answer tests + rule scenarios.

The reference has no shogi engine (games/__init__.py:31 reserves the id), so
the CPU oracle is pinned by public perft counts and hand-built positions;
the device kernel is held bit-exact to it (tests/test_gpu_shogi.py).
"""

import numpy as np
import pytest

MATSURI = "l6nl/5+P1gk/2np1S3/p1p4Pp/3P2Sp1/1PPb2P1P/P5GS1/R8/LN4bKL w RGgsn5p 1"
MAXPOS = "R8/2K1S1SSk/4B4/9/9/9/9/9/1L1L1L3 b RBGSNLP3g3n17p 1"


def test_perft_start(oracle):
    assert [oracle.ShogiBatch.perft(None, d) for d in (1, 2, 3)] == [30, 900, 25470]


def test_perft_matsuri_and_max(oracle):
    assert [oracle.ShogiBatch.perft(MATSURI, d) for d in (1, 2)] == [207, 28684]
    assert oracle.ShogiBatch.perft(MAXPOS, 1) == 593


@pytest.mark.slow
def test_perft_deep(oracle):
    assert oracle.ShogiBatch.perft(None, 4) == 719731
    assert oracle.ShogiBatch.perft(MATSURI, 3) == 4809015


def _one(oracle, sfen):
    b = oracle.ShogiBatch(1).init(77)
    b.set_sfen(0, sfen)
    return b, b.columns()


def test_uchifuzume_is_illegal(oracle):
    drop_p_1_8 = 20 * 81 + 17
    _, c = _one(oracle, "8k/9/7GN/9/9/9/9/9/K8 b P 1")
    m = c["legal_action_mask"][0]
    assert not m[drop_p_1_8]                      # pawn-drop mate
    assert m[20 * 81 + 4 * 9 + 4]                 # other pawn drops fine
    _, c = _one(oracle, "8k/9/7G1/9/9/9/9/9/K8 b P 1")
    assert c["legal_action_mask"][0][drop_p_1_8]  # king can escape -> legal


def test_nifu_and_must_promote(oracle):
    _, c = _one(oracle, "4k4/P8/9/9/9/9/9/9/4K4 b P 1")
    m = c["legal_action_mask"][0]
    col0 = [20 * 81 + r * 9 + 0 for r in range(1, 9)]
    assert not any(m[a] for a in col0)            # nifu on file 9
    assert m[20 * 81 + 4 * 9 + 1]
    assert m[(0 + 10) * 81 + 0] and not m[0 * 81 + 0]   # pawn to the last rank must promote


def test_no_legal_moves_loses(oracle):
    _, c = _one(oracle, "8k/7G1/7G1/9/9/9/9/9/K8 w - 1")   # white king mated (gold on 1,7 covered)
    assert c["terminated"][0]
    p2r = c["player_to_role"][0]
    white = int(np.flatnonzero(p2r == 1)[0])
    assert c["rewards"][0, white] == -1.0


def test_random_play_invariants(oracle):
    s = oracle.Session("shogi", 32, 5)
    for t in range(260):
        c = s.b.columns()
        live = ~(c["terminated"] | c["truncated"])
        assert (c["legal_action_mask"][live].sum(axis=1) > 0).all()
        assert (c["rewards"].sum(axis=1) == 0).all()
        obs = c["observation"]
        assert (obs[..., 7].sum(axis=(1, 2)) == 1).all() and (obs[..., 31 + 7].sum(axis=(1, 2)) == 1).all()
        assert s.step(s.sample_random_actions(c)) == -1


def test_lance_slide_is_not_a_knight_code(oracle):
    # after 1. P-9f (pawn (6,0)->(5,0)) the lance on (8,0) may slide up two squares: direction UP (0)
    b = oracle.ShogiBatch(1).init(3)
    b.set_sfen(0, "lnsgkgsnl/1r5b1/ppppppppp/9/9/P8/1PPPPPPPP/1B5R1/LNSGKGSNL b - 1")
    m = b.columns()["legal_action_mask"][0]
    assert m[0 * 81 + 6 * 9 + 0] and m[0 * 81 + 7 * 9 + 0]
    assert not m[9 * 81 + 6 * 9 + 0]          # (the knight reaches (6,0) with code 8, legitimately)
