"""Chess oracle pinning: perft known-answer tests + rule scenarios.

The reference has no chess engine (games/__init__.py:23 reserves the id), so
the CPU oracle is pinned by public perft counts (chessprogramming wiki) and
by hand-built terminal positions; the device kernel is then held bit-exact
to the oracle (tests/test_gpu_chess.py).
"""

import numpy as np
import pytest

START = "rnbqkbnr/pppppppp/8/8/8/8/PPPPPPPP/RNBQKBNR w KQkq - 0 1"
PERFT = [
    (START, [20, 400, 8902, 197281]),
    ("r3k2r/p1ppqpb1/bn2pnp1/3PN3/1p2P3/2N2Q1p/PPPBBPPP/R3K2R w KQkq -", [48, 2039, 97862]),
    ("8/2p5/3p4/KP5r/1R3p1k/8/4P1P1/8 w - -", [14, 191, 2812, 43238]),
    ("r3k2r/Pppp1ppp/1b3nbN/nP6/BBP1P3/q4N2/Pp1P2PP/R2Q1RK1 w kq - 0 1", [6, 264, 9467]),
    ("rnbq1k1r/pp1Pbppp/2p5/8/2B5/8/PPP1NnPP/RNBQK2R w KQ - 1 8", [44, 1486, 62379]),
    ("r4rk1/1pp1qppp/p1np1n2/2b1p1B1/2B1P1b1/P1NP1N2/1PP1QPPP/R4RK1 w - - 0 10", [46, 2079, 89890]),
]


@pytest.mark.parametrize("fen,counts", PERFT)
def test_perft(oracle, fen, counts):
    assert [oracle.ChessBatch.perft(fen, d + 1) for d in range(len(counts))] == counts


@pytest.mark.slow
def test_perft_deep(oracle):
    assert oracle.ChessBatch.perft(START, 5) == 4865609
    assert oracle.ChessBatch.perft(PERFT[1][0], 4) == 4085603


def _one(oracle, fen):
    b = oracle.ChessBatch(1)
    b.init(123)
    b.set_fen(0, fen)
    return b, b.columns()


def test_opening_mask_has_20_moves(oracle):
    b = oracle.ChessBatch(2).init(5)
    c = b.columns()
    assert (c["legal_action_mask"].sum(axis=1) == 20).all()
    # e2e4 = from e2 (12) plane N dist 2 = 1; g1f3 = from g1 (6), knight (+2,-1) = plane 63
    assert c["legal_action_mask"][0, 12 * 73 + 1] and c["legal_action_mask"][0, 6 * 73 + 63]


def test_checkmate_is_terminal_with_rewards(oracle):
    b, c = _one(oracle, "rnb1kbnr/pppp1ppp/8/4p3/6Pq/5P2/PPPPP2P/RNBQKBNR w KQkq - 1 3")   # fool's mate
    assert c["terminated"][0] and c["legal_action_mask"][0].sum() == 0
    p2r = c["player_to_role"][0]
    white = int(np.flatnonzero(p2r == 0)[0])
    assert c["rewards"][0, white] == -1.0 and c["rewards"][0, 1 - white] == 1.0


def test_stalemate_and_insufficient_are_draws(oracle):
    for fen in ("7k/5Q2/6K1/8/8/8/8/8 b - - 0 1", "8/8/8/4k3/8/8/2B5/4K3 w - - 0 1",
                "8/8/2b5/4k3/8/8/2B5/4K3 w - - 0 1"):
        _, c = _one(oracle, fen)
        assert c["terminated"][0] and (c["rewards"][0] == 0).all(), fen
    _, c = _one(oracle, "8/8/1b6/4k3/8/8/2B5/4K3 w - - 0 1")   # bishops on opposite colours: play on
    assert not c["terminated"][0]


def test_fifty_move_rule(oracle):
    _, c = _one(oracle, "4k3/8/8/8/8/8/4P3/R3K3 w - - 100 80")
    assert c["terminated"][0]
    _, c = _one(oracle, "4k3/8/8/8/8/8/4P3/R3K3 w - - 99 80")
    assert not c["terminated"][0]


def test_threefold_repetition_by_knight_shuffle(oracle):
    b = oracle.ChessBatch(1).init(9)
    # Ng1-f3, Ng8-f6, Nf3-g1, Nf6-g8 twice -> start position occurs a third time
    seq = [6 * 73 + 63, 6 * 73 + 63]   # mover-frame: g1->f3 for white, g8->f6 for black (flipped)
    back = 21 * 73 + 59                # f3 -> g1 : (-2,+1) knight = plane 56+3
    cycle = [6 * 73 + 63, 6 * 73 + 63, back, back]
    for i, a in enumerate(cycle * 2):
        c = b.columns(with_obs=False)
        assert not c["terminated"][0], i
        assert b.step(np.array([a]), 0) == -1
    c = b.columns()
    assert c["terminated"][0] and (c["rewards"][0] == 0).all()
    obs = c["observation"][0]
    assert obs[:, :, 12].all() and obs[:, :, 13].all()   # current position repeated twice before


def test_random_play_invariants(oracle):
    s = oracle.Session("chess", 64, 3)
    for t in range(300):
        c = s.b.columns()
        live = ~(c["terminated"] | c["truncated"])
        assert (c["legal_action_mask"][live].sum(axis=1) > 0).all()
        assert (c["rewards"].sum(axis=1) == 0).all()
        obs = c["observation"]
        # exactly one own king and one opponent king plane set at t=0
        assert (obs[..., 5].sum(axis=(1, 2)) == 1).all() and (obs[..., 11].sum(axis=(1, 2)) == 1).all()
        assert s.step(s.sample_random_actions(c)) == -1
