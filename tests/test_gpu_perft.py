"""Device perft: the chess and shogi step kernels expand known-answer positions level by level.

The reference has no chess / shogi engine (games/__init__.py:23,31 reserve the ids; the rules are
prose in PAPER.md:781-856 and 1278-1354), so the kernels are pinned here by public perft counts
(chessprogramming wiki: start position, Kiwipete, positions 3-6; shogi: start position, the
"matsuri" position, the 593-move position) run ON THE DEVICE, not only in the CPU oracle:

* a batch of one slot per root is started from the FEN / SFEN (``bbk_<game>_load``);
* every level, each parent row is replicated once per legal action with ``bbk_copy_rows`` (all
  columns, private state and the in-place history ring / position log), and ONE batched step
  launch plays every child's action;
* the node count of level d+1 is the sum of the popcounts of level d's legal masks: the KATs
  below are asserted at every depth;
* every node of every level (or a seeded sample of 20,000 rows on the biggest levels) is compared
  with the oracle replaying the same action path from the same root: legal mask, every column,
  the device fingerprint (blake2b over the columns and ``Core.encode()``, ``core.py:417-434``),
  and the full observation tensor on levels up to 4,096 rows (and a 4,096-row sample above).
"""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.core import resolve
from paper_2303_17503_b200.games._device import Lineage

pytestmark = pytest.mark.gpu

KEY = 0x5EED
COLS = ("current_player", "legal_action_mask", "rewards", "terminated", "truncated", "step_count", "player_to_role")

CHESS_START = "rnbqkbnr/pppppppp/8/8/8/8/PPPPPPPP/RNBQKBNR w KQkq - 0 1"
KIWIPETE = "r3k2r/p1ppqpb1/bn2pnp1/3PN3/1p2P3/2N2Q1p/PPPBBPPP/R3K2R w KQkq -"
POS3 = "8/2p5/3p4/KP5r/1R3p1k/8/4P1P1/8 w - -"
POS4 = "r3k2r/Pppp1ppp/1b3nbN/nP6/BBP1P3/q4N2/Pp1P2PP/R2Q1RK1 w kq - 0 1"
POS5 = "rnbq1k1r/pp1Pbppp/2p5/8/2B5/8/PPP1NnPP/RNBQK2R w KQ - 1 8"
POS6 = "r4rk1/1pp1qppp/p1np1n2/2b1p1B1/2B1P1b1/P1NP1N2/1PP1QPPP/R4RK1 w - - 0 10"

# (position, perft counts for depth 1..D); the last depth is counted from the popcounts of the
# deepest materialised level, so level D-1 is stepped on the device and compared with the oracle
CHESS_KATS = [
    (CHESS_START, [20, 400, 8902, 197281]),
    (KIWIPETE, [48, 2039, 97862]),
    (POS3, [14, 191, 2812, 43238]),
    (POS4, [6, 264, 9467]),
    (POS5, [44, 1486, 62379]),
    (POS6, [46, 2079, 89890]),
]
# one level deeper (the deepest level stepped on the device holds 9,467-197,281 rows)
CHESS_DEEP = [
    (CHESS_START, 4865609),   # level 4 = 197,281 device rows
    (KIWIPETE, 4085603),
    (POS3, 674624),
    (POS4, 422333),
    (POS5, 2103487),
    (POS6, 3894594),
]

SHOGI_START = "lnsgkgsnl/1r5b1/ppppppppp/9/9/9/PPPPPPPPP/1B5R1/LNSGKGSNL b - 1"
MATSURI = "l6nl/5+P1gk/2np1S3/p1p4Pp/3P2Sp1/1PPb2P1P/P5GS1/R8/LN4bKL w RGgsn5p 1"
MAXPOS = "R8/2K1S1SSk/4B4/9/9/9/9/9/1L1L1L3 b RBGSNLP3g3n17p 1"
SHOGI_KATS = [
    (SHOGI_START, [30, 900, 25470, 719731]),
    (MATSURI, [207, 28684, 4809015]),
    (MAXPOS, [593, None]),   # perft(2) unpublished: the level is stepped and held to the oracle only
]

SAMPLE_ROWS = 20000
OBS_ROWS = 4096


def _oracle_batch(oracle, game, n):
    return oracle.ChessBatch(n) if game == "chess" else oracle.ShogiBatch(n)


def _check_level(oracle, game, root, v, paths, rng):
    """Compare device level v (row i reached by paths[:, i] from root) with the oracle."""
    n = v.n
    rows = np.arange(n) if n <= SAMPLE_ROWS else np.sort(rng.choice(n, SAMPLE_ROWS, replace=False))
    m = len(rows)
    ob = _oracle_batch(oracle, game, m)
    root_key = oracle._child(KEY, 0)   # device: slot key child(key, slot0 + 0) of the root slot
    ob.init(KEY, 0, slot_keys=np.full(m, root_key, dtype=np.uint64))
    for i in range(m):
        (ob.set_fen if game == "chess" else ob.set_sfen)(i, root)
    for d in range(paths.shape[0]):
        assert ob.step(paths[d, rows], 0) == -1, f"oracle rejected level-{d + 1} actions"
    with_obs = m <= OBS_ROWS
    oc = ob.columns(with_obs=with_obs)
    for c in COLS:
        got = np.asarray(getattr(v, c))[rows]
        exp = oc[c]
        if got.dtype == np.bool_:
            got, exp = got.astype(np.uint8), exp.astype(np.uint8)
        if not np.array_equal(got, exp):
            bad = np.argwhere(got != exp)[:5]
            raise AssertionError(f"{game} {root!r} level {paths.shape[0]}: {c} differs at {bad.tolist()}")
    fp_dev = v.kern.fingerprints(v)[rows]
    fp_orc = np.frombuffer(b"".join(ob.fingerprints(oc)), dtype=np.uint8).reshape(m, 16)
    bad = np.flatnonzero((fp_dev != fp_orc).any(axis=1))
    assert not len(bad), f"{game} {root!r} level {paths.shape[0]}: fingerprint (encode) differs at rows {rows[bad[:5]]}"
    obs_rows = np.arange(m) if with_obs else np.sort(rng.choice(m, min(OBS_ROWS, m), replace=False))
    if not with_obs:   # observation on a sample: replay only those rows
        ob2 = _oracle_batch(oracle, game, len(obs_rows))
        ob2.init(KEY, 0, slot_keys=np.full(len(obs_rows), root_key, dtype=np.uint64))
        for i in range(len(obs_rows)):
            (ob2.set_fen if game == "chess" else ob2.set_sfen)(i, root)
        for d in range(paths.shape[0]):
            assert ob2.step(paths[d, rows[obs_rows]], 0) == -1
        exp_obs = ob2.columns(with_obs=True)["observation"]
    else:
        exp_obs = oc["observation"]
    got_obs = v.dev.observation[rows[obs_rows]].cpu().numpy()
    if not np.array_equal(got_obs, exp_obs):
        idx = np.argwhere(got_obs != exp_obs)[:5]
        raise AssertionError(f"{game} {root!r} level {paths.shape[0]}: observation differs at {idx.tolist()}")
    # Core.encode() bytes themselves on a few rows (the fingerprint already covers all of them)
    for j in rng.choice(m, min(8, m), replace=False):
        st = v.kern.state_at(resolve(game), v, int(rows[j]), v.limit)
        assert st.core.encode() == ob.encode(int(j))


def expand(kern, gdef, v):
    """Level d -> d+1: replicate each parent row once per legal action (bbk_copy_rows), then one
    batched step launch. Returns (children batch, parent index per child, action per child)."""
    import torch

    from paper_2303_17503_b200.search import copy_rows
    from paper_2303_17503_b200 import _native as nat

    parents, actions = np.nonzero(v.legal_action_mask)
    n2 = len(parents)
    w = kern.new_v(n2, 0, v.device, v.t, v.limit, obs=True)
    w.store = v.store.like(n2)
    w.store.lineage = Lineage(w.uid)
    src = torch.from_numpy(parents.astype(np.int32)).to(v.device)
    copy_rows(kern.row_tensors(v), kern.row_tensors(w), src, None, n2, nat.stream_handle(v.device))
    out = kern.step(gdef, w, actions.astype(np.int64), bb.RngKey(1), v.limit)
    return out, parents, actions


def run_perft(oracle, game, root, counts, extra=None):
    gdef = resolve(game)
    kern = gdef.batch_kernel
    rng = np.random.default_rng(len(root))
    v = kern.load(gdef, [root], key=KEY)
    _check_level(oracle, game, root, v, np.zeros((0, 1), np.int64), rng)
    paths = np.zeros((0, 1), np.int64)
    levels = len(counts) - 1 + (extra is not None)
    for d in range(levels):
        nodes = int(np.asarray(v.legal_action_mask).sum())
        assert counts[d] is None or nodes == counts[d], f"{game} {root!r}: perft({d + 1}) = {nodes}, expected {counts[d]}"
        v, parents, actions = expand(kern, gdef, v)
        paths = np.concatenate([paths[:, parents], actions[None, :]], axis=0)
        _check_level(oracle, game, root, v, paths, rng)
    total = int(np.asarray(v.legal_action_mask).sum())
    exp = extra if extra is not None else counts[-1]
    assert exp is None or total == exp, f"{game} {root!r}: perft({levels + 1}) = {total}, expected {exp}"


@pytest.mark.parametrize("fen,counts", CHESS_KATS, ids=["start", "kiwipete", "pos3", "pos4", "pos5", "pos6"])
def test_chess_device_perft(oracle, fen, counts):
    run_perft(oracle, "chess", fen, counts)


@pytest.mark.parametrize("fen,count", CHESS_DEEP, ids=["start", "kiwipete", "pos3", "pos4", "pos5", "pos6"])
def test_chess_device_perft_one_deeper(oracle, fen, count):
    run_perft(oracle, "chess", fen, dict(CHESS_KATS)[fen], extra=count)


@pytest.mark.parametrize("sfen,counts", SHOGI_KATS, ids=["start", "matsuri", "max593"])
def test_shogi_device_perft(oracle, sfen, counts):
    run_perft(oracle, "shogi", sfen, counts)


def test_loaded_positions_match_oracle_rule_positions(oracle):
    """Hand-built rule positions of the oracle tests (mate, stalemate, insufficient material,
    fifty-move rule, castling through check, en-passant pins, underpromotions) loaded on the device
    in one batch: every column, encode and observation equal to the oracle's set_fen."""
    fens = [
        "rnb1kbnr/pppp1ppp/8/4p3/6Pq/5P2/PPPPP2P/RNBQKBNR w KQkq - 1 3",   # fool's mate
        "7k/5Q2/6K1/8/8/8/8/8 b - - 0 1",                                  # stalemate
        "8/8/8/4k3/8/8/2B5/4K3 w - - 0 1",                                 # K+B vs K
        "8/8/2b5/4k3/8/8/2B5/4K3 w - - 0 1",                               # same-colour bishops
        "8/8/1b6/4k3/8/8/2B5/4K3 w - - 0 1",                               # opposite bishops: play on
        "4k3/8/8/8/8/8/4P3/R3K3 w - - 100 80",                             # fifty-move rule
        "4k3/8/8/8/8/8/4P3/R3K3 w - - 99 80",
        "r3k2r/8/8/8/8/8/8/R3K2R w KQkq - 0 1",                            # both castlings
        "r3k2r/8/8/8/8/5q2/8/R3K2R w KQkq - 0 1",                          # O-O through check
        "r3k2r/8/8/8/8/3q4/8/R3K2R w KQkq - 0 1",                          # O-O-O through check
        "1r2k3/8/8/8/8/8/8/R3K2R w KQ - 0 1",                              # O-O-O: b1 attacked only
        "8/8/8/KPp4r/8/8/8/7k w - c6 0 2",                                 # horizontal ep pin
        "8/8/8/8/k1pP3R/8/8/4K3 b - d3 0 1",                               # ep pin (black)
        "4k3/8/8/2KpP3/8/8/8/8 w - d6 0 1",                                # ep capture of the checker
        "n1n5/PPPk4/8/8/8/8/4Kppp/5N1N b - - 0 1",                         # underpromotion captures
        "n1n5/PPPk4/8/8/8/8/4Kppp/5N1N w - - 0 1",
        KIWIPETE, POS3, POS4, POS5, POS6,
    ]
    gdef = resolve("chess")
    v = gdef.batch_kernel.load(gdef, fens, key=KEY)
    ob = oracle.ChessBatch(len(fens))
    ob.init(KEY, 0)
    for i, f in enumerate(fens):
        ob.set_fen(i, f)
    oc = ob.columns()
    for c in COLS + ("observation",):
        got, exp = np.asarray(getattr(v, c)), oc[c]
        if got.dtype == np.bool_:
            got, exp = got.astype(np.uint8), exp.astype(np.uint8)
        assert np.array_equal(got, exp), c
    for i in range(len(fens)):
        assert v.kern.state_at(gdef, v, i, v.limit).core.encode() == ob.encode(i), fens[i]
    assert v.terminated[0] and v.terminated[1] and v.terminated[2] and v.terminated[3] and v.terminated[5]
    assert not v.terminated[4] and not v.terminated[6]
    # under-promotion planes present for the b7 pawn capturing a8 / c8 (mover frame, white)
    m = v.legal_action_mask[15]
    assert m[49 * 73 + 64 + 0] and m[49 * 73 + 64 + 2] and m[49 * 73 + 64 + 3 * 2 + 2]


def test_loaded_shogi_rule_positions_match_oracle(oracle):
    sfens = [
        "8k/9/7GN/9/9/9/9/9/K8 b P 1",            # pawn-drop mate (uchifuzume) is illegal
        "8k/9/7G1/9/9/9/9/9/K8 b P 1",            # ... legal when the king escapes
        "k8/9/9/9/9/9/9/9/8K b 2P 1",             # nifu: pawns in hand, free files
        "k8/9/9/9/4P4/9/9/9/8K b P 1",            # nifu on file 5
        "4k4/9/9/9/9/9/9/9/4K4 b L 1",            # lance drops not on the last rank
        "4k4/9/9/9/9/9/9/9/4K4 b N 1",            # knight drops not on the last two ranks
        "4k4/4P4/9/9/9/9/9/9/4K4 w - 1",          # check by a pawn
        "lnsgkgsnl/1r5b1/ppppppppp/9/9/2P6/PP1PPPPPP/1B5R1/LNSGKGSNL w - 1",
        MATSURI, MAXPOS,
    ]
    gdef = resolve("shogi")
    v = gdef.batch_kernel.load(gdef, sfens, key=KEY)
    ob = oracle.ShogiBatch(len(sfens))
    ob.init(KEY, 0)
    for i, s in enumerate(sfens):
        ob.set_sfen(i, s)
    oc = ob.columns()
    for c in COLS + ("observation",):
        got, exp = np.asarray(getattr(v, c)), oc[c]
        if got.dtype == np.bool_:
            got, exp = got.astype(np.uint8), exp.astype(np.uint8)
        assert np.array_equal(got, exp), c
    for i in range(len(sfens)):
        assert v.kern.state_at(gdef, v, i, v.limit).core.encode() == ob.encode(i), sfens[i]
    assert not v.legal_action_mask[0][20 * 81 + 17] and v.legal_action_mask[1][20 * 81 + 17]
    assert int(v.legal_action_mask[9].sum()) == 593


def test_loaded_positions_then_random_play_match_oracle(oracle):
    """Random play from the perft positions (not only the start position): 64 slots cycling the
    roots, 120 steps, bit-exact every step (the slot keys drive resets into the start position)."""
    for game, roots in (("chess", [KIWIPETE, POS3, POS4, POS5, POS6]), ("shogi", [MATSURI, MAXPOS, SHOGI_START])):
        gdef = resolve(game)
        kern = gdef.batch_kernel
        n = 64
        pos = [roots[i % len(roots)] for i in range(n)]
        v = kern.load(gdef, pos, key=KEY)
        ob = _oracle_batch(oracle, game, n)
        ob.init(KEY, 0)
        for i, p in enumerate(pos):
            (ob.set_fen if game == "chess" else ob.set_sfen)(i, p)
        for t in range(120):
            oc = ob.columns(with_obs=(t % 10 == 0))
            for c in COLS:
                got, exp = np.asarray(getattr(v, c)), oc[c]
                if got.dtype == np.bool_:
                    got, exp = got.astype(np.uint8), exp.astype(np.uint8)
                assert np.array_equal(got, exp), (game, t, c)
            if t % 10 == 0:
                assert np.array_equal(v.observation, oc["observation"]), (game, t)
            akey = oracle._child(KEY, 1000 + t)
            a = oracle.random_actions(oc["legal_action_mask"], akey)
            skey = oracle._child(KEY, 2000 + t)
            v = kern.step(gdef, v, a, skey, v.limit)
            assert ob.step(a, skey) == -1
