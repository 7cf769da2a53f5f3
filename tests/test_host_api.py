"""Host-side API contract (no GPU): registry, specs, errors, key schedule (reference test_core.py:10-50)."""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.games._device import Lineage

EXPECTED = {
    "go_9x9": (2, (9, 9, 17), 82),
    "go_19x19": (2, (19, 19, 17), 362),
    "backgammon": (2, (34,), 156),
    "chess": (2, (8, 8, 119), 4672),
    "shogi": (2, (9, 9, 119), 2187),
    # the reference's small engines (games/*.py specs)
    "tic_tac_toe": (2, (3, 3, 2), 9),
    "connect_four": (2, (6, 7, 2), 7),
    "othello": (2, (8, 8, 2), 65),
    "hex": (2, (11, 11, 4), 122),
    "2048": (1, (4, 4, 31), 4),
    "kuhn_poker": (2, (7,), 4),
    "leduc_holdem": (2, (34,), 3),
}


def test_registry_has_the_hot_path_and_small_games():
    assert set(bb.available_games()) == set(EXPECTED)


@pytest.mark.parametrize("game_id", sorted(EXPECTED))
def test_specs_match_table(game_id):
    spec = bb.game_spec(game_id)
    assert (spec.num_players, spec.observation_shape, spec.num_actions) == EXPECTED[game_id]


def test_reserved_and_unknown_ids():
    for game_id in ("gardner_chess", "bridge_bidding", "animal_shogi", "minatar_breakout"):
        assert bb.game_spec(game_id).num_actions > 0
        with pytest.raises(bb.UnsupportedGame):
            bb.batch_init(game_id, bb.RngKey(0), 2)
    with pytest.raises(bb.UnsupportedGame):
        bb.game_spec("parcheesi")


def test_empty_batch_rejected_before_any_device_work():
    with pytest.raises(bb.EmptyBatch):
        bb.batch_init("go_9x9", bb.RngKey(0), 0)


def test_self_capture_variant_and_other_sizes():
    from paper_2303_17503_b200.games import go

    g = go.make_game(9, allow_self_capture=True)
    assert g.batch_kernel.allow_self_capture and g.spec.game_id == "go_9x9"
    assert not go.GAME.batch_kernel.allow_self_capture
    assert go.make_game(13).spec.num_actions == 170
    assert go.make_game(7).spec.num_actions == 50
    for bad in (4, 21):
        with pytest.raises(bb.UnsupportedGame):
            go.make_game(bad)


def test_lineage_allows_head_and_recent_branches():
    lin = Lineage(1)
    assert lin.depth(1) == 0
    lin.advance(1, 2)
    lin.advance(2, 3)
    assert lin.depth(3) == 0 and lin.depth(2) == 1 and lin.depth(1) == 2 and lin.depth(99) > 2
    lin.advance(2, 4)          # branch from the predecessor: 3 is dropped
    assert lin.depth(4) == 0 and lin.depth(2) == 1 and lin.depth(3) > 2


def test_lineage_reports_what_falls_off_the_trail():
    lin = Lineage(1)
    assert lin.advance(1, 2) == [] and lin.advance(2, 3) == [] and lin.advance(3, 4) == []
    assert lin.trail == [3, 2, 1]                     # append-only: the full trail
    assert lin.mark_batch_step(2) == [1]              # a batch step keeps two predecessors
    assert lin.mark_batch_step(2) == []
    assert lin.advance(4, 5) == [2] and lin.trail == [4, 3]
    assert lin.advance(4, 6) == [5] and lin.trail == [4, 3]   # branch in place: the old head goes
    assert lin.drop([4]) == [4] and lin.trail == [3]


def test_release_gives_held_batches_their_own_store():
    """DeviceKernel.release: a live batch that leaves the trail gets a private store copy and its
    own lineage; dead batches and batches reusing a uid slot (the bench's ping-pong) are skipped."""
    import gc

    from paper_2303_17503_b200.games._device import DeviceKernel

    class Store:
        def __init__(self, rows):
            self.rows, self.lineage = rows, None

        def clone_rows(self):
            return Store(list(self.rows))

    class B:
        def __init__(self, uid, t, store):
            self.uid, self.t, self.store = uid, t, store

    class K(DeviceKernel):
        ready = []

        def private_store_ready(self, w):
            self.ready.append(w.uid)

    k = K()
    shared = Store([7, 8])
    shared.lineage = lin = Lineage(1)
    held = [B(1, 0, shared)]
    lin.track(held[0])
    for u in range(2, 6):
        b = B(u, u - 1, shared)
        lin.advance(u - 1, u, 2, u - 1)
        lin.track(b)
        held.append(b)
    lin.mark_batch_step(2)
    gone = lin.advance(5, 6, 2, 5)
    held[2].uid = 99                                  # object reused under another uid: not this batch
    del held[1]
    gc.collect()
    k.release(lin, [1, 2, 3] + gone)
    b1 = held[0]
    assert b1.store is not shared and b1.store.rows == [7, 8] and b1.store.lineage.head == 1
    assert b1.store.lineage.depth(1) == 0 and k.ready == [1] and k.snapshots == 1
    assert held[1].store is shared                    # the reused object keeps the shared store


def test_session_key_schedule_matches_reference_formula():
    # bench.py:54-83: init root.child(0), actions before step t root.child(2t-1), step t root.child(2t)
    root = bb.RngKey(0)
    assert root.child(0).state != root.child(1).state
    assert bb.RngKey(0).state == 0xE220A8397B1DCDAF


def test_output_wire_parser_roundtrip():
    """unpack_outputs reads the binary batch-outputs format (header + 64-B aligned fields)."""
    import json
    import struct

    from paper_2303_17503_b200.session import _WIRE_MAGIC, unpack_outputs

    a = np.arange(6, dtype=np.float32).reshape(2, 3)
    m = np.array([[True, False]], dtype=bool)
    hdr = json.dumps({"game_id": "x", "n": 2, "fields": {"observations": ["float32", [2, 3], 0, 24],
                                                         "legal_action_mask": ["bool", [1, 2], 64, 2]}}).encode()
    pre = _WIRE_MAGIC + struct.pack("<I", len(hdr)) + hdr
    base = (len(pre) + 63) // 64 * 64
    buf = bytearray(base + 66)
    buf[:len(pre)] = pre
    buf[base:base + 24] = a.tobytes()
    buf[base + 64:base + 66] = m.tobytes()
    o = unpack_outputs(bytes(buf))
    assert np.array_equal(o["observations"], a) and np.array_equal(o["legal_action_mask"], m)
    with pytest.raises(ValueError):
        unpack_outputs(b"XXXX" + bytes(60))


def test_bench_config_results_and_csv(tmp_path):
    """bench.py:32-60, 118-150 mirrors: validation, thread resolution and the CSV writers."""
    from paper_2303_17503_b200.session import resolve_threads

    with pytest.raises(ValueError):
        bb.bench_run(bb.BenchConfig("go_9x9", 0, 10))
    with pytest.raises(ValueError):
        bb.bench_run(bb.BenchConfig("go_9x9", 4, 0))
    assert resolve_threads("auto") >= 1 and resolve_threads(3) == 3
    with pytest.raises(ValueError):
        resolve_threads(0)
    r = bb.BenchResult("go_9x9", 8, 10, 0, 1, 0.125, 640.0, 3)
    p = tmp_path / "b.csv"
    bb.write_results([r], p)
    lines = p.read_text().splitlines()
    assert lines[0] == "game_id,batch_size,total_steps,seed,threads,wall_seconds,samples_per_second,episodes_completed"
    assert lines[1] == "go_9x9,8,10,0,1,0.125,640.0,3"
    bb.write_results_long([r], tmp_path / "l.csv")
    assert len((tmp_path / "l.csv").read_text().splitlines()) == 5
    with pytest.raises(bb.IoError):
        bb.write_results([r], tmp_path / "missing" / "x.csv")
    # match results (bench.py:162-170): the kind follows the row type
    from paper_2303_17503_b200.agents import MatchResult

    m = tmp_path / "m.csv"
    bb.write_results([MatchResult("tic_tac_toe", "random", "mcts", 3, 5, 2)], m)
    assert m.read_text().splitlines() == ["game_id,agent_a,agent_b,wins_a,wins_b,draws", "tic_tac_toe,random,mcts,3,5,2"]


def _toy_kernel():
    import torch

    from paper_2303_17503_b200.games._device import DeviceKernel

    class Toy(DeviceKernel):
        game_id, num_actions, obs_shape = "toy", 4, (3,)

        def alloc_private(self, v):
            v.priv.board = torch.zeros((v.n, 5), dtype=torch.uint8, device=v.device)

    return Toy()


def test_dead_batch_buffers_are_recycled_only_when_unreferenced():
    """new_v reuses a dead batch's buffers (e2e host overhead) but never ones still referenced."""
    import gc

    import torch

    k = _toy_kernel()
    v = k.new_v(8, 0, torch.device("cpu"), 0, 10)
    ids = (id(v.dev.rewards), id(v.priv.board))
    del v
    gc.collect()
    w = k.new_v(8, 0, torch.device("cpu"), 1, 10)
    assert (id(w.dev.rewards), id(w.priv.board)) == ids            # recycled
    assert k.new_v(4, 0, torch.device("cpu"), 0, 10).n == 4       # other shape: fresh
    pool = next(iter(k._pools.values()))
    for hold in (lambda x: x.dev.rewards, lambda x: x.dev.rewards[1:3], lambda x: x.priv.board.numpy(),
                 lambda x: torch.utils.dlpack.to_dlpack(x.dev.observation)):
        pool.clear()
        keep = hold(w)
        del w
        gc.collect()
        assert pool == []                                           # a live reference blocks reuse
        w = k.new_v(8, 0, torch.device("cpu"), 1, 10)
        del keep
    del w
    gc.collect()
    assert len(pool) == 1
