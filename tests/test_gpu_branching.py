"""Value semantics of device states (reference core.py:1-7: states are immutable values and step is
a pure function) under the shared per-trajectory history stores (Go superko, chess ring, shogi key
log), plus the host-side thread-safety of the shared kernel objects.

* scalar trajectories (core.init / core.step) never auto-reset, so their stores are append-only:
  ANY earlier state can be stepped again (the reference's mcts_agent re-steps stored node states),
  and the original trajectory stays steppable afterwards;
* batch trajectories share the store with the newest batch and its last predecessors (Go two,
  chess / shogi one); a held batch that falls further behind gets a private store first, so it
  stays steppable too (DeviceKernel.release), and a loop that drops its batches never pays that;
* search() and slicing honour the same rule.
"""

import threading

import numpy as np
import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.agents import random_actions

pytestmark = pytest.mark.gpu

GAMES = ("go_9x9", "go_19x19", "chess", "shogi", "backgammon")


def _walk(game, key, n_steps):
    st = [bb.init(game, key.child(0))]
    acts = []
    for t in range(1, n_steps + 1):
        s = st[-1]
        if s.terminated or s.truncated:
            break
        legal = np.flatnonzero(s.legal_action_mask)
        a = int(legal[key.child(2 * t).randint(len(legal))])
        acts.append(a)
        st.append(bb.step(s, a, key.child(2 * t + 1)))
    return st, acts


@pytest.mark.parametrize("game", GAMES)
def test_scalar_states_branch_at_any_depth(game):
    key = bb.RngKey(41)
    states, acts = _walk(game, key, 40)
    assert len(states) > 12
    for j in (1, 4, len(states) // 2):   # re-step an old state with a different legal action
        s = states[j]
        legal = np.flatnonzero(s.legal_action_mask)
        a = int(legal[-1])
        got = bb.step(s, a, key.child(2 * (j + 1) + 1))
        # reference semantics: identical to replaying the same actions from a fresh init
        r = bb.init(game, key.child(0))
        for t, b in enumerate(acts[:j], start=1):
            r = bb.step(r, b, key.child(2 * t + 1))
        want = bb.step(r, a, key.child(2 * (j + 1) + 1))
        assert bb.state_fingerprint(got) == bb.state_fingerprint(want), (game, j)
        assert np.array_equal(bb.observe(got, 0), bb.observe(want, 0))
    # ... and the original trajectory is untouched: its head steps on like before
    head = states[-1]
    if not (head.terminated or head.truncated):
        a = int(np.flatnonzero(head.legal_action_mask)[0])
        bb.step(head, a, key.child(999))
        states2, _ = _walk(game, key, len(states) - 1)
        for x, y in zip(states, states2):
            assert bb.state_fingerprint(x) == bb.state_fingerprint(y)


@pytest.mark.parametrize("game,keep", [("go_9x9", 2), ("go_19x19", 2), ("chess", 1), ("shogi", 1)])
def test_batch_states_branch_at_any_depth(game, keep):
    """Every held batch stays steppable: within keep of the head it branches off the shared store;
    a held batch that falls further behind was given a store of its own before its history could
    be overwritten (DeviceKernel.release). Each branch equals a from-scratch replay."""
    root = bb.RngKey(3)
    kern = bb.core.resolve(game).batch_kernel
    b = [bb.batch_init(game, root.child(0), 64)]
    s0 = kern.snapshots
    T = 12
    for t in range(1, T + 1):
        b.append(bb.batch_step(b[-1], random_actions(b[-1], root.child(2 * t - 1)), root.child(2 * t)))
    assert kern.snapshots - s0 == T - keep   # every held batch older than keep was copied once
    for d in (keep, keep + 1, T // 2, T):
        src = b[-1 - d]
        acts = random_actions(src, root.child(777 + d))
        got = bb.batch_step(src, acts, root.child(778))
        r = bb.batch_init(game, root.child(0), 64)
        for t in range(1, T + 1 - d):
            r = bb.batch_step(r, random_actions(r, root.child(2 * t - 1)), root.child(2 * t))
        want = bb.batch_step(r, acts, root.child(778))
        assert bb.batch_fingerprint(got) == bb.batch_fingerprint(want), (game, d)
        assert np.array_equal(got.observation, want.observation)
    # the head's trajectory is untouched by all of that and steps on like a fresh replay
    nxt = bb.batch_step(b[-1], random_actions(b[-1], root.child(11)), root.child(12))
    r = bb.batch_init(game, root.child(0), 64)
    for t in range(1, T + 1):
        r = bb.batch_step(r, random_actions(r, root.child(2 * t - 1)), root.child(2 * t))
    assert bb.batch_fingerprint(nxt) == bb.batch_fingerprint(
        bb.batch_step(r, random_actions(r, root.child(11)), root.child(12)))


@pytest.mark.parametrize("game", ["go_19x19", "chess", "shogi"])
def test_a_loop_that_drops_its_batches_copies_no_store(game):
    """The copy is paid only by held batches: the reference's step loop (and the result fetcher that
    keeps the previous batch until its copies land) never triggers one."""
    root = bb.RngKey(5)
    kern = bb.core.resolve(game).batch_kernel
    b = bb.batch_init(game, root.child(0), 256)
    fetch = bb.ResultFetcher(256, 2)
    s0 = kern.snapshots
    for t in range(1, 40):
        b = bb.batch_step(b, random_actions(b, root.child(2 * t - 1)), root.child(2 * t))
        fetch.fetch(b)
    fetch.drain()
    assert kern.snapshots == s0


def test_scalar_chess_states_older_than_the_ring_window_stay_steppable():
    """A scalar chess trajectory keeps its states on one 128-ply ring; states the caller holds get
    their own ring before the head is far enough ahead to overwrite their window."""
    key = bb.RngKey(8)
    states, acts = _walk("chess", key, 70)
    assert len(states) > 60
    for j in (2, 20):
        s = states[j]
        a = int(np.flatnonzero(s.legal_action_mask)[-1])
        got = bb.step(s, a, key.child(5000 + j))
        r = bb.init("chess", key.child(0))
        for t, x in enumerate(acts[:j], start=1):
            r = bb.step(r, x, key.child(2 * t + 1))
        want = bb.step(r, a, key.child(5000 + j))
        assert bb.state_fingerprint(got) == bb.state_fingerprint(want), j
        assert np.array_equal(bb.observe(got, 0), bb.observe(want, 0))


def test_search_on_a_predecessor_batch_equals_search_before_stepping():
    from paper_2303_17503_b200.agents import mcts_actions

    root = bb.RngKey(9)
    b = bb.batch_init("go_9x9", root.child(0), 16)
    for t in range(1, 30):
        b = bb.batch_step(b, random_actions(b, root.child(2 * t - 1)), root.child(2 * t))
    live = ~(b.terminated | b.truncated)
    assert live.all()
    before = np.asarray(mcts_actions(b, root.child(100), 8))
    b1 = bb.batch_step(b, random_actions(b, root.child(101)), root.child(102))
    b2 = bb.batch_step(b1, random_actions(b1, root.child(103)), root.child(104))
    after = np.asarray(mcts_actions(b, root.child(100), 8))   # b is two steps behind now
    assert np.array_equal(before, after)
    bb.batch_step(b2, random_actions(b2, root.child(105)), root.child(106))
    later = np.asarray(mcts_actions(b, root.child(100), 8))   # three behind: b has its own store
    assert np.array_equal(before, later)


def test_threads_stepping_the_same_game_match_a_sequential_run():
    """One kernel object per game is shared by every caller: launches from several threads (each
    with its own fused next-actions buffer) must not see each other's pointers."""
    import torch

    def run(seed, out, idx):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            sess = bb.BatchSession("go_9x9", 512, seed)
            prints = []
            for _ in range(40):
                sess.step(sess.sample_random_actions())
                prints.append(bb.batch_fingerprint(sess.batch))
        out[idx] = prints

    seq = [None] * 4
    for i in range(4):
        run(i, seq, i)
    par = [None] * 4
    th = [threading.Thread(target=run, args=(i, par, i)) for i in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert par == seq


def test_random_actions_into_pinned_buffer_is_synchronised_and_copied():
    import torch

    root = bb.RngKey(4)
    b = bb.batch_init("chess", root.child(0), 4096)
    buf = torch.empty(4096, dtype=torch.int64).pin_memory()
    nxt = bb.batch_step(b, random_actions(b, root.child(1)), root.child(2), next_key=root.child(3), next_actions=buf)
    got = random_actions(nxt, root.child(3))
    want = np.asarray(nxt._v.kern.random_actions(nxt._v, root.child(3)).cpu())
    assert np.array_equal(got, want)
    assert not np.shares_memory(got, buf.numpy())
