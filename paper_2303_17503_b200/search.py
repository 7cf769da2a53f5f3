"""Batched UCT search on the device: reference ``agents.mcts_agent`` (agents.py:49-131) for many
root states at once.

One search per root; all searches advance one simulation at a time through the kernels of
``csrc/mcts.cu`` and the game's own step kernel:

  select   (bbk_mcts_select)   UCB descent + random untried expansion, one thread per search
  expand   (bbk_copy_rows + step kernel + bbk_copy_rows)   parent rows of the node pool ->
           staging batch -> one step -> child rows back into the pool
  rollout  (bbk_mcts_rollout_actions + step kernel + bbk_mcts_latch)*   uniform random play to
           the end of the episode; the host polls a finished-search counter every few steps
  backup   (bbk_mcts_backup)

The node pool is an ordinary batch of the game's state with ``n_search * (simulations + 1)``
slots (node k of search s in row ``s * (simulations + 1) + k``), so any engine whose step kernel
exists can be searched. Each search draws from its own MT19937 stream seeded like
``random.Random(key.state)`` in the reference's order, and UCB is evaluated with the
reference's double-precision operation order, so the chosen actions equal ``mcts_agent``'s.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as nat
from .core import TerminalStep, UnsupportedGame


def _torch():
    import torch

    return torch


def check_searchable(gdef) -> None:
    """mcts_agent's game restriction (agents.py:81-82)."""
    if gdef.chance_in_step or not gdef.perfect_information or gdef.spec.num_players != 2:
        raise UnsupportedGame(f"mcts_agent does not support {gdef.game_id}")


def _unit(t) -> int:
    rb = t[0].numel() * t.element_size() if t.shape[0] else 0
    for u in (16, 8, 4):
        if rb % u == 0 and t.data_ptr() % u == 0:
            return u
    return 1


def copy_rows(src_tensors, dst_tensors, src_idx, dst_idx, n: int, stream) -> None:
    """dst[dst_idx[i]] = src[src_idx[i]] for every per-slot tensor pair (bbk_copy_rows)."""
    for idx in (src_idx, dst_idx):
        if idx is not None and (idx.dtype != _torch().int32 or not idx.is_contiguous()):
            raise ValueError("bbk_copy_rows takes contiguous int32 row indices")
    pairs = list(zip(src_tensors, dst_tensors))
    for k in range(0, len(pairs), nat.ROW_COPY_MAX):
        chunk = pairs[k:k + nat.ROW_COPY_MAX]
        rs = nat.RowCopySet()
        rs.count = len(chunk)
        for j, (s, d) in enumerate(chunk):
            if not (s.is_contiguous() and d.is_contiguous()) or s.shape[1:] != d.shape[1:] or s.dtype != d.dtype:
                raise ValueError("row copy between incompatible tensors")
            rb = s[0].numel() * s.element_size()
            rs.t[j].src = s.data_ptr()
            rs.t[j].dst = d.data_ptr()
            rs.t[j].row_bytes = rb
            rs.t[j].unit = min(_unit(s), _unit(d))
        nat.check(nat.lib().bbk_copy_rows(ctypes.byref(rs), nat.ptr(src_idx), nat.ptr(dst_idx), n, stream),
                  "bbk_copy_rows")


class SearchPool:
    """Device buffers of n_search concurrent searches of `simulations` simulations each:
    the tree arrays (bbk_mcts_tree), the node pool and two staging batches. Reusable for
    every search with the same template batch layout, n_search and simulations."""

    def __init__(self, kern, template, n_search: int, simulations: int):
        torch = _torch()
        self.kern = kern
        self.n = int(n_search)
        self.sims = max(1, int(simulations))
        self.M = self.sims + 1
        self.device = template.device
        self.limit = template.limit
        dev, n, M = self.device, self.n, self.M
        A = kern.num_actions
        W = (A + 31) // 32
        i32 = torch.int32
        self.mt = torch.empty((n, 625), dtype=i32, device=dev)
        self.visits = torch.empty((n, M), dtype=i32, device=dev)
        self.value_sum = torch.empty((n, M), dtype=torch.float64, device=dev)
        self.parent = torch.empty((n, M), dtype=i32, device=dev)
        self.first_child = torch.empty((n, M), dtype=i32, device=dev)
        self.last_child = torch.empty((n, M), dtype=i32, device=dev)
        self.next_sibling = torch.empty((n, M), dtype=i32, device=dev)
        self.action = torch.empty((n, M), dtype=i32, device=dev)
        self.role = torch.empty((n, M), dtype=torch.uint8, device=dev)
        self.untried = torch.empty((n, M, W), dtype=i32, device=dev)
        self.untried_count = torch.empty((n, M), dtype=i32, device=dev)
        self.next_node = torch.empty(n, dtype=i32, device=dev)
        self.leaf = torch.empty(n, dtype=i32, device=dev)
        self.tree = nat.MctsTree(n, M, A, W, *(nat.ptr(t) for t in (
            self.mt, self.visits, self.value_sum, self.parent, self.first_child, self.last_child, self.next_sibling,
            self.action, self.role, self.untried, self.untried_count, self.next_node, self.leaf)))
        # per-simulation scratch
        self.src_row = torch.empty(n, dtype=i32, device=dev)
        self.dst_row = torch.empty(n, dtype=i32, device=dev)
        self.new_id = torch.empty(n, dtype=i32, device=dev)
        self.act = torch.empty(n, dtype=torch.int64, device=dev)
        self.done = torch.empty(n, dtype=torch.uint8, device=dev)
        self.ret = torch.empty((n, 2), dtype=torch.float32, device=dev)
        self.count = torch.empty(1, dtype=torch.int64, device=dev)
        self.best = torch.empty(n, dtype=torch.int64, device=dev)
        self.root_dst = (torch.arange(n, dtype=i32, device=dev) * M).contiguous()
        logs = [0.0] + [math.log(v) for v in range(1, M + 1)]   # Python math.log: the reference's libm
        self.logtab = torch.tensor(logs, dtype=torch.float64, device=dev)
        # node pool and staging (a and b share one per-env store: a rollout is one trajectory)
        self.pool = kern.new_v_like(template, n * M)
        self.sa = kern.new_v_like(template, n)
        self.sb = kern.new_v_like(template, n, store=False)
        self.sb.store = self.sa.store
        self.pool_rows = kern.row_tensors(self.pool)
        self.graphs = {}

    def graph(self, key, fn) -> None:
        """Replay the CUDA graph of `fn`'s launches (captured on first use) on the current stream.
        Every pointer the launches use belongs to this pool, so the capture stays valid."""
        torch = _torch()
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.graph(g, stream=side):
                fn()
            torch.cuda.current_stream(self.device).wait_stream(side)
            self.graphs[key] = g
        g.replay()

    def fits(self, kern, template, n_search, simulations) -> bool:
        return (kern is self.kern and n_search == self.n and max(1, int(simulations)) == self.sims
                and template.device == self.device and template.limit == self.limit
                and [tuple(t.shape[1:]) for t in kern.row_tensors(template)] ==
                [tuple(t.shape[1:]) for t in self.pool_rows])


SHORT_CHUNK, LONG_CHUNK = 4, 32   # rollout moves between finished-search polls (even: ping-pong parity)


def _latch(v, sel, want, p, stream) -> None:
    d = v.dev
    nat.check(nat.lib().bbk_mcts_latch(nat.ptr(d.terminated), nat.ptr(d.truncated), nat.ptr(d.rewards),
                                       nat.ptr(d.player_to_role), nat.ptr(sel), int(want), p.n, nat.ptr(p.done),
                                       nat.ptr(p.ret), nat.ptr(p.count), stream), "bbk_mcts_latch")


def search(v, rows, key_states, simulations: int = 32, *, exploration: float = math.sqrt(2.0),
           value_transform: tuple = (1.0, 0.0), pool: SearchPool | None = None, stats: dict | None = None,
           graphs: bool = True):
    """mcts_agent(state_at(v, rows[s]), RngKey(key_states[s]), simulations, ...) for every s, on the device.

    Returns the chosen actions as a CUDA int64 tensor [len(rows)]. Rows must be unfinished slots
    of batch v (mcts_agent raises TerminalStep otherwise; checked by the caller). ``stats``, if
    given, accumulates the batched steps taken (``expand_steps``, ``rollout_steps``). With
    ``graphs`` the per-simulation launch sequence and the rollout chunks replay as CUDA graphs
    captured once per pool (the loop is otherwise bound by host launch overhead)."""
    torch = _torch()
    kern = v.kern
    L = nat.lib()
    n = len(rows)
    sims = max(1, int(simulations))
    if pool is None or not pool.fits(kern, v, n, sims):
        pool = SearchPool(kern, v, n, sims)
    p = pool
    dev = v.device
    stream = nat.stream_handle(dev)
    scale, offset = value_transform
    c = exploration * scale   # agents.py:84
    tree = ctypes.byref(p.tree)
    rows_t = torch.as_tensor(np.asarray(rows, dtype=np.int32)).to(dev)
    keys = torch.as_tensor(np.asarray([int(k) & ((1 << 64) - 1) for k in key_states], dtype=np.uint64)
                           .view(np.int64)).to(dev)
    # roots: v rows -> staging a -> pool rows s * M; untried sets from the staging masks
    depth = kern.branch_depth(v)   # > 0: v branches off a shared store that its descendants moved on
    copy_rows(kern.row_tensors(v), kern.row_tensors(p.sa), rows_t, None, n, stream)
    if depth > 0 and hasattr(kern, "rebuild_filters"):
        kern.rebuild_filters(p.sa)   # the store rows may carry entries of v's descendants
    copy_rows(kern.row_tensors(p.sa), p.pool_rows, None, p.root_dst, n, stream)
    nat.check(L.bbk_mcts_seed(tree, nat.ptr(keys), stream), "bbk_mcts_seed")
    sa, sb = p.sa, p.sb
    nat.check(L.bbk_mcts_untried(tree, nat.ptr(sa.dev.legal_action_mask), nat.ptr(sa.dev.current_player),
                                 nat.ptr(sa.dev.player_to_role), None, stream), "bbk_mcts_untried")
    limit = v.limit
    sa_rows, sb_rows = kern.row_tensors(sa), kern.row_tensors(sb)

    def prologue():   # selection, expansion step, first latches (one simulation, up to the rollout)
        st = nat.stream_handle(dev)
        nat.check(L.bbk_mcts_select(tree, float(c), nat.ptr(p.logtab), nat.ptr(p.src_row), nat.ptr(p.dst_row),
                                    nat.ptr(p.act), nat.ptr(p.new_id), st), "bbk_mcts_select")
        copy_rows(p.pool_rows, sa_rows, p.src_row, None, n, st)
        p.done.zero_()
        p.count.zero_()
        _latch(sa, p.new_id, 0, p, st)        # finished leaves score themselves
        kern.raw_step(sa, sb, p.act, limit)   # expansion step (agents.py:106)
        copy_rows(sb_rows, p.pool_rows, None, p.dst_row, n, st)
        nat.check(L.bbk_mcts_untried(tree, nat.ptr(sb.dev.legal_action_mask), nat.ptr(sb.dev.current_player),
                                     nat.ptr(sb.dev.player_to_role), nat.ptr(p.new_id), st), "bbk_mcts_untried")
        _latch(sb, p.new_id, 1, p, st)

    def rollout(k):   # k rollout moves (k even: the live batch is back in sb afterwards)
        st = nat.stream_handle(dev)
        cur, nxt = sb, sa
        for _ in range(k):
            nat.check(L.bbk_mcts_rollout_actions(tree, nat.ptr(cur.dev.legal_action_mask), nat.ptr(p.done),
                                                 nat.ptr(p.act), st), "bbk_mcts_rollout_actions")
            kern.raw_step(cur, nxt, p.act, limit)
            _latch(nxt, None, 1, p, st)
            cur, nxt = nxt, cur

    run_pro = (lambda: p.graph(("pro", float(c)), prologue)) if graphs else prologue
    prev = 0
    for _ in range(sims):
        run_pro()
        t = 0
        while int(p.count.item()) < n:
            k = LONG_CHUNK if t + LONG_CHUNK <= 0.75 * prev else SHORT_CHUNK
            if graphs:
                p.graph(("roll", k), lambda: rollout(k))
            else:
                rollout(k)
            t += k
        prev = max(prev, t)
        if stats is not None:
            stats["expand_steps"] = stats.get("expand_steps", 0) + 1
            stats["rollout_steps"] = stats.get("rollout_steps", 0) + t
        nat.check(L.bbk_mcts_backup(tree, nat.ptr(p.ret), float(scale), float(offset), stream), "bbk_mcts_backup")
    nat.check(L.bbk_mcts_best(tree, nat.ptr(p.best), stream), "bbk_mcts_best")
    return p.best.clone()


def mcts_agent(state, key, simulations: int = 32, *, exploration: float = math.sqrt(2.0),
               value_transform: tuple = (1.0, 0.0)) -> int:
    """reference agents.mcts_agent (agents.py:63-123) for one state of a device batch."""
    from .rng import key_state

    gdef = state.game
    check_searchable(gdef)
    if state.terminated or state.truncated:
        raise TerminalStep("cannot search from a finished state")
    if state._v is None:
        raise UnsupportedGame("mcts_agent needs a state of a device batch")
    out = search(state._v, [state._i], [key_state(key)], simulations, exploration=exploration,
                 value_transform=value_transform)
    return int(out[0].item())


def mcts_actions(batch, key, simulations: int = 32, *, exploration: float = math.sqrt(2.0),
                 value_transform: tuple = (1.0, 0.0), pool: SearchPool | None = None) -> np.ndarray:
    """Batched mcts_agent: slot i gets ``mcts_agent(states[i], key.child(slot0 + i), simulations)``
    (the key convention of agents.random_actions, agents.py:33-46); finished slots get 0."""
    from .rng import child_states, key_state

    v = batch._v
    check_searchable(batch.game)
    fin = np.asarray(v.terminated, dtype=bool) | np.asarray(v.truncated, dtype=bool)
    live = np.flatnonzero(~fin)
    out = np.zeros(v.n, dtype=np.int64)
    if live.size:
        ks = child_states(key_state(key), v.n, v.slot0)[live]
        res = search(v, live.tolist(), ks.tolist(), simulations, exploration=exploration,
                     value_transform=value_transform, pool=pool)
        out[live] = res.cpu().numpy()
    return out
