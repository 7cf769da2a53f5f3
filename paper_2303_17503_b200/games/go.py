"""Go (Tromp-Taylor, positional superko) on the device.

Drop-in for reference ``games/go.py``: ``make_game(size, komi)`` returns a
``GameDef`` with the same spec (``go_{N}x{N}``, obs (N, N, 17), N*N+1
actions, max_steps 512; go.py:282-290) whose ``batch_kernel`` runs
``csrc/go.cu`` through ``bbk_go_*`` (include/bbk.h).

Device state per slot (besides the public columns):
  pat[PS] int16   transposed 8-deep board history (bit 2t/2t+1: black/white
                  stone in boards_hist[t]); replaces ``board`` + ``boards_hist``
  lab[PS] int16   chain label per stone (a point of its chain), kept incrementally
  hash, hist_xor int64 (u64), hist_len int32, role_to_move, pass_count u8
and a per-lineage append-only superko store: history[hist_cap] u64 and an
8192-bit Bloom filter. The store is shared along a trajectory; a batch up
to two steps behind the head can still be stepped (the store is cloned and
the filters rebuilt), older ones raise ``StaleBatch``.
"""

from __future__ import annotations

import numpy as np

from .. import _native as nat
from ..core import GameDef, GameSpec, StaleBatch, UnsupportedGame
from ._device import DeviceKernel, DeviceV, Lineage, _torch

HISTORY_PLANES = 8
SIZES = (5, 7, 9, 11, 13, 15, 17, 19)   # step_kernel<N> instantiations (csrc/go.cu dispatch_step)


class GoCoreView:
    """Host view of one slot with the reference Core's fields (go.py:83-111)."""

    __slots__ = ("board", "role_to_move", "terminal", "rewards", "mask", "pass_count", "hash", "hist_xor",
                 "hist_len", "boards_hist", "_src", "_history")

    def __init__(self, board, role_to_move, terminal, rewards, mask, pass_count, hash_, hist_xor, hist_len,
                 boards_hist):
        self.board = board
        self.role_to_move = role_to_move
        self.terminal = terminal
        self.rewards = rewards
        self.mask = mask
        self.pass_count = pass_count
        self.hash = hash_
        self.hist_xor = hist_xor
        self.hist_len = hist_len
        self.boards_hist = boards_hist
        self._src = None
        self._history = None

    @property
    def history(self) -> frozenset:
        """The superko set (reference ``Core.history``, go.py:83-100): the slot's prefix of the
        device history store, read on first access. Raises StaleBatch when the batch is too far
        behind its lineage for the shared store to still hold its prefix."""
        if self._history is None:
            if self._src is None:
                raise AttributeError("history: core view is not attached to a device batch")
            v, i = self._src
            self._history = v.kern.history_of(v, i, self.hist_len)
        return self._history

    def encode(self) -> bytes:
        """Byte-identical to reference Core.encode (go.py:103-111)."""
        return (
            self.board
            + bytes([self.role_to_move, self.pass_count])
            + self.hash.to_bytes(8, "little")
            + self.hist_xor.to_bytes(8, "little")
            + self.hist_len.to_bytes(2, "little")
            + b"".join(self.boards_hist)
        )


class GoStore:
    """Per-env state shared IN PLACE along a lineage: the append-only superko history, its Bloom /
    stone-count filter, and the chain labels of the lineage head's board (a step writes only the
    labels it changes; a branch rebuilds them from the branching batch's board, bbk_go_relabel)."""

    def __init__(self, history, bloom, lab, hist_cap: int):
        self.history = history
        self.bloom = bloom
        self.lab = lab
        self.hist_cap = hist_cap
        self.lineage = None

    def row_tensors(self):
        return [self.history, self.bloom, self.lab]

    def like(self, n: int) -> "GoStore":
        torch = _torch()
        return GoStore(torch.empty((n, self.hist_cap), dtype=torch.int64, device=self.history.device),
                       torch.empty((n,) + tuple(self.bloom.shape[1:]), dtype=self.bloom.dtype,
                                   device=self.bloom.device),
                       torch.empty((n,) + tuple(self.lab.shape[1:]), dtype=self.lab.dtype, device=self.lab.device),
                       self.hist_cap)

    def clone_rows(self, rows=slice(None)) -> "GoStore":
        return GoStore(self.history[rows].clone(), self.bloom[rows].clone(), self.lab[rows].clone(), self.hist_cap)

    def struct(self) -> nat.GoStore:
        st = self.__dict__.get("_struct")
        if st is None:
            st = self._struct = nat.GoStore(nat.ptr(self.history), nat.ptr(self.bloom), nat.ptr(self.lab),
                                            self.hist_cap)
        return st


def _with_store(v: DeviceV, store) -> DeviceV:
    """A shallow stand-in of v whose store is `store` (v's private state, the copy's filters)."""
    from types import SimpleNamespace

    return SimpleNamespace(store=store, priv=v.priv, n=v.n, device=v.device)


class GoKernel(DeviceKernel):
    def __init__(self, size: int, komi: float = 6.5, allow_self_capture: bool = False):
        if size not in SIZES:
            raise UnsupportedGame(f"go size {size} has no device kernel (odd sizes 5..19 are instantiated)")
        self.size = size
        self.komi = float(komi)
        self.allow_self_capture = bool(allow_self_capture)
        self.cells = size * size
        self.num_actions = self.cells + 1
        self.obs_shape = (size, size, 2 * HISTORY_PLANES + 1)
        self.game_id = f"go_{size}x{size}"
        self.pat_stride = (self.cells + 7) & ~7

    @property
    def filter_words(self) -> int:
        """u32 words of one env's superko filter row (Bloom + stone-count pairs), as the loaded
        library sizes it per board (bbk_go_filter_words)."""
        fw = self.__dict__.get("_filter_words")
        if fw is None:
            fw = self._filter_words = int(nat.lib().bbk_go_filter_words(self.size))
            if fw <= 0:
                raise UnsupportedGame(f"go size {self.size}: no superko filter layout in the library")
        return fw

    def alloc_private(self, v: DeviceV) -> None:
        torch = _torch()
        n, dev = v.n, v.device
        p = v.priv
        p.pat = torch.empty((n, self.pat_stride), dtype=torch.int16, device=dev)
        p.hash = torch.empty(n, dtype=torch.int64, device=dev)
        p.hist_xor = torch.empty(n, dtype=torch.int64, device=dev)
        p.hist_len = torch.empty(n, dtype=torch.int32, device=dev)
        p.role_to_move = torch.empty(n, dtype=torch.uint8, device=dev)
        p.pass_count = torch.empty(n, dtype=torch.uint8, device=dev)

    def state_struct(self, v: DeviceV) -> nat.GoState:
        st = v.__dict__.get("_gostate")   # private tensors are fixed per batch: build once
        if st is not None:
            return st
        p = v.priv
        st = v._gostate = nat.GoState(nat.ptr(p.pat), nat.ptr(p.hash), nat.ptr(p.hist_xor),
                                      nat.ptr(p.hist_len), nat.ptr(p.role_to_move), nat.ptr(p.pass_count))
        return st

    def new_store(self, n: int, limit: int, device) -> GoStore:
        torch = _torch()
        cap = int(limit) + 2
        hist = torch.empty((n, cap), dtype=torch.int64, device=device)
        bloom = torch.empty((n, self.filter_words), dtype=torch.int32, device=device)
        lab = torch.empty((n, self.pat_stride), dtype=torch.int16, device=device)   # written before read
        return GoStore(hist, bloom, lab, cap)

    def launch_init(self, v: DeviceV, ks: int, sk) -> None:
        v.store = self.new_store(v.n, v.limit, v.device)
        v.store.lineage = Lineage(v.uid).track(v)
        cols, st, store = self.out_cols(v), self.state_struct(v), v.store.struct()
        nat.check(nat.lib().bbk_go_init(self.size, cols, st, store, v.n, v.slot0, ks, nat.ptr(sk), v.limit,
                                        nat.stream_handle(v.device)), "bbk_go_init")

    branch_keep = 2   # a live slot's history prefix survives two batch steps (see history_of)

    def private_store_ready(self, w: DeviceV) -> None:
        self.rebuild_filters(w)

    def rebuild_filters(self, w: DeviceV) -> None:
        """Recompute w's store from w's own state after a branch copied a store that later steps may
        have changed: the Bloom / count-pair filters from its history prefixes (bbk_go_rebuild_bloom)
        and the chain labels from its board (bbk_go_relabel)."""
        st, stream = w.store.struct(), nat.stream_handle(w.device)
        nat.check(nat.lib().bbk_go_rebuild_bloom(self.size, st, nat.ptr(w.priv.hist_len), w.n, stream),
                  "bbk_go_rebuild_bloom")
        nat.check(nat.lib().bbk_go_relabel(self.size, st, nat.ptr(w.priv.pat), w.n, stream), "bbk_go_relabel")

    def prepare_step(self, v: DeviceV, out: DeviceV) -> None:
        store = v.store
        if out.limit + 2 > store.hist_cap:
            raise ValueError("max_steps exceeds the history capacity of this batch")
        depth = self.branch_depth(v)
        if depth > 0:
            # branch: private copy of the history, filters rebuilt for v's lengths; the
            # original lineage keeps its store (and stays steppable)
            old = store.lineage
            store = store.clone_rows()
            store.lineage = Lineage(v.uid, v.t, old.append_only)
            self.rebuild_filters(_with_store(v, store))
        out.store = store
        self.advance_lineage(store.lineage, v, out)

    def launch_step(self, v, out, a, ks, sk, limit) -> None:
        nat.check(nat.lib().bbk_go_step(self.size, self.komi, int(self.allow_self_capture), self.cols(v), self.state_struct(v), self.out_cols(out),
                                        self.state_struct(out), out.store.struct(), nat.ptr(a), v.n, v.slot0, ks,
                                        nat.ptr(sk), limit, nat.stream_handle(v.device)), "bbk_go_step")

    fp_code = 0

    def launch_fingerprint(self, v, scratch, stride, lens, out) -> None:
        nat.check(nat.lib().bbk_go_fingerprint(self.size, self.cols(v), self.state_struct(v), v.n, nat.ptr(scratch),
                                               stride, nat.ptr(lens), nat.ptr(out), nat.stream_handle(v.device)),
                  "bbk_go_fingerprint")

    def launch_observe(self, v, i, roles, out) -> None:
        nat.check(nat.lib().bbk_go_observe(self.size, nat.ptr(v.priv.pat[i:i + 1]), nat.ptr(roles), nat.ptr(out), 1,
                                           nat.stream_handle(v.device)), "bbk_go_observe")

    def observe_at(self, gdef, v, i, role):
        if v.dev.observation is not None and int(role) == int(self.host_snapshot(v)["role_to_move"][i]):
            return v.observation[i].copy()
        return super().observe_at(gdef, v, i, role)

    def slice_store(self, v: DeviceV, w: DeviceV, i: int) -> None:
        depth = self.branch_depth(v)
        s = v.store
        w.store = s.clone_rows(slice(i, i + 1))
        w.store.lineage = Lineage(w.uid, w.t).track(w)
        if depth > 0:
            self.rebuild_filters(w)

    def history_of(self, v: DeviceV, i: int, hist_len: int) -> frozenset:
        """Slot i's superko set: entries [0, hist_len) of v's history store. A live slot's prefix
        survives in the shared store while the batch is at most two steps behind the lineage head (a
        reset rewrites entry 0 with the same value 0, the next placement entry 1); a held batch
        that falls further behind gets a store of its own first (DeviceKernel.release)."""
        self.branch_depth(v)   # raises StaleBatch when the store may no longer hold v's prefix
        row = v.store.history[i, :hist_len].cpu().numpy().view(np.uint64)
        return frozenset(int(x) for x in row)

    def state_at(self, gdef, v, i, limit):
        st = super().state_at(gdef, v, i, limit)
        st.core._src = (v, i)
        return st

    def core_view(self, s, i, p2r, rewards, mask, terminal):
        pat = s["pat"][i].view(np.uint16)[: self.cells].astype(np.uint32)
        step = int(s["step_count"][i])
        nbh = min(step + 1, HISTORY_PLANES)
        boards = []
        for t in range(nbh):
            b = ((pat >> (2 * t)) & 1) + 2 * ((pat >> (2 * t + 1)) & 1)
            boards.append(b.astype(np.uint8).tobytes())
        bits = 0 if (terminal or s["truncated"][i]) else int.from_bytes(
            np.packbits(mask, bitorder="little").tobytes(), "little")
        return GoCoreView(
            board=boards[0],
            role_to_move=int(s["role_to_move"][i]),
            terminal=terminal,
            rewards=self.role_rewards(p2r, rewards),
            mask=bits,
            pass_count=int(s["pass_count"][i]),
            hash_=int(s["hash"][i]) & ((1 << 64) - 1),
            hist_xor=int(s["hist_xor"][i]) & ((1 << 64) - 1),
            hist_len=int(s["hist_len"][i]),
            boards_hist=tuple(boards),
        )


def make_game(size: int = 9, komi: float = 6.5, allow_self_capture: bool = False) -> GameDef:
    """Device twin of reference go.make_game (go.py:114-290)."""
    cells = size * size
    return GameDef(
        spec=GameSpec(f"go_{size}x{size}", 2, (size, size, 2 * HISTORY_PLANES + 1), cells + 1),
        max_steps=512,
        batch_kernel=GoKernel(size, komi, allow_self_capture),
    )


GAME = make_game(9)
GAME19 = make_game(19)
