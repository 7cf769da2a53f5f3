"""Device implementation of the reference's ``batch_kernel`` plugin protocol.

The reference (core.py:88, 346-348, 366-368, 276-282; template
games/tictactoe.py:71-198) expects an object with ``init(gdef, key, n,
limit) -> V``, ``step(gdef, v, acts, key, limit) -> V`` and
``state_at(gdef, v, i, limit) -> EnvState``, where ``V`` exposes numpy
columns ``current_player, legal_action_mask, rewards, terminated,
truncated, step_count, player_to_role``. Here ``V`` (``DeviceV``) owns CUDA
tensors; the numpy columns are lazy host copies, and ``v.dev`` exposes the
tensors themselves. Each game subclass only declares its private state and
the C-ABI calls.
"""

from __future__ import annotations

import ctypes as C
import sys
import threading
import weakref
from types import SimpleNamespace

import numpy as np

from .. import _native as nat
from ..core import EnvState, IllegalAction, ShapeMismatch
from ..rng import key_state

INT32_MAX = 2**31 - 1


def _torch():
    import torch

    return torch


_UID = [0]
_UID_LOCK = threading.Lock()
_POOLS_LOCK = threading.RLock()   # re-entrant: a finalizer (_recycle) may run inside a locked region (GC)
# per-thread fused outputs of the launch being built (the kernel objects are shared per game)
_TLS = threading.local()


def _next_uid() -> int:
    with _UID_LOCK:
        _UID[0] += 1
        return _UID[0]


class Lineage:
    """Which batches of a trajectory may still be stepped.

    Games with an in-place per-env history (Go superko store, chess/shogi
    repetition rings) share it along a trajectory. ``head`` is the newest
    batch, ``trail`` its predecessors (newest first), ``head_t`` the head's
    step index. Stepping the head is the fast path; stepping a predecessor is a
    branch: the game copies the store first, so the original trajectory stays
    steppable (reference states are pure values, core.py:1-7).

    ``append_only``: no step of this lineage could have auto-reset a slot (only
    scalar ``core.step`` calls, which refuse finished states, advanced it). Every
    predecessor's history prefix is then still intact, so any of them can be
    branched (the trail is kept in full). Once a batch step runs, resets may have
    rewritten a slot's history, and only the last ``keep`` predecessors stay
    branchable in the shared store (the games' depth limits).

    A batch that falls off the trail while the caller still holds it is not lost:
    ``mark_batch_step`` / ``advance`` / ``drop`` return the uids they removed, and
    the kernel gives each batch still alive (``track`` keeps weak references) a
    private copy of the store BEFORE the next launch can overwrite its history
    (DeviceKernel.release). Every state therefore stays steppable at any depth, as
    reference states are (core.py:1-7); the copy is paid only by batches that are
    held, never by a loop that drops its predecessors. StaleBatch remains only for a
    uid the lineage never saw.
    """

    def __init__(self, uid: int, t: int = 0, append_only: bool = True):
        self.head = uid
        self.head_t = t
        self.trail: list[int] = []
        self.append_only = append_only
        self.refs: dict[int, weakref.ref] = {}

    def track(self, v) -> "Lineage":
        """Remember batch v weakly (see release)."""
        self.refs[v.uid] = weakref.ref(v)
        return self

    def depth(self, uid: int) -> int:
        if uid == self.head:
            return 0
        try:
            return self.trail.index(uid) + 1
        except ValueError:
            return 1 << 30

    def _removed(self, before: list[int]) -> list[int]:
        now = set(self.trail)
        now.add(self.head)
        return [u for u in before if u not in now]

    def mark_batch_step(self, keep: int = 2) -> list[int]:
        if not self.append_only:
            return []
        before = list(self.trail)
        self.append_only = False
        self.trail = self.trail[:keep]
        return self._removed(before)

    def advance(self, parent: int, child: int, keep: int = 2, child_t: int | None = None) -> list[int]:
        before = [self.head] + self.trail
        lim = None if self.append_only else keep
        if parent == self.head:
            self.trail = ([parent] + self.trail)[:lim]
        else:   # branch in place: the old head (and anything newer than parent) is dropped
            i = self.trail.index(parent)
            self.trail = self.trail[i:] if lim is None else self.trail[i:i + lim]
        self.head = child
        if child_t is not None:
            self.head_t = child_t
        return self._removed(before)

    def drop(self, uids) -> list[int]:
        """Take uids off the trail (a game whose store wraps, chess.RingKernel.window)."""
        gone = set(uids)
        before = list(self.trail)
        self.trail = [u for u in self.trail if u not in gone]
        return self._removed(before)


class DeviceV:
    """Struct-of-arrays device state of one batch (reference V, tictactoe.py:74-79)."""

    _COLS = ("current_player", "legal_action_mask", "rewards", "terminated", "truncated", "step_count",
             "player_to_role", "observation")

    def __init__(self, kern, n: int, slot0: int, device, t: int, limit: int):
        self.kern = kern
        self.n = n
        self.slot0 = slot0
        self.device = device
        self.t = t              # batch steps since batch_init along this lineage
        self.limit = limit
        self.dev = SimpleNamespace()
        self.priv = SimpleNamespace()
        self.store = None
        self.uid = _next_uid()
        self._host = {}
        self.next_actions = None     # fused agents.random_actions output of the producing call
        self.next_key = None

    # lazily materialised host columns (the reference reads them via getattr)
    def _h(self, name):
        arr = self._host.get(name)
        if arr is None:
            t = getattr(self.dev, name)
            arr = t.cpu().numpy()
            arr.flags.writeable = False
            self._host[name] = arr
        return arr

    current_player = property(lambda self: self._h("current_player"))
    legal_action_mask = property(lambda self: self._h("legal_action_mask"))
    rewards = property(lambda self: self._h("rewards"))
    terminated = property(lambda self: self._h("terminated"))
    truncated = property(lambda self: self._h("truncated"))
    step_count = property(lambda self: self._h("step_count"))
    player_to_role = property(lambda self: self._h("player_to_role"))
    observation = property(lambda self: self._h("observation"))

    def priv_host(self, name):
        key = "priv." + name
        arr = self._host.get(key)
        if arr is None:
            arr = getattr(self.priv, name).cpu().numpy()
            self._host[key] = arr
        return arr


# BBK_ZERO_COPY=0: copy pinned host action buffers to the device instead of reading them in place
ZERO_COPY = __import__("os").environ.get("BBK_ZERO_COPY", "1") != "0"
POOL_DEPTH = 2        # dead batches' buffer sets kept per (n, device, obs, stream)
_CACHED = ("_cols", "_gostate")   # ctypes structs of fixed column pointers, valid with the buffers


def _recycle(pool: list, vd: dict) -> None:
    """Finalizer of a DeviceV: return its column and private buffers to the pool when nothing else
    references them (no Python alias, view, DLPack export or numpy view of any tensor).

    A recycled buffer set is handed to the next new_v on the same stream, so stream order makes
    the reuse safe exactly as for torch's caching allocator. This removes the ~16 allocations and
    the pointer-struct rebuild from every public step call (the e2e path's host overhead).
    """
    dev, priv = vd.get("dev"), vd.get("priv")
    if dev is None or priv is None:
        return
    use_count = _torch()._C._storage_Use_Count
    for ns in (dev, priv):
        for t in vars(ns).values():
            # references: the namespace, the loop variable, getrefcount's argument
            if t is not None and (sys.getrefcount(t) != 3 or use_count(t.untyped_storage()._cdata) != 2):
                return
    with _POOLS_LOCK:
        if len(pool) < POOL_DEPTH:
            pool.append((dev, priv, {k: vd[k] for k in _CACHED if k in vd}))


class DeviceKernel:
    """Common host logic; subclasses implement the game-specific C-ABI calls."""

    game_id = ""
    num_actions = 0
    num_players = 2
    obs_shape: tuple = ()

    # ------------------------------------------------------------ allocation
    def new_v(self, n: int, slot0: int, device, t: int, limit: int, obs: bool = True) -> DeviceV:
        """A batch state of n slots: buffers recycled from a dead batch of the same shape on the same
        stream when one is pooled (see _recycle), else freshly allocated."""
        torch = _torch()
        v = DeviceV(self, n, slot0, device, t, limit)
        stream = nat.stream_handle(device) if torch.device(device).type == "cuda" else 0
        pkey = (n, device, obs, stream)
        with _POOLS_LOCK:
            pool = self.__dict__.setdefault("_pools", {}).setdefault(pkey, [])
            got = pool.pop() if pool else None
        if got is not None:
            v.dev, v.priv, cached = got
            v.__dict__.update(cached)
        else:
            self._alloc_columns(v, obs)
        weakref.finalize(v, _recycle, pool, v.__dict__).atexit = False
        return v

    def _alloc_columns(self, v: DeviceV, obs: bool) -> None:
        torch = _torch()
        n, device = v.n, v.device
        d = v.dev
        d.observation = torch.empty((n,) + tuple(self.obs_shape), dtype=torch.float32, device=device) if obs else None
        d.legal_action_mask = torch.empty((n, self.num_actions), dtype=torch.bool, device=device)
        d.rewards = torch.empty((n, self.num_players), dtype=torch.float32, device=device)
        d.terminated = torch.empty(n, dtype=torch.bool, device=device)
        d.truncated = torch.empty(n, dtype=torch.bool, device=device)
        d.current_player = torch.empty(n, dtype=torch.int32, device=device)
        d.step_count = torch.empty(n, dtype=torch.int32, device=device)
        d.player_to_role = torch.empty((n, self.num_players), dtype=torch.int8, device=device)
        self.alloc_private(v)

    def alloc_private(self, v: DeviceV) -> None:
        raise NotImplementedError

    @staticmethod
    def cols(v: DeviceV, fused: tuple | None = None) -> nat.Cols:
        """Column pointers; `fused` = (next_key_state, next_actions tensor, episodes tensor) or None.

        The column tensors of a DeviceV never change, so the struct is built once per batch and
        only the fused fields are filled in per call (host overhead of the public step path)."""
        base = v.__dict__.get("_cols")
        if base is None:
            d = v.dev
            base = nat.Cols(nat.ptr(d.observation), nat.ptr(d.legal_action_mask), nat.ptr(d.rewards),
                            nat.ptr(d.terminated), nat.ptr(d.truncated), nat.ptr(d.current_player),
                            nat.ptr(d.step_count), nat.ptr(d.player_to_role), None, 0, None)
            v._cols = base
        if fused is None:
            return base
        nk, na, ep = fused
        c = nat.Cols.from_buffer_copy(base)
        c.next_actions = nat.ptr(na)
        c.next_key = int(nk) & ((1 << 64) - 1)
        c.episodes = nat.ptr(ep)
        return c

    @staticmethod
    def _device(device):
        torch = _torch()
        if device is None:
            if not torch.cuda.is_available():
                raise nat.NativeUnavailable("no CUDA device: the engines run only on the GPU (no CPU fallback)")
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device(device)

    @staticmethod
    def _slot_keys(slot_keys, device):
        if slot_keys is None:
            return None
        torch = _torch()
        arr = np.asarray([int(k) & ((1 << 64) - 1) for k in slot_keys], dtype=np.uint64).view(np.int64)
        return torch.from_numpy(arr).to(device)

    # -------------------------------------------------------- protocol: init
    def init(self, gdef, key, n: int, limit: int, slot_keys=None, slot0: int = 0, device=None,
             obs: bool = True, next_key=None, next_actions=None, episodes=None) -> DeviceV:
        device = self._device(device)
        v = self.new_v(n, slot0, device, 0, limit, obs)
        sk = self._slot_keys(slot_keys, device)
        ks = 0 if key is None else key_state(key)
        _TLS.fused = self._fused_args(v, next_key, next_actions, episodes)
        try:
            self.launch_init(v, ks, sk)
        finally:
            _TLS.fused = None
        return v

    def _fused_args(self, v, next_key, next_actions, episodes):
        """Optional fused outputs of a launch (bbk_cols.next_actions / next_key / episodes)."""
        if next_key is None and episodes is None:
            return None
        torch = _torch()
        if next_key is not None and next_actions is None:
            next_actions = torch.empty(v.n, dtype=torch.int64, device=v.device)
        elif next_actions is not None:
            ok_place = next_actions.device == v.device or (next_actions.device.type == "cpu" and next_actions.is_pinned())
            if (next_actions.dtype != torch.int64 or tuple(next_actions.shape) != (v.n,) or not ok_place
                    or not next_actions.is_contiguous()):
                raise ShapeMismatch(f"next_actions must be a contiguous int64 [{v.n}] tensor on {v.device} "
                                    "or in pinned host memory")
        if next_key is not None:
            v.next_actions = next_actions
            v.next_key = key_state(next_key)
        return (0 if next_key is None else key_state(next_key), next_actions if next_key is not None else None,
                episodes)

    def out_cols(self, v: DeviceV) -> nat.Cols:
        return self.cols(v, getattr(_TLS, "fused", None))

    # -------------------------------------------------------- protocol: step
    def as_actions(self, actions, v: DeviceV):
        torch = _torch()
        if isinstance(actions, torch.Tensor):
            a = actions
            if a.device != v.device or a.dtype != torch.int64:
                pinned = a.device.type == "cpu" and a.dtype == torch.int64 and a.is_pinned()
                if pinned and ZERO_COPY and a.dim() == 1 and a.is_contiguous():
                    # zero-copy: page-locked host memory is device-addressable (UVA), so the step
                    # kernel reads each slot's action over PCIe itself, prefetched with the slot's
                    # state; the caller must not rewrite the buffer before the step's results are
                    # read, as with any CUDA async copy
                    if a.shape[0] != v.n:
                        raise ShapeMismatch(f"expected {v.n} actions, got shape {tuple(a.shape)}")
                    return a
                # otherwise a pinned buffer is copied asynchronously on the launch stream
                a = a.to(device=v.device, dtype=torch.int64, non_blocking=pinned)
        else:
            arr = np.ascontiguousarray(np.asarray(actions, dtype=np.int64))
            a = torch.from_numpy(arr).to(v.device)
        if a.dim() != 1 or a.shape[0] != v.n:
            raise ShapeMismatch(f"expected {v.n} actions, got shape {tuple(a.shape)}")
        return a.contiguous()

    def validate(self, v: DeviceV, a) -> None:
        """IllegalAction with the lowest offending live slot (tictactoe.py:111-121)."""
        torch = _torch()
        bkey = (v.device, nat.stream_handle(v.device))
        with _POOLS_LOCK:   # one result word per (device, stream); bbk_check_actions stores it (no fill launch)
            bad = self.__dict__.setdefault("_bad", {}).get(bkey)
            if bad is None:
                bad = self._bad[bkey] = torch.empty(1, dtype=torch.int32, device=v.device)
        d = v.dev
        nat.check(nat.lib().bbk_check_actions(nat.ptr(d.legal_action_mask), nat.ptr(d.terminated),
                                              nat.ptr(d.truncated), nat.ptr(a), v.n, self.num_actions,
                                              nat.ptr(bad), nat.stream_handle(v.device)), "bbk_check_actions")
        slot = int(bad.item())
        if slot != INT32_MAX:
            act = int(a[slot].item())
            raise IllegalAction(f"slot {slot}: illegal action {act} in {self.game_id}", action=act, slot=slot)

    def step(self, gdef, v: DeviceV, actions, key, limit: int, validate: bool = True, slot_keys=None,
             out: DeviceV | None = None, next_key=None, next_actions=None, episodes=None,
             scalar: bool = False) -> DeviceV:
        """``scalar``: the caller guarantees no slot of v is finished (core.step), so no slot
        resets and the trajectory's history store stays append-only (see Lineage)."""
        a = self.as_actions(actions, v)
        if validate:
            self.validate(v, a)
        if v.store is not None and not scalar:
            lin = v.store.lineage
            self.release(lin, lin.mark_batch_step(self.branch_keep))
        sk = self._slot_keys(slot_keys, v.device)
        ks = 0 if key is None else key_state(key)
        if out is None:
            out = self.new_v(v.n, v.slot0, v.device, v.t + 1, limit, v.dev.observation is not None)
        else:
            out.t = v.t + 1
            out.limit = limit
            out.uid = _next_uid()
            out._host = {}
            out.next_actions = None
            out.next_key = None
        self.prepare_step(v, out)
        _TLS.fused = self._fused_args(out, next_key, next_actions, episodes)
        try:
            self.launch_step(v, out, a, ks, sk, limit)
        finally:
            _TLS.fused = None
        return out

    def prepare_step(self, v: DeviceV, out: DeviceV) -> None:
        """Hook for games with shared in-place stores (Go, chess, shogi)."""
        out.store = v.store

    # ------------------------------------------------ branching (shared per-env stores)
    branch_keep = 2   # predecessors a batch-stepped lineage keeps branchable in the shared store
    window = None     # steps a trail entry of an append-only lineage stays intact (None: unbounded)
    snapshots = 0     # batches given a private store by release (a count for the tests)

    def advance_lineage(self, lin: Lineage, v: DeviceV, out: DeviceV) -> None:
        """out (stepped from v) becomes lin's head; live batches that fall off the trail get a
        private store before out's launch (release)."""
        gone = lin.advance(v.uid, out.uid, self.branch_keep, out.t)
        lin.track(out)
        if self.window is not None and lin.append_only:
            old = []
            for u in lin.trail:
                r = lin.refs.get(u)
                w = None if r is None else r()
                if w is None or w.uid != u or out.t - w.t > self.window:
                    old.append(u)
            if old:
                gone += lin.drop(old)
        self.release(lin, gone)

    def release(self, lin: Lineage, uids: list) -> None:
        """Batches that left lin's trail: each one still alive gets a private copy of the store
        now, while its history is intact (the trail invariant) and before the next launch can
        overwrite it, and becomes the head of its own lineage. So every state the caller holds
        stays steppable (reference value semantics, core.py:1-7) at the price of one store copy
        per held batch; a loop that drops its predecessors never pays it."""
        for u in uids:
            r = lin.refs.pop(u, None)
            w = None if r is None else r()
            if w is None or w.uid != u or w.store is None or w.store.lineage is not lin:
                continue
            store = w.store.clone_rows()
            store.lineage = Lineage(w.uid, w.t).track(w)
            w.store = store
            self.private_store_ready(w)
            self.snapshots += 1

    def private_store_ready(self, w: DeviceV) -> None:
        """Game hook: make a copied store consistent with w (Go: filters and chain labels)."""

    def branch_depth(self, v: DeviceV) -> int:
        """How far v is behind the head of its store's lineage (0 = head). StaleBatch only for a
        batch its lineage cannot account for (release keeps every live batch on a trail or in a
        store of its own)."""
        from ..core import StaleBatch

        if v.store is None or v.store.lineage is None:
            return 0
        lin = v.store.lineage
        d = lin.depth(v.uid)
        if d == 0:
            return 0
        if d >= (1 << 30) or (d > self.branch_keep and not lin.append_only):
            raise StaleBatch(f"{self.game_id}: batch is not on its trajectory's trail (its history store may "
                             "have been overwritten)")
        self.check_branch(v, lin)
        return d

    def check_branch(self, v: DeviceV, lin: Lineage) -> None:
        """Game hook: extra validity conditions of a branch (chess: ring wrap)."""

    # ----------------------------------------------------- protocol: state_at
    def host_snapshot(self, v: DeviceV) -> dict:
        snap = v._host.get("__snap")
        if snap is None:
            snap = {c: getattr(v, c) for c in DeviceV._COLS if c != "observation"}
            snap.update(self.private_host(v))
            v._host["__snap"] = snap
        return snap

    def private_host(self, v: DeviceV) -> dict:
        return {k: t.cpu().numpy() for k, t in vars(v.priv).items()}

    # -------------------------------------------------- device fingerprints
    fp_code = -1   # bbk_fingerprint_stride game code

    def fingerprints(self, v: DeviceV):
        """core.state_fingerprint of every slot, computed on the device: uint8 [n, 16] (host)."""
        torch = _torch()
        stride = int(nat.lib().bbk_fingerprint_stride(self.fp_code, int(getattr(self, "size", 0))))
        scratch = torch.empty((v.n, stride), dtype=torch.uint8, device=v.device)
        lens = torch.empty(v.n, dtype=torch.int32, device=v.device)
        out = torch.empty((v.n, 16), dtype=torch.uint8, device=v.device)
        self.launch_fingerprint(v, scratch, stride, lens, out)
        return out.cpu().numpy()

    def launch_fingerprint(self, v, scratch, stride, lens, out) -> None:
        raise NotImplementedError

    def state_at(self, gdef, v: DeviceV, i: int, limit: int) -> EnvState:
        s = self.host_snapshot(v)
        term = bool(s["terminated"][i])
        trunc = bool(s["truncated"][i])
        rewards = s["rewards"][i].copy()
        rewards.flags.writeable = False
        mask = s["legal_action_mask"][i].copy()
        mask.flags.writeable = False
        p2r = tuple(int(x) for x in s["player_to_role"][i])
        core = self.core_view(s, i, p2r, rewards, mask, term)
        return EnvState(
            current_player=int(s["current_player"][i]),
            legal_action_mask=mask,
            rewards=rewards,
            terminated=term,
            truncated=trunc,
            step_count=int(s["step_count"][i]),
            player_to_role=p2r,
            core=core,
            game=gdef,
            max_steps=limit,
            _v=v,
            _i=i,
        )

    def core_view(self, s: dict, i: int, p2r, rewards, mask, terminal):
        raise NotImplementedError

    @staticmethod
    def role_rewards(p2r, rewards) -> tuple:
        rr = [0.0] * len(p2r)
        for p in range(len(p2r)):
            rr[p2r[p]] = float(rewards[p])
        return tuple(rr)

    # ----------------------------------------------------------- observation
    def observe_at(self, gdef, v: DeviceV, i: int, role: int) -> np.ndarray:
        torch = _torch()
        roles = torch.full((1,), int(role), dtype=torch.uint8, device=v.device)
        out = torch.empty((1,) + tuple(self.obs_shape), dtype=torch.float32, device=v.device)
        self.launch_observe(v, i, roles, out)
        arr = out[0].cpu().numpy()
        return arr

    # ---------------------------------------------------------------- slicing
    def slice(self, gdef, v: DeviceV, i: int) -> DeviceV:
        """One-slot copy of slot i (scalar API on a batch state)."""
        w = self.new_v(1, v.slot0 + i, v.device, v.t, v.limit, v.dev.observation is not None)
        for name in DeviceV._COLS:
            src = getattr(v.dev, name)
            if src is not None:
                getattr(w.dev, name).copy_(src[i:i + 1])
        for name, t in vars(v.priv).items():
            getattr(w.priv, name).copy_(t[i:i + 1])
        self.slice_store(v, w, i)
        return w

    def slice_store(self, v: DeviceV, w: DeviceV, i: int) -> None:
        pass

    # ------------------------------------------------------------- sampling
    def random_actions(self, v: DeviceV, key, out=None):
        """agents.random_actions on the device (agents.py:33-46)."""
        torch = _torch()
        if out is None:
            out = torch.empty(v.n, dtype=torch.int64, device=v.device)
        nat.check(nat.lib().bbk_random_actions(nat.ptr(v.dev.legal_action_mask), v.n, self.num_actions,
                                               key_state(key), v.slot0, nat.ptr(out),
                                               nat.stream_handle(v.device)), "bbk_random_actions")
        return out

    # ---------------------------------------------- whole-row copies (search pools)
    def row_tensors(self, v: DeviceV) -> list:
        """Every per-slot tensor of a batch's state (columns except the observation, private
        state, per-env stores), leading dimension n: what a slot IS, for bbk_copy_rows."""
        d = v.dev
        out = [d.legal_action_mask, d.rewards, d.terminated, d.truncated, d.current_player, d.step_count,
               d.player_to_role]
        out += list(vars(v.priv).values())
        if v.store is not None:
            out += v.store.row_tensors()
        return out

    def new_v_like(self, v: DeviceV, n: int, store: bool = True) -> DeviceV:
        """A batch of n slots with v's state layout (no observation), with its own stores."""
        w = self.new_v(n, 0, v.device, v.t, v.limit, obs=False)
        w.store = None if (v.store is None or not store) else v.store.like(n)
        return w

    def raw_step(self, v: DeviceV, out: DeviceV, a, limit: int, slot_keys=None) -> None:
        """The step kernel on buffers the caller owns: no validation, no lineage bookkeeping;
        v and out share v's per-env store (updated in place)."""
        out.store = v.store
        out._host = {}
        _TLS.fused = None
        self.launch_step(v, out, a, 0, slot_keys, limit)

    # subclasses
    def launch_init(self, v, ks, sk):
        raise NotImplementedError

    def launch_step(self, v, out, a, ks, sk, limit):
        raise NotImplementedError

    def launch_observe(self, v, i, roles, out):
        raise NotImplementedError
