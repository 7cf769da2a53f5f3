"""ORACLE -- test infrastructure, not product code.

CPU restatement of the reference's hot path (reference
``pkg/src/boardbatch/games/go.py``, ``games/backgammon.py``, ``core.py``)
compiled from ``oracle/orc_*.c`` into ``oracle/liborc.so``. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module; the product path in
``paper_2303_17503_b200`` never does.

Parity pinning: Go and backgammon are pinned against golden fingerprints
produced by the reference itself (``tests/golden/make_golden.py``). Chess and
shogi have no reference engine: they are pinned by perft
known-answer tests and documented as "parity unpinned" against the reference.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import struct
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64


def build() -> str:
    """Compile liborc.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liborc.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liborc.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        for g in ("go", "bg", "chess", "shogi"):
            if not hasattr(L, f"orc_{g}_step"):
                continue
            getattr(L, f"orc_{g}_init").argtypes = [_P, _U64, _I64, _P]
            getattr(L, f"orc_{g}_step").argtypes = [_P, _P, _U64, _I64, _P]
            getattr(L, f"orc_{g}_step").restype = _I64
            getattr(L, f"orc_{g}_columns").argtypes = [_P] * 9
            getattr(L, f"orc_{g}_encode").argtypes = [_P, _I64, _P]
            getattr(L, f"orc_{g}_encode").restype = C.c_int
            getattr(L, f"orc_{g}_observe").argtypes = [_P, _I64, C.c_int, _P]
            getattr(L, f"orc_{g}_free").argtypes = [_P]
        L.orc_go_new.argtypes = [C.c_int, C.c_double, C.c_int, _I64, C.c_int]
        L.orc_go_new.restype = _P
        L.orc_go_set_board.argtypes = [_P, _I64, _P, C.c_int]
        L.orc_go_scalars.argtypes = [_P, _I64, _P]
        L.orc_bg_new.argtypes = [_I64, C.c_int]
        L.orc_bg_new.restype = _P
        if hasattr(L, "orc_chess_new"):
            L.orc_chess_new.argtypes = [_I64, C.c_int]
            L.orc_chess_new.restype = _P
            L.orc_chess_perft.argtypes = [C.c_char_p, C.c_int]
            L.orc_chess_perft.restype = C.c_uint64
            L.orc_chess_set_fen.argtypes = [_P, _I64, C.c_char_p]
            L.orc_chess_set_fen.restype = C.c_int
        if hasattr(L, "orc_shogi_new"):
            L.orc_shogi_new.argtypes = [_I64, C.c_int]
            L.orc_shogi_new.restype = _P
            L.orc_shogi_perft.argtypes = [C.c_char_p, C.c_int]
            L.orc_shogi_perft.restype = C.c_uint64
            L.orc_shogi_set_sfen.argtypes = [_P, _I64, C.c_char_p]
            L.orc_shogi_set_sfen.restype = C.c_int
        if hasattr(L, "omp_set_num_threads"):
            pass
        _LIB = L
    return _LIB


def set_threads(n: int) -> None:
    """OpenMP thread count for the oracle's slot loop."""
    try:
        gomp = C.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(C.c_int(int(n)))
    except OSError:
        os.environ["OMP_NUM_THREADS"] = str(int(n))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def fingerprint(game_id: str, cur: int, step: int, term: bool, trunc: bool, p2r, rewards, mask, enc: bytes) -> bytes:
    """Same digest as reference core.state_fingerprint (core.py:417-434)."""
    h = hashlib.blake2b(digest_size=16)
    h.update(game_id.encode())
    h.update(struct.pack("<iiBB", int(cur), int(step), bool(term), bool(trunc)))
    h.update(bytes(int(x) & 0xFF for x in p2r))
    h.update(np.asarray(rewards, dtype=np.float32).tobytes())
    h.update(np.packbits(np.asarray(mask, dtype=bool)).tobytes())
    h.update(enc)
    return h.digest()


class _Batch:
    """Mutable oracle batch: init/step with the reference's per-slot key rules."""

    prefix = ""
    num_actions = 0
    obs_shape: tuple = ()
    game_id = ""

    def __init__(self, handle, n: int):
        self.h = handle
        self.n = n
        self.L = lib()

    def __del__(self):
        try:
            getattr(self.L, f"orc_{self.prefix}_free")(self.h)
        except Exception:
            pass

    def init(self, key_state: int, slot0: int = 0, slot_keys=None):
        sk = None if slot_keys is None else np.ascontiguousarray(slot_keys, dtype=np.uint64)
        getattr(self.L, f"orc_{self.prefix}_init")(self.h, key_state, slot0, _ptr(sk))
        return self

    def step(self, actions, key_state: int, slot0: int = 0, slot_keys=None) -> int:
        acts = np.ascontiguousarray(actions, dtype=np.int64)
        assert acts.shape == (self.n,)
        sk = None if slot_keys is None else np.ascontiguousarray(slot_keys, dtype=np.uint64)
        return int(getattr(self.L, f"orc_{self.prefix}_step")(self.h, _ptr(acts), key_state, slot0, _ptr(sk)))

    def columns(self, with_obs: bool = True) -> dict:
        n, A = self.n, self.num_actions
        out = {
            "observation": np.empty((n,) + self.obs_shape, np.float32) if with_obs else None,
            "legal_action_mask": np.empty((n, A), np.uint8),
            "rewards": np.empty((n, 2), np.float32),
            "terminated": np.empty(n, np.uint8),
            "truncated": np.empty(n, np.uint8),
            "current_player": np.empty(n, np.int32),
            "step_count": np.empty(n, np.int32),
            "player_to_role": np.empty((n, 2), np.int8),
        }
        getattr(self.L, f"orc_{self.prefix}_columns")(
            self.h, _ptr(out["observation"]), _ptr(out["legal_action_mask"]), _ptr(out["rewards"]),
            _ptr(out["terminated"]), _ptr(out["truncated"]), _ptr(out["current_player"]),
            _ptr(out["step_count"]), _ptr(out["player_to_role"]))
        out["legal_action_mask"] = out["legal_action_mask"].view(np.bool_)
        out["terminated"] = out["terminated"].view(np.bool_)
        out["truncated"] = out["truncated"].view(np.bool_)
        if not with_obs:
            del out["observation"]
        return out

    def encode(self, i: int) -> bytes:
        buf = np.empty(1 << 16, np.uint8)
        ln = getattr(self.L, f"orc_{self.prefix}_encode")(self.h, i, _ptr(buf))
        return buf[:ln].tobytes()

    def observe(self, i: int, role: int) -> np.ndarray:
        out = np.empty(self.obs_shape, np.float32)
        getattr(self.L, f"orc_{self.prefix}_observe")(self.h, i, role, _ptr(out))
        return out

    def fingerprints(self, cols=None) -> list[bytes]:
        c = cols if cols is not None else self.columns(with_obs=False)
        return [
            fingerprint(self.game_id, c["current_player"][i], c["step_count"][i], c["terminated"][i],
                        c["truncated"][i], c["player_to_role"][i], c["rewards"][i],
                        c["legal_action_mask"][i], self.encode(i))
            for i in range(self.n)
        ]

    def batch_fingerprint(self, cols=None) -> bytes:
        h = hashlib.blake2b(digest_size=16)
        for f in self.fingerprints(cols):
            h.update(f)
        return h.digest()


class GoBatch(_Batch):
    prefix = "go"

    def __init__(self, size: int, n: int, max_steps: int = 512, komi: float = 6.5, self_capture: bool = False):
        h = lib().orc_go_new(size, komi, int(self_capture), n, max_steps)
        if not h:
            raise ValueError("bad go oracle configuration")
        super().__init__(h, n)
        self.size = size
        self.num_actions = size * size + 1
        self.obs_shape = (size, size, 17)
        self.game_id = f"go_{size}x{size}"

    def set_board(self, i: int, board, role: int):
        b = np.ascontiguousarray(board, dtype=np.uint8)
        self.L.orc_go_set_board(self.h, i, _ptr(b), role)

    def scalars(self, i: int) -> dict:
        out = np.empty(6, np.int64)
        self.L.orc_go_scalars(self.h, i, _ptr(out))
        return dict(role_to_move=int(out[0]), pass_count=int(out[1]), terminal=bool(out[2]),
                    hash=int(out[3]) & ((1 << 64) - 1), hist_xor=int(out[4]) & ((1 << 64) - 1),
                    hist_len=int(out[5]))


class BackgammonBatch(_Batch):
    prefix = "bg"
    num_actions = 156
    obs_shape = (34,)
    game_id = "backgammon"

    def __init__(self, n: int, max_steps: int = 1024):
        super().__init__(lib().orc_bg_new(n, max_steps), n)


def random_actions(mask: np.ndarray, key_state: int, slot0: int = 0) -> np.ndarray:
    """agents.random_actions (reference agents.py:33-46), numpy restatement."""
    from_mask = np.asarray(mask, dtype=bool)
    n = from_mask.shape[0]
    idx = np.arange(slot0 + 1, slot0 + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(key_state) + idx * np.uint64(0x9E3779B97F4A7C15)
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    counts = from_mask.sum(axis=1).astype(np.uint64)
    draws = x % np.maximum(counts, np.uint64(1))
    cum = np.cumsum(from_mask, axis=1, dtype=np.int64)
    actions = (cum <= draws[:, None].astype(np.int64)).sum(axis=1)
    actions[counts == 0] = 0
    return actions.astype(np.int64)


def make(game_id: str, n: int, max_steps: int | None = None, self_capture: bool = False) -> _Batch:
    if game_id.startswith("go_"):
        size = int(game_id[3:].split("x")[0])
        return GoBatch(size, n, 512 if max_steps is None else max_steps, self_capture=self_capture)
    if game_id == "backgammon":
        return BackgammonBatch(n, 1024 if max_steps is None else max_steps)
    if game_id == "chess":
        return ChessBatch(n, 256 if max_steps is None else max_steps)
    if game_id == "shogi":
        return ShogiBatch(n, 256 if max_steps is None else max_steps)
    raise KeyError(game_id)


class ChessBatch(_Batch):
    prefix = "chess"
    num_actions = 4672
    obs_shape = (8, 8, 119)
    game_id = "chess"

    def __init__(self, n: int, max_steps: int = 256):
        super().__init__(lib().orc_chess_new(n, max_steps), n)

    def set_fen(self, i: int, fen: str):
        assert self.L.orc_chess_set_fen(self.h, i, fen.encode()) == 0

    @staticmethod
    def perft(fen: str, depth: int) -> int:
        return int(lib().orc_chess_perft(fen.encode(), depth))


class ShogiBatch(_Batch):
    prefix = "shogi"
    num_actions = 2187
    obs_shape = (9, 9, 119)
    game_id = "shogi"

    def __init__(self, n: int, max_steps: int = 256):
        super().__init__(lib().orc_shogi_new(n, max_steps), n)

    def set_sfen(self, i: int, sfen: str):
        assert self.L.orc_shogi_set_sfen(self.h, i, sfen.encode()) == 0

    @staticmethod
    def perft(sfen, depth: int) -> int:
        return int(lib().orc_shogi_perft(None if sfen is None else sfen.encode(), depth))


class Session:
    """BatchSession key schedule (reference bench.py:54-83) over an oracle batch."""

    def __init__(self, game_id: str, n: int, seed: int, max_steps: int | None = None, slot0: int = 0,
                 self_capture: bool = False):
        from_seed = _mix64((seed + 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
        self.root = from_seed
        self.slot0 = slot0
        self.b = make(game_id, n, max_steps, self_capture)
        self.b.init(_child(self.root, 0), slot0)
        self.t = 0

    def sample_random_actions(self, cols=None) -> np.ndarray:
        c = cols if cols is not None else self.b.columns(with_obs=False)
        return random_actions(c["legal_action_mask"], _child(self.root, 2 * self.t + 1), self.slot0)

    def step(self, actions) -> int:
        bad = self.b.step(actions, _child(self.root, 2 * (self.t + 1)), self.slot0)
        if bad < 0:
            self.t += 1
        return bad


def _mix64(x: int) -> int:
    M = (1 << 64) - 1
    x &= M
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & M
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def _child(state: int, i: int) -> int:
    return _mix64((state + (i + 1) * 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
