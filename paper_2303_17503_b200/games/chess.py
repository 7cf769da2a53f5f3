"""Chess on the device (reserved id ``chess`` in the reference, games/__init__.py:23).

There is no reference engine: rules, observation and action encodings follow
PAPER.md:781-856 (AlphaZero 8x8x119 observation, 64x73 actions, +1/-1/0)
with the conventions recorded in DESIGN.md §3.3. The CPU twin is
oracle/orc_chess.c (perft-pinned); parity against the reference is
"unpinned" for chess.

Device state per slot: board[64] piece codes, misc[8] (stm, castling, ep,
half-move clock, repetition), and a per-lineage in-place ring of the last
128 plies (packed boards + meta) for the repetition rule and the 8-step
observation history.
"""

from __future__ import annotations

import numpy as np

from .. import _native as nat
from ..core import GameDef, GameSpec, StaleBatch
from ..rng import key_state
from ._device import DeviceKernel, DeviceV, Lineage, _torch

HIST_BYTES = 128 * 32 + 128 * 4

_FEN_TYPES = {"p": 1, "n": 2, "b": 3, "r": 4, "q": 5, "k": 6}


def parse_fen(fen: str) -> tuple[bytes, bytes]:
    """FEN -> (board[64] piece codes colour << 3 | P1 N2 B3 R4 Q5 K6, a1 = 0; misc[8] = side to move,
    castling bits (1 K, 2 Q, 4 k, 8 q), en-passant square (int8, -1 none), half-move clock).

    The layout bbk_chess_load takes (DESIGN.md §3.3 conventions; same reading as the oracle's
    test hook orc_chess_set_fen). Raises ValueError on a malformed placement field."""
    parts = fen.split()
    board = bytearray(64)
    r, f = 7, 0
    for ch in parts[0]:
        if ch == "/":
            r, f = r - 1, 0
        elif ch.isdigit():
            f += int(ch)
        else:
            t = _FEN_TYPES.get(ch.lower())
            if t is None or not (0 <= r < 8 and 0 <= f < 8):
                raise ValueError(f"bad FEN placement: {parts[0]!r}")
            board[r * 8 + f] = (8 if ch.islower() else 0) | t
            f += 1
    stm = 1 if len(parts) > 1 and parts[1] == "b" else 0
    castle = 0
    for ch in parts[2] if len(parts) > 2 else "":
        castle |= {"K": 1, "Q": 2, "k": 4, "q": 8}.get(ch, 0)
    ep = -1
    if len(parts) > 3 and parts[3] != "-":
        ep = (int(parts[3][1]) - 1) * 8 + (ord(parts[3][0]) - ord("a"))
    half = int(parts[4]) if len(parts) > 4 else 0
    return bytes(board), bytes([stm, castle, ep & 0xFF, min(half, 255), 0, 0, 0, 0])


class RingStore:
    """In-place per-env history ring shared along a trajectory."""

    def __init__(self, hist):
        self.hist = hist
        self.lineage = None

    def row_tensors(self):
        return [self.hist]

    def like(self, n: int) -> "RingStore":
        torch = _torch()
        return RingStore(torch.empty((n,) + tuple(self.hist.shape[1:]), dtype=self.hist.dtype,
                                     device=self.hist.device))

    def clone_rows(self, rows=slice(None)) -> "RingStore":
        return RingStore(self.hist[rows].clone())


class ChessCoreView:
    __slots__ = ("board", "role_to_move", "castling", "ep", "halfmove", "rep", "terminal", "rewards", "mask")

    def __init__(self, board, role_to_move, castling, ep, halfmove, rep, terminal, rewards, mask):
        self.board = board
        self.role_to_move = role_to_move
        self.castling = castling
        self.ep = ep
        self.halfmove = halfmove
        self.rep = rep
        self.terminal = terminal
        self.rewards = rewards
        self.mask = mask

    def encode(self) -> bytes:
        """board[64] + stm + castling + ep + half-move clock + repetition (oracle orc_chess_encode)."""
        return self.board + bytes([self.role_to_move, self.castling, self.ep & 0xFF, self.halfmove, self.rep])


class RingKernel(DeviceKernel):
    """Shared logic of games with a per-env in-place history ring (chess, shogi)."""

    prefix = ""
    hist_bytes = 0
    board_bytes = 0
    misc_bytes = 8

    def alloc_private(self, v: DeviceV) -> None:
        torch = _torch()
        v.priv.board = torch.empty((v.n, self.board_bytes), dtype=torch.uint8, device=v.device)
        v.priv.misc = torch.empty((v.n, self.misc_bytes), dtype=torch.uint8, device=v.device)

    def state_struct(self, v: DeviceV, i: int | None = None):
        S = nat.ChessState if self.prefix == "chess" else nat.ShogiState
        if i is None:
            return S(nat.ptr(v.priv.board), nat.ptr(v.priv.misc), nat.ptr(v.store.hist))
        return S(nat.ptr(v.priv.board[i:i + 1]), nat.ptr(v.priv.misc[i:i + 1]), nat.ptr(v.store.hist[i:i + 1]))

    def launch_init(self, v, ks, sk):
        v.store = self.alloc_store(v)
        v.store.lineage = Lineage(v.uid).track(v)
        fn = getattr(nat.lib(), f"bbk_{self.prefix}_init")
        nat.check(fn(self.out_cols(v), self.state_struct(v), v.n, v.slot0, ks, nat.ptr(sk), v.limit,
                     nat.stream_handle(v.device)), f"bbk_{self.prefix}_init")

    def parse_position(self, text: str) -> tuple[bytes, bytes]:
        raise NotImplementedError

    def alloc_store(self, v):
        torch = _torch()
        return RingStore(torch.empty((v.n, self.hist_bytes), dtype=torch.uint8, device=v.device))

    def load(self, gdef, positions, key=None, limit: int | None = None, slot0: int = 0, device=None,
             obs: bool = True) -> DeviceV:
        """A batch whose slot i starts from positions[i] (FEN / SFEN text or a (board, misc) byte pair):
        step_count 0, empty history, player_to_role from the slot key as in init (bbk_<game>_load).

        There is no reference counterpart (the reference has no chess / shogi engine); this is the
        device twin of the oracle's set_fen / set_sfen test hooks and what the device perft and
        rule-position tests drive."""
        torch = _torch()
        pairs = [self.parse_position(p) if isinstance(p, str) else p for p in positions]
        if not pairs:
            from ..core import EmptyBatch

            raise EmptyBatch("no positions")
        limit = gdef.max_steps if limit is None else int(limit)
        device = self._device(device)
        n = len(pairs)
        boards = torch.tensor(np.frombuffer(b"".join(b for b, _ in pairs), dtype=np.uint8).reshape(n, -1)).to(device)
        misc = torch.tensor(np.frombuffer(b"".join(m for _, m in pairs), dtype=np.uint8).reshape(n, -1)).to(device)
        if boards.shape[1] != self.board_bytes or misc.shape[1] != self.misc_bytes:
            raise ValueError(f"{self.game_id}: positions must be {self.board_bytes} + {self.misc_bytes} bytes")
        v = self.new_v(n, slot0, device, 0, limit, obs)
        v.store = self.alloc_store(v)
        v.store.lineage = Lineage(v.uid).track(v)
        fn = getattr(nat.lib(), f"bbk_{self.prefix}_load")
        nat.check(fn(self.cols(v), self.state_struct(v), nat.ptr(boards), nat.ptr(misc), n, slot0,
                     0 if key is None else key_state(key), None, limit, nat.stream_handle(device)),
                  f"bbk_{self.prefix}_load")
        return v

    branch_keep = 1   # after a batch step only the newest batch's predecessor is branchable

    def prepare_step(self, v, out):
        depth = self.branch_depth(v)
        store = v.store
        if depth > 0:   # branch: private copy, the original trajectory stays steppable
            old = store.lineage
            store = RingStore(store.hist.clone())
            store.lineage = Lineage(v.uid, v.t, old.append_only)
        out.store = store
        self.advance_lineage(store.lineage, v, out)

    def launch_step(self, v, out, a, ks, sk, limit):
        fn = getattr(nat.lib(), f"bbk_{self.prefix}_step")
        nat.check(fn(self.cols(v), self.state_struct(v), self.out_cols(out), self.state_struct(out), nat.ptr(a), v.n,
                     v.slot0, ks, nat.ptr(sk), limit, nat.stream_handle(v.device)), f"bbk_{self.prefix}_step")

    def launch_fingerprint(self, v, scratch, stride, lens, out) -> None:
        fn = getattr(nat.lib(), f"bbk_{self.prefix}_fingerprint")
        nat.check(fn(self.cols(v), self.state_struct(v), v.n, nat.ptr(scratch), stride, nat.ptr(lens), nat.ptr(out),
                     nat.stream_handle(v.device)), f"bbk_{self.prefix}_fingerprint")

    def launch_observe(self, v, i, roles, out):
        fn = getattr(nat.lib(), f"bbk_{self.prefix}_observe")
        nat.check(fn(self.state_struct(v, i), nat.ptr(v.dev.step_count[i:i + 1]), nat.ptr(roles), nat.ptr(out), 1,
                     nat.stream_handle(v.device)), f"bbk_{self.prefix}_observe")

    def observe_at(self, gdef, v, i, role):
        s = self.host_snapshot(v)
        if v.dev.observation is not None and int(role) == int(s["misc"][i][0]):
            return v.observation[i].copy()
        return super().observe_at(gdef, v, i, role)

    def private_host(self, v):
        return {"board": v.priv.board.cpu().numpy(), "misc": v.priv.misc.cpu().numpy()}

    def slice_store(self, v, w, i):
        self.branch_depth(v)   # StaleBatch if stepping v's descendants overwrote its history
        w.store = RingStore(v.store.hist[i:i + 1].clone())
        w.store.lineage = Lineage(w.uid, w.t).track(w)


class ChessKernel(RingKernel):
    game_id = "chess"
    prefix = "chess"
    fp_code = 2
    num_actions = 4672
    obs_shape = (8, 8, 119)
    hist_bytes = HIST_BYTES
    board_bytes = 64

    def parse_position(self, text):
        return parse_fen(text)

    # A trail entry t of an append-only (scalar) lineage reads plies [t + 1 - M, t] of the ring,
    # M <= 101 (a live state's half-move clock is below 100), so it is intact while the head is
    # fewer than 128 - 101 + 1 = 28 plies ahead; older entries still held get their own ring
    # first (DeviceKernel.advance_lineage / release), with two plies of margin.
    window = 25

    def check_branch(self, v, lin):
        """The 128-ply ring is reused modulo 128: stepping v reads plies [t + 1 - M, t] (M = the
        half-move window, at least the 7 observation plies), which later plies of the lineage
        overwrite once the head is 128 plies past the window's start."""
        from ..core import StaleBatch

        hm = int(v.priv.misc[:, 3].max().item())
        M = max(hm + 1, 7)
        if lin.head_t - (v.t + 1 - M) >= 128:
            raise StaleBatch("chess: the repetition ring no longer holds this batch's history (more than 128 "
                             "plies behind)")

    def core_view(self, s, i, p2r, rewards, mask, terminal):
        m = s["misc"][i]
        bits = 0 if (terminal or s["truncated"][i]) else int.from_bytes(
            np.packbits(mask, bitorder="little").tobytes(), "little")
        return ChessCoreView(bytes(s["board"][i]), int(m[0]), int(m[1]), (int(m[2]) ^ 0x80) - 0x80, int(m[3]),
                             int(m[4]), terminal, self.role_rewards(p2r, rewards), bits)


GAME = GameDef(
    spec=GameSpec("chess", 2, (8, 8, 119), 4672),
    max_steps=256,
    batch_kernel=ChessKernel(),
)
