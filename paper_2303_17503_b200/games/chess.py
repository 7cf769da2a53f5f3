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
from ._device import DeviceKernel, DeviceV, Lineage, _torch

HIST_BYTES = 128 * 32 + 128 * 4


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
        torch = _torch()
        v.store = RingStore(torch.empty((v.n, self.hist_bytes), dtype=torch.uint8, device=v.device))
        v.store.lineage = Lineage(v.uid)
        fn = getattr(nat.lib(), f"bbk_{self.prefix}_init")
        nat.check(fn(self.out_cols(v), self.state_struct(v), v.n, v.slot0, ks, nat.ptr(sk), v.limit,
                     nat.stream_handle(v.device)), f"bbk_{self.prefix}_init")

    def prepare_step(self, v, out):
        lin = v.store.lineage
        depth = lin.depth(v.uid)
        if depth > 1:
            raise StaleBatch(f"{self.game_id}: only the newest batch and its predecessor can be stepped "
                             "(the repetition ring is shared in place)")
        out.store = v.store
        lin.advance(v.uid, out.uid)

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
        w.store = RingStore(v.store.hist[i:i + 1].clone())
        w.store.lineage = Lineage(w.uid)


class ChessKernel(RingKernel):
    game_id = "chess"
    prefix = "chess"
    fp_code = 2
    num_actions = 4672
    obs_shape = (8, 8, 119)
    hist_bytes = HIST_BYTES
    board_bytes = 64

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
