"""Shogi on the device (reserved id ``shogi`` in the reference, games/__init__.py:31).

There is no reference engine: rules, observation (dlshogi-style 119 planes)
and action encoding (81 destinations x 27 directions incl. 7 drops) follow
PAPER.md:1278-1354 with the conventions in DESIGN.md §3.4. CPU twin:
oracle/orc_shogi.c (perft-pinned); parity against the reference is
"unpinned" for shogi.

Device state per slot: board[96] absolute piece codes, misc[16] (hands,
side to move, repetition count) and a per-lineage in-place log of 64-bit
position keys by ply (four-fold repetition).
"""

from __future__ import annotations

from .. import _native as nat
from ..core import GameDef, GameSpec
from ._device import DeviceV, Lineage, _torch
from .chess import RingKernel, RingStore  # noqa: F401


_SFEN_TYPES = {"p": 1, "l": 2, "n": 3, "s": 4, "g": 5, "b": 6, "r": 7, "k": 8}
_PROMOTE = {1: 9, 2: 10, 3: 11, 4: 12, 6: 13, 7: 14}
_HAND = "plnsgbr"


def parse_sfen(sfen: str) -> tuple[bytes, bytes]:
    """SFEN -> (board[96] absolute codes owner << 4 | FU1 KY2 KE3 GI4 KI5 KA6 HI7 OU8 TO9 NY10 NK11
    NG12 UM13 RY14, square r*9+c with r = 0 the top rank and c = 0 file 9; misc[16] = hands [2][7]
    (FU KY KE GI KI KA HI), side to move (1 = White / gote), 0).

    The layout bbk_shogi_load takes (same reading as orc_shogi_set_sfen)."""
    parts = sfen.split()
    board = bytearray(96)
    r = c = 0
    prom = False
    for ch in parts[0]:
        if ch == "/":
            r, c = r + 1, 0
        elif ch.isdigit():
            c += int(ch)
        elif ch == "+":
            prom = True
        else:
            t = _SFEN_TYPES.get(ch.lower())
            if t is None or r > 8 or c > 8 or (prom and t not in _PROMOTE):
                raise ValueError(f"bad SFEN placement: {parts[0]!r}")
            board[r * 9 + c] = (16 if ch.islower() else 0) | (_PROMOTE[t] if prom else t)
            c, prom = c + 1, False
    misc = bytearray(16)
    misc[14] = 1 if len(parts) > 1 and parts[1] == "w" else 0
    cnt = 0
    for ch in parts[2] if len(parts) > 2 else "-":
        if ch == "-":
            break
        if ch.isdigit():
            cnt = cnt * 10 + int(ch)
            continue
        if ch.lower() not in _HAND:
            raise ValueError(f"bad SFEN hand: {parts[2]!r}")
        misc[(7 if ch.islower() else 0) + _HAND.index(ch.lower())] += cnt or 1
        cnt = 0
    return bytes(board), bytes(misc)


class ShogiCoreView:
    __slots__ = ("board", "hands", "role_to_move", "rep", "terminal", "rewards", "mask")

    def __init__(self, board, hands, role_to_move, rep, terminal, rewards, mask):
        self.board = board
        self.hands = hands
        self.role_to_move = role_to_move
        self.rep = rep
        self.terminal = terminal
        self.rewards = rewards
        self.mask = mask

    def encode(self) -> bytes:
        """board[81] + hands[2][7] + side to move + repetition count (oracle orc_shogi_encode)."""
        return self.board + self.hands + bytes([self.role_to_move, self.rep])


class ShogiKernel(RingKernel):
    game_id = "shogi"
    prefix = "shogi"
    fp_code = 3
    num_actions = 2187
    obs_shape = (9, 9, 119)
    board_bytes = 96
    misc_bytes = 16

    def state_struct(self, v: DeviceV, i: int | None = None):
        h = v.store.hist
        if i is None:
            return nat.ShogiState(nat.ptr(v.priv.board), nat.ptr(v.priv.misc), nat.ptr(h), h.shape[1])
        return nat.ShogiState(nat.ptr(v.priv.board[i:i + 1]), nat.ptr(v.priv.misc[i:i + 1]), nat.ptr(h[i:i + 1]),
                              h.shape[1])

    def parse_position(self, text):
        return parse_sfen(text)

    def alloc_store(self, v):
        torch = _torch()
        # per env: position keys by ply (max_steps + 2) then a 2048-bit repetition Bloom filter (32 x u64)
        return RingStore(torch.empty((v.n, int(v.limit) + 2 + 32), dtype=torch.int64, device=v.device))

    def launch_init(self, v, ks, sk):
        v.store = self.alloc_store(v)
        v.store.lineage = Lineage(v.uid).track(v)
        nat.check(nat.lib().bbk_shogi_init(self.out_cols(v), self.state_struct(v), v.n, v.slot0, ks, nat.ptr(sk), v.limit,
                                           nat.stream_handle(v.device)), "bbk_shogi_init")

    def prepare_step(self, v, out):
        if out.limit + 2 + 32 > v.store.hist.shape[1]:
            raise ValueError("max_steps exceeds the position-log capacity of this batch")
        super().prepare_step(v, out)

    def observe_at(self, gdef, v, i, role):
        s = self.host_snapshot(v)
        if v.dev.observation is not None and int(role) == int(s["misc"][i][14]):
            return v.observation[i].copy()
        return super(RingKernel, self).observe_at(gdef, v, i, role)

    def core_view(self, s, i, p2r, rewards, mask, terminal):
        import numpy as np

        m = s["misc"][i]
        bits = 0 if (terminal or s["truncated"][i]) else int.from_bytes(
            np.packbits(mask, bitorder="little").tobytes(), "little")
        return ShogiCoreView(bytes(s["board"][i][:81]), bytes(m[:14]), int(m[14]), int(m[15]), terminal,
                             self.role_rewards(p2r, rewards), bits)


GAME = GameDef(
    spec=GameSpec("shogi", 2, (9, 9, 119), 2187),
    max_steps=256,
    batch_kernel=ShogiKernel(),
)
