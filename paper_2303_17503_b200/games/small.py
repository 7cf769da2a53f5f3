"""The reference's small engines on the device.

Drop-ins for reference games/tictactoe.py, connect_four.py, othello.py,
hexgame.py, play2048.py, kuhn_poker.py and leduc_holdem.py: same specs,
max_steps, chance / information flags and Core.encode bytes, with every
init / step running ``csrc/small.cu`` (one thread per slot) through the
``bbk_small_*`` entry points of include/bbk.h. Each slot's Core lives in a
48-byte blob whose layout is documented per engine in csrc/small.cuh; the
host views below decode it for ``state_at`` / ``Core.encode``.
"""

from __future__ import annotations

import numpy as np

from .. import _native as nat
from ..core import GameDef, GameSpec
from ._device import DeviceKernel, DeviceV, _torch

STATE_BYTES = 48   # BBK_SMALL_STATE_BYTES


def _le(b: bytes) -> int:
    return int.from_bytes(b, "little")


class SmallCoreView:
    """Host view of one slot's Core: ``encode()`` (byte-identical to the reference) and the
    engine's fields by their reference names."""

    def __init__(self, code: int, blob: bytes, terminal: bool, rewards, mask: int):
        self._code = code
        self._b = blob
        self.terminal = terminal
        self.rewards = rewards
        self.mask = mask

    # ---- reference Core fields
    _ROLE_BYTE = {0: 9, 1: 16, 2: 16, 3: 37, 5: 9, 6: 8}   # 2048 has one role

    @property
    def role_to_move(self) -> int:
        return 0 if self._code == 4 else self._b[self._ROLE_BYTE[self._code]]

    def __getattr__(self, name):
        b, c = self.__dict__["_b"], self.__dict__["_code"]
        if c in (0, 4) and name == "board":
            return tuple(b[:9]) if c == 0 else tuple(b[:16])
        if c in (1, 2) and name in ("bb0", "bb1"):
            return _le(b[0:8]) if name == "bb0" else _le(b[8:16])
        if c == 1 and name == "heights":
            occ = _le(b[0:8]) | _le(b[8:16])
            return tuple(bin((occ >> (7 * col)) & 0x7F).count("1") for col in range(7))
        if c == 2 and name == "pass_count":
            return b[17]
        if c == 3:
            if name in ("bb0", "bb1"):
                return _le(b[0:16]) if name == "bb0" else _le(b[16:32])
            if name == "move_number":
                return _le(b[32:36])
            if name == "swapped":
                return bool(b[36])
        if c == 4 and name == "score":
            return _le(b[16:24])
        if c == 5:
            if name == "hands":
                return (b[0], b[1])
            if name == "history":
                return tuple(b[2:2 + b[6]])
            if name == "extra":
                return (b[7], b[8])
        if c == 6:
            fields = {"hands": (b[0], b[1]), "public": b[2] - 1, "round": b[3], "raises": b[4],
                      "committed": (b[5], b[6]), "acted": b[7]}
            if name in fields:
                return fields[name]
        raise AttributeError(name)

    def encode(self) -> bytes:
        b, c = self._b, self._code
        if c == 0:                       # tictactoe.py:32-33
            return b[:10]
        if c == 1:                       # connect_four.py:38-43
            return b[0:7] + b[8:15] + b[16:17]
        if c == 2:                       # othello.py:95-100
            return b[0:16] + bytes([b[16], b[17]])
        if c == 3:                       # hexgame.py:62-67
            return b[0:32] + bytes([b[37], b[32], b[36]])
        if c == 4:                       # play2048.py:91-92
            return b[0:24]
        if c == 5:                       # kuhn_poker.py:33-34
            return b[0:2] + b[2:2 + b[6]] + b"\xff" + b[7:9]
        return b[0:9]                    # leduc_holdem.py:38-45


class SmallKernel(DeviceKernel):
    fp_code = 4

    def __init__(self, code: int, game_id: str, num_actions: int, obs_shape: tuple, num_players: int = 2):
        self.code = code
        self.game_id = game_id
        self.num_actions = num_actions
        self.obs_shape = obs_shape
        self.num_players = num_players

    def alloc_private(self, v: DeviceV) -> None:
        torch = _torch()
        v.priv.blob = torch.empty((v.n, STATE_BYTES), dtype=torch.uint8, device=v.device)

    def launch_init(self, v, ks, sk) -> None:
        nat.check(nat.lib().bbk_small_init(self.code, self.out_cols(v), nat.ptr(v.priv.blob), v.n, v.slot0, ks,
                                           nat.ptr(sk), v.limit, nat.stream_handle(v.device)), "bbk_small_init")

    def launch_step(self, v, out, a, ks, sk, limit) -> None:
        nat.check(nat.lib().bbk_small_step(self.code, self.cols(v), nat.ptr(v.priv.blob), self.out_cols(out),
                                           nat.ptr(out.priv.blob), nat.ptr(a), v.n, v.slot0, ks, nat.ptr(sk), limit,
                                           nat.stream_handle(v.device)), "bbk_small_step")

    def launch_observe(self, v, i, roles, out) -> None:
        nat.check(nat.lib().bbk_small_observe(self.code, nat.ptr(v.priv.blob[i:i + 1]),
                                              nat.ptr(v.dev.terminated[i:i + 1]), nat.ptr(roles), nat.ptr(out), 1,
                                              nat.stream_handle(v.device)), "bbk_small_observe")

    def launch_fingerprint(self, v, scratch, stride, lens, out) -> None:
        nat.check(nat.lib().bbk_small_fingerprint(self.code, self.cols(v), nat.ptr(v.priv.blob), v.n,
                                                  nat.ptr(scratch), stride, nat.ptr(lens), nat.ptr(out),
                                                  nat.stream_handle(v.device)), "bbk_small_fingerprint")

    def core_view(self, s, i, p2r, rewards, mask, terminal):
        bits = 0 if (terminal or s["truncated"][i]) else int.from_bytes(
            np.packbits(mask, bitorder="little").tobytes(), "little")
        return SmallCoreView(self.code, bytes(s["blob"][i]), terminal, self.role_rewards(p2r, rewards), bits)


def _game(code, game_id, players, obs_shape, actions, **flags) -> GameDef:
    return GameDef(spec=GameSpec(game_id, players, obs_shape, actions), max_steps=256,
                   batch_kernel=SmallKernel(code, game_id, actions, obs_shape, players), **flags)


TIC_TAC_TOE = _game(0, "tic_tac_toe", 2, (3, 3, 2), 9)
CONNECT_FOUR = _game(1, "connect_four", 2, (6, 7, 2), 7)
OTHELLO = _game(2, "othello", 2, (8, 8, 2), 65)
HEX = _game(3, "hex", 2, (11, 11, 4), 122)
PLAY_2048 = _game(4, "2048", 1, (4, 4, 31), 4, chance_in_step=True)
KUHN_POKER = _game(5, "kuhn_poker", 2, (7,), 4, perfect_information=False)
LEDUC_HOLDEM = _game(6, "leduc_holdem", 2, (34,), 3, chance_in_step=True, perfect_information=False)

GAMES = (TIC_TAC_TOE, CONNECT_FOUR, OTHELLO, HEX, PLAY_2048, KUHN_POKER, LEDUC_HOLDEM)
