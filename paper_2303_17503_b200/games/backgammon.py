"""Backgammon on the device.

Drop-in for reference ``games/backgammon.py`` (GameSpec("backgammon", 2,
(34,), 156), max_steps 1024, chance_in_step; backgammon.py:227-233). The
kernel (``csrc/backgammon.cu``) keeps 36 bytes of state per slot:
points[24] int8 and misc[12] = bar0 bar1 off0 off1 role d1 d2 rem0..3 nrem.
"""

from __future__ import annotations

from .. import _native as nat
from ..core import GameDef, GameSpec
from ._device import DeviceKernel, DeviceV, _torch


class BgCoreView:
    """Host view with the reference Core's fields (backgammon.py:98-119)."""

    __slots__ = ("points", "bar", "off", "role_to_move", "dice", "remaining", "terminal", "rewards", "mask")

    def __init__(self, points, bar, off, role_to_move, dice, remaining, terminal, rewards, mask):
        self.points = points
        self.bar = bar
        self.off = off
        self.role_to_move = role_to_move
        self.dice = dice
        self.remaining = remaining
        self.terminal = terminal
        self.rewards = rewards
        self.mask = mask

    def encode(self) -> bytes:
        """Byte-identical to reference Core.encode (backgammon.py:113-119)."""
        pts = bytes((v + 16) & 0xFF for v in self.points)
        rem = tuple(self.remaining) + (0,) * (4 - len(self.remaining))
        return pts + bytes((self.bar[0], self.bar[1], self.off[0], self.off[1], self.role_to_move,
                            self.dice[0], self.dice[1]) + rem)


class BackgammonKernel(DeviceKernel):
    game_id = "backgammon"
    num_actions = 156
    obs_shape = (34,)

    def alloc_private(self, v: DeviceV) -> None:
        torch = _torch()
        v.priv.points = torch.empty((v.n, 24), dtype=torch.int8, device=v.device)
        v.priv.misc = torch.empty((v.n, 12), dtype=torch.uint8, device=v.device)

    @staticmethod
    def state_struct(v: DeviceV, i: int | None = None) -> nat.BgState:
        if i is None:
            return nat.BgState(nat.ptr(v.priv.points), nat.ptr(v.priv.misc))
        return nat.BgState(nat.ptr(v.priv.points[i:i + 1]), nat.ptr(v.priv.misc[i:i + 1]))

    fp_code = 1

    def launch_fingerprint(self, v, scratch, stride, lens, out) -> None:
        nat.check(nat.lib().bbk_bg_fingerprint(self.cols(v), self.state_struct(v), v.n, nat.ptr(scratch), stride,
                                               nat.ptr(lens), nat.ptr(out), nat.stream_handle(v.device)),
                  "bbk_bg_fingerprint")

    def launch_init(self, v, ks, sk):
        nat.check(nat.lib().bbk_bg_init(self.out_cols(v), self.state_struct(v), v.n, v.slot0, ks, nat.ptr(sk), v.limit,
                                        nat.stream_handle(v.device)), "bbk_bg_init")

    def launch_step(self, v, out, a, ks, sk, limit):
        nat.check(nat.lib().bbk_bg_step(self.cols(v), self.state_struct(v), self.out_cols(out), self.state_struct(out),
                                        nat.ptr(a), v.n, v.slot0, ks, nat.ptr(sk), limit,
                                        nat.stream_handle(v.device)), "bbk_bg_step")

    def launch_observe(self, v, i, roles, out):
        nat.check(nat.lib().bbk_bg_observe(self.state_struct(v, i), nat.ptr(roles), nat.ptr(out), 1,
                                           nat.stream_handle(v.device)), "bbk_bg_observe")

    def core_view(self, s, i, p2r, rewards, mask, terminal):
        m = s["misc"][i]
        nrem = int(m[11])
        bits = 0 if (terminal or s["truncated"][i]) else int.from_bytes(
            __import__("numpy").packbits(mask, bitorder="little").tobytes(), "little")
        return BgCoreView(
            points=tuple(int(x) for x in s["points"][i]),
            bar=(int(m[0]), int(m[1])),
            off=(int(m[2]), int(m[3])),
            role_to_move=int(m[4]),
            dice=(int(m[5]), int(m[6])),
            remaining=tuple(int(x) for x in m[7:7 + nrem]),
            terminal=terminal,
            rewards=self.role_rewards(p2r, rewards),
            mask=bits,
        )


GAME = GameDef(
    spec=GameSpec("backgammon", 2, (34,), 156),
    max_steps=1024,
    chance_in_step=True,
    batch_kernel=BackgammonKernel(),
)
