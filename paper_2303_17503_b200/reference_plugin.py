"""Reference-side hook-in: run the reference's own engines' batch path on the B200 kernels.

This is the binding a ``boardbatch`` maintainer adds, as a module: it
re-registers the reference's registered games with ``core.register(dataclasses.replace(GAME,
batch_kernel=K))`` (reference ``core.py:126-128``), where ``K`` implements the reference's
``batch_kernel`` protocol (``core.py:88``; ``init`` ``core.py:346-348``, ``step``
``core.py:366-368``, ``state_at`` ``core.py:276-282``; template ``games/tictactoe.py:71-198``) over
this package's device kernels. Nothing in the reference changes; only ``batch_init`` /
``batch_step`` / ``Batch.states`` of the registered games now run on the GPU.

``K.state_at`` returns the reference's own ``EnvState`` carrying the reference module's own
``Core`` class, rebuilt from the device state, so every reference code path that consumes a
kernel-produced state — the scalar ``step`` (``go.apply`` reads ``core.an`` and
``core.history``, ``go.py:232,253-254``), ``observe``, ``render``, agents, fingerprints — works
unchanged (as ``tictactoe.py:171-198`` does for its numpy kernel). Errors raised by the device path
are re-raised as the reference's exception classes.

Use::

    pytest -p paper_2303_17503_b200.reference_plugin <reference tests>   # pytest plugin
    import paper_2303_17503_b200.reference_plugin as p; p.install()     # or at startup

``BBK_PLUGIN_GAMES`` (comma-separated ids) limits which games are re-registered.
"""

from __future__ import annotations

import dataclasses
import inspect
import os
import sys

import numpy as np

from . import core as ours
from .core import resolve as _resolve_ours

# reference game id -> (reference module name, reference GameDef attribute)
REFERENCE_GAMES = {
    "tic_tac_toe": "tictactoe",
    "connect_four": "connect_four",
    "othello": "othello",
    "hex": "hexgame",
    "go_9x9": "go",
    "2048": "play2048",
    "backgammon": "backgammon",
    "kuhn_poker": "kuhn_poker",
    "leduc_holdem": "leduc_holdem",
}


def _ref():
    import boardbatch
    import boardbatch.core as rcore

    return boardbatch, rcore


class _CoreBuilder:
    """Our host core view -> an instance of the reference module's ``Core`` class."""

    def __init__(self, game_id: str, module):
        self.game_id = game_id
        self.mod = module
        self.Core = module.Core
        self.params = [p for p in inspect.signature(self.Core.__init__).parameters if p != "self"]
        if game_id.startswith("go_"):
            size = int(game_id[3:].split("x")[0])
            self._nbrs = module._neighbor_table(size)
            self._zob = module._zobrist(size)

    def __call__(self, view, st):
        g = self.game_id
        if g == "2048":
            # the reference Core caches its four slides; _finish recomputes them from the board
            # (play2048.py:90-99) with the last transition's reward
            return self.mod._finish(tuple(view.board), int(view.score), int(view.rewards[0]))
        if g.startswith("go_"):
            # go.py:83-111: `history` is the superko set (device store prefix), `an` the cached
            # analysis of the current board (go.py:45-80)
            an = self.mod._analyse(view.board, self._nbrs, self._zob)
            return self.Core(view.board, view.role_to_move, view.terminal, view.rewards, view.mask,
                             view.pass_count, view.hash, view.hist_xor, view.history, view.boards_hist, an)
        vals = []
        for p in self.params:
            x = getattr(view, p.rstrip("_"))   # constructor args `round_`, `hash_` name fields
            if g == "tic_tac_toe" and p == "board":
                x = bytes(x)
            vals.append(x)
        return self.Core(*vals)


class ReferenceKernel:
    """The reference's ``batch_kernel`` protocol over this package's device kernel for one game."""

    def __init__(self, game_id: str, ref_gdef):
        self.game_id = game_id
        self.ours = _resolve_ours(game_id)
        self.kern = self.ours.batch_kernel
        import importlib

        self.build_core = _CoreBuilder(game_id, importlib.import_module(f"boardbatch.games.{REFERENCE_GAMES[game_id]}"))
        self.ref_gdef = ref_gdef

    # protocol -----------------------------------------------------------------------------
    def init(self, gdef, key, n, limit):
        with _translated_errors():
            return self.kern.init(self.ours, key, int(n), int(limit))

    def step(self, gdef, v, actions, key, limit):
        with _translated_errors():
            return self.kern.step(self.ours, v, np.asarray(actions, dtype=np.int64), key, int(limit))

    def state_at(self, gdef, v, i, limit):
        _, rcore = _ref()
        with _translated_errors():
            s = self.kern.state_at(self.ours, v, int(i), int(limit))
            core = self.build_core(s.core, s)
        return rcore.EnvState(
            current_player=s.current_player,
            legal_action_mask=s.legal_action_mask,
            rewards=s.rewards,
            terminated=s.terminated,
            truncated=s.truncated,
            step_count=s.step_count,
            player_to_role=s.player_to_role,
            core=core,
            game=gdef,
            max_steps=limit,
        )


class _translated_errors:
    """Re-raise this package's errors as the reference's classes (same names, core.py:24-58)."""

    def __enter__(self):
        return self

    def __exit__(self, et, ev, tb):
        if ev is None or not isinstance(ev, ours.EngineError):
            return False
        _, rcore = _ref()
        cls = getattr(rcore, type(ev).__name__, None)
        if cls is None:
            return False
        if type(ev).__name__ == "IllegalAction":
            raise cls(str(ev), action=ev.action, slot=ev.slot) from ev
        raise cls(str(ev)) from ev


def install(games=None) -> list[str]:
    """Re-register the reference's engines with device kernels; returns the ids re-registered."""
    _, rcore = _ref()
    env = os.environ.get("BBK_PLUGIN_GAMES")
    if games is None:
        games = env.split(",") if env else list(REFERENCE_GAMES)
    done = []
    for gid in games:
        gdef = rcore.resolve(gid)
        if isinstance(gdef.batch_kernel, ReferenceKernel):
            done.append(gid)
            continue
        rgd = dataclasses.replace(gdef, batch_kernel=None)
        kern = ReferenceKernel(gid, rgd)
        rcore.register(dataclasses.replace(gdef, batch_kernel=kern))
        done.append(gid)
    return done


# pytest plugin hook (pytest -p paper_2303_17503_b200.reference_plugin)
def pytest_configure(config):
    games = install()
    config._bbk_plugin_games = games
    print(f"boardbatch B200 plugin: device batch_kernel for {', '.join(games)}", file=sys.stderr, flush=True)


def pytest_report_header(config):
    return [f"boardbatch B200 plugin: device batch_kernel for {', '.join(getattr(config, '_bbk_plugin_games', []))}"]
