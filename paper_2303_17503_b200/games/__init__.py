"""Device engines and the game registry (reference games/__init__.py:1-36).

Registered here: the north-star games go_9x9, go_19x19, backgammon, chess,
shogi, and the reference's small engines (tic_tac_toe, connect_four,
othello, hex, 2048, kuhn_poker, leduc_holdem; games/small.py). The
remaining reserved ids keep their metadata (``game_spec`` works) and raise
``UnsupportedGame`` on use.
"""

from ..core import GameSpec, register, reserve
from . import backgammon, go, small

register(go.GAME)
register(go.GAME19)
register(backgammon.GAME)
for _g in small.GAMES:
    register(_g)

try:
    from . import chess as _chess
    register(_chess.GAME)
except ImportError:  # pragma: no cover
    _chess = None
try:
    from . import shogi as _shogi
    register(_shogi.GAME)
except ImportError:  # pragma: no cover
    _shogi = None

_RESERVED = (
    GameSpec("tic_tac_toe", 2, (3, 3, 2), 9),
    GameSpec("connect_four", 2, (6, 7, 2), 7),
    GameSpec("othello", 2, (8, 8, 2), 65),
    GameSpec("hex", 2, (11, 11, 4), 122),
    GameSpec("2048", 1, (4, 4, 31), 4),
    GameSpec("kuhn_poker", 2, (7,), 4),
    GameSpec("leduc_holdem", 2, (34,), 3),
    GameSpec("animal_shogi", 2, (4, 3, 194), 132),
    GameSpec("bridge_bidding", 4, (480,), 38),
    GameSpec("chess", 2, (8, 8, 119), 4672),
    GameSpec("gardner_chess", 2, (5, 5, 115), 1225),
    GameSpec("minatar_asterix", 1, (10, 10, 4), 5),
    GameSpec("minatar_breakout", 1, (10, 10, 4), 3),
    GameSpec("minatar_freeway", 1, (10, 10, 7), 3),
    GameSpec("minatar_seaquest", 1, (10, 10, 10), 6),
    GameSpec("minatar_space_invaders", 1, (10, 10, 6), 4),
    GameSpec("shogi", 2, (9, 9, 119), 2187),
    GameSpec("sparrow_mahjong", 3, (11, 15), 11),
)

from ..core import _ENGINES  # noqa: E402

for _spec in _RESERVED:
    if _spec.game_id not in _ENGINES:
        reserve(_spec)
