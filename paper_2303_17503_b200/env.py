"""pgx-style facade: ``make(env_id)``, ``env.init(key)``, ``env.step(state, action)``.

The State fields named by the north star (current_player, observation,
legal_action_mask, rewards, terminated, truncated) are CUDA tensors with a
leading batch axis, like Pgx's vmapped states. Keys follow the reference's
BatchSession schedule (bench.py:54-83): ``init(seed)`` uses
root.child(0); the t-th ``step`` without an explicit key uses
root.child(2t); ``random_action(state)`` uses root.child(2t+1).
"""

from __future__ import annotations

from .core import Batch, batch_init, batch_step, resolve
from .rng import RngKey


class State:
    """Batched environment state (device tensors) over a Batch."""

    __slots__ = ("_batch", "_root", "_t")

    def __init__(self, batch: Batch, root: RngKey, t: int):
        self._batch = batch
        self._root = root
        self._t = t

    @property
    def batch(self) -> Batch:
        return self._batch

    current_player = property(lambda s: s._batch.device.current_player)
    observation = property(lambda s: s._batch.device.observation)
    legal_action_mask = property(lambda s: s._batch.device.legal_action_mask)
    rewards = property(lambda s: s._batch.device.rewards)
    terminated = property(lambda s: s._batch.device.terminated)
    truncated = property(lambda s: s._batch.device.truncated)
    step_count = property(lambda s: s._batch.device.step_count)
    player_to_role = property(lambda s: s._batch.device.player_to_role)

    def __len__(self) -> int:
        return self._batch.size


class Env:
    def __init__(self, env_id: str, batch_size: int = 1, max_steps: int | None = None):
        self.gdef = resolve(env_id)
        self.id = self.gdef.game_id
        self.batch_size = batch_size
        self.max_steps = max_steps

    num_players = property(lambda s: s.gdef.spec.num_players)
    num_actions = property(lambda s: s.gdef.spec.num_actions)
    observation_shape = property(lambda s: s.gdef.spec.observation_shape)

    def init(self, key, batch_size: int | None = None) -> State:
        root = key if isinstance(key, RngKey) else RngKey(int(key))
        n = self.batch_size if batch_size is None else batch_size
        return State(batch_init(self.gdef, root.child(0), n, max_steps=self.max_steps, next_key=root.child(1)), root, 0)

    def step(self, state: State, action, key: RngKey | None = None, validate: bool = True) -> State:
        k = key if key is not None else state._root.child(2 * (state._t + 1))
        nk = state._root.child(2 * (state._t + 1) + 1)
        return State(batch_step(state._batch, action, k, validate=validate, next_key=nk), state._root, state._t + 1)

    def random_action(self, state: State):
        from .agents import random_actions_device

        return random_actions_device(state._batch, state._root.child(2 * state._t + 1))


def make(env_id: str, batch_size: int = 1, max_steps: int | None = None) -> Env:
    return Env(env_id, batch_size=batch_size, max_steps=max_steps)
