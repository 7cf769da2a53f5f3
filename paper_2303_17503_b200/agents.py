"""Random-policy sampling (reference agents.py:25-46) on the device."""

from __future__ import annotations

import numpy as np

from .core import EnvState, TerminalStep
from .rng import RngKey


def random_agent(state: EnvState, key: RngKey) -> int:
    """Uniform draw over the mask-true actions (agents.py:25-30)."""
    if state.terminated or state.truncated:
        raise TerminalStep("cannot pick an action in a finished state")
    legal = np.flatnonzero(state.legal_action_mask)
    return int(legal[key.randint(len(legal))])


def random_actions_device(batch, key: RngKey, out=None):
    """Per-slot uniform legal actions as a CUDA int64 tensor (no host copy).

    Slot i receives exactly ``random_agent(states[i], key.child(slot0 + i))``;
    finished slots get 0 (agents.py:33-46), computed by bbk_random_actions.
    """
    v = batch._v
    if out is None and v.next_actions is not None and v.next_key == key.state:
        return v.next_actions   # already sampled by the fused step/init kernel from the same mask and key
    return v.kern.random_actions(v, key, out)


def random_actions(batch, key: RngKey) -> np.ndarray:
    """Host-array version with the reference's return type (agents.py:33-46)."""
    return random_actions_device(batch, key).cpu().numpy()


class RolloutResult:
    """First-episode outcome of every slot of a batched random rollout."""

    __slots__ = ("game_id", "returns", "lengths", "steps")

    def __init__(self, game_id, returns, lengths, steps):
        self.game_id = game_id
        self.returns = returns      # float32 [n, players], rewards by player at the episode's end
        self.lengths = lengths      # int32 [n], steps of the episode (step_count when it ended)
        self.steps = steps          # batch steps taken until every slot had finished once


def rollout(game, n: int, seed: int, *, max_steps: int | None = None, check_every: int = 16) -> RolloutResult:
    """Uniform-random rollouts to the end of the episode for n slots (agents.py:113-116, batched).

    Every slot plays the reference's random policy on the BatchSession key schedule
    (bench.py:54-83) -- the same trajectories as the reference's own ``BatchSession`` +
    ``random_actions`` loop -- until its first episode ends. The step kernel samples the next
    actions itself, ``bbk_latch_finished`` records each slot's first outcome on the device, and the
    host only polls a finished-slot counter every ``check_every`` steps.
    """
    import torch

    from . import _native as nat
    from .session import BatchSession

    sess = BatchSession(game, n, seed, max_steps=max_steps, validate=False)
    v0 = sess.batch._v
    dev = v0.device
    players = sess.gdef.spec.num_players
    done = torch.zeros(n, dtype=torch.uint8, device=dev)
    ret = torch.zeros((n, players), dtype=torch.float32, device=dev)
    length = torch.zeros(n, dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = nat.stream_handle(dev)
    t = 0
    while True:
        b = sess.step(sess.sample_random_actions())
        d = b.device
        nat.check(nat.lib().bbk_latch_finished(nat.ptr(d.terminated), nat.ptr(d.truncated), nat.ptr(d.rewards),
                                               nat.ptr(d.step_count), players, n, nat.ptr(done), nat.ptr(ret),
                                               nat.ptr(length), nat.ptr(count), stream), "bbk_latch_finished")
        t += 1
        if t % check_every == 0 or t >= (max_steps or sess.gdef.max_steps) + 1:
            if int(count.item()) >= n:
                break
    return RolloutResult(sess.gdef.game_id, ret.cpu().numpy(), length.cpu().numpy(), t)
