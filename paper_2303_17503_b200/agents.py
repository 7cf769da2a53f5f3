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
