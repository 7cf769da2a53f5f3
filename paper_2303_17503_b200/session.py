"""Benchmark harness mirror: BatchSession / batch_outputs / bench_run.

Reference pkg/src/boardbatch/bench.py:54-141. The key schedule is the
reference's: init uses root.child(0), step t (1-based) uses root.child(2t),
random actions before step t use root.child(2t-1).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .agents import random_actions_device
from .core import Batch, batch_init, batch_step, resolve
from .rng import RngKey


class BatchSession:
    """A batched environment driven from one root seed (bench.py:54-83)."""

    def __init__(self, game, batch_size: int, seed: int, *, max_steps: int | None = None, workers: int = 1,
                 validate: bool = True):
        self.gdef = resolve(game)
        self.root = RngKey(seed)
        self.workers = workers
        self.validate = validate
        self.batch: Batch = batch_init(self.gdef, self.root.child(0), batch_size, max_steps=max_steps,
                                       next_key=self.root.child(1))
        self.t = 0

    def sample_random_actions(self):
        """Device tensor of actions (bench.py:73-74)."""
        return random_actions_device(self.batch, self.root.child(2 * self.t + 1))

    def step(self, actions) -> Batch:
        batch = batch_step(self.batch, actions, self.root.child(2 * (self.t + 1)), validate=self.validate,
                           next_key=self.root.child(2 * (self.t + 1) + 1))
        self.t += 1
        self.batch = batch
        return batch


def batch_outputs(batch: Batch) -> dict:
    """Per-field host arrays, observations for each slot's current player (bench.py:86-97)."""
    return {
        "observations": batch.observation,
        "rewards": batch.rewards,
        "terminated": batch.terminated,
        "truncated": batch.truncated,
        "current_player": batch.current_player,
        "legal_action_mask": batch.legal_action_mask,
    }


@dataclass(frozen=True)
class BenchResult:
    game_id: str
    batch_size: int
    total_steps: int
    seed: int
    threads: int
    wall_seconds: float
    samples_per_second: float
    episodes_completed: int


def bench_run(game_id: str, batch_size: int, total_steps: int, seed: int = 0) -> BenchResult:
    """Random-policy batched stepping with auto-reset (bench.py:109-141), on the GPU."""
    import torch

    sess = BatchSession(game_id, batch_size, seed, validate=False)
    episodes = torch.zeros(1, dtype=torch.int64, device=sess.batch._v.device)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(total_steps):
        acts = sess.sample_random_actions()
        b = sess.step(acts)
        episodes += (b.device.terminated | b.device.truncated).sum()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return BenchResult(sess.gdef.game_id, batch_size, total_steps, seed, 1, wall,
                       batch_size * total_steps / max(wall, 1e-9), int(episodes.item()))
