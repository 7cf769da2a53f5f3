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


OUTPUT_FIELDS = ("observations", "rewards", "terminated", "truncated", "current_player", "legal_action_mask")


def batch_outputs(batch: Batch, *, device: bool = False) -> dict:
    """Per-field arrays, observations for each slot's current player (bench.py:86-97).

    ``device=False`` (the reference contract): host numpy arrays. ``device=True``: the
    batch's own CUDA tensors, zero copy; ``legal_action_mask`` is bool.
    """
    if device:
        d = batch.device
        return {
            "observations": d.observation,
            "rewards": d.rewards,
            "terminated": d.terminated,
            "truncated": d.truncated,
            "current_player": d.current_player,
            "legal_action_mask": d.legal_action_mask,
        }
    return {
        "observations": batch.observation,
        "rewards": batch.rewards,
        "terminated": batch.terminated,
        "truncated": batch.truncated,
        "current_player": batch.current_player,
        "legal_action_mask": batch.legal_action_mask,
    }


def batch_outputs_dlpack(batch: Batch) -> dict:
    """DLPack capsules of the device outputs (zero copy; consumable by any DLPack framework)."""
    from torch.utils.dlpack import to_dlpack

    return {k: to_dlpack(t) for k, t in batch_outputs(batch, device=True).items()}


_WIRE_MAGIC = b"BBKO"
_WIRE_ALIGN = 64


def pack_outputs(batch: Batch) -> bytes:
    """Binary wire form of batch_outputs (the JSON `.tolist()` of the reference's trace/serve is
    unusable at GB-sized observations): b"BBKO" | u32 header length | JSON header
    {field: [dtype, shape, offset, nbytes]} | 64-byte aligned raw little-endian fields. The device
    fields are copied once each into one pinned host buffer.
    """
    import json
    import struct

    import torch

    dev = batch_outputs(batch, device=True)
    layout, off = {}, 0
    for k in OUTPUT_FIELDS:
        t = dev[k]
        nbytes = t.numel() * t.element_size()
        layout[k] = [str(t.dtype).replace("torch.", ""), list(t.shape), off, nbytes]
        off = (off + nbytes + _WIRE_ALIGN - 1) // _WIRE_ALIGN * _WIRE_ALIGN
    hdr = json.dumps({"game_id": batch.game.game_id, "n": batch.size, "fields": layout}).encode()
    pre = _WIRE_MAGIC + struct.pack("<I", len(hdr)) + hdr
    base = (len(pre) + _WIRE_ALIGN - 1) // _WIRE_ALIGN * _WIRE_ALIGN
    host = torch.empty(base + off, dtype=torch.uint8, pin_memory=True)
    host[:len(pre)] = torch.frombuffer(bytearray(pre), dtype=torch.uint8)
    host[len(pre):base] = 0
    for k in OUTPUT_FIELDS:
        t = dev[k].contiguous().view(-1).view(torch.uint8)
        o = base + layout[k][2]
        host[o:o + t.numel()].copy_(t, non_blocking=True)
    torch.cuda.current_stream(dev["rewards"].device).synchronize()
    return host.numpy().tobytes()


def unpack_outputs(buf) -> dict:
    """Inverse of pack_outputs: numpy arrays (views into ``buf``) keyed like batch_outputs."""
    import json
    import struct

    mv = memoryview(buf)
    if bytes(mv[:4]) != _WIRE_MAGIC:
        raise ValueError("not a batch-outputs wire buffer")
    (hl,) = struct.unpack("<I", mv[4:8])
    hdr = json.loads(bytes(mv[8:8 + hl]))
    base = (8 + hl + _WIRE_ALIGN - 1) // _WIRE_ALIGN * _WIRE_ALIGN
    out = {}
    for k, (dtype, shape, off, nbytes) in hdr["fields"].items():
        a = np.frombuffer(mv, dtype=np.dtype(dtype), count=nbytes // np.dtype(dtype).itemsize, offset=base + off)
        out[k] = a.reshape(shape)
    return out


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
