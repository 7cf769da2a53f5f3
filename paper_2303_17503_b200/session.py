"""Benchmark harness mirror: BatchSession / batch_outputs / bench_run.

Reference pkg/src/boardbatch/bench.py:54-141. The key schedule is the
reference's: init uses root.child(0), step t (1-based) uses root.child(2t),
random actions before step t use root.child(2t-1).
"""

from __future__ import annotations

import csv
import os
import time
from dataclasses import dataclass

import numpy as np

from .agents import random_actions_device
from .core import Batch, EngineError, batch_init, batch_step, resolve
from .rng import RngKey


class ResultFetcher:
    """The per-step host read of a batch's results -- rewards, terminated, truncated and
    current_player, what the reference's bench loop consumes every step (bench.py:121-129) --
    without stalling the device: double-buffered pinned host buffers filled on a copy stream by one
    native call (bbk_fetch_async: event record, stream wait, the copies, a done event) after the
    step's launch. ``fetch(batch)`` queues batch's copies and returns the PREVIOUS batch's results as
    numpy arrays (None on the first call), so the host runs one step behind the GPU; ``drain()``
    returns the last one."""

    FIELDS = ("rewards", "terminated", "truncated", "current_player")

    def __init__(self, n: int, num_players: int, device=None):
        import ctypes

        import torch

        from . import _native as nat

        self._torch, self._nat, self._C = torch, nat, ctypes
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        shapes = {"rewards": ((n, num_players), torch.float32), "terminated": ((n,), torch.bool),
                  "truncated": ((n,), torch.bool), "current_player": ((n,), torch.int32)}
        self.host = [{f: torch.empty(shp, dtype=dt, pin_memory=True) for f, (shp, dt) in shapes.items()}
                     for _ in range(2)]
        self._dst = [(ctypes.c_void_p * 4)(*[h[f].data_ptr() for f in self.FIELDS]) for h in self.host]
        self._bytes = (ctypes.c_int64 * 4)(*[self.host[0][f].numel() * self.host[0][f].element_size()
                                             for f in self.FIELDS])
        self.copy = torch.cuda.Stream(self.device)
        self.after = [torch.cuda.Event() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]
        for ev in self.after + self.done:   # materialise the CUDA events (handles for the native call)
            ev.record(self.copy)
        self._t = 0
        self._pending = None

    def _read(self, slot: int) -> dict:
        self.done[slot].synchronize()
        return {f: self.host[slot][f].numpy() for f in self.FIELDS}

    def fetch(self, batch):
        nat = self._nat
        d = batch.device
        slot = self._t & 1
        src = (self._C.c_void_p * 4)(*[getattr(d, f).data_ptr() for f in self.FIELDS])
        nat.check(nat.lib().bbk_fetch_async(4, self._dst[slot], src, self._bytes, nat.stream_handle(self.device),
                                            self.copy.cuda_stream, self.after[slot].cuda_event,
                                            self.done[slot].cuda_event), "bbk_fetch_async")
        # batch stays referenced until its copies are waited for: its buffers must not be recycled
        # (stream-ordered reuse covers the main stream only, not the copy stream)
        prev, self._pending = self._pending, (slot, batch)
        self._t += 1
        return None if prev is None else self._read(prev[0])

    def drain(self):
        prev, self._pending = self._pending, None
        return None if prev is None else self._read(prev[0])


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


class IoError(EngineError):
    """Output path cannot be written (bench.py:28-29)."""


@dataclass(frozen=True)
class BenchConfig:
    """bench.py:32-39: what bench_run measures."""

    game_id: str
    batch_size: int
    total_steps: int
    seed: int = 0
    worker_threads: int | str = 1   # accepted for compatibility: the GPU grid replaces the thread pool
    output_path: str | None = None


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


def resolve_threads(worker_threads) -> int:
    """bench.py:54-60."""
    if worker_threads == "auto":
        return os.cpu_count() or 1
    threads = int(worker_threads)
    if threads < 1:
        raise ValueError("worker_threads must be >= 1 or 'auto'")
    return threads


def bench_run(config: BenchConfig) -> BenchResult:
    """Random-policy batched stepping with auto-reset (bench.py:63-97), on the GPU.

    Wall time covers the step loop only (synchronised at both ends); the random policy is the
    fused in-kernel sampler and episodes are counted on the device.
    """
    import torch

    if config.batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    if config.total_steps < 1:
        raise ValueError("total_steps must be >= 1")
    threads = resolve_threads(config.worker_threads)
    sess = BatchSession(config.game_id, config.batch_size, config.seed, validate=False)
    episodes = torch.zeros(1, dtype=torch.int64, device=sess.batch._v.device)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(config.total_steps):
        b = sess.step(sess.sample_random_actions())
        episodes += (b.device.terminated | b.device.truncated).sum()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    samples = config.batch_size * config.total_steps
    return BenchResult(sess.gdef.game_id, config.batch_size, config.total_steps, config.seed, threads, wall,
                       samples / max(wall, 1e-9), int(episodes.item()))


_BENCH_FIELDS = ("game_id", "batch_size", "total_steps", "seed", "threads", "wall_seconds", "samples_per_second",
                 "episodes_completed")
_MATCH_FIELDS = ("game_id", "agent_a", "agent_b", "wins_a", "wins_b", "draws")


def _fmt(v):
    return repr(v) if isinstance(v, float) else v   # floats round-trip exactly


def write_results(results, path, kind: str | None = None) -> None:
    """CSV of BenchResults or agents.MatchResults with the reference's fixed headers
    (bench.py:158-179; the kind defaults from the first row's type)."""
    rows = list(results)
    if kind is None:
        kind = "matches" if rows and hasattr(rows[0], "wins_a") else "bench"
    if kind not in ("bench", "matches"):
        raise ValueError(f"unknown result kind {kind!r}")
    fields = _MATCH_FIELDS if kind == "matches" else _BENCH_FIELDS
    try:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(fields)
            for row in rows:
                w.writerow([_fmt(getattr(row, f)) for f in fields])
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc


def write_results_long(results, path) -> None:
    """Long format, one metric per row (bench.py:138-150)."""
    try:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(("game_id", "batch_size", "seed", "threads", "metric", "value"))
            for row in results:
                for metric in ("total_steps", "wall_seconds", "samples_per_second", "episodes_completed"):
                    w.writerow((row.game_id, row.batch_size, row.seed, row.threads, metric, _fmt(getattr(row, metric))))
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc
