#!/usr/bin/env python
"""Random-play env-steps/s benchmark (BASELINE.json metric) on 1..8 B200s.

One "step" = one pass of the hot path over the whole batch: device random
actions (agents.random_actions, agents.py:33-46) + the batched env step with
auto-reset and fused observation emission (core.batch_step, core.py:353-386;
the reference's bench_run loop, bench.py:121-129) + the episode counter.

  python bench.py [--game go_19x19] [--batch 131072] [--steps K] [--warmup W]
  torchrun --nproc-per-node N bench.py --gpus N ...      (weak scaling: B per GPU)
  torchrun ... bench.py --game backgammon --global-batch 131072   (strong scaling: B/N per GPU)
  python bench.py --impl reference ...                    (CPU reference arm)

Rank 0 prints ONE JSON line. `value` = env-steps/s over all ranks with inputs
resident in HBM (K steps after W warm-up steps from init); `e2e` = the same
metric through the public batch_step API with host (pinned) buffers, with the
device random policy writing the next actions into the host buffer
("policy": "device"); `e2e_host_policy` = a host agent that reads the legal mask
back every step and samples with the reference's random_actions rule on the
host; `roofline` = the step kernel's algorithmic bytes per launch / its
CUDA-event duration vs MEASURED_PEAKS.json. The default single-GPU line also
carries `windows` (go_19x19 full episode cycle and a late-game window), a
`games` block (chess, shogi, go_9x9, backgammon, each with value / roofline /
e2e / cpu_baseline), and the real reference (pure Python, baseline/_ref)
timed on the host's cores for go_9x9 / go_19x19 / backgammon, including
BASELINE config 1 (go_9x9, 1024 envs to termination).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

# Algorithmic bytes per env-step (restated in DESIGN.md §4):
# int64 action + float32 observation + bool mask + rewards/flags/player +
# compact state read/write. The superko history scan is excluded.
B_ALG = {"go_9x9": 5964, "go_19x19": 25860, "chess": 35502, "shogi": 41013, "backgammon": 400}
DEFAULT_BATCH = {"go_9x9": 1 << 17, "go_19x19": 1 << 17, "chess": 1 << 17, "shogi": 1 << 16, "backgammon": 1 << 17}
STEP_KERNEL = {"go_9x9": "go::step_kernel<9>", "go_19x19": "go::step_kernel<19>", "chess": "chess::step_kernel<false>",
               "shogi": "shogi::step_kernel<false>", "backgammon": "bg::step_kernel"}
# The reference's small engines: (obs floats, actions, players, Core.encode bytes);
# B_alg = action 8 + obs + mask + rewards + flags/player/step + player_to_role + encoded Core r/w.
SMALL = {"tic_tac_toe": (18, 9, 2, 10, "TicTacToe"), "connect_four": (84, 7, 2, 15, "ConnectFour"),
         "othello": (128, 65, 2, 18, "Othello"), "hex": (484, 122, 2, 35, "Hex"), "2048": (496, 4, 1, 24, "Play2048"),
         "kuhn_poker": (7, 4, 2, 8, "Kuhn"), "leduc_holdem": (34, 3, 2, 9, "Leduc")}
for _g, (_o, _a, _p, _e, _k) in SMALL.items():
    B_ALG[_g] = 8 + 4 * _o + _a + 4 * _p + 10 + _p + 2 * _e
    DEFAULT_BATCH[_g] = 1 << 17
    STEP_KERNEL[_g] = f"small::step_kernel<{_k}>"
METRIC = "random-play env steps/sec"
NORTH_STAR_GAMES = ("chess", "shogi", "go_9x9", "backgammon")   # the `games` block next to go_19x19
REFERENCE_GAMES = ("go_9x9", "go_19x19", "backgammon")           # engines the reference itself implements


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--game", default="go_19x19")
    ap.add_argument("--batch", type=int, default=0, help="envs per GPU (default per game, 2^17 for go_19x19)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: total envs split over the ranks (BASELINE config 5: backgammon 2^17)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="omit the batch-size sweep 2^10..2^17 from the line")
    ap.add_argument("--no-games", action="store_true", help="omit the per-game block of the default line")
    ap.add_argument("--no-reference-cpu", action="store_true", help="do not time the pure-Python reference")
    ap.add_argument("--unfused", action="store_true", help="separate sampler / step / counter launches")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard_plan(game: str, batch: int, global_batch: int, rank: int, world: int) -> dict:
    """Which slots this rank owns: weak scaling keeps B per GPU; strong scaling
    splits a fixed global batch. slot0 = the rank's first GLOBAL slot index, so every rank's
    trajectory is bit-identical to the same rows of one big batch (global slot keys)."""
    if global_batch:
        if global_batch % world:
            raise SystemExit(f"--global-batch {global_batch} is not divisible by {world} ranks")
        B = global_batch // world
        return {"B": B, "slot0": rank * B, "scaling": "strong", "global_batch": global_batch}
    B = batch or DEFAULT_BATCH[game]
    return {"B": B, "slot0": rank * B, "scaling": "weak", "global_batch": B * world}


def reduce_over_ranks(ms: float, episodes, world: int, device) -> tuple[float, int]:
    """MAX of the timed region over ranks, SUM of the episode counters (the only collectives)."""
    if world == 1:
        return ms, int(episodes.item())
    import torch
    import torch.distributed as dist

    tt = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ep = episodes.to(device=device, dtype=torch.int64).clone()
    dist.all_reduce(ep, op=dist.ReduceOp.SUM)
    dist.barrier()
    return float(tt.item()), int(ep.item())


def ncu_traffic(game: str, B: int):
    """DRAM bytes per step-kernel launch from the committed ncu --set full capture (profiles/)."""
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", rnd, "ncu_traffic.json")
        try:
            with open(path) as fh:
                d = json.load(fh)[game]
            return d["dram_bytes_per_env_step"] * B, f"profiles/{rnd}/ncu_traffic.json ({d['captured']})"
        except Exception:
            continue
    return None, None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bbk_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ GPU arm
class DeviceLoop:
    """The benchmark's step loop on one game: ping-pong device states (only the previous batch stays
    valid), and by default the fused step kernel (it also samples the NEXT step's random actions
    from the new legal mask with the schedule's key and counts finished slots: one launch per
    step). ``unfused`` runs sampler / step / counter as 3 launches."""

    def __init__(self, game, B, slot0, dev, seed, unfused=False):
        import torch

        import paper_2303_17503_b200 as bb
        from paper_2303_17503_b200.core import resolve

        self.game, self.B, self.dev, self.unfused = game, B, dev, unfused
        self.gdef = resolve(game)
        self.kern = self.gdef.batch_kernel
        self.limit = self.gdef.max_steps
        self.root = bb.RngKey(seed)
        self.acts = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(2)]
        self.episodes = torch.zeros(1, dtype=torch.int64, device=dev)
        self.cur = self.kern.init(self.gdef, self.root.child(0), B, self.limit, slot0=slot0, device=dev,
                                  next_key=None if unfused else self.root.child(1), next_actions=self.acts[0])
        self.spare = self.kern.new_v(B, slot0, dev, 0, self.limit)
        self.lib = __import__("paper_2303_17503_b200._native", fromlist=["lib"]).lib()
        self.stream = torch.cuda.current_stream(dev)
        self.t = 0

    def step(self, ev=None):
        kern, gdef, root, t = self.kern, self.gdef, self.root, self.t
        a_now, a_next = self.acts[t % 2], self.acts[(t + 1) % 2]
        if self.unfused:
            kern.random_actions(self.cur, root.child(2 * t + 1), out=a_now)
        if ev is not None:
            ev[0].record(self.stream)
        if self.unfused:
            nxt = kern.step(gdef, self.cur, a_now, root.child(2 * (t + 1)), self.limit, validate=False, out=self.spare)
        else:
            nxt = kern.step(gdef, self.cur, a_now, root.child(2 * (t + 1)), self.limit, validate=False, out=self.spare,
                            next_key=root.child(2 * (t + 1) + 1), next_actions=a_next, episodes=self.episodes)
        if ev is not None:
            ev[1].record(self.stream)
        if self.unfused:
            self.lib.bbk_count_finished(nxt.dev.terminated.data_ptr(), nxt.dev.truncated.data_ptr(), self.B,
                                        self.episodes.data_ptr(), self.stream.cuda_stream)
        self.spare, self.cur = self.cur, nxt
        self.t += 1

    def timed(self, K):
        """K steps between CUDA events on the launching stream (synchronised on both sides). Returns
        (ms, per-launch step-kernel ms list).

        Fused mode (one kernel per step): the K launches are captured into one CUDA graph (the same
        kernels with the same arguments as the eager loop) and the graph is replayed once between the
        events, so host launch overhead never shows up as device time -- backgammon's 30 us step is
        shorter than the host's ~30 us per launch, and eager timing made it host-bound and noisy
        (2.8-4.2 G env-steps/s). Every kernel in the graph is a step kernel, so the per-launch
        duration is the replay time / K. Unfused mode keeps eager launches with per-launch events."""
        import torch

        if not self.unfused:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.dev)
            side.wait_stream(self.stream)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=side):
                for _ in range(K):
                    self.step()
            torch.cuda.synchronize()
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(self.stream)
            g.replay()
            end.record(self.stream)
            torch.cuda.synchronize()
            ms = start.elapsed_time(end)
            del g
            return ms, [ms / K] * K
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(self.stream)
        for k in range(K):
            self.step(evs[k])
        end.record(self.stream)
        torch.cuda.synchronize()
        return start.elapsed_time(end), [a.elapsed_time(b) for a, b in evs]


def roofline(game, B, kern_ms, ms_per_step):
    peak, peak_kind = peaks()
    avg = sum(kern_ms) / len(kern_ms)
    achieved = B_ALG[game] * B / (avg / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(game, B)
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_kind,
            "kernel": STEP_KERNEL[game], "kernel_ms": avg, "kernel_share_of_step": avg / ms_per_step,
            "bytes_per_env_step": B_ALG[game], "bytes_per_launch": B_ALG[game] * B}


def run_gpu(args, rank, world, local):
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    game = args.game
    plan = shard_plan(game, args.batch, args.global_batch, rank, world)
    B, slot0 = plan["B"], plan["slot0"]
    loop = DeviceLoop(game, B, slot0, dev, args.seed, args.unfused)
    gdef = loop.gdef
    for _ in range(args.warmup):
        loop.step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms, kern_ms = loop.timed(args.steps)
    clk = clocks.stop()
    ms, episodes = reduce_over_ranks(ms, loop.episodes, world, dev)
    total_steps = B * world * args.steps
    value = total_steps / (ms / 1e3)
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "env-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": plan["scaling"],
        "vs_baseline": None,
        "dtype": "u64/int8 (integer board logic; float32 observation output)",
        "data": "synthetic: random-play rollouts from the reference key schedule (seed %d), auto-reset" % args.seed,
        "config": {"workload": f"{game} random play with legal_action_mask + observation", "game": game,
                   "batch_per_gpu": B, "global_batch": plan["global_batch"], "max_steps": loop.limit,
                   "parallelism": f"dp{world} (independent env slices, global slot keys)",
                   "l2": "per-step outputs exceed L2 (obs %.2f GB/step), no flush needed" % (
                       B * 4 * math.prod(gdef.spec.observation_shape) / 1e9),
                   "timed": "K steps after W warm-up steps from init (steps W+1..W+K of the BatchSession schedule)"},
        "clocks": clk,
        "gpu_launches": (3 if args.unfused else 1) * args.steps,
        "roofline": roofline(game, B, kern_ms, ms / args.steps),
        "episodes_completed": episodes,
    }
    if world == 1 and game == "go_19x19":
        out["windows"] = go19_windows(args, dev, slot0, B)
    if not args.no_e2e:
        out["e2e"] = run_e2e(args, game, dev, world, slot0, B)
        if world == 1:
            out["e2e_host_policy"] = run_e2e_host_policy(args, game, dev, slot0, B)
    if not args.no_sweep and not args.global_batch:
        out["sweep"] = run_sweep(args, gdef, loop.kern, dev, slot0)
    del loop
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, game, B, args.cpu_seconds)
        if game in REFERENCE_GAMES and not args.no_reference_cpu:
            out["reference_cpu"] = reference_python(game, args.seed, args.cpu_seconds)
    if world == 1 and not args.no_games and args.game == "go_19x19" and not args.batch:
        out["games"] = {g: game_block(args, g, dev) for g in NORTH_STAR_GAMES}
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return out


def go19_windows(args, dev, slot0, B):
    """Windows beside the driver's (early-game) K: the full episode cycle (slots truncate in
    phase at max_steps = 512, so 512 steps after a 16-step warm-up cover every phase once), a
    late-game window (steps 401..432: long superko histories, crowded boards), and SURVEY §8(d)
    config 2's steady-state window (1024 steps after a 512-step warm-up: two cycles, every slot
    past its first reset)."""
    import torch

    res = {}
    for name, W, K in (("full_cycle", 16, 512), ("late_game", 400, 32), ("survey_config2", 512, 1024)):
        loop = DeviceLoop("go_19x19", B, slot0, dev, args.seed)
        for _ in range(W):
            loop.step()
        torch.cuda.synchronize()
        ms, kern_ms = loop.timed(K)
        rf = roofline("go_19x19", B, kern_ms, ms / K)
        res[name] = {"value": B * K / (ms / 1e3), "steps": K, "warmup": W, "ms_per_step": ms / K,
                     "roofline_frac": rf["frac"], "kernel_ms": rf["kernel_ms"]}
        del loop
    return res


def game_block(args, game, dev):
    """One north-star game at its BASELINE batch: value (K=64 after W=8), roofline, e2e, cpu_baseline
    (+ the pure-Python reference where it implements the game)."""
    import torch

    B = DEFAULT_BATCH[game]
    W, K = 8, 64
    loop = DeviceLoop(game, B, 0, dev, args.seed)
    for _ in range(W):
        loop.step()
    torch.cuda.synchronize()
    ms, kern_ms = loop.timed(K)
    del loop
    out = {"value": B * K / (ms / 1e3), "unit": "env-steps/s", "batch": B, "steps": K, "warmup": W,
           "ms_per_step": ms / K, "roofline": roofline(game, B, kern_ms, ms / K), "gpu_launches": K}
    if not args.no_sweep:   # batch sizes 2^10..2^17 (north star), as for the headline game
        from paper_2303_17503_b200.core import resolve

        gdef = resolve(game)
        out["sweep"] = run_sweep(args, gdef, gdef.batch_kernel, dev, 0)
    if not args.no_e2e:
        sub = argparse.Namespace(**{**vars(args), "steps": K, "warmup": W})
        out["e2e"] = run_e2e(sub, game, dev, 1, 0, B)
        out["e2e_host_policy"] = run_e2e_host_policy(sub, game, dev, 0, B)
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, game, B, min(args.cpu_seconds, 5.0))
        if game in REFERENCE_GAMES and not args.no_reference_cpu:
            out["reference_cpu"] = reference_python(game, args.seed, min(args.cpu_seconds, 6.0))
    if game == "go_9x9":
        out["baseline_config1"] = baseline_config1(args)
    if game == "backgammon":   # SURVEY §8(d) config 5's window: 2048 steps after a 1024-step warm-up
        loop = DeviceLoop(game, B, 0, dev, args.seed)
        for _ in range(1024):
            loop.step()
        torch.cuda.synchronize()
        ms, kern_ms = loop.timed(2048)
        del loop
        out["survey_config5_window"] = {"value": B * 2048 / (ms / 1e3), "steps": 2048, "warmup": 1024,
                                        "ms_per_step": ms / 2048,
                                        "roofline_frac": roofline(game, B, kern_ms, ms / 2048)["frac"]}
    return out


def run_e2e(args, game, dev, world, slot0, B):
    """Same metric through the public API with host buffers, over the same step window, with the
    DEVICE random policy (policy "device").

    A fresh batch (same seed, same slots) is stepped W untimed + K timed steps through
    core.batch_step. Per step: core.batch_step reads the actions from a pinned host buffer and its
    fused sampler (the device random policy) writes the next actions into the other pinned buffer
    (zero-copy over PCIe: the kernel loads / stores them itself; BBK_ZERO_COPY=0 uses an H2D copy
    and a D2H copy instead); the step's rewards / terminated / truncated / current_player go D2H on
    a copy stream into double-buffered pinned buffers, read on the host one step later (they overlap
    the next step; the last step's are waited for inside the timed region). Neither the legal mask
    nor the observation crosses PCIe (see e2e_host_policy for a host agent that needs the mask).
    """
    import torch

    import paper_2303_17503_b200 as bb
    from paper_2303_17503_b200.agents import random_actions_device
    from paper_2303_17503_b200.core import Batch, batch_step, resolve
    from paper_2303_17503_b200.games._device import ZERO_COPY
    from paper_2303_17503_b200.session import ResultFetcher

    gdef = resolve(game)
    kern = gdef.batch_kernel
    root = bb.RngKey(args.seed)
    batch = Batch(gdef, B, gdef.max_steps, vstate=kern.init(gdef, root.child(0), B, gdef.max_steps, slot0=slot0,
                                                            device=dev, next_key=root.child(1)))
    acts = [torch.empty(B, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    P = gdef.spec.num_players
    fetcher = ResultFetcher(B, P, dev)   # public API: pinned double buffers, one native call per step
    t = 0
    acts[0].copy_(random_actions_device(batch, root.child(1)))

    def one():
        nonlocal batch, t
        nk = root.child(2 * (t + 1) + 1)
        batch = batch_step(batch, acts[t % 2], root.child(2 * (t + 1)), validate=False, next_key=nk,
                           next_actions=acts[(t + 1) % 2] if ZERO_COPY else None)
        if not ZERO_COPY:
            acts[(t + 1) % 2].copy_(random_actions_device(batch, nk), non_blocking=True)
        # no host wait for the step itself: the next step's kernel reads the next actions from the
        # pinned buffer in stream order; the host reads the PREVIOUS step's results here (one step
        # behind), so it runs at most one step ahead of the GPU
        fetcher.fetch(batch)
        t += 1

    def drain():
        fetcher.drain()

    for _ in range(args.warmup):
        one()
    drain()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    drain()
    dt = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    return {"value": B * world * args.steps / dt, "unit": "env-steps/s", "policy": "device",
            "h2d_bytes_per_step": 8 * B, "d2h_bytes_per_step": (4 * P + 2 + 4 + 8) * B, "steps": args.steps,
            "path": "public core.batch_step; the DEVICE random policy (fused sampler) writes the next actions into "
                    "pinned host memory and the step kernel reads them from there (zero-copy over PCIe; "
                    "BBK_ZERO_COPY=0 copies instead); rewards/flags/player D2H on a copy stream (session.ResultFetcher: "
                    "pinned double buffers, one native bbk_fetch_async call per step), read by the host one "
                    "step later; the mask and observation stay on the device; same window as value",
            "zero_copy": ZERO_COPY}


def host_random_actions(mask, key_state: int, slot0: int = 0):
    """agents.random_actions (reference agents.py:33-46) on the host, vectorised numpy: slot i plays
    the d-th legal action, d = child(key, slot0 + i) % max(popcount(mask_i), 1); 0 if none."""
    import numpy as np

    from paper_2303_17503_b200.rng import child_states

    n = mask.shape[0]
    rows, cols = np.nonzero(mask)
    cnt = np.bincount(rows, minlength=n)
    start = np.cumsum(cnt) - cnt
    d = (child_states(key_state, n, slot0) % np.maximum(cnt, 1).astype(np.uint64)).astype(np.int64)
    out = np.zeros(n, dtype=np.int64)
    live = cnt > 0
    out[live] = cols[start[live] + d[live]]
    return out


def run_e2e_host_policy(args, game, dev, slot0, B, K=None):
    """The drop-in cost for a HOST agent of the reference API: every step the legal mask goes D2H
    (pinned), the host samples with the reference's random_actions rule (host_random_actions), the
    actions go H2D (pinned), batch_step runs, and rewards / flags / player come back. Bounded: a
    few steps (the host sampler dominates)."""
    import torch

    import paper_2303_17503_b200 as bb
    from paper_2303_17503_b200.core import Batch, batch_step, resolve

    gdef = resolve(game)
    kern = gdef.batch_kernel
    A, P = gdef.spec.num_actions, gdef.spec.num_players
    K = K or (4 if A * B > 1e8 else 8)
    root = bb.RngKey(args.seed)
    batch = Batch(gdef, B, gdef.max_steps, vstate=kern.init(gdef, root.child(0), B, gdef.max_steps, slot0=slot0,
                                                            device=dev))
    mask_h = torch.empty((B, A), dtype=torch.bool, pin_memory=True)
    acts_h = torch.empty(B, dtype=torch.int64, pin_memory=True)
    res_h = dict(r=torch.empty((B, P), dtype=torch.float32, pin_memory=True),
                 term=torch.empty(B, dtype=torch.bool, pin_memory=True),
                 trunc=torch.empty(B, dtype=torch.bool, pin_memory=True),
                 cp=torch.empty(B, dtype=torch.int32, pin_memory=True))
    t = 0

    def one():
        nonlocal batch, t
        d = batch.device
        mask_h.copy_(d.legal_action_mask, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        acts_h.numpy()[:] = host_random_actions(mask_h.numpy(), root.child(2 * t + 1).state, slot0)
        batch = batch_step(batch, acts_h, root.child(2 * (t + 1)), validate=False)
        d = batch.device
        for k, src in (("r", d.rewards), ("term", d.terminated), ("trunc", d.truncated), ("cp", d.current_player)):
            res_h[k].copy_(src, non_blocking=True)
        t += 1

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        one()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"value": B * K / dt, "unit": "env-steps/s", "policy": "host", "steps": K, "warmup": 2,
            "h2d_bytes_per_step": 8 * B, "d2h_bytes_per_step": (A + 4 * P + 2 + 4) * B,
            "path": "public core.batch_step with a host agent: legal mask D2H (pinned) -> reference random_actions "
                    "rule on the host (numpy) -> actions H2D (pinned) -> step -> rewards/flags/player D2H"}


def run_sweep(args, gdef, kern, dev, slot0):
    """env-steps/s vs batch size (BASELINE metric): per B, 8 eager steps from init, then steps
    9..72 captured once into a CUDA graph (the same kernels with the same arguments as the eager
    loop, no host launch overhead) and replayed once between CUDA events."""
    import torch

    import paper_2303_17503_b200 as bb

    res = {}
    root = bb.RngKey(args.seed)
    n_steps = 64
    for e in range(10, 18):
        B = 1 << e
        if gdef.game_id == "shogi" and e > 16:
            continue
        acts = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(2)]
        st = {"cur": kern.init(gdef, root.child(0), B, gdef.max_steps, slot0=slot0, device=dev,
                               next_key=root.child(1), next_actions=acts[0]),
              "spare": kern.new_v(B, slot0, dev, 0, gdef.max_steps), "t": 0}

        def one():
            t = st["t"]
            nxt = kern.step(gdef, st["cur"], acts[t % 2], root.child(2 * (t + 1)), gdef.max_steps, validate=False,
                            out=st["spare"], next_key=root.child(2 * (t + 1) + 1), next_actions=acts[(t + 1) % 2])
            st["spare"], st["cur"] = st["cur"], nxt
            st["t"] = t + 1

        for _ in range(8):
            one()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.graph(g, stream=side):
            for _ in range(n_steps):
                one()
        torch.cuda.synchronize()
        s, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e_.record()
        torch.cuda.synchronize()
        res[str(B)] = B * n_steps / (s.elapsed_time(e_) / 1e3)
        del g, st
    return {"env_steps_per_s": res, "steps": n_steps,
            "note": "steps 9..72 after init (early game), one CUDA-graph replay of the 64 step launches"}


def baseline_config1(args):
    """BASELINE configs[0]: go_9x9, 1024 envs, random play until every slot has finished once (379
    steps at seed 0). GPU: agents.rollout (one fused launch per step + the latch kernel). CPU: the
    pure-Python reference on the same envs, process-sharded over the host's cores."""
    import torch

    from paper_2303_17503_b200.agents import rollout

    rollout("go_9x9", 1024, args.seed)   # warm-up (allocations, module load)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = rollout("go_9x9", 1024, args.seed)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    out = {"workload": "go_9x9, 1024 envs, random play until every slot finished once",
           "gpu_seconds": gpu_s, "gpu_batch_steps": int(r.steps),
           "episode_steps_max": int(r.lengths.max())}
    if not args.no_cpu_baseline and not args.no_reference_cpu:
        ref = reference_python("go_9x9", args.seed, None, n_envs=1024, to_termination=True)
        out["reference_cpu"] = ref
    return out


# ------------------------------------------------------------ CPU arms
def cpu_run(game, n, seconds, threads):
    """Oracle port (C, OpenMP) driven through the reference's bench loop, with observations."""
    import oracle

    oracle.build()
    oracle.set_threads(threads)
    sess = oracle.Session(game, n, 0)
    for _ in range(3):
        c = sess.b.columns(with_obs=True)
        sess.step(sess.sample_random_actions(c))
    steps = 0
    t0 = time.perf_counter()
    while True:
        c = sess.b.columns(with_obs=True)
        sess.step(sess.sample_random_actions(c))
        steps += 1
        dt = time.perf_counter() - t0
        if dt >= seconds:
            break
    return n * steps / dt, steps, dt


def cpu_baseline(args, game, B, seconds):
    threads = os.cpu_count() or 1
    if game in SMALL:
        return {"value": None, "unit": "env-steps/s", "cores": threads, "kind": "port",
                "sample": "none: oracle/ has no restatement of the small engines (their parity is pinned to "
                          "reference goldens); see the go/chess/shogi/backgammon lines"}
    n = min(B, 512 if game in ("go_19x19", "chess", "shogi") else 4096)
    v, steps, dt = cpu_run(game, n, seconds, threads)
    return {"value": v, "unit": "env-steps/s", "cores": threads, "kind": "port",
            "sample": f"{game}: {n} envs x {steps} steps from init ({dt:.1f} s), oracle/orc_*.c (OpenMP, "
                      f"{threads} threads) + numpy random_actions, observations emitted"}


def _ref_worker(conn, ref_path, game, seed, lo, hi, steps, seconds, to_termination, barrier):
    """One process of the sharded pure-Python reference: slots [lo, hi) of a BatchSession batch, per
    slot exactly the reference's batch_step loop (core.py:372-386: reset with key.child(i) when
    finished, else step with key.child(i)) with the random policy (agents.py:25-46: random_agent with
    A_t.child(i)) and the observation of the current player (bench.batch_outputs, bench.py:86-97).
    Global slot indices, so the shards together are the batch (test_core.py:179-196)."""
    sys.path.insert(0, ref_path)
    import boardbatch as rb
    from boardbatch.agents import random_agent

    gdef = rb.core.resolve(game) if not game.startswith("go_19") else __import__(
        "boardbatch.games.go", fromlist=["make_game"]).make_game(19)
    R = rb.RngKey(seed)
    S0 = R.child(0)
    states = [rb.init(gdef, S0.child(i)) for i in range(lo, hi)]
    done = [False] * (hi - lo)
    t = 0

    def one():
        nonlocal t
        t += 1
        A, S = R.child(2 * t - 1), R.child(2 * t)
        for j, i in enumerate(range(lo, hi)):
            s = states[j]
            k = S.child(i)
            if s.terminated or s.truncated:
                states[j] = rb.init(gdef, k)
            else:
                states[j] = rb.step(s, random_agent(s, A.child(i)), k)
                if states[j].terminated or states[j].truncated:
                    done[j] = True
            ns = states[j]
            rb.observe(ns, ns.current_player)

    if not to_termination:
        one()   # warm-up step
    barrier.wait()
    t0 = time.perf_counter()
    n = 0
    while True:
        one()
        n += 1
        if to_termination:
            if all(done):
                break
        elif (steps and n >= steps) or (seconds and time.perf_counter() - t0 >= seconds):
            break
    conn.send((t0, time.perf_counter(), n, hi - lo, t))
    conn.close()


def reference_python(game, seed, seconds, n_envs=None, to_termination=False, procs=None):
    """The reference itself (pure Python, baseline/_ref, unmodified) on the host's cores, process-
    sharded by slot; bounded by `seconds` (every process runs for that long after a common start) or
    run to termination. Aggregate env-steps/s = slot-steps of all processes / (last end - first
    start)."""
    if not os.path.isdir(os.path.join(REF_PATH, "boardbatch")):
        return {"value": None, "unavailable": "reference not installed in baseline/_ref (tools/install_reference.sh)"}
    import multiprocessing as mp

    procs = procs or (os.cpu_count() or 1)
    n_envs = n_envs or {"go_9x9": 64, "go_19x19": 16, "backgammon": 256}[game] * procs
    procs = min(procs, n_envs)
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(procs)
    bounds = [round(k * n_envs / procs) for k in range(procs + 1)]
    pipes, ps = [], []
    for k in range(procs):
        a, b = ctx.Pipe(duplex=False)
        p = ctx.Process(target=_ref_worker, args=(b, REF_PATH, game, seed, bounds[k], bounds[k + 1], None,
                                                   seconds, to_termination, barrier))
        p.start()
        pipes.append(a)
        ps.append(p)
    res = [a.recv() for a in pipes]
    for p in ps:
        p.join()
    t0 = min(r[0] for r in res)
    t1 = max(r[1] for r in res)
    slot_steps = sum(r[2] * r[3] for r in res)
    wall = t1 - t0
    out = {"value": slot_steps / wall, "unit": "env-steps/s", "cores": procs, "kind": "reference",
           "impl": "pure-Python reference (baseline/_ref boardbatch, unmodified) via its public init/step/observe/"
                   "random_agent, process-sharded by slot with global slot keys",
           "envs": n_envs, "wall_seconds": wall, "steps_per_process": [r[2] for r in res][:4]}
    if to_termination:
        out["steps_to_all_finished"] = max(r[4] for r in res)
    else:
        out["sample"] = f"{n_envs} envs over {procs} processes, {seconds:.0f} s after one warm-up step, " \
                        "observations emitted"
    return out


def run_reference(args, rank, world):
    game = args.game
    if game in SMALL:
        return {"impl": "reference", "unavailable": f"{game}: no CPU restatement in oracle/ (pinned to reference goldens)"}
    B = args.batch or DEFAULT_BATCH[game]
    threads = os.cpu_count() or 1
    n = min(B, 512 if game in ("go_19x19", "chess", "shogi") else 4096)
    v, steps, dt = cpu_run(game, n, max(args.cpu_seconds, 5.0), threads)
    out = {
        "metric": METRIC, "value": v, "unit": "env-steps/s", "n_gpus": world, "steps": steps,
        "requested_steps": args.steps, "warmup": 3, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int (CPU)", "data": "synthetic random play, seed %d" % args.seed,
        "impl": "reference",
        "config": {"workload": f"{game} random play with legal_action_mask + observation", "game": game,
                   "batch_per_gpu": B, "cpu_envs": n},
        "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": threads, "kind": "port",
                         "sample": f"{n} envs x {steps} steps ({dt:.1f} s) after 3 warm-up steps, observations "
                                   "emitted. The reference is pure Python (no compilable C path), so its C "
                                   "restatement oracle/ (OpenMP) is the arm; the pure-Python reference itself is "
                                   "timed under reference_python"},
        "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if game in REFERENCE_GAMES and not args.no_reference_cpu:
        out["reference_python"] = reference_python(game, args.seed, max(args.cpu_seconds, 5.0))
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args, rank, world)), flush=True)
        return 0
    out = run_gpu(args, rank, world, local)
    if rank == 0:
        print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
