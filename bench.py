#!/usr/bin/env python
"""Random-play env-steps/s benchmark (BASELINE.json metric) on 1..8 B200s.

One "step" = one pass of the hot path over the whole batch: device random
actions (agents.random_actions, agents.py:33-46) + the batched env step with
auto-reset and fused observation emission (core.batch_step, core.py:353-386;
the reference's bench_run loop, bench.py:121-129) + the episode counter.

  python bench.py [--game go_19x19] [--batch 131072] [--steps K] [--warmup W]
  torchrun --nproc-per-node N bench.py --gpus N ...      (weak scaling: B per GPU)
  python bench.py --impl reference ...                    (CPU reference arm)

Rank 0 prints ONE JSON line. `value` = env-steps/s over all ranks with
inputs resident in HBM; `e2e` = the same metric through the public
batch_step API with host (pinned) action buffers and a per-step host read of
rewards/terminated/truncated/current_player; `roofline` = the step kernel's
algorithmic bytes per launch / its CUDA-event duration vs MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic bytes per env-step (restated in DESIGN.md §4):
# int64 action + float32 observation + bool mask + rewards/flags/player +
# compact state read/write. The superko history scan is excluded.
B_ALG = {"go_9x9": 5964, "go_19x19": 25860, "chess": 35502, "shogi": 41013, "backgammon": 400}
DEFAULT_BATCH = {"go_9x9": 1 << 17, "go_19x19": 1 << 17, "chess": 1 << 17, "shogi": 1 << 16, "backgammon": 1 << 17}
STEP_KERNEL = {"go_9x9": "go::step_kernel<9>", "go_19x19": "go::step_kernel<19>", "chess": "chess::step_kernel",
               "shogi": "shogi::step_kernel", "backgammon": "bg::step_kernel"}
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--game", default="go_19x19")
    ap.add_argument("--batch", type=int, default=0, help="envs per GPU (default per game, 2^17 for go_19x19)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="omit the batch-size sweep 2^10..2^17 from the line")
    ap.add_argument("--unfused", action="store_true", help="separate sampler / step / counter launches")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


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
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
def run_gpu(args, rank, world, local):
    import torch

    import paper_2303_17503_b200 as bb
    from paper_2303_17503_b200.core import resolve

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    game = args.game
    gdef = resolve(game)
    kern = gdef.batch_kernel
    B = args.batch or DEFAULT_BATCH[game]
    limit = gdef.max_steps
    root = bb.RngKey(args.seed)
    slot0 = rank * B   # global slot index: bit-identical to one big batch

    # ping-pong device states: only the previous batch stays valid in bench mode.
    # Fused loop (default): each step kernel also samples the NEXT step's random actions from
    # the new legal mask (agents.random_actions with the schedule's key) and counts finished
    # slots, so one step = one launch. --unfused runs sampler / step / counter as 3 launches.
    acts = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(2)]
    episodes = torch.zeros(1, dtype=torch.int64, device=dev)
    cur = kern.init(gdef, root.child(0), B, limit, slot0=slot0, device=dev,
                    next_key=None if args.unfused else root.child(1), next_actions=acts[0])
    spare = kern.new_v(B, slot0, dev, 0, limit)
    lib = __import__("paper_2303_17503_b200._native", fromlist=["lib"]).lib()
    stream = torch.cuda.current_stream(dev)
    t = 0

    def one_step(ev=None):
        nonlocal cur, spare, t
        a_now, a_next = acts[t % 2], acts[(t + 1) % 2]
        if args.unfused:
            kern.random_actions(cur, root.child(2 * t + 1), out=a_now)
        if ev is not None:
            ev[0].record(stream)
        if args.unfused:
            nxt = kern.step(gdef, cur, a_now, root.child(2 * (t + 1)), limit, validate=False, out=spare)
        else:
            nxt = kern.step(gdef, cur, a_now, root.child(2 * (t + 1)), limit, validate=False, out=spare,
                            next_key=root.child(2 * (t + 1) + 1), next_actions=a_next, episodes=episodes)
        if ev is not None:
            ev[1].record(stream)
        if args.unfused:
            lib.bbk_count_finished(nxt.dev.terminated.data_ptr(), nxt.dev.truncated.data_ptr(), B,
                                   episodes.data_ptr(), stream.cuda_stream)
        spare, cur = cur, nxt
        t += 1

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for k in range(args.steps):
        one_step(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    kern_ms = [a.elapsed_time(b) for a, b in evs]
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.all_reduce(episodes, op=dist.ReduceOp.SUM)
        dist.barrier()
    total_steps = B * world * args.steps
    value = total_steps / (ms / 1e3)
    avg_kern_ms = sum(kern_ms) / len(kern_ms)
    peak, peak_kind = peaks()
    achieved = B_ALG[game] * B / (avg_kern_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(game, B)
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "env-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64/int8 (integer board logic; float32 observation output)",
        "data": "synthetic: random-play rollouts from the reference key schedule (seed %d), auto-reset" % args.seed,
        "config": {"workload": f"{game} random play with legal_action_mask + observation", "game": game,
                   "batch_per_gpu": B, "global_batch": B * world, "max_steps": limit,
                   "parallelism": f"dp{world} (independent env slices, global slot keys)",
                   "l2": "per-step outputs exceed L2 (obs %.2f GB/step)" % (B * 4 * __import__("math").prod(
                       gdef.spec.observation_shape) / 1e9),
                   "timed": "K steps after W warm-up steps from init (step t of the BatchSession schedule)"},
        "clocks": clk,
        "gpu_launches": (3 if args.unfused else 1) * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_kind,
                     "kernel": STEP_KERNEL[game], "kernel_ms": avg_kern_ms,
                     "kernel_share_of_step": avg_kern_ms / (ms / args.steps),
                     "bytes_per_env_step": B_ALG[game]},
        "episodes_completed": int(episodes.item()),
    }
    if not args.no_e2e:
        out["e2e"] = run_e2e(args, gdef, kern, root, dev, world, slot0, B)
    if not args.no_sweep:
        out["sweep"] = run_sweep(args, gdef, kern, dev, slot0)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, game, B, args.cpu_seconds)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return out


def run_e2e(args, gdef, kern, root, dev, world, slot0, B):
    """Same metric through the public API with host buffers, over the same step window.

    A fresh batch (same seed, same slots) is stepped W untimed + K timed steps through
    core.batch_step. Per step: core.batch_step reads the host agent's actions from a pinned host
    buffer and its fused sampler writes the device random policy's next actions into the other
    pinned buffer (zero-copy over PCIe: the kernel loads / stores them itself; BBK_ZERO_COPY=0 uses
    an H2D copy and a D2H copy instead); the step's rewards / terminated / truncated /
    current_player go D2H on a copy stream into double-buffered pinned buffers, read on the host one
    step later (they overlap the next step; the last step's are waited for inside the timed region).
    """
    import torch

    from paper_2303_17503_b200.agents import random_actions_device
    from paper_2303_17503_b200.core import Batch, batch_step

    batch = Batch(gdef, B, gdef.max_steps, vstate=kern.init(gdef, root.child(0), B, gdef.max_steps, slot0=slot0,
                                                            device=dev, next_key=root.child(1)))
    # the host agent's action buffers (pinned, ping-pong): step t reads acts[t % 2] in place and its
    # fused sampler writes the next actions into acts[(t + 1) % 2] (zero-copy both ways)
    acts = [torch.empty(B, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    P = gdef.spec.num_players
    host = [dict(r=torch.empty((B, P), dtype=torch.float32, pin_memory=True),
                 term=torch.empty(B, dtype=torch.bool, pin_memory=True),
                 trunc=torch.empty(B, dtype=torch.bool, pin_memory=True),
                 cp=torch.empty(B, dtype=torch.int32, pin_memory=True)) for _ in range(2)]
    main = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    pending = []      # (batch whose results are in flight, copy-stream event, host buffer set)
    t = 0

    acts[0].copy_(random_actions_device(batch, root.child(1)))

    def read(entry):
        entry[1].synchronize()    # step t's rewards / flags / current player are now in host memory

    from paper_2303_17503_b200.games._device import ZERO_COPY

    def one():
        nonlocal batch, t
        nk = root.child(2 * (t + 1) + 1)
        batch = batch_step(batch, acts[t % 2], root.child(2 * (t + 1)), validate=False, next_key=nk,
                           next_actions=acts[(t + 1) % 2] if ZERO_COPY else None)
        if not ZERO_COPY:
            acts[(t + 1) % 2].copy_(random_actions_device(batch, nk), non_blocking=True)
        d = batch.device
        h = host[t % 2]
        done = torch.cuda.Event()
        done.record(main)
        copy.wait_event(done)
        with torch.cuda.stream(copy):
            h["r"].copy_(d.rewards, non_blocking=True)
            h["term"].copy_(d.terminated, non_blocking=True)
            h["trunc"].copy_(d.truncated, non_blocking=True)
            h["cp"].copy_(d.current_player, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        main.synchronize()        # the next actions are in host memory
        if pending:
            read(pending.pop())
        pending.append((batch, ev, h))
        t += 1

    def drain():
        while pending:
            read(pending.pop())

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

        tt = torch.tensor([dt], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    return {"value": B * world * args.steps / dt, "unit": "env-steps/s", "h2d_bytes_per_step": 8 * B,
            "d2h_bytes_per_step": (4 * P + 2 + 4 + 8) * B, "steps": args.steps,
            "path": "public core.batch_step: the step kernel reads the host agent's actions from pinned host "
                    "memory and writes the next actions there (zero-copy over PCIe; BBK_ZERO_COPY=0 copies "
                    "instead); rewards/flags/player D2H on a copy stream, read by the host one step later; "
                    "same window as value (fresh init, W warm-up, K timed)",
            "zero_copy": ZERO_COPY}


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


# ------------------------------------------------------------ CPU arms
def cpu_run(game, n, seconds, threads):
    """Oracle port (C, OpenMP) driven through the reference's bench loop, with observations."""
    import oracle

    oracle.build()
    oracle.set_threads(threads)
    sess = oracle.Session(game, n, 0)
    # warm-up a few steps, then time whole steps until `seconds` elapse
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
            "sample": f"{game}: {n} envs x {steps} steps from init ({dt:.1f} s), oracle/orc_*.c (OpenMP) + "
                      "numpy random_actions, observations emitted"}


def run_reference(args, rank, world):
    game = args.game
    if game in SMALL:
        return {"impl": "reference", "unavailable": f"{game}: no CPU restatement in oracle/ (pinned to reference goldens)"}
    B = args.batch or DEFAULT_BATCH[game]
    threads = os.cpu_count() or 1
    n = min(B, 512 if game in ("go_19x19", "chess", "shogi") else 4096)
    v, steps, dt = cpu_run(game, n, max(args.cpu_seconds, 5.0), threads)
    return {
        "metric": METRIC, "value": v, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int (CPU)", "data": "synthetic random play, seed %d" % args.seed,
        "impl": "reference",
        "config": {"workload": f"{game} random play with legal_action_mask + observation", "game": game,
                   "batch_per_gpu": B},
        "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": threads, "kind": "port",
                         "sample": f"{n} envs x {steps} steps ({dt:.1f} s); reference is pure Python "
                                   "(no compilable C path), so the C restatement oracle/ is timed"},
        "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


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
