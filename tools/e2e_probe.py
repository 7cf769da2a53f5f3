"""Breakdown of the e2e step (bench.py run_e2e) at the default batch: where the gap to the device
step time goes (host Python in batch_step, H2D, kernel, D2H, sync)."""

import json
import sys
import time

import torch

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.agents import random_actions_device
from paper_2303_17503_b200.core import Batch, batch_step, resolve


def main(game="go_19x19", B=1 << 17, W=16, K=128):
    gdef = resolve(game)
    kern = gdef.batch_kernel
    root = bb.RngKey(0)
    dev = torch.device("cuda", 0)
    batch = Batch(gdef, B, gdef.max_steps, vstate=kern.init(gdef, root.child(0), B, gdef.max_steps, device=dev,
                                                            next_key=root.child(1)))
    P = gdef.spec.num_players
    host_act = torch.empty(B, dtype=torch.int64, pin_memory=True)
    host_r = torch.empty((B, P), dtype=torch.float32, pin_memory=True)
    host_term = torch.empty(B, dtype=torch.bool, pin_memory=True)
    host_trunc = torch.empty(B, dtype=torch.bool, pin_memory=True)
    host_cp = torch.empty(B, dtype=torch.int32, pin_memory=True)
    host_act.copy_(random_actions_device(batch, root.child(1)))
    st = {"t": 0, "py": 0.0, "py2": 0.0}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    acc = [0.0, 0.0, 0.0]

    def one(timed):
        t = st["t"]
        s = torch.cuda.current_stream()
        if timed:
            ev[0].record(s)
        p0 = time.perf_counter()
        nb = batch_step(st["b"], host_act, root.child(2 * (t + 1)), validate=False, next_key=root.child(2 * (t + 1) + 1))
        p1 = time.perf_counter()
        if timed:
            ev[1].record(s)
        d = nb.device
        host_r.copy_(d.rewards, non_blocking=True)
        host_term.copy_(d.terminated, non_blocking=True)
        host_trunc.copy_(d.truncated, non_blocking=True)
        host_cp.copy_(d.current_player, non_blocking=True)
        host_act.copy_(random_actions_device(nb, root.child(2 * (t + 1) + 1)), non_blocking=True)
        p2 = time.perf_counter()
        if timed:
            ev[2].record(s)
        s.synchronize()
        if timed:
            acc[0] += ev[0].elapsed_time(ev[1])
            acc[1] += ev[1].elapsed_time(ev[2])
            st["py"] += p1 - p0
            st["py2"] += p2 - p1
        st["b"] = nb
        st["t"] = t + 1

    st["b"] = batch
    for _ in range(W):
        one(False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        one(False)
    wall = (time.perf_counter() - t0) / K
    for _ in range(K):
        one(True)
    print(json.dumps({"game": game, "B": B, "e2e_ms_per_step": wall * 1e3,
                      "events_h2d+kernel_ms": acc[0] / K, "events_d2h_ms": acc[1] / K,
                      "py_batch_step_ms": st["py"] / K * 1e3, "py_copies_ms": st["py2"] / K * 1e3}))


if __name__ == "__main__":
    for g in (sys.argv[1:] or ["go_19x19", "chess"]):
        main(g, B=(1 << 16) if g == "shogi" else (1 << 17))
