"""Host-side cost per public step call (µs), with a batch small enough that the GPU is never the
bottleneck: batch_step alone, and batch_step + the e2e loop's result copies on a copy stream.

usage (GPU box): python tools/host_cost.py [game] [B] [K]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2303_17503_b200 as bb  # noqa: E402
from paper_2303_17503_b200.core import Batch, batch_step, resolve  # noqa: E402


def main():
    game = sys.argv[1] if len(sys.argv) > 1 else "backgammon"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
    gdef = resolve(game)
    kern = gdef.batch_kernel
    root = bb.RngKey(0)
    dev = torch.device("cuda", 0)
    acts = [torch.empty(B, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    batch = Batch(gdef, B, gdef.max_steps, vstate=kern.init(gdef, root.child(0), B, gdef.max_steps, device=dev,
                                                            next_key=root.child(1), next_actions=acts[0]))
    torch.cuda.synchronize()

    def loop(n, copies):
        nonlocal batch
        P = gdef.spec.num_players
        h = dict(r=torch.empty((B, P), dtype=torch.float32, pin_memory=True),
                 term=torch.empty(B, dtype=torch.bool, pin_memory=True),
                 trunc=torch.empty(B, dtype=torch.bool, pin_memory=True),
                 cp=torch.empty(B, dtype=torch.int32, pin_memory=True))
        main_s = torch.cuda.current_stream(dev)
        copy = torch.cuda.Stream(dev)
        t0 = time.perf_counter()
        for t in range(n):
            batch = batch_step(batch, acts[t % 2], root.child(2 * (t + 1)), validate=False,
                               next_key=root.child(2 * (t + 1) + 1), next_actions=acts[(t + 1) % 2])
            if copies:
                d = batch.device
                done = torch.cuda.Event()
                done.record(main_s)
                copy.wait_event(done)
                with torch.cuda.stream(copy):
                    h["r"].copy_(d.rewards, non_blocking=True)
                    h["term"].copy_(d.terminated, non_blocking=True)
                    h["trunc"].copy_(d.truncated, non_blocking=True)
                    h["cp"].copy_(d.current_player, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        return (t1 - t0) / n * 1e6

    loop(50, False)
    a = loop(K, False)
    b = loop(K, True)
    print(f"{game} B={B}: batch_step host {a:.1f} us/call; + result copies {b:.1f} us/step")


if __name__ == "__main__":
    main()
