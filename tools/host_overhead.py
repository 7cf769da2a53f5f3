"""cProfile of the public step path (batch_step with a pinned host action buffer), per game."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cProfile
import pstats
import time

import torch

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.agents import random_actions_device

B = int(os.environ.get("B", 1 << 17))
for g in (sys.argv[1:] or ["go_19x19", "chess"]):
    sess = bb.BatchSession(g, B, 0, validate=False)
    b = sess.batch
    host = torch.empty(B, dtype=torch.int64, pin_memory=True)
    root = bb.RngKey(0)
    for t in range(20):
        host.copy_(random_actions_device(b, root.child(2 * t + 1)))
        b = bb.batch_step(b, host, root.child(2 * (t + 1)), validate=False, next_key=root.child(2 * (t + 1) + 1))
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for t in range(20, 120):
        host.copy_(random_actions_device(b, root.child(2 * t + 1)))
        b = bb.batch_step(b, host, root.child(2 * (t + 1)), validate=False, next_key=root.child(2 * (t + 1) + 1))
    pr.disable()
    torch.cuda.synchronize()
    print(g, "per step us", (time.perf_counter() - t0) / 100 * 1e6)
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
