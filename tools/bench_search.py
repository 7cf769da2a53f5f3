"""Throughput of the batched UCT search (search.py) on one GPU, and of the reference's scalar
mcts_agent on this host's CPU for comparison (build container only: --reference).

    python tools/bench_search.py [--configs go_9x9:1024:32,connect_four:4096:64] [--reference]

Device lines: searches/s (whole batch of searches, each `sims` simulations, divided by the
CUDA-event time of the whole search), simulations/s and batched env-steps/s of the expansion and
rollout steps. Reference line: the same search on the reference, one state at a time.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def roots(game, n, seed=0, t=8):
    import paper_2303_17503_b200 as bb

    sess = bb.BatchSession(game, n, seed)
    for _ in range(t):
        sess.step(sess.sample_random_actions())
    return sess.batch


def device(game, n, sims, reps=3):
    import torch

    import paper_2303_17503_b200 as bb
    from paper_2303_17503_b200 import search

    batch = roots(game, n)
    v = batch._v
    fin = (v.dev.terminated | v.dev.truncated).cpu().numpy()
    rows = [i for i in range(n) if not fin[i]]
    keys = [bb.RngKey(7).child(i).state for i in rows]
    pool = search.SearchPool(v.kern, v, len(rows), sims)
    search.search(v, rows, keys, sims, pool=pool)   # warm-up
    best = None
    for _ in range(reps):
        st = {}
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        search.search(v, rows, keys, sims, pool=pool, stats=st)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        if best is None or sec < best[0]:
            best = (sec, st)
    sec, st = best
    steps = (st["expand_steps"] + st["rollout_steps"]) * len(rows)
    return {"impl": "device", "game": game, "searches": len(rows), "sims": sims, "seconds": round(sec, 4),
            "searches_per_s": round(len(rows) / sec, 1), "simulations_per_s": round(len(rows) * sims / sec, 1),
            "batched_steps": st["expand_steps"] + st["rollout_steps"], "env_steps_per_s": round(steps / sec, 1)}


def reference(game, n, sims, budget_s=20.0):
    sys.path.insert(0, "/root/reference/pkg/src")
    import boardbatch as rb
    from boardbatch.agents import mcts_agent
    from boardbatch.bench import BatchSession

    gdef = game
    if game == "go_19x19":
        from boardbatch.games import go
        gdef = go.make_game(19)
    sess = BatchSession(gdef, n, 0)
    for _ in range(8):
        sess.step(sess.sample_random_actions())
    states = [s for s in sess.batch.states if not (s.terminated or s.truncated)]
    t0 = time.perf_counter()
    done = 0
    for i, s in enumerate(states):
        mcts_agent(s, rb.RngKey(7).child(i), sims)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    sec = time.perf_counter() - t0
    return {"impl": "reference", "game": game, "searches": done, "sims": sims, "seconds": round(sec, 2),
            "searches_per_s": round(done / sec, 3), "simulations_per_s": round(done * sims / sec, 1), "cores": 1,
            "host": "build container CPU (the reference is not on the GPU box)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="go_9x9:1024:32,go_19x19:256:16,connect_four:4096:64,othello:2048:32,"
                                          "hex:2048:32,tic_tac_toe:8192:64")
    ap.add_argument("--reference", action="store_true")
    a = ap.parse_args()
    for spec in a.configs.split(","):
        game, n, sims = spec.split(":")
        fn = reference if a.reference else device
        print(json.dumps(fn(game, int(n), int(sims))), flush=True)


if __name__ == "__main__":
    main()
