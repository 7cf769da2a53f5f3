"""Small-batch probe: eager (host-launched) step loop vs the same 64-step window replayed as a CUDA graph.

Per game and batch 2^10..2^17: W=8 eager steps from init, then steps 9..72 timed with CUDA events
(a) launched from Python one by one (bench.py's sweep) and (b) captured once into a CUDA graph on a
fresh batch at the same point of the schedule and replayed (no host launch overhead).
"""

import json
import sys

import torch

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.core import resolve


def window(game, B, graph):
    gdef = resolve(game)
    kern = gdef.batch_kernel
    root = bb.RngKey(0)
    dev = torch.device("cuda", 0)
    acts = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(2)]
    cur = kern.init(gdef, root.child(0), B, gdef.max_steps, device=dev, next_key=root.child(1), next_actions=acts[0])
    spare = kern.new_v(B, 0, dev, 0, gdef.max_steps)
    st = {"cur": cur, "spare": spare, "t": 0}

    def one():
        t = st["t"]
        nxt = kern.step(gdef, st["cur"], acts[t % 2], root.child(2 * (t + 1)), gdef.max_steps, validate=False,
                        out=st["spare"], next_key=root.child(2 * (t + 1) + 1), next_actions=acts[(t + 1) % 2])
        st["spare"], st["cur"] = st["cur"], nxt
        st["t"] = t + 1

    for _ in range(8):
        one()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=side):
            for _ in range(64):
                one()
        torch.cuda.synchronize()
        s.record()
        g.replay()
        e.record()
    else:
        s.record()
        for _ in range(64):
            one()
        e.record()
    torch.cuda.synchronize()
    return B * 64 / (s.elapsed_time(e) / 1e3)


def main():
    games = sys.argv[1:] or ["go_19x19", "chess", "shogi"]
    for g in games:
        res = {}
        for ex in range(10, 18):
            if g == "shogi" and ex > 16:
                continue
            B = 1 << ex
            res[B] = (window(g, B, False) / 1e6, window(g, B, True) / 1e6)
        print(json.dumps({"game": g, "eager_vs_graph_Msteps": res}))


if __name__ == "__main__":
    main()
