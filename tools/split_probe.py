"""Would a split step pay? Go step without the observation stream on the main stream, pipelined
with the previous step's observation emission (bbk_go_observe) on a side stream, vs the fused step.

usage (GPU box): python tools/split_probe.py [game] [B] [W] [K]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    game = sys.argv[1] if len(sys.argv) > 1 else "go_19x19"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
    W = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    K = int(sys.argv[4]) if len(sys.argv) > 4 else 64
    dev = torch.device("cuda:0")
    loop = bench.DeviceLoop(game, B, 0, dev, 0)
    for _ in range(W):
        loop.step()
    ms_full, _ = loop.timed(K)
    kern, lib = loop.kern, loop.lib
    loop.spare = kern.new_v(B, 0, dev, 0, loop.limit, False)
    for _ in range(2):
        loop.step()
    obs = [torch.empty((B,) + tuple(kern.obs_shape), dtype=torch.float32, device=dev) for _ in range(2)]
    side = torch.cuda.Stream(dev)
    main = loop.stream
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(main)
    for k in range(K):
        loop.step()                       # step t (no observation) on the main stream
        v = loop.cur
        done = torch.cuda.Event()
        done.record(main)
        side.wait_event(done)             # observation of step t on the side stream, overlapping step t+1
        lib.bbk_go_observe(kern.size, v.priv.pat.data_ptr(), v.priv.role_to_move.data_ptr(), obs[k % 2].data_ptr(), B,
                           side.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(side)
        main.wait_event(ev) if k % 2 == 1 else None   # the observation buffers are double-buffered
    main.wait_stream(side)
    end.record(main)
    torch.cuda.synchronize()
    ms_split = start.elapsed_time(end)
    print(json.dumps({"game": game, "B": B, "fused_ms": ms_full / K, "split_ms": ms_split / K}))


if __name__ == "__main__":
    main()
