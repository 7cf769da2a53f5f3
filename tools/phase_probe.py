"""Split a Go step's time: full fused step vs the same step without the observation stream vs the
observation stream alone (bbk_go_observe over the same batch). Tells whether the logic and the
emission overlap across warps (full ~ max) or add up (full ~ sum).

usage (GPU box): python tools/phase_probe.py [game] [B] [warmup] [K]
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
    # same trajectory position, outputs without the observation column
    kern, lib = loop.kern, loop.lib
    noobs = [kern.new_v(B, 0, dev, 0, loop.limit, False) for _ in range(2)]
    loop.spare = noobs[0]
    for _ in range(2):   # the ping-pong pair becomes observation-free
        loop.step()
    ms_noobs, _ = loop.timed(K)
    size = kern.size
    obs = torch.empty((B,) + tuple(kern.obs_shape), dtype=torch.float32, device=dev)
    v = loop.cur
    st = loop.stream.cuda_stream
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        lib.bbk_go_observe(size, v.priv.pat.data_ptr(), v.priv.role_to_move.data_ptr(), obs.data_ptr(), B, st)
    torch.cuda.synchronize()
    start.record(loop.stream)
    for _ in range(K):
        lib.bbk_go_observe(size, v.priv.pat.data_ptr(), v.priv.role_to_move.data_ptr(), obs.data_ptr(), B, st)
    end.record(loop.stream)
    torch.cuda.synchronize()
    ms_obs = start.elapsed_time(end)
    start.record(loop.stream)
    for _ in range(K):
        obs.fill_(1.0)
    end.record(loop.stream)
    torch.cuda.synchronize()
    ms_fill = start.elapsed_time(end)
    print(json.dumps({"game": game, "B": B, "full_ms": ms_full / K, "no_obs_ms": ms_noobs / K,
                      "observe_only_ms": ms_obs / K, "fill_same_bytes_ms": ms_fill / K,
                      "observe_gbs": obs.numel() * 4 / (ms_obs / K) / 1e6, "fill_gbs": obs.numel() * 4 / (ms_fill / K) / 1e6}))


if __name__ == "__main__":
    main()
