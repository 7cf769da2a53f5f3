"""Write-only HBM bandwidth probe (the store-dominated side of every step kernel's traffic).

Times torch fill_ (a pure float4 store stream) and copy_ (read + write) over buffers larger than
L2 with CUDA events, best of 10. Used to read the step kernels' roofline fraction against the
write-only ceiling as well as the copy peak in MEASURED_PEAKS.json.
"""

import json

import torch


def best(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) / 1e3)
    return min(out)


def main():
    res = {}
    for gb in (1, 4):
        n = gb * (1 << 30) // 4
        x = torch.empty(n, dtype=torch.float32, device="cuda")
        y = torch.empty_like(x)
        t = best(lambda: x.fill_(1.0))
        res[f"fill_{gb}GiB_GBs"] = 4 * n / t / 1e9
        t = best(lambda: y.copy_(x))
        res[f"copy_{gb}GiB_GBs"] = 8 * n / t / 1e9
        del x, y
    print(json.dumps(res))


if __name__ == "__main__":
    main()
