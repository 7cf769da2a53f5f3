"""Copy a tools/gpu_measure.sh pass from gpurun_out/ into profiles/<round>/ and (re)write the
bench / ncu numbers at the top of profiles/<round>/SUMMARY.md (the hand-written history below the
marker line is kept).

usage: python tools/summarize.py r01
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
MARK = "<!-- history -->"
GAMES = [("go19", "go_19x19", "go_19x19 (default window)", 131072, "-s 250"),
         ("chess", "chess", "chess", 131072, "-s 100"),
         ("shogi", "shogi", "shogi (B=2^16)", 65536, "-s 100"),
         ("backgammon", "backgammon", "backgammon", 131072, "-s 100"),
         ("go_9x9", "go_9x9", "go_9x9", 131072, "-s 60")]


def line(path):
    with open(path) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def main():
    rnd = sys.argv[1]
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    specs = []
    # a pass run with NCU=0 keeps the previous captures (kernels unchanged since)
    have_ncu = all(os.path.exists(os.path.join(OUT, f"ncu_{g}.ncu-rep")) for _, g, *_ in GAMES)
    for short, game, _, B, s in GAMES if have_ncu else []:
        rep = os.path.join(OUT, f"ncu_{game}.ncu-rep")
        specs.append(f"{game}={rep}:{B}:ncu --set full --clock-control none -k regex:step_kernel {s} -c 1 (mid-episode launch)")
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(dst, f"ncu_raw_{game}.csv"), "w") as fh:
            fh.write(raw)
    if have_ncu:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_traffic.py"),
                        os.path.join(dst, "ncu_traffic.json")] + specs, check=True, capture_output=True)
    for short, *_ in GAMES + [("reference",)]:
        shutil.copy(os.path.join(OUT, f"bench_{short}.json"), os.path.join(dst, f"bench_{short}.json"))
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(dst, "go19_launches.csv"))
    t = json.load(open(os.path.join(dst, "ncu_traffic.json")))
    rows = []
    for short, key, name, B, _ in GAMES:
        d = line(os.path.join(dst, f"bench_{short}.json"))
        v = t[key]
        rows.append(f"| {name} | {d['value'] / 1e6:.1f} M | {d['ms_per_step']:.3f} | {d['roofline']['frac']:.3f} | "
                    f"{d['e2e']['value'] / 1e6:.1f} M | {v['dram_bytes_per_env_step']:,.0f} | {v['b_alg']:,} | "
                    f"{v['issue_active_pct']:.0f} % | {v['warp_inst_per_env_step']:,.0f} |")
    go = line(os.path.join(dst, "bench_go19.json"))
    for name, w in go.get("windows", {}).items():
        rows.insert(1, f"| go_19x19 window `{name}` (W={w['warmup']}, K={w['steps']}) | {w['value'] / 1e6:.1f} M | "
                       f"{w['ms_per_step']:.3f} | {w['roofline_frac']:.3f} | | | | | |")
    ref = line(os.path.join(dst, "bench_reference.json"))
    sweeps = []
    for short, key, *_ in GAMES[:3]:
        sw = line(os.path.join(dst, f"bench_{short}.json"))["sweep"]["env_steps_per_s"]
        sweeps.append(f"| {key} | " + " | ".join(f"{sw[str(1 << e)] / 1e6:.1f} M" if str(1 << e) in sw else "-"
                                                 for e in range(10, 18)) + " |")
    head = f"""# {rnd} measurement pass (tools/gpu_measure.sh on one B200; tools/summarize.py)

`python bench.py` defaults: B = 2^17 per GPU (shogi 2^16), W = 8, K = 128 (the per-game lines of
tools/gpu_measure.sh: K = 256), fused step kernel (one launch per step incl. next-step random actions and the episode
counter), SM clock {go['clocks']['sm_mhz']:.0f} MHz (max {go['clocks']['sm_max_mhz']:.0f}), throttle reasons {go['clocks']['reasons']}.
Roofline = B_alg x B / step-kernel CUDA-event time vs the measured {go['roofline']['peak']} GB/s copy peak
(MEASURED_PEAKS.json).

| game | env-steps/s | step ms | kernel frac of HBM roofline | e2e (host actions + host read) | DRAM B / env-step (ncu) | B_alg | issue active | warp-inst / env-step |
|---|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + """

Batch sweep (env-steps/s, steps 9..72 after init as one CUDA-graph replay, part of every default bench line):

| B | 2^10 | 2^11 | 2^12 | 2^13 | 2^14 | 2^15 | 2^16 | 2^17 |
|---|---|---|---|---|---|---|---|---|
""" + "\n".join(sweeps) + f"""

CPU baseline on the same box ({go['cpu_baseline']['cores']} host cores, oracle/ C port with OpenMP, observations emitted):
go_19x19 {go['cpu_baseline']['value'] / 1e3:.0f} k env-steps/s; `--impl reference` arm {ref['value'] / 1e3:.0f} k env-steps/s.

ncu (`ncu_raw_*.csv`, `ncu_traffic.json`): one mid-episode launch per game, `--set full --clock-control
none`; `go19_launches.csv` is the launch list of a short default bench (`--metrics
gpu__time_duration.sum`): the step kernel is the only kernel in the timed loop.

"""
    small = []
    for g in ("tic_tac_toe", "connect_four", "othello", "hex", "2048", "kuhn_poker", "leduc_holdem"):
        src = os.path.join(OUT, f"bench_{g}.json")
        if os.path.exists(src):
            shutil.copy(src, os.path.join(dst, f"bench_{g}.json"))
        src = os.path.join(dst, f"bench_{g}.json")   # a pass run with SMALL=0 keeps the previous lines
        if os.path.exists(src):
            d = line(src)
            small.append(f"| {g} | {d['value'] / 1e6:,.1f} M | {d['roofline']['frac']:.3f} | "
                         f"{d['e2e']['value'] / 1e6:,.1f} M | {d['roofline']['bytes_per_env_step']:,} |")
    if small:
        head += """The reference's small engines (SURVEY §8f rank 4; thread per slot, B = 2^17, parity pinned to
reference goldens, no CPU oracle):

| game | env-steps/s | kernel frac of HBM roofline | e2e | B_alg |
|---|---|---|---|---|
""" + "\n".join(small) + "\n\n"
    path = os.path.join(dst, "SUMMARY.md")
    tail = ""
    if os.path.exists(path):
        old = open(path).read()
        if MARK in old:
            tail = old[old.index(MARK):]
    open(path, "w").write(head + (tail or MARK + "\n"))
    print(head)


if __name__ == "__main__":
    main()
