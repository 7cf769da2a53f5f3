"""Summarise `ncu --set full` captures of the step kernels into profiles/<round>/ncu_traffic.json.

usage: python tools/ncu_traffic.py <out.json> <game>=<file.ncu-rep>:<batch>:<note> ...
Reads the raw page of each report (one captured launch) and records DRAM bytes per launch and per
env-step, issue activity, occupancy and instruction counts; bench.py reads dram_bytes_per_env_step
for its roofline `traffic` field.
"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import B_ALG  # noqa: E402

METRICS = {
    "gpu__time_duration.sum": "kernel",
    "dram__bytes_read.sum": "rd",
    "dram__bytes_write.sum": "wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_per_sm",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "lanes_per_inst",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "inst",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k, name in METRICS.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            out[name] = v * SCALE.get(units[i], 1.0)
    return out


def main():
    dst = sys.argv[1]
    res = {}
    for spec in sys.argv[2:]:
        game, rest = spec.split("=", 1)
        rep, batch, note = rest.split(":", 2)
        B = int(batch)
        m = raw(rep)
        dram = m["rd"] + m["wr"]
        res[game] = {
            "batch": B,
            "kernel_s": m["kernel"],
            "dram_bytes_per_launch": dram,
            "dram_bytes_per_env_step": dram / B,
            "b_alg": B_ALG[game],
            "traffic_over_alg": dram / B / B_ALG[game],
            "dram_pct_peak": m.get("dram_pct_peak"),
            "issue_active_pct": m.get("issue_active_pct"),
            "warps_per_sm": m.get("warps_per_sm"),
            "lanes_per_inst": m.get("lanes_per_inst"),
            "regs": m.get("regs"),
            "warp_inst_per_env_step": m["inst"] / B,
            "captured": note,
        }
    with open(dst, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
