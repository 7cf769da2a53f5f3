"""Per-source-line stall samples / instructions / lane efficiency from an ncu source-page CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
hdr = None
agg, inst, thr, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 10:
        continue
    if r[0] in ("Line No", "Address", "# Address"):
        hdr = r
        continue
    if not r[0].isdigit():
        continue
    k = (cur_file, int(r[0]))
    src[k] = r[1].strip()
    num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
    agg[k] += num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    inst[k] += num(r[hdr.index("Instructions Executed")])
    thr[k] += num(r[hdr.index("Thread Instructions Executed")])
tot, ti = sum(agg.values()), sum(inst.values())
print(f"samples {tot}  warp-instructions {ti}  lane-eff {sum(thr.values()) / max(ti, 1):.1f}")
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {100 * inst[k] / ti:5.1f}%i eff{thr[k] / max(inst[k], 1):5.1f} {k[0]}:{k[1]:<4d} {src[k][:80]}")
