"""Per-CUDA-line stall samples (total and by reason), warp-instructions and lane efficiency.

Input: `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` output.
usage: ncu_srclines.py file.csv [top] [reason ...]   (reason e.g. stall_no_inst stall_short_sb)
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
reasons = sys.argv[3:] or ["stall_no_inst", "stall_short_sb", "stall_wait", "stall_long_sb", "stall_mio"]
hdr = None
cur = None
S, I, T = collections.Counter(), collections.Counter(), collections.Counter()
R = {r: collections.Counter() for r in reasons}
src = {}
num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 10:
        continue
    if r[0].isdigit():
        cur = int(r[0])
        src[cur] = r[1].strip()[:90]
        continue
    if cur is None or not r[2].startswith("0x"):
        continue
    S[cur] += num(r[4])
    I[cur] += num(r[7])
    T[cur] += num(r[8])
    for k in reasons:
        R[k][cur] += num(r[hdr.index(k)])
tot, ti = sum(S.values()), sum(I.values())
print(f"samples {tot} warp-inst {ti} " + " ".join(f"{k}={sum(R[k].values()) / max(tot, 1) * 100:.1f}%" for k in reasons))
print(f"{'line':>5} {'samp%':>6} {'inst%':>6} {'lanes':>5} " + " ".join(f"{k[6:]:>8}" for k in reasons))
for ln, v in S.most_common(top):
    print(f"{ln:5d} {v / tot * 100:6.2f} {I[ln] / ti * 100:6.2f} {T[ln] / max(I[ln], 1):5.1f} "
          + " ".join(f"{R[k][ln] / tot * 100:8.2f}" for k in reasons) + "  " + src.get(ln, ""))
