"""Stall samples / instructions aggregated over named line ranges of one source file (ncu source CSV)."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
fname = sys.argv[2]
ranges = [(n, int(a), int(b)) for n, a, b in (x.split(":") for x in sys.argv[3:])]
cur, hdr = None, None
agg, inst, tot_s, tot_i = collections.Counter(), collections.Counter(), 0, 0
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]; continue
    if len(r) < 10: continue
    if r[0] in ("Line No", "Address", "# Address"): hdr = r; continue
    if not r[0].isdigit(): continue
    num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
    s = num(r[hdr.index("Warp Stall Sampling (All Samples)")]); i = num(r[hdr.index("Instructions Executed")])
    if hdr[0] != "Line No": continue
    tot_s += s; tot_i += i
    name = "other:" + cur
    if cur == fname:
        ln = int(r[0])
        name = next((n for n, a, b in ranges if a <= ln <= b), "other:" + fname)
    agg[name] += s; inst[name] += i
for k, v in agg.most_common():
    print(f"{k:24s} samples {100 * v / tot_s:5.1f}%  inst {100 * inst[k] / tot_i:5.1f}%")
