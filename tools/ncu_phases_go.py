"""Aggregate ncu source-page samples / warp-instructions of go.cu by phase (line ranges)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
phases = [(int(a), int(b), n) for a, b, n in (x.split(":") for x in sys.argv[2].split(","))]
hdr = None; cur = None; curfile = None
S, I = collections.Counter(), collections.Counter()
num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r; continue
    if r and r[0].startswith("File"):
        curfile = r[0]; continue
    if hdr is None or len(r) < 10:
        continue
    if r[0].isdigit():
        cur = int(r[0]); continue
    if cur is None or not r[2].startswith("0x"):
        continue
    S[cur] += num(r[4]); I[cur] += num(r[7])
tot, ti = sum(S.values()), sum(I.values())
agg_s, agg_i = collections.Counter(), collections.Counter()
for ln in S:
    name = next((n for a, b, n in phases if a <= ln <= b), "other")
    agg_s[name] += S[ln]; agg_i[name] += I[ln]
for name, v in agg_s.most_common():
    print(f"{name:14s} samples {v / tot * 100:5.1f}%  inst {agg_i[name] / ti * 100:5.1f}%")
