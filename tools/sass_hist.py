"""Summarise an ncu source page (--page source --csv --print-source sass): runs of SASS with equal
execution counts, their share of issued instructions and of stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
h = rows[1]
ia, isrc, ie, iss = (h.index(k) for k in ["Address", "Source", "Instructions Executed",
                                           "Warp Stall Sampling (All Samples)"])
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[ia], 16), r[isrc].strip(), int(r[ie]), int(r[iss])))
    except ValueError:
        pass
tot = sum(d[2] for d in data)
tots = sum(d[3] for d in data) or 1
print(f"total warp-instructions {tot/1e9:.3f} G, stall samples {tots}")
segs, cur = [], None
for a, s, n, ss in data:
    if cur and cur[2] == n:
        cur[1] = a; cur[3] += 1; cur[4] += ss
    else:
        if cur:
            segs.append(cur)
        cur = [a, a, n, 1, ss, s]
segs.append(cur)
base = data[0][0]
for s0, s1, n, cnt, ss, src in segs:
    if n * cnt > tot * thr or ss > tots * 0.02:
        print(f"{s0-base:6x}-{s1-base:6x} {n/1e6:9.2f}M x {cnt:4d} = {100*n*cnt/tot:5.2f}%  stall {100*ss/tots:5.2f}%  {src[:48]}")
