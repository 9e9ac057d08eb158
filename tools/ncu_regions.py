"""Summarise an ncu --page source --csv dump: stall reasons per code region.
usage: python tools/ncu_regions.py src.csv [block]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 200
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = Counter()
for d in data:
    for r in reasons:
        tot[r] += I(d[r])
print("total", sum(tot.values()), tot.most_common(8))
for b in range(0, len(data), blk):
    seg = data[b:b + blk]
    c = Counter()
    for d in seg:
        for r in reasons:
            c[r] += I(d[r])
    s = sum(c.values())
    ins = sum(I(d["Instructions Executed"]) for d in seg)
    if s > 200:
        top = max(seg, key=lambda d: I(d["Warp Stall Sampling (All Samples)"]))
        print(f"{b:6d} samp={s:7d} instr={ins:9d} {[(k[6:], v) for k, v in c.most_common(3)]} | {top['Source'].strip()[:50]}")
