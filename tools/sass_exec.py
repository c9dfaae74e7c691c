"""Summarise an `ncu --page source --csv --print-source sass` dump: executed warp instructions
by opcode and the hottest basic-block ranges (python tools/sass_exec.py dump.csv [top])."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) > ix and r[ix].replace('.', '').isdigit()]
tot = sum(float(r[ix]) for r in body)
samp = sum(float(r[isamp] or 0) for r in body)
by_op = Counter()
for r in body:
    op = r[1].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    by_op[o.split(".")[0]] += float(r[ix])
print(f"total warp instructions {tot:.0f}, stall samples {samp:.0f}")
for o, n in by_op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{o:12s} {n:12.0f} {n / tot:6.1%}")
