"""Per-CUDA-line executed warp instructions and stall samples of one kernel in an ncu report
(`--import-source on`): python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, timeout=600).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr = None, None
data, samp, src = defaultdict(float), defaultdict(float), {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ix, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ix or not (r[0] and r[0].isdigit()):
        continue
    k = (cur, int(r[0]))
    src[k] = r[1]
    num = lambda x: float(x) if x.replace(".", "").isdigit() else 0.0
    data[k] += num(r[ix])
    samp[k] += num(r[isamp])
tot, ts = sum(data.values()), sum(samp.values())
print(f"warp instructions {tot:.0f}, stall samples {ts:.0f}")
for k in sorted(data, key=lambda k: -data[k])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{k[0][:12]:12s}:{k[1]:5d} {data[k] / tot:6.2%} {samp[k] / max(ts, 1):6.2%}  {src[k].strip()[:96]}")
