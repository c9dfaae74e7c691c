"""Stall-reason breakdown by SASS region of one kernel in an ncu report (source page).
    python tools/ncu_stalls.py REPORT LAUNCH_INDEX [region_size]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
step = int(sys.argv[3]) if len(sys.argv) > 3 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx), "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][1][:90])
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
# the page can repeat the listing; keep the first copy
n = len(data)
for k in range(1, n // 2 + 1):
    if n % k == 0 and data[:k] == data[k:2 * k]:
        data = data[:k]
        break
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = [hdr.index(h) for h in names]
isrc = hdr.index("Source")
tot = [0] * len(ci)
print("region  samples  " + " ".join(h.replace("stall_", "")[:9] for h in names))
for a in range(0, len(data), step):
    blk = data[a:a + step]
    v = [sum(int(r[c] or 0) for r in blk) for c in ci]
    tot = [x + y for x, y in zip(tot, v)]
    if sum(v) > 0.01 * 1:
        print(f"{a:5d} {sum(v):7d}  " + " ".join(f"{x:9d}" for x in v) + "  " + blk[0][isrc].strip()[:40])
print("total", sum(tot), dict((h.replace('stall_', ''), x) for h, x in zip(names, tot) if x))
