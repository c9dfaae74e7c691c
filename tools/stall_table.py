"""Per-launch warp-stall breakdown (share of samples by reason) for every kernel in an ncu
--set full report with source counters.   python tools/stall_table.py REPORT [n_launches]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 31
names = ["wait", "long_sb", "short_sb", "mio", "barrier", "math", "not_selected", "selected", "branch_resolving",
         "sleep", "no_inst", "dispatch", "lg", "membar", "tex", "drain", "misc"]
print("launch,kernel,samples," + ",".join(names))
for i in range(n):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(i), "--launch-count", "1",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        break
    kname = rows[0][1][:60].replace(",", ";") if rows[0] and len(rows[0]) > 1 else "?"
    hdr = rows[1]
    data = [r for r in rows[2:] if r and r[0].startswith("0x")]
    m = len(data)
    for k in range(1, m // 2 + 1):
        if m % k == 0 and data[:k] == data[k:2 * k]:
            data = data[:k]
            break
    tot = {}
    for nm in names:
        col = "stall_" + nm
        cands = [h for h in hdr if h.lower().startswith(col) and "Not Issued" not in h]
        if not cands:
            continue
        c = hdr.index(cands[0])
        tot[nm] = sum(int(r[c] or 0) for r in data)
    s = sum(tot.values()) or 1
    print(f"{i},{kname},{s}," + ",".join(f"{tot.get(nm, 0) / s:.3f}" for nm in names), flush=True)
