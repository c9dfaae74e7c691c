"""Per-launch table from ncu --csv --metrics logs: python tools/attr_table.py A.csv [B.csv]
(time in us, instructions per SM; B: the same workload under another PS_TC_DBG)."""
import csv
import sys


def load(fn):
    lines = open(fn).read().splitlines()
    s = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[s:]))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    d = {}
    for r in rows[1:]:
        if len(r) <= ix["Metric Value"]:
            continue
        k = int(r[ix["ID"]])
        d.setdefault(k, {"name": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = r[ix["Metric Value"]].replace(",", "")
    return d


a = load(sys.argv[1])
b = load(sys.argv[2]) if len(sys.argv) > 2 else None
tot = [0.0, 0.0]
for k in sorted(a):
    n = a[k]["name"]
    n = n[n.find("<"):n.find(">") + 1]
    t0 = float(a[k]["gpu__time_duration.sum"]) / 1e3
    t1 = float(b[k]["gpu__time_duration.sum"]) / 1e3 if b else 0.0
    ins = float(a[k].get("sm__inst_executed.sum", 0)) / 148 / 1e3
    tot[0] += t0
    tot[1] += t1
    print(f"{k:3d} {n:28s} {t0:8.1f} {t1:8.1f}  inst/SM {ins:8.1f}k")
print(f"total {tot[0]:.1f} {tot[1]:.1f}")
