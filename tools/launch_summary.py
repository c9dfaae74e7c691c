"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of `bench.py
--steps 1 --warmup W`: per-kernel device time over the LAST step (the timed one), found as
the launches from the last esdf build to its select, and each kernel's share of that step.

    python tools/launch_summary.py gpurun_out/launches.csv [out.csv]
"""
import csv
import re
import sys
from collections import OrderedDict


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.reader(lines):
        if r[0] == "ID" or len(r) < 15:
            continue
        rows.append((int(r[0]), r[4], float(r[-1])))
    return rows


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("ps::", "")


def main():
    rows = load(sys.argv[1])
    starts = [i for i, (_, n, _) in enumerate(rows) if short(n).startswith("esdf_")]
    # ... up to its select launch (bench.py's post-run seed check samples again after the step)
    ends = [i for i, (_, n, _) in enumerate(rows) if i >= starts[-1] and short(n).startswith("select_kernel")]
    step = rows[starts[-1]:(ends[-1] + 1 if ends else len(rows))]
    tot = sum(t for _, _, t in step)
    agg = OrderedDict()
    for _, n, t in step:
        k = short(n)
        c, s = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, s + t)
    out = [f"# last timed step: {len(step)} launches, {tot / 1e6:.2f} ms summed device time (ncu serialised, cold)"]
    out.append("kernel,launches,total_ms,share")
    for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k},{c},{s / 1e6:.3f},{s / tot:.4f}")
    text = "\n".join(out)
    print(text)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")


if __name__ == "__main__":
    main()
