"""SASS instruction histogram of the in-tree library, per kernel family, with the Blackwell-specific
opcodes that prove the tcgen05 / TMA / CTA-pair paths (UTCHMMA, UTCBAR, LDTM, UTMALDG, UTMASTG,
FFMA2 ...).  python tools/sass_hist.py [lib] > profiles/<round>_sass_hist.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

lib = sys.argv[1] if len(sys.argv) > 1 else str(Path(__file__).resolve().parents[1] / "paper_2410_16727_b200/_build/libps_b200.so")
out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fam = None
hist = collections.defaultdict(collections.Counter)
for ln in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        name = m.group(1)
        for key in ("unet_tc_kernel", "unet_persist_kernel", "conv_tc_kernel", "bl_refine_kernel", "esdf_cull_kernel",
                    "select_kernel", "enc_", "ref_", "guide_kernel", "metrics_kernel", "optimize_kernel", "cost_kernel"):
            if key in name:
                fam = key.rstrip("_")
                break
        else:
            fam = "other"
        hist[fam]["#functions"] += 1
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
    if m and fam:
        op = m.group(2)
        hist[fam][op.split(".")[0]] += 1
        if op.startswith(("UTC", "UTMA", "LDTM", "STTM", "UBLKCP", "UTMACCTL")):
            hist[fam][op] += 1
KEY = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAPF", "FFMA2", "FADD2", "FMUL2", "MUFU", "SYNCS",
       "ELECT", "LDG", "STG", "LDS", "STS", "SHFL", "FFMA", "BAR"]
print(f"# cuobjdump -sass {Path(lib).name}: opcode counts per kernel family (static instructions)")
for f, c in sorted(hist.items()):
    print(f"\n[{f}] functions={c['#functions']} total={sum(v for k, v in c.items() if not k.startswith('#') and '.' not in k)}")
    print("  key: " + ", ".join(f"{k}={c[k]}" for k in KEY if c[k]))
    detail = sorted(((k, v) for k, v in c.items() if "." in k), key=lambda kv: -kv[1])
    if detail:
        print("  tcgen05/TMA forms: " + ", ".join(f"{k}={v}" for k, v in detail[:16]))
    top = [(k, v) for k, v in c.most_common() if not k.startswith("#") and "." not in k][:14]
    print("  top: " + ", ".join(f"{k}={v}" for k, v in top))
