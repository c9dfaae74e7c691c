"""Memory-side summary of an ncu --set full report (refinement / ESDF kernels): duration,
DRAM bytes and GB/s, L2 (LTS) bytes and GB/s, L1 / L2 hit rates, against the B200 peaks in
MEASURED_PEAKS.json.   python tools/ncu_memory.py report.ncu-rep [out.csv]"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

M = {
    "us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "l2_sectors": "lts__t_sectors.sum",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit%": "lts__t_sector_hit_rate.pct",
    "l1_hit%": "l1tex__t_sector_hit_rate.pct",
    "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-3, "ns": 1e-3,
         "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = r[0], r[1], r[2:]
    root = Path(__file__).resolve().parents[1]
    try:
        peaks = json.loads((root / "MEASURED_PEAKS.json").read_text())
        hbm = peaks.get("hbm_gbs") or 7700.0
    except Exception:
        hbm = 7700.0
    lines = ["kernel,us,dram_rd_GB,dram_wr_GB,dram_GBps,dram_frac_of_measured_peak,l2_GB,l2_GBps,l2_throughput%,l2_hit%,l1_hit%,issue%"]
    for row in rows:
        v = {}
        for k, m in M.items():
            if m not in hdr:
                v[k] = float("nan")
                continue
            i = hdr.index(m)
            x = float(row[i].replace(",", "")) if row[i] not in ("", "n/a") else float("nan")
            v[k] = x * SCALE.get(units[i], 1)
        us = v["us"]
        gb = lambda b: b / 1e9
        dram = (v["dram_rd"] + v["dram_wr"]) / (us * 1e-6) / 1e9
        l2b = v["l2_sectors"] * 32
        l2 = l2b / (us * 1e-6) / 1e9
        name = row[hdr.index("Kernel Name")].split("(")[0].replace(",", ";")
        lines.append(f"{name},{us:.1f},{gb(v['dram_rd']):.3f},{gb(v['dram_wr']):.3f},{dram:.0f},{dram / hbm:.3f},"
                     f"{gb(l2b):.3f},{l2:.0f},{v['l2_pct']:.1f},{v['l2_hit%']:.1f},{v['l1_hit%']:.1f},{v['issue%']:.1f}")
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(text)
    print(text, end="")


if __name__ == "__main__":
    main()
