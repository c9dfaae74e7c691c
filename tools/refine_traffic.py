"""DRAM traffic per launch of the refinement (and ESDF build) kernels from an ncu --set full capture
of the bench step, written to profiles/<round>_refine_traffic.json for bench.py's
roofline_refine.traffic.   python tools/refine_traffic.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units, rows = r[0], r[1], r[2:]
    ik = hdr.index("Kernel Name")
    c = {k: hdr.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                                   "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct")}
    per = {}
    for row in rows:
        name = row[ik].split("(")[0].replace("void ", "")
        v = lambda k: float(row[c[k]].replace(",", "")) * SCALE.get(units[c[k]], 1.0)
        per.setdefault(name, {"dram_read_bytes": v("dram__bytes_read.sum"), "dram_write_bytes": v("dram__bytes_write.sum"),
                              "us": v("gpu__time_duration.sum") / (1e3 if units[c["gpu__time_duration.sum"]] == "nsecond" else 1),
                              "l2_hit_pct": v("lts__t_sector_hit_rate.pct"), "l1_hit_pct": v("l1tex__t_sector_hit_rate.pct")})
    ref = [k for k in per if "bl_refine" in k]
    res = {"source": rep, "note": "ncu --set full of one bench step (1024 problems x 32 seeds, bricked ESDFs, "
                                  "diffusion seeds); per-launch DRAM bytes", "kernels": per}
    if ref:
        d = per[ref[0]]
        res["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
    open(out, "w").write(json.dumps(res, indent=1))
    print(json.dumps({k: round((v["dram_read_bytes"] + v["dram_write_bytes"]) / 1e9, 3) for k, v in per.items()}))


if __name__ == "__main__":
    main()
