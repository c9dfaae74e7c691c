"""DRAM traffic of one U-Net forward from an ncu --set full capture of tools/profile_unet.py
(all unet_tc launches + the per-step film/state kernels of one forward), written to
profiles/<round>_unet_traffic.json for bench.py's roofline.traffic (bytes per sampler call =
per-forward bytes x denoising steps).

    python tools/unet_traffic.py gpurun_out/prof_unet.ncu-rep profiles/r01_unet_traffic.json
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units, rows = r[0], r[1], r[2:]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ik = hdr.index("Kernel Name")
    cols = {k: hdr.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    per = []
    for row in rows:
        name = row[ik].split("(")[0].replace("void ", "")
        rd = float(row[cols["dram__bytes_read.sum"]].replace(",", "")) * scale[units[cols["dram__bytes_read.sum"]]]
        wr = float(row[cols["dram__bytes_write.sum"]].replace(",", "")) * scale[units[cols["dram__bytes_write.sum"]]]
        per.append({"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr})
    total = sum(p["dram_read_bytes"] + p["dram_write_bytes"] for p in per)
    res = {"source": rep, "launches": len(per), "dram_bytes_per_forward": total, "per_launch": per,
           "note": "ncu --set full, one forward at 1024 problems x 32 seeds, T=32 (tools/profile_unet.py)"}
    open(out, "w").write(json.dumps(res, indent=1))
    print(f"{len(per)} launches, {total / 1e9:.3f} GB DRAM per forward")


if __name__ == "__main__":
    main()
