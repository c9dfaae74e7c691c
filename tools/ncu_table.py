"""Per-launch table from an ncu --set full report: time, DRAM bytes, tensor-pipe and issue
utilisation.   python tools/ncu_table.py gpurun_out/prof_unet.ncu-rep [out.csv]"""
import csv
import io
import subprocess
import sys

COLS = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tc_hmma%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tc%"),
        ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uni%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("lts__t_bytes.sum", "l2_bytes"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs")]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = r[0], r[1], r[2:]
    have = [(c, n) for c, n in COLS if c in hdr]
    tc_cols = [h for h in hdr if "pipe_tensor" in h and "pct" in h]
    lines = [",".join(n for _, n in have)]
    for row in rows:
        vals = []
        for c, n in have:
            v = row[hdr.index(c)]
            u = units[hdr.index(c)]
            if n == "kernel":
                v = v.split("(")[0].replace("void ", "").replace("ps::", "").replace(",", ";")
            elif u in ("Mbyte", "Gbyte", "Kbyte", "byte"):
                mult = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u]
                v = f"{float(v.replace(',', '')) * mult:.1f}MB"
            elif u == "ms":
                v = f"{float(v) * 1e3:.1f}"
            vals.append(v)
        lines.append(",".join(vals))
    text = "\n".join(lines)
    print(text)
    print("# tensor-pipe metric columns available:", tc_cols[:8], file=sys.stderr)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")


if __name__ == "__main__":
    main()
