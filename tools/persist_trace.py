"""Critical path of the persistent small-batch sampler from a PS_PERSIST_TRACE dump.
Run:  PS_NO_GRAPH=1 PS_PERSIST=1 PS_PERSIST_TRACE=gpurun_out/trace.bin python tools/persist_trace.py --run P S
Read: python tools/persist_trace.py gpurun_out/trace.bin [step]
Per layer (one step): units, layer span (last publish - previous layer's last publish),
and medians / maxima of: wait (counter seen - previous last publish), A load (first chunk
landed - counter seen), MMA (accumulator ready - first chunk), epilogue (publish - ready),
and the pipeline-0 MMA warp's issue loop (last commit - first chunk)."""
import sys
import numpy as np


def load(path):
    with open(path, "rb") as f:
        grid, cap, nl, ns = np.frombuffer(f.read(16), np.int32)
        units = np.frombuffer(f.read(4 * nl), np.int32)
        tr = np.frombuffer(f.read(), np.uint64).reshape(grid, cap, 20).astype(np.int64)
    return grid, cap, nl, ns, units, tr


def main():
    if sys.argv[1] == "--run":
        import os
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import torch
        from paper_2410_16727_b200 import spec, synth
        from paper_2410_16727_b200.sampler import SeedSampler
        P, S = int(sys.argv[2]), int(sys.argv[3])
        s1 = SeedSampler(spec.random_model(), mode=1)
        rng = np.random.default_rng(0)
        cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
        q0 = synth.make_problems(P, seed=3).q_start
        fa = s1.film(cond)
        for _ in range(2):
            s1.sample(fa, q0, S)
        torch.cuda.synchronize()
        return
    grid, cap, nl, ns, units, tr = load(sys.argv[1])
    step = int(sys.argv[2]) if len(sys.argv) > 2 else ns // 2
    # rebuild each CTA's unit sequence
    rec = {}   # (step, layer) -> list of stamps
    for c in range(grid):
        j = 0
        for s in range(ns):
            for l in range(nl):
                for u in range(c, units[l], grid):
                    rec.setdefault((s, l), []).append(tr[c, j])
                    j += 1
    prev_last = None
    tot = 0
    print(f"grid {grid}, {nl} layers, step {step}")
    print("layer units  span_us  wait_med wait_max  A_med  A_max  mma_med mma_max  epi_med epi_max  issue_loop_us")
    if step > 0:
        prev_last = max(r[3] for r in rec[(step - 1, nl - 1)])
    t_start = prev_last
    for l in range(nl):
        r = np.array(rec[(step, l)])
        last = r[:, 3].max()
        w = (r[:, 0] - prev_last) / 1e3 if prev_last is not None else np.zeros(len(r))
        a_ = (r[:, 1] - r[:, 0]) / 1e3
        m = (r[:, 2] - r[:, 1]) / 1e3
        e = (r[:, 3] - r[:, 2]) / 1e3
        span = (last - prev_last) / 1e3 if prev_last is not None else float("nan")
        print(f"{l:5d} {units[l]:5d} {span:8.2f} {np.median(w):8.2f} {w.max():8.2f} {np.median(a_):6.2f} {a_.max():6.2f}"
              f" {np.median(m):7.2f} {m.max():7.2f} {np.median(e):7.2f} {e.max():7.2f}  {np.median(r[:, 11] - r[:, 1]) / 1e3:7.2f}")
        prev_last = last
    if t_start is not None:
        print(f"step total {(prev_last - t_start) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
