"""Sampler time for P problems x 32 seeds in one call vs n_split concurrent calls on separate streams
(each with its own workspace); results must be identical (shard invariance)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import spec, synth  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 128
params = spec.random_model()
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
q0 = torch.as_tensor(synth.make_problems(P, seed=1).q_start).cuda()
res = {}
ref = None
for n_split in (1, 2, 4):
    smps = [SeedSampler(params, mode=1) for _ in range(n_split)]
    streams = [torch.cuda.Stream() for _ in range(n_split)]
    m = P // n_split
    fas = [smps[i].film(cond[i * m:(i + 1) * m]) for i in range(n_split)]
    outs = [torch.empty((m * 32, 32, 7), device="cuda") for _ in range(n_split)]

    def run():
        cur = torch.cuda.current_stream()
        for i in range(n_split):
            streams[i].wait_stream(cur)
            with torch.cuda.stream(streams[i]):
                smps[i].sample(fas[i], q0[i * m:(i + 1) * m], 32, p0=i * m, out=outs[i])
        for i in range(n_split):
            cur.wait_stream(streams[i])

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run()
    e1.record()
    torch.cuda.synchronize()
    full = torch.cat(outs).cpu().numpy()
    if ref is None:
        ref = full
    res[n_split] = {"ms": e0.elapsed_time(e1) / 3, "identical": bool(np.array_equal(full, ref))}
    del smps
    torch.cuda.empty_cache()
print(json.dumps({"P": P, **{str(k): v for k, v in res.items()}}))
