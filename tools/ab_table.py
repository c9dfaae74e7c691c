import sys
sys.path.insert(0, 'tools')
from launch_summary import load, short
a = load('gpurun_out/fwd_launches.csv')[-31:]
b = load('gpurun_out/fwd_launches_b.csv')[-31:]
for (_, n, t), (_, _, t2) in zip(a, b):
    print(f"{short(n):36s} {t/1e3:7.1f} {t2/1e3:7.1f}")
print("sum", sum(r[2] for r in a) / 1e3, sum(r[2] for r in b) / 1e3)
