"""Compare two dump_sample.py npz files bit for bit."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
ok = True
for k in a.files:
    same = np.array_equal(a[k], b[k])
    d = np.abs(a[k].astype(np.float64) - b[k]).max()
    print(f"{k}: {'bitwise equal' if same else 'DIFFERENT'} (max |d| {d:.3e})")
    ok &= same
sys.exit(0 if ok else 1)
