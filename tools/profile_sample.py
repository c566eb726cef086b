"""Measure a random sample of sweep instances one batch at a time and save
per-instance times + descriptors (gpurun_out/profile_sample.npz)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1412_6986_b200 as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 240.0
_, table, perm = bench.workload(0)
rows = perm[1000:1000 + n]
rec = table.records(rows)
out = []
t0 = time.time()
for k in range(0, n, 8):
    out.append(L.measure_records(rec[k:k + 8]))
    if time.time() - t0 > budget:
        rec = rec[: k + 8]
        break
res = np.concatenate(out)
np.savez(os.path.join(ROOT, "gpurun_out", "profile_sample.npz"), rec=rec[: len(res)], res=res)
print("measured", len(res), "in", time.time() - t0)
