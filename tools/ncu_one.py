"""Run one instance (fill, K1, K2, digest) -- a short target for ncu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402

for arg in sys.argv[1:]:
    rec = np.array([[int(x) for x in arg.split(",")]], dtype=np.int32)
    r = L.measure_records(rec)
    print(arg, "t_base", r["t_base_ms"][0], "t_opt", r["t_opt_ms"][0], "mism", r["mismatches"][0],
          "kid", r["kernel_id"][0], "S", r["nstages"][0], flush=True)
