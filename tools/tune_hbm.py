"""Kernel-shape sweep on the HBM-leg instances (bench.hbm_records): each
(U, D, min CTAs/SM) of the baseline and (U, group stages, min CTAs/SM) of the
optimized variant, L2 flushed before each variant, median of `reps` runs;
every run is digest-checked against the automatic choice.

    python tools/tune_hbm.py [reps]
"""
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402
from bench import hbm_records  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
recs = hbm_records()
out = {}
auto = L.measure_records(np.repeat(recs, reps, axis=0))
for k, r in enumerate(recs):
    m = auto[k * reps:(k + 1) * reps]
    out[str(k)] = {"record": r.tolist(), "auto": {"base_ms": float(np.median(m["t_base_ms"])),
                                                  "opt_ms": float(np.median(m["t_opt_ms"])), "kid": int(m["kernel_id"][0]),
                                                  "S": int(m["nstages"][0])}, "base": [], "opt": []}
for U, D, mb in itertools.product((1, 2, 4, 8), (1, 2, 3), (2, 3, 4, 6, 8)):
    res = L.measure_records(np.repeat(recs, reps, axis=0), tune=(U, D, mb, 0, 0, 0), skip_opt=True)
    for k in range(len(recs)):
        m = res[k * reps:(k + 1) * reps]
        ok = bool((m["digest_base"] == auto["digest_base"][k * reps]).all()) and bool((m["status"] == 0).all())
        out[str(k)]["base"].append({"U": U, "D": D, "minb": mb, "ms": float(np.median(m["t_base_ms"])), "ok": ok})
for U, S, mb in itertools.product((1, 2, 4, 8), (1, 2, 3, 4), (0, 2, 4, 8)):
    res = L.measure_records(np.repeat(recs, reps, axis=0), tune=(0, 0, 0, U, S, mb))
    for k in range(len(recs)):
        m = res[k * reps:(k + 1) * reps]
        ok = bool((m["digest_opt"] == auto["digest_base"][k * reps]).all()) and bool((m["status"] == 0).all())
        out[str(k)]["opt"].append({"U": U, "S": S, "minb": mb, "ms": float(np.median(m["t_opt_ms"])), "ok": ok})
for k, v in out.items():
    b = min(v["base"], key=lambda e: e["ms"] if e["ok"] else 1e9)
    o = min(v["opt"], key=lambda e: e["ms"] if e["ok"] else 1e9)
    print(k, v["record"][15:], "auto", v["auto"], "best base", b, "best opt", o, flush=True)
    print("   bad:", [e for e in v["base"] + v["opt"] if not e["ok"]][:4])
json.dump(out, open(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/tune_hbm.json", "w"), indent=0)
