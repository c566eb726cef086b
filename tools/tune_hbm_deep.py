"""Deeper rings than tools/tune_hbm.py tried: K2 group stages S up to 16,
K1 prefetch depth D up to 6, on the full-chip HBM legs (bench.hbm_records
1..3), L2 flushed before each variant, median of `reps`; every run
digest-checked against the automatic choice.   python tools/tune_hbm_deep.py [reps] [out.json]"""
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402
from bench import hbm_records  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
recs = hbm_records()[1:]
rep = np.repeat(recs, reps, axis=0)
auto = L.measure_records(rep)
out = {"records": recs.tolist(), "auto": [], "opt": [], "base": []}
for k in range(len(recs)):
    m = auto[k * reps:(k + 1) * reps]
    out["auto"].append({"base_ms": float(np.median(m["t_base_ms"])), "opt_ms": float(np.median(m["t_opt_ms"])),
                        "S": int(m["nstages"][0])})
for U, S, mb in itertools.product((1, 2, 4), (4, 6, 8, 12, 16), (0, 2, 4)):
    try:
        res = L.measure_records(rep, tune=(0, 0, 0, U, S, mb))
    except Exception as e:  # a shape that does not fit
        out["opt"].append({"U": U, "S": S, "minb": mb, "err": str(e)[:80]})
        continue
    for k in range(len(recs)):
        m = res[k * reps:(k + 1) * reps]
        ok = bool((m["digest_opt"] == auto["digest_base"][k * reps]).all()) and bool((m["status"] == 0).all())
        out["opt"].append({"leg": k, "U": U, "S": S, "minb": mb, "ms": float(np.median(m["t_opt_ms"])), "ok": ok,
                           "S_used": int(m["nstages"][0])})
for U, D, mb in itertools.product((2, 4, 8), (2, 3, 4, 6), (4, 6, 8)):
    try:
        res = L.measure_records(rep, tune=(U, D, mb, 0, 0, 0), skip_opt=True)
    except Exception as e:
        out["base"].append({"U": U, "D": D, "minb": mb, "err": str(e)[:80]})
        continue
    for k in range(len(recs)):
        m = res[k * reps:(k + 1) * reps]
        ok = bool((m["digest_base"] == auto["digest_base"][k * reps]).all()) and bool((m["status"] == 0).all())
        out["base"].append({"leg": k, "U": U, "D": D, "minb": mb, "ms": float(np.median(m["t_base_ms"])), "ok": ok})
for k in range(len(recs)):
    bo = sorted([e for e in out["opt"] if e.get("leg") == k and e["ok"]], key=lambda e: e["ms"])[:3]
    bb = sorted([e for e in out["base"] if e.get("leg") == k and e["ok"]], key=lambda e: e["ms"])[:3]
    print(k, "auto", out["auto"][k], "\n   best opt", bo, "\n   best base", bb, flush=True)
json.dump(out, open(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/tune_hbm_deep.json", "w"), indent=0)
