"""Kernel-shape sweep on given instances (records as comma lists): the
baseline's (U, D, min CTAs/SM) and the optimized variant's (U, group stages,
min CTAs/SM), L2 flushed, median of `reps`; every run digest-checked against
the automatic choice.
    python tools/tune_records.py OUT.json REPS REC [REC ...]"""
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402

out_path, reps = sys.argv[1], int(sys.argv[2])
recs = np.array([[int(x) for x in a.split(",")] for a in sys.argv[3:]], dtype=np.int32)
auto = L.measure_records(np.repeat(recs, reps, axis=0))
out = {}
for k, r in enumerate(recs):
    m = auto[k * reps:(k + 1) * reps]
    out[str(k)] = {"record": r.tolist(), "auto": {"base_ms": float(np.median(m["t_base_ms"])),
                                                  "opt_ms": float(np.median(m["t_opt_ms"])),
                                                  "kid": int(m["kernel_id"][0]), "G": int(m["nstages"][0])},
                   "base": [], "opt": []}
for U, D, mb in itertools.product((2, 4, 8, 16), (1, 3), (0, 4, 8)):
    res = L.measure_records(np.repeat(recs, reps, axis=0), tune=(U, D, mb, 0, 0, 0), skip_opt=True)
    for k in range(len(recs)):
        m = res[k * reps:(k + 1) * reps]
        ok = bool((m["digest_base"] == auto["digest_base"][k * reps]).all()) and bool((m["status"] == 0).all())
        out[str(k)]["base"].append({"U": U, "D": D, "minb": mb, "ms": float(np.median(m["t_base_ms"])), "ok": ok})
for U, G, mb in itertools.product((1, 2, 4, 8), (1, 2), (0, 4)):
    res = L.measure_records(np.repeat(recs, reps, axis=0), tune=(0, 0, 0, U, G, mb))
    for k in range(len(recs)):
        m = res[k * reps:(k + 1) * reps]
        ok = bool((m["digest_opt"] == auto["digest_base"][k * reps]).all()) and bool((m["status"] == 0).all())
        out[str(k)]["opt"].append({"U": U, "G": G, "minb": mb, "ms": float(np.median(m["t_opt_ms"])), "ok": ok})
for k, v in out.items():
    b = min(v["base"], key=lambda e: e["ms"] if e["ok"] else 1e9)
    o = min(v["opt"], key=lambda e: e["ms"] if e["ok"] else 1e9)
    print(k, v["record"][4:], "auto", v["auto"], "\n   best base", b, "\n   best opt", o, flush=True)
json.dump(out, open(out_path, "w"), indent=0)
