"""Summarise a measured-sweep directory pulled back from the GPU box
(run.json, verify.json, study.json, labels.npz) into one JSON.
    python tools/dla_summary.py gpurun_out/r02_dla100k profiles/r02_dla100k_summary.json"""
import json
import os
import sys

import numpy as np

d = sys.argv[1]
run = json.loads(open(os.path.join(d, "run.json")).read().strip().splitlines()[-1])
ver = json.load(open(os.path.join(d, "verify.json")))
study = json.load(open(os.path.join(d, "study.json"))) if os.path.exists(os.path.join(d, "study.json")) else None
lab = np.load(os.path.join(d, "labels.npz"))
sp = lab["measured_speedup"]
ok = lab["t_base_ms"] > 0
feas = lab["t_opt_ms"] > 0
out = {
    "workload": "BASELINE configs[2]: dense-linear-algebra family (xy_reuse, x_reuse_row/col, y_reuse_row/col) of "
                "SamplingSpec(max_instances=1_000_000, seed=0), seeded random sample, both variants per instance, "
                "1 B200, launches of <= 74 CTAs in SM partitions (green contexts), whole-device launches L2-flushed",
    "instances": int(run["rows"]), "measure_s": run["measure_s"], "prepare_s": run["prepare_s"],
    "instances_per_s": run.get("instances_per_s"),
    "verified_bitwise_k1_eq_k2": run["verified"], "k1_k2_mismatched": run["mismatched"],
    "optimized_infeasible": int((ok & ~feas).sum()), "failed": int((~ok).sum()),
    "oracle_check": {k: ver[k] for k in ("instances", "mismatched", "cells", "seconds")},
    "measured_speedup": {"beneficial_frac": float((sp[feas] > 1).mean()), "min": float(sp[feas].min()),
                         "p10": float(np.percentile(sp[feas], 10)), "median": float(np.median(sp[feas])),
                         "p90": float(np.percentile(sp[feas], 90)), "max": float(sp[feas].max())},
    "kernel_time_s": {"baseline": float(lab["t_base_ms"][ok].sum() / 1e3),
                      "optimized": float(lab["t_opt_ms"][feas].sum() / 1e3)},
}
if study:
    out["rf_study"] = study
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
