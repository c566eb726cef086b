"""Concurrent (SM-partition) vs isolated per-instance times on a sweep sample.

The measurement contract lets launches of <= 74 CTAs run several at a time
in disjoint SM partitions (LMT_MEASURE_CONCURRENT). This checks that each
such instance's time matches its isolated time (alone on the chip, L2
flushed before each variant) -- the condition for the labels to be the
same. Writes a JSON summary.

    python tools/conc_validate.py N OUT.json
"""
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/conc_validate.json"
tab = L.select_instance_table(L.SamplingSpec(max_instances=1_000_000, seed=0))
rng = np.random.default_rng(2024)
rows = np.sort(rng.choice(len(tab), size=n * 3, replace=False))
rec = tab.records(rows)
ctas = (rec[:, 15] // rec[:, 17]) * (rec[:, 16] // rec[:, 18])
cost = L.sweep.launch_cost(rec)
sel = (ctas <= 74) & (cost < 0.6)
rec = rec[sel][:n]
L.prepare_records(rec, concurrent=True)
t0 = time.perf_counter()
iso = L.measure_records(rec)
t_iso = time.perf_counter() - t0
t0 = time.perf_counter()
con = L.measure_records(rec, concurrent=True)
t_con = time.perf_counter() - t0
t0 = time.perf_counter()
iso2 = L.measure_records(rec)
t_iso2 = time.perf_counter() - t0
summary = {"instances": int(len(rec)), "wall_isolated_s": t_iso, "wall_concurrent_s": t_con,
           "wall_isolated_repeat_s": t_iso2, "speedup_wall": t_iso / t_con,
           "in_partitions": int((con["lane_sms"] > 0).sum()), "partitions": L._lib.partitions()}
for col in ("t_base_ms", "t_opt_ms"):
    ok = (iso[col] > 0) & (con[col] > 0)
    r = con[col][ok] / iso[col][ok]
    r2 = iso2[col][ok] / iso[col][ok]  # isolated run-to-run noise, for scale
    big = iso[col][ok] >= 1.0
    summary[col] = {
        "n": int(ok.sum()), "ratio_median": float(np.median(r)), "ratio_p05": float(np.percentile(r, 5)),
        "ratio_p95": float(np.percentile(r, 95)), "within_3pct": float((np.abs(r - 1) <= 0.03).mean()),
        "within_3pct_ge_1ms": float((np.abs(r[big] - 1) <= 0.03).mean()) if big.any() else None,
        "time_weighted_ratio": float(con[col][ok].sum() / iso[col][ok].sum()),
        "iso_repeat_ratio_median": float(np.median(r2)),
        "iso_repeat_within_3pct": float((np.abs(r2 - 1) <= 0.03).mean()),
    }
lab_i = iso["t_base_ms"] / np.where(iso["t_opt_ms"] > 0, iso["t_opt_ms"], np.nan)
lab_c = con["t_base_ms"] / np.where(con["t_opt_ms"] > 0, con["t_opt_ms"], np.nan)
okl = np.isfinite(lab_i) & np.isfinite(lab_c)
summary["label_agreement"] = float(((lab_i[okl] > 1) == (lab_c[okl] > 1)).mean())
summary["digests_equal"] = bool((iso["digest_base"] == con["digest_base"]).all())
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
json.dump(summary, open(out, "w"), indent=1)
np.savez(out.replace(".json", ".npz"), rec=rec, iso=iso, con=con, iso2=iso2)
print(json.dumps(summary, indent=1))
