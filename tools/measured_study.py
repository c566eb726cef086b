"""The paper's experiment on B200 labels from a finished run_sweep output
directory (the same computation as `run_sweep --study`, one process):
train the random forest on a seeded 10 % of the rows and evaluate the
held-out 90 % (count-based and penalty-weighted accuracy),
once with the reference's modelled labels and once with the speedups measured
on the B200. Writes DIR/study.json and prints it.

    python tools/measured_study.py DIR [--max-instances N] [--seed S]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("dir")
    ap.add_argument("--max-instances", type=int, default=None)
    ap.add_argument("--seed", type=int, default=None)
    a = ap.parse_args(argv)
    summ = {}
    if os.path.exists(os.path.join(a.dir, "summary.json")):
        summ = json.load(open(os.path.join(a.dir, "summary.json")))
    max_inst = a.max_instances or summ.get("max_instances", 1_000_000)
    seed = a.seed if a.seed is not None else summ.get("seed", 0)
    lab = np.load(os.path.join(a.dir, "labels.npz"))
    labels = np.stack([lab["row"].astype(np.float64), lab["t_base_ms"], lab["t_opt_ms"], lab["mismatches"],
                       lab["status"]], 1)
    table = L.select_instance_table(L.SamplingSpec(max_instances=max_inst, seed=seed))
    L.study.run_rank(a.dir, table, labels, labels[:, 0].astype(np.int64), 0, seed, threads=os.cpu_count() or 1)
    print(json.dumps(L.study.merge(a.dir, table, labels, 1, seed), indent=1))


if __name__ == "__main__":
    main()
