"""The paper's experiment on B200 labels: from a run_sweep output directory,
train the random forest on a seeded 10 % of the rows and evaluate the
held-out 90 % (count-based and penalty-weighted accuracy),
once with the reference's modelled labels and once with the speedups measured
on the B200. Prints one JSON object.

    python tools/measured_study.py DIR
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402


def main(d):
    lab = np.load(os.path.join(d, "labels.npz"))
    rows = L.read_rows(os.path.join(d, "dataset.csv"))
    X = np.stack([r.features.to_array() for r in rows])
    model = np.array([r.speedup for r in rows])
    # measured labels in dataset row order (labels.npz is sorted by row, as is the csv)
    meas = lab["measured_speedup"][: len(rows)]
    assert len(meas) == len(rows)
    tr, he = L.dataset.split_indices(len(rows), 0.10, 0)
    out = {"rows": len(rows), "train": int(len(tr)), "held_out": int(len(he)),
           "measured_beneficial_frac": float((meas > 1.0).mean()),
           "model_beneficial_frac": float((model > 1.0).mean()),
           "model_vs_measured_decision_agreement": float(((model > 1.0) == (meas > 1.0)).mean())}
    for name, y in (("modelled_labels", model), ("measured_labels", meas)):
        f = L.train_arrays(X[tr], np.array([L.speedup_to_target(v) for v in y[tr]]),
                           L.Hyperparams(num_trees=20, features_per_node=4, seed=0), L.FEATURE_NAMES, threads=8)
        pred = L.predict(f, X[he])
        rep = L.evaluate(pred > 1.0, y[he])
        out[name] = {"count_accuracy": rep.count_accuracy, "penalty_weighted_accuracy": rep.penalty_weighted_accuracy,
                     "min_score": rep.min_score, "confusion": [rep.true_optimize, rep.false_optimize, rep.true_leave,
                                                               rep.false_leave]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
