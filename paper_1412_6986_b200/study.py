"""The paper's experiment on a measured sweep (SURVEY 8(e)
"after the gather"): train the random forest on a seeded 10 % of the
instances and score its decisions on the other 90 % (count-based and
penalty-weighted accuracy, metrics.evaluate), once on the reference's
modelled labels and once on the speedups measured on the B200.

Distributed form (run_sweep --study): after the label all-gather every rank
holds all labels; each rank featurises the study set (K4, deterministic),
draws the same split (dataset.split_indices) and trains the same forests
(native trainer, bit-identical to forest.train and independent of the thread
count), so no model is broadcast. Each rank then predicts (K3) only the
held-out rows it measured and writes them to DIR/rankRRR/study_pred.npz;
rank 0 merges the files in row order and evaluates. The result is the same
for any number of ranks.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np

HP = dict(num_trees=20, features_per_node=4)
STUDY_FRACTION = 0.10


def study_set(table, labels: np.ndarray):
    """Rows of a gathered label matrix (run_sweep: row, t_base_ms, t_opt_ms,
    mismatches, status) that enter the study: measured without failure (the
    optimized variant may be infeasible: label 0.0, cost_model.py:154-157),
    no output mismatch, a dataset row (not invalid / unsupported). Returns
    (rows, X, modelled, measured) in row order."""
    from .access_analysis import features_records
    from .dataset import STATUS_INVALID, STATUS_UNSUPPORTED

    lab = labels[np.argsort(labels[:, 0], kind="stable")]
    rows = lab[:, 0].astype(np.int64)
    tb, to = lab[:, 1], lab[:, 2]
    mism, st = lab[:, 3], lab[:, 4]
    keep = ((st == 0) | (st == 2)) & (tb > 0) & (mism <= 0)
    rows, tb, to = rows[keep], tb[keep], to[keep]
    measured = np.where(to > 0, tb / np.where(to > 0, to, 1.0), 0.0)
    fb = features_records(table.records(rows))
    ok = (fb.status != STATUS_INVALID) & (fb.status != STATUS_UNSUPPORTED)  # DatasetArrays.ok: infeasible stays (0.0)
    return rows[ok], fb.X[ok], fb.label[ok], measured[ok]


def train(X, speedups, seed: int, threads: int):
    from . import forest as F
    from .access_analysis import FEATURE_NAMES

    y = np.array([F.speedup_to_target(float(v)) for v in speedups])
    return F.train_arrays(X, y, F.Hyperparams(seed=seed, **HP), FEATURE_NAMES, threads=threads)


def report(pred, speedups) -> dict:
    from .metrics import evaluate

    rep = evaluate(np.asarray(pred) > 1.0, np.asarray(speedups))
    return {"count_accuracy": rep.count_accuracy, "penalty_weighted_accuracy": rep.penalty_weighted_accuracy,
            "min_score": rep.min_score,
            "confusion": [rep.true_optimize, rep.false_optimize, rep.true_leave, rep.false_leave]}


def run_rank(out_dir: str, table, labels: np.ndarray, my_rows: np.ndarray, rank: int, seed: int = 0,
             threads: int = 1) -> dict:
    """One rank's part: featurise, split, train both forests, predict this
    rank's held-out rows, write rankRRR/study_pred.npz. Returns timings."""
    from .forest import predict

    t0 = time.perf_counter()
    rows, X, modelled, measured = study_set(table, labels)
    t_feat = time.perf_counter() - t0
    from .dataset import split_indices

    tr, he = split_indices(len(rows), STUDY_FRACTION, seed)
    he = np.sort(he)
    mine = he[np.isin(rows[he], my_rows)]
    out = {"idx": mine}
    t_train = t_pred = 0.0
    for name, y in (("modelled", modelled), ("measured", measured)):
        t1 = time.perf_counter()
        f = train(X[tr], y[tr], seed, threads)
        t_train += time.perf_counter() - t1
        t1 = time.perf_counter()
        out[name] = predict(f, X[mine]) if len(mine) else np.zeros(0)
        t_pred += time.perf_counter() - t1
    rdir = os.path.join(out_dir, f"rank{rank:03d}")
    os.makedirs(rdir, exist_ok=True)
    tmp = os.path.join(rdir, "study_pred.tmp.npz")
    np.savez(tmp, **out)
    os.replace(tmp, os.path.join(rdir, "study_pred.npz"))
    return {"study_rows": int(len(rows)), "train_rows": int(len(tr)), "held_out_mine": int(len(mine)),
            "k4_s": t_feat, "train_s": t_train, "k3_predict_s": t_pred}


def merge(out_dir: str, table, labels: np.ndarray, world: int, seed: int = 0) -> dict:
    """Rank 0 after a barrier: the held-out predictions of every rank in row
    order, scored; writes DIR/study.json."""
    from .dataset import split_indices

    rows, X, modelled, measured = study_set(table, labels)
    tr, he = split_indices(len(rows), STUDY_FRACTION, seed)
    he = np.sort(he)
    pos = {int(i): k for k, i in enumerate(he)}
    pm = np.full(len(he), np.nan)
    pr = np.full(len(he), np.nan)
    for r in range(world):
        z = np.load(os.path.join(out_dir, f"rank{r:03d}", "study_pred.npz"))
        k = np.array([pos[int(i)] for i in z["idx"]], dtype=np.int64)
        pm[k], pr[k] = z["modelled"], z["measured"]
    if np.isnan(pm).any() or np.isnan(pr).any():
        raise RuntimeError("study: some held-out rows were predicted by no rank")
    res = {"rows": int(len(rows)), "train": int(len(tr)), "held_out": int(len(he)), "ranks": world,
           "measured_beneficial_frac": float((measured > 1.0).mean()) if len(rows) else 0.0,
           "model_beneficial_frac": float((modelled > 1.0).mean()) if len(rows) else 0.0,
           "model_vs_measured_decision_agreement":
               float(((modelled > 1.0) == (measured > 1.0)).mean()) if len(rows) else 0.0,
           "modelled_labels": report(pm, modelled[he]), "measured_labels": report(pr, measured[he])}
    with open(os.path.join(out_dir, "study.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    return res
