"""Config 4 fixture (BASELINE.json configs[3]) generated with the REFERENCE in
the build container:

  rows  = dataset.build_dataset(SamplingSpec(max_instances=100_000, seed=0))   (modelled labels)
  train, held = cli.split_rows(rows, 0.10, seed=0)
  forest = forest.train(train, Hyperparams(num_trees=20, features_per_node=4, seed=0))

Writes forest_sweep100k.txt.gz (the `lmforest 1` model) and
forest_sweep100k_eval.npz: the held-out row indices into the selection, the
reference's predictions for every 8th held-out row, and a digest of all of
them. bench.py and tests/test_gpu_parity.py rebuild X on the GPU (K4) from the
product's own selection and check predictions against these.

    python tests/golden/make_forest_sweep.py
"""

import gzip
import hashlib
import os
import sys

import numpy as np

REF = os.environ.get("LMTUNE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from lmtune import cli, dataset, forest  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    spec = dataset.SamplingSpec(max_instances=100_000, seed=0)
    res = dataset.build_dataset(spec, threads=1)
    assert not res.skips, res.skips[:3]
    rows = res.rows
    idx = np.arange(len(rows))
    train_i, held_i = cli.split_rows(list(idx), 0.10, 0)
    train = [rows[i] for i in train_i]
    held = [rows[i] for i in held_i]
    f = forest.train(train, forest.Hyperparams(num_trees=20, features_per_node=4, seed=0))
    tmp = os.path.join(OUT, "forest_sweep100k.txt")
    forest.save(f, tmp)
    with open(tmp, "rb") as src, gzip.open(tmp + ".gz", "wb", compresslevel=9) as dst:
        dst.write(src.read())
    os.unlink(tmp)
    X = np.stack([r.features.to_array() for r in held])
    pred = forest.predict(f, X)
    np.savez_compressed(os.path.join(OUT, "forest_sweep100k_eval.npz"), train_idx=np.array(train_i, dtype=np.int64),
                        held_idx=np.array(held_i, dtype=np.int64), pred_every8=pred[::8],
                        pred_sha256=np.frombuffer(hashlib.sha256(pred.tobytes()).digest(), dtype=np.uint8),
                        X_sha256=np.frombuffer(hashlib.sha256(X.tobytes()).digest(), dtype=np.uint8),
                        speedup_every8=np.array([r.speedup for r in held[::8]]))
    print("rows", len(rows), "train", len(train), "held", len(held), "nodes", sum(len(t.feature) for t in f.trees))


if __name__ == "__main__":
    main()
