"""One pass of config 4's GPU work (an ncu target): K4 features of the 90k
held-out rows, K3 forest means over them, and GPU training of the forest on
the 10% (lmt_rf_train_gpu)."""
import gzip
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402

g = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
ev = np.load(os.path.join(g, "forest_sweep100k_eval.npz"))
with gzip.open(os.path.join(g, "forest_sweep100k.txt.gz"), "rb") as fh, \
        tempfile.NamedTemporaryFile(suffix=".txt", delete=False) as out:
    out.write(fh.read())
forest = L.load(out.name)
t = L.select_instance_table(L.SamplingSpec(max_instances=100_000, seed=0))
fb = L.features_records(t.records(ev["held_idx"]))
m = L.forest.predict_mean(forest, fb.X)
tr = L.features_records(t.records(ev["train_idx"]))
y = np.array([L.speedup_to_target(s) for s in tr.label])
f2 = L.train_arrays_gpu(tr.X, y, L.Hyperparams(num_trees=20, features_per_node=4, seed=0))
print("rows", len(m), "nodes", sum(len(x.feature) for x in f2.trees))
