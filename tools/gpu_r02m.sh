#!/bin/bash
OUT=gpurun_out/${1:-r02m}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -15 $OUT/pytest.log
timeout 900 python tools/real_summary.py $OUT/real_summary.json > $OUT/real_summary.txt 2>&1
cat $OUT/real_summary.txt
timeout 600 python - > $OUT/rftrain.txt 2>&1 <<'PY'
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1412_6986_b200 as L
ev = np.load("tests/golden/forest_sweep100k_eval.npz")
t = L.select_instance_table(L.SamplingSpec(max_instances=100_000, seed=0))
tr = L.features_records(t.records(ev["train_idx"]))
y = np.array([L.speedup_to_target(s) for s in tr.label])
hp = L.Hyperparams(num_trees=20, features_per_node=4, seed=0)
L.train_arrays_gpu(tr.X[:500], y[:500], hp)
for k in range(3):
    t0 = time.perf_counter(); g = L.train_arrays_gpu(tr.X, y, hp); t1 = time.perf_counter()
    c = L.train_arrays(tr.X, y, hp, threads=16); t2 = time.perf_counter()
    same = all(np.array_equal(a.threshold, b.threshold) and np.array_equal(a.value, b.value) for a, b in zip(g.trees, c.trees))
    print(f"gpu {t1-t0:.3f}s cpu16 {t2-t1:.3f}s rows {len(y)} nodes {sum(len(x.feature) for x in g.trees)} same {same}", flush=True)
PY
cat $OUT/rftrain.txt
