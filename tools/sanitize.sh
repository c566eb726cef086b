#!/bin/bash
# compute-sanitizer over small instances of every kernel family: memcheck
# (K0-K5), racecheck + synccheck (K2's TMA/mbarrier staging, K5 tiles).
#   gpurun -- bash tools/sanitize.sh r01san
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
cat > /tmp/san_cases.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1412_6986_b200 as L
recs = np.array([
    [64,64,64,64,0,4,4,0,1,3,2,1,1,1,1,32,32,8,8],        # xy_reuse rect1
    [64,64,64,64,3,2,4,2,2,5,3,2,1,1,2,32,32,32,1],       # y_reuse_row star2 (vec rows)
    [64,64,32,32,5,2,2,1,2,20,18,20,18,11,9,32,32,4,8],  # no_reuse ctx-wrap
    [64,64,32,512,4,2,4,0,1,3,2,1,1,1,1,512,2,512,1],    # wide TMA
    [64,64,64,64,6,2,3,0,3,3,2,1,1,1,1,32,32,8,4],       # radius 3
    [1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,32,8],  # memory-bound: unit-group stream, group stages
    [256,256,256,256,0,4,4,1,1,5,3,2,1,1,1,32,64,8,4],    # xy_reuse, partial groups
], dtype=np.int32)
L.prepare_records(recs)
r = L.measure_records(recs)
print("measure", r["mismatches"].tolist(), r["status"].tolist())
r = L.measure_records(recs, concurrent=True)
print("measure concurrent", r["mismatches"].tolist(), r["status"].tolist())
r = L.measure_records(recs, regblock=True)
print("measure regblock", r["mismatches"].tolist(), r["status"].tolist())
fb = L.features_records(recs)
print("features", fb.status.tolist())
f = L.forest.synthetic_forest(ntrees=5, nodes_per_tree=301, seed=1)
print("rf", L.forest.predict_mean(f, np.random.default_rng(0).normal(0, 1000, size=(100, 18)))[:2])
R = L.real
small = [R.RealInstance(0, 64, 16, 4, tile=16), R.RealInstance(0, 128, 32, 8, tile=64),
         R.RealInstance(1, 64, 16, 8, tile=16), R.RealInstance(2, 64, 16, 4, tile=1, radius=2),
         R.RealInstance(2, 64, 16, 4, tile=4, radius=3), R.RealInstance(3, 512, 64, 1, tile=16),
         R.RealInstance(3, 512, 32, 1, tile=32)]
print("real", R.measure(small)["mismatches"].tolist())
ev = np.load("tests/golden/forest_eval.npz")
X, y = ev["X"][:300], np.array([L.speedup_to_target(v) for v in ev["speedup"][:300]])
g = L.train_arrays_gpu(X, y, L.Hyperparams(num_trees=2, features_per_node=4, seed=1))
print("rf train gpu", [len(t.feature) for t in g.trees])
PY
python /tmp/san_cases.py > $OUT/plain.log 2>&1   # warm the JIT cache outside the tools
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_cases.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/$tool.log
done
tail -4 $OUT/plain.log $OUT/memcheck.log $OUT/racecheck.log $OUT/synccheck.log
