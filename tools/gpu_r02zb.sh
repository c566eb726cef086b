#!/bin/bash
OUT=gpurun_out/${1:-r02zb}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
timeout 900 python tools/real_summary.py $OUT/real_summary.json > $OUT/real_summary.txt 2>&1; cat $OUT/real_summary.txt
timeout 600 python - <<'PY'
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1412_6986_b200 as L
ev = np.load("tests/golden/forest_sweep100k_eval.npz")
t = L.select_instance_table(L.SamplingSpec(max_instances=100_000, seed=0))
rec = t.records(ev["held_idx"])
for k in range(3):
    t0 = time.perf_counter(); L.features_records(rec); print("features", len(rec), time.perf_counter() - t0, flush=True)
L.measure_records(t.records(np.arange(8)), concurrent=True)
for k in range(3):
    t0 = time.perf_counter(); L.features_records(rec); print("features after partitions", time.perf_counter() - t0, flush=True)
PY
timeout 1800 python bench.py --no-rf --no-real --no-hbm --cpu-seconds 5 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'n', d['instances_timed'], 'kernel_ms', d['kernel_ms'], 'oracle', d['oracle_checked'], d['oracle_mismatched'], d['e2e']['oracle_mismatched'])"
