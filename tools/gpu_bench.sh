#!/bin/bash
# Parity tests, smoke and the default bench line (no ncu).
TAG=${1:-r01bench}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py --dump $OUT/bench_sample.npz > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
for f in $OUT/pytest_gpu.log $OUT/smoke.log $OUT/bench.err; do tail -n 2 $f; done
python -c "import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'kernel_ms', d['kernel_ms'], 'step_ms_total', d['step_ms_total'], 'e2e', d['e2e']['value'], 'floor', d['launch_floor']['frac'])"
