#!/bin/bash
# memory-bound launch policy from the deep sweep: GPU tests + default bench
OUT=gpurun_out/${TAG:-r02s15}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
S=$(date +%s); timeout 2400 python bench.py --dump $OUT/bench_sample.npz > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$? wall_s=$(( $(date +%s) - S ))" >> $OUT/bench.err
tail -n 2 $OUT/pytest_gpu.log; tail -n 2 $OUT/bench.err
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'oracle', d['oracle_checked'], d['oracle_mismatched'])
for c in d['hbm_leg']['cases']: print(c['case'], round(c['baseline']['frac'],3), round(c['optimized']['frac'],3), c['verified'])"
