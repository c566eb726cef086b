#!/bin/bash
# Parity tests, then the bench's device-timed value next to its end-to-end
# (host buffers) number on the default workload.
TAG=${1:-r01e2e}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -n 3 $OUT/pytest.log
timeout 900 python bench.py --no-cpu --no-rf --no-real > $OUT/bench.json 2> $OUT/bench.err
python -c "import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'floor', d['launch_floor']['frac'])"
