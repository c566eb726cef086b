#!/bin/bash
OUT=gpurun_out/${1:-r02s}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
python tools/ncu_real.py 3,4096,32,1,32,0 3,4096,64,1,32,0 3,4096,128,1,32,0
timeout 1200 python bench.py --steps 2 --warmup 1 --batch 256 --no-rf --no-real --no-hbm --cpu-seconds 5 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
tail -3 $OUT/bench.err; python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'oracle', d['oracle_checked'], d['oracle_mismatched'], d['e2e']['oracle_checked'], d['e2e']['oracle_mismatched'])"
