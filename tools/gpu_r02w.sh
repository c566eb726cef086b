#!/bin/bash
OUT=gpurun_out/${1:-r02w}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
C1=1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,16,16
H16=2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,2048,2048,32,8
H64=2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,1024,1024,32,8
P16=2048,2048,8192,8192,5,1,1,0,0,0,0,0,0,0,0,2048,2048,32,8
python tools/ncu_one.py $C1 $H16 $H64 $P16 $C1 $H16 $H64 $P16
bash tools/ncu_src.sh ${1}_H16 $H16 > /dev/null 2>&1
timeout 1800 python bench.py --no-rf --no-real --no-hbm --cpu-seconds 5 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'kernel_ms', d['kernel_ms'], 'oracle', d['oracle_checked'], d['oracle_mismatched'], d['e2e']['oracle_mismatched'])"
