#!/bin/bash
OUT=gpurun_out/${1:-r02w}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
bash tools/ncu_src.sh ${1}_H16 2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,2048,2048,32,8 > /dev/null 2>&1
timeout 1800 python bench.py --no-rf --no-real --no-hbm --cpu-seconds 5 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'kernel_ms', d['kernel_ms'], 'oracle', d['oracle_checked'], d['oracle_mismatched'], d['e2e']['oracle_mismatched'])"
