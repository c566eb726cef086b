#!/bin/bash
OUT=gpurun_out/${1:-r02zd}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
timeout 2400 python bench.py --no-real --no-hbm --cpu-seconds 5 --dump $OUT/bench_sample.npz > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'n', d['instances_timed'], 'kernel_ms', d['kernel_ms'], 'oracle', d['oracle_checked'], d['oracle_mismatched'], d['e2e']['oracle_mismatched']); print({k:d['rf'][k] for k in ('k3_rows_per_s','predict_e2e_rows_per_s','k4_features_rows_per_s','train_s')})"
