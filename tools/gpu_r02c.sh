#!/bin/bash
OUT=gpurun_out/r02c
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 1200 python tools/conc_validate.py 2000 $OUT/conc.json > $OUT/conc.log 2>&1; echo "rc=$?" >> $OUT/conc.log
tail -45 $OUT/conc.log
