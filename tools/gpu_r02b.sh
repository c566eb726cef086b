#!/bin/bash
# round 2: GPU tests on the new measurement engine, concurrency validation, a short bench
OUT=gpurun_out/r02b
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 900 python tools/conc_validate.py 400 $OUT/conc.json > $OUT/conc.log 2>&1; echo "rc=$?" >> $OUT/conc.log
tail -40 $OUT/conc.log
timeout 900 python bench.py --steps 2 --warmup 1 --batch 96 --no-rf --no-real --cpu-seconds 8 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
tail -3 $OUT/bench.err; head -c 3000 $OUT/bench.json
