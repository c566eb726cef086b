#!/bin/bash
# round 2 re-entry: GPU tests, smoke, concurrency validation, a short bench, green-context probe
OUT=gpurun_out/r02d
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 900 python tools/conc_validate.py 400 $OUT/conc.json > $OUT/conc.log 2>&1; echo "rc=$?" >> $OUT/conc.log
tail -40 $OUT/conc.log
timeout 1200 python bench.py --steps 2 --warmup 1 --batch 96 --no-rf --no-real --cpu-seconds 8 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
tail -5 $OUT/bench.err; head -c 4000 $OUT/bench.json
