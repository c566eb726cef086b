#!/bin/bash
# full GPU tests + smoke on the final code
OUT=gpurun_out/r02s10; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python tools/real_summary.py $OUT/real.json > $OUT/real.txt 2>&1
tail -n 3 $OUT/pytest_gpu.log; tail -n 2 $OUT/smoke.log; cat $OUT/real.txt
