#!/bin/bash
OUT=gpurun_out/${1:-r02f}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 1200 python tools/tune_hbm.py 5 $OUT/tune_hbm.json > $OUT/tune.log 2>&1; echo "rc=$?" >> $OUT/tune.log
cat $OUT/tune.log
