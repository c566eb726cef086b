#!/bin/bash
OUT=gpurun_out/${1:-r02l}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 900 python tools/real_summary.py $OUT/real_summary.json > $OUT/real_summary.txt 2>&1
cat $OUT/real_summary.txt
