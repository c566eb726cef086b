#!/bin/bash
# K5 round: matrixMul fragment double-buffering, convolution interior paths; FFMA issue-form probe
OUT=gpurun_out/r02s3
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fpi tools/probes/fp_issue.cu && /tmp/fpi > $OUT/fp_issue.txt 2>&1
timeout 600 python -m pytest tests/test_real.py -x -q -m gpu > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
timeout 600 python tools/real_summary.py $OUT/real.json > $OUT/real.txt 2>&1
timeout 900 bash tools/ncu_real.sh r02s3/ncu 1,1024,16,16,64,0 1,1024,8,4,32,0 2,8192,32,8,4,1 > $OUT/ncu_real.log 2>&1
tail -3 $OUT/pytest.log; cat $OUT/real.txt; cat $OUT/fp_issue.txt
