#!/bin/bash
# K5: convolution optimized staging (aligned 128-bit rows, warp-local rows, two-phase column staging); 64-wide CC=2 matrixMul tiles
OUT=gpurun_out/r02s5
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py -x -q -m gpu > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
for i in 1 2; do python tools/ncu_real.py 1,1024,32,8,64,0 1,1024,32,16,64,0 1,1024,16,16,64,0 2,8192,32,8,4,1 2,8192,32,8,4,2 2,8192,32,8,1,1; done > $OUT/times.txt 2>&1
timeout 600 python tools/real_summary.py $OUT/real.json > $OUT/real.txt 2>&1
tail -3 $OUT/pytest.log; cat $OUT/times.txt $OUT/real.txt
