#!/bin/bash
# K5 MVT ring kernels (concurrent kernel 1 / kernel 2) and compile-time matrixMul tiles
OUT=gpurun_out/r02s2
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_real.py -x -q -m gpu > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
timeout 600 python tools/real_summary.py $OUT/real.json > $OUT/real.txt 2>&1
timeout 900 bash tools/ncu_real.sh r02s2/ncu 3,4096,32,1,32,0 3,4096,64,1,32,0 1,1024,16,16,64,0 1,1024,16,8,64,0 > $OUT/ncu_real.log 2>&1
python tools/src_hot.py $OUT/ncu/source.csv.gz 30 > $OUT/src_hot.txt 2>&1
tail -3 $OUT/pytest.log; cat $OUT/real.txt
