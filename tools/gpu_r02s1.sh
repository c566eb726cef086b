#!/bin/bash
# session re-entry check: GPU tests + ncu of the K5 MVT / matrixMul shapes
OUT=gpurun_out/r02s1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
timeout 900 bash tools/ncu_real.sh r02s1/ncu 3,4096,32,1,32,0 3,4096,64,1,32,0 1,1024,16,16,64,0 > $OUT/ncu_real.log 2>&1
python tools/src_hot.py $OUT/ncu/source.csv.gz 40 > $OUT/src_hot.txt 2>&1
tail -3 $OUT/pytest.log
