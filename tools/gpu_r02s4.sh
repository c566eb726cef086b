#!/bin/bash
# K5 MVT: y by one bulk copy
OUT=gpurun_out/r02s4
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_real.py -x -q -m gpu > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
for i in 1 2; do python tools/ncu_real.py 3,4096,32,1,32,0 3,4096,32,1,16,0 3,4096,64,1,32,0 3,4096,64,1,16,0 3,4096,128,1,32,0; done > $OUT/times.txt 2>&1
tail -3 $OUT/pytest.log; cat $OUT/times.txt
