#!/bin/bash
# MVT kernel 1 with two-box stages on whole-SM workgroups
OUT=gpurun_out/r02s11; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
for i in 1 2 3; do python tools/ncu_real.py 3,4096,32,1,32,0 3,4096,32,1,16,0 3,4096,64,1,32,0 3,4096,64,1,16,0 3,4096,128,1,32,0; done > $OUT/times.txt 2>&1
tail -3 $OUT/pytest.log; cat $OUT/times.txt
