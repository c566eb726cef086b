#!/bin/bash
OUT=gpurun_out/${1:-r02z}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
python tools/ncu_real.py 3,4096,32,1,32,0 3,4096,64,1,32,0 3,4096,128,1,32,0 3,4096,32,1,16,0 3,4096,512,1,32,0
timeout 900 python tools/real_summary.py $OUT/real_summary.json > $OUT/real_summary.txt 2>&1; cat $OUT/real_summary.txt
bash tools/ncu_real.sh ${1}_mvt 3,4096,32,1,32,0 > /dev/null 2>&1
