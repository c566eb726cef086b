#!/bin/bash
# matrixMul 8 x 8 register tile
OUT=gpurun_out/r02s9; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
for i in 1 2; do python tools/ncu_real.py 1,1024,8,8,64,0 1,1024,16,16,64,0; done > $OUT/times.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_matmul_opt88" -o $OUT/prof python tools/ncu_real.py 1,1024,8,8,64,0 > $OUT/ncu.log 2>&1
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1; gzip -f $OUT/raw.csv; rm -f $OUT/prof.ncu-rep
tail -3 $OUT/pytest.log; cat $OUT/times.txt
