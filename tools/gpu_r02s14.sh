#!/bin/bash
OUT=gpurun_out/r02s14; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python tools/tune_hbm_deep.py 5 $OUT/tune_hbm_deep.json > $OUT/tune.txt 2>&1
cat $OUT/tune.txt | tail -12
