#!/bin/bash
# ncu --set full of K5 instances: gpurun -- bash tools/ncu_real.sh TAG INST...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python tools/ncu_real.py "$@" > $OUT/times.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mvt|k_conv|k_matmul|k_transpose" \
   -o $OUT/prof python tools/ncu_real.py "$@" > $OUT/ncu.log 2>&1
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>&1
gzip -f $OUT/raw.csv $OUT/source.csv
mv $OUT/prof.ncu-rep /tmp/ 2>/dev/null
cat $OUT/times.txt
