#!/bin/bash
# ncu --set full + SASS source page of one instance's kernels (both variants)
#   gpurun -- bash tools/ncu_src.sh TAG RECORD [TUNE]
TAG=$1; REC=$2
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python tools/ncu_one.py $REC > $OUT/times.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmt_kernel -c 2 \
   -o $OUT/prof python tools/ncu_one.py $REC > $OUT/ncu.log 2>&1
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>&1
gzip -f $OUT/raw.csv $OUT/source.csv
mv $OUT/prof.ncu-rep /tmp/ 2>/dev/null
cat $OUT/times.txt
