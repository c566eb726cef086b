#!/bin/bash
# ncu --set full of the HBM-leg instances (both variants): DRAM bytes, L2 hit
# rate, bank conflicts, occupancy.   gpurun -- bash tools/ncu_hbm.sh TAG
TAG=${1:-r02_hbm}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
C1=1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,16,16
H16=2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,2048,2048,32,8
H64=2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,1024,1024,32,8
P16=2048,2048,8192,8192,5,1,1,0,0,0,0,0,0,0,0,2048,2048,32,8
python tools/ncu_one.py $C1 $H16 $H64 $P16 $C1 $H16 $H64 $P16 > $OUT/times.txt 2>&1
for c in C1 H16 P16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmt_kernel -c 2 \
     -o $OUT/prof_$c python tools/ncu_one.py ${!c} > $OUT/ncu_$c.log 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page raw --csv > $OUT/raw_$c.csv 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/details_$c.csv 2>&1
  gzip -f $OUT/raw_$c.csv
  mv $OUT/prof_$c.ncu-rep /tmp/ 2>/dev/null
done
cat $OUT/times.txt
