#!/bin/bash
# ncu --set full on reduced-size proxies of the largest remaining gaps:
#   P788 xy_reuse 64x64 star1, 2 CTAs of 512 (opt 1.65x floor)  out 512^2
#   P745 y_reuse_row 64x8 star2, 2 CTAs of 512 (base 14x floor) out 2048x128
TAG=${1:-r01gap}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
P788=2048,2048,512,512,0,64,64,2,1,6,44,13,0,2,4,256,4,128,4
P745=2048,2048,128,2048,3,64,8,2,2,17,1,1,10,0,2,512,2,256,2
python tools/ncu_one.py $P788 $P745 > $OUT/times.txt 2>&1
for c in P788 P745; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lmt_kernel" -c 2 \
     -o $OUT/prof_$c python tools/ncu_one.py ${!c} > $OUT/ncu_$c.log 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/details_$c.csv 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page source --csv --print-source sass > $OUT/source_$c.csv 2>&1
  gzip -f $OUT/source_$c.csv
  mv $OUT/prof_$c.ncu-rep /tmp/ 2>/dev/null
done
cat $OUT/times.txt
