#!/bin/bash
# ncu --set full on reduced-size proxies of the largest remaining gaps:
#   P429 xy_reuse 64x64 diamond0, 32 CTAs of 16 threads (out 512^2 proxy)
#   P249 xy_reuse 64x64 diamond1, 8 CTAs of 512 (out 256x2048 proxy)
TAG=${1:-r01gap}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
P429=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
P249=2048,2048,256,2048,0,64,64,1,1,44,10,13,1,3,2,2048,2,256,2
python tools/ncu_one.py $P429 $P249 > $OUT/times.txt 2>&1
for c in P429 P249; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lmt_kernel" -c 2 \
     -o $OUT/prof_$c python tools/ncu_one.py ${!c} > $OUT/ncu_$c.log 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/details_$c.csv 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page source --csv --print-source sass > $OUT/source_$c.csv 2>&1
  gzip -f $OUT/source_$c.csv
  mv $OUT/prof_$c.ncu-rep /tmp/ 2>/dev/null
done
cat $OUT/times.txt
