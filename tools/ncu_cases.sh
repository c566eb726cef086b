#!/bin/bash
# Full ncu captures of representative instances (both variants each):
#   A latency-bound small grid (xy_reuse 64x64, 512 workitems, out 512^2 proxy)
#   B tiny workgroups, huge grid (xy_reuse 16x16 star1, wg 2x1)
#   C cfg1 (memory-bound 5-point stencil, 1024^2)
#   D two 1024-thread CTAs (x_reuse_row 64x2 rect1)
#   E four 256-thread CTAs, one column of workitems (xy_reuse 64x64, out 1024^2 proxy)
TAG=${1:-r01c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
B=2048,2048,2048,2048,0,16,16,2,1,6,44,13,0,2,4,256,2048,2,1
C=1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,16,16
D=2048,2048,2048,2048,1,64,2,0,1,17,24,8,12,4,0,16,128,8,128
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
I=2048,2048,2048,2048,0,32,16,0,1,35,19,6,13,4,4,128,4,64,2
K=2048,2048,1024,1024,0,32,32,1,1,33,28,10,2,3,2,4,128,1,64
CASES=${CASES:-A B C D E}
python tools/ncu_one.py $A $B $C $D $E $I $K > $OUT/times.txt 2>&1
for c in $CASES; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_synth|lmt_kernel" -c 2 \
     -o $OUT/prof_$c python tools/ncu_one.py ${!c} > $OUT/ncu_$c.log 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page raw --csv > $OUT/raw_$c.csv 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/details_$c.csv 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page source --csv --print-source sass > $OUT/source_$c.csv 2>&1
  gzip -f $OUT/source_$c.csv $OUT/raw_$c.csv
  mv $OUT/prof_$c.ncu-rep /tmp/ 2>/dev/null
done
ls -la $OUT
cat $OUT/times.txt
