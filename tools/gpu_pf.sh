#!/bin/bash
# Prefetch-distance experiment on the representative instances.
TAG=${1:-r01g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
B=2048,2048,2048,2048,0,16,16,2,1,6,44,13,0,2,4,256,2048,2,1
D=2048,2048,2048,2048,1,64,2,0,1,17,24,8,12,4,0,16,128,8,128
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
F=2048,2048,2048,2048,5,8,1,0,1,16,36,10,9,4,4,16,512,4,128
G=2048,2048,2048,2048,3,32,8,0,2,10,34,12,4,1,3,128,16,32,8
for pf in 0 4 8 16; do
  LMT_PF=$pf timeout 600 python tools/ncu_one.py $A $B $D $E $F $G > $OUT/pf$pf.txt 2>&1
done
for pf in 0 4 8 16; do echo "PF=$pf"; cat $OUT/pf$pf.txt; done
