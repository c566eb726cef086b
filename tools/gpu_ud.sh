#!/bin/bash
# (U, D) experiment on the representative instances.
TAG=${1:-r01h}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
B=2048,2048,2048,2048,0,16,16,2,1,6,44,13,0,2,4,256,2048,2,1
D=2048,2048,2048,2048,1,64,2,0,1,17,24,8,12,4,0,16,128,8,128
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
G=2048,2048,2048,2048,3,32,8,0,2,10,34,12,4,1,3,128,16,32,8
H=2048,2048,1024,1024,0,32,32,0,2,37,9,9,5,4,4,16,64,1,1
for cfg in "auto auto" "8 3" "8 2" "4 2" "4 1" "2 3"; do
  set -- $cfg
  if [ $1 = auto ]; then unset LMT_FORCE_U LMT_FORCE_D; else export LMT_FORCE_U=$1 LMT_FORCE_D=$2; fi
  echo "== U=$1 D=$2" >> $OUT/ud.txt
  timeout 600 python tools/ncu_one.py $A $B $D $E $G $H >> $OUT/ud.txt 2>&1
done
cat $OUT/ud.txt
