#!/bin/bash
# Optimized variant: U work units per group vs staging overlap (S >= 2U) on
# shapes whose shared memory allows only S = U at U = 8.
TAG=${1:-r01optu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
P788=2048,2048,512,512,0,64,64,2,1,6,44,13,0,2,4,256,4,128,4
P249=2048,2048,256,2048,0,64,64,1,1,44,10,13,1,3,2,2048,2,256,2
H=2048,2048,1024,1024,0,32,32,0,2,37,9,9,5,4,4,16,64,1,1
K=2048,2048,1024,1024,0,32,32,1,1,33,28,10,2,3,2,4,128,1,64
G=2048,2048,2048,2048,3,32,8,0,2,10,34,12,4,1,3,128,16,32,8
for cfg in "auto" "8" "4" "2"; do
  if [ $cfg = auto ]; then unset LMT_FORCE_U; else export LMT_FORCE_U=$cfg; fi
  echo "== U=$cfg" >> $OUT/optu.txt
  timeout 600 python tools/ncu_one.py $A $E $P788 $P249 $H $K $G >> $OUT/optu.txt 2>&1
done
cat $OUT/optu.txt | awk '/^==/{print; next} {print $3, $5, $9, $11}'
