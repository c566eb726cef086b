#!/bin/bash
# Loop-body size experiment: with LMT_SHARE the step bodies are long, and
# U x D unrolled steps can exceed the 32 KB instruction cache on launches
# with few CTAs. Times representative shapes at forced (U, D).
TAG=${1:-r01icache}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
H=2048,2048,1024,1024,0,32,32,0,2,37,9,9,5,4,4,16,64,1,1
I=2048,2048,2048,2048,0,32,16,0,1,35,19,6,13,4,4,128,4,64,2
K=2048,2048,1024,1024,0,32,32,1,1,33,28,10,2,3,2,4,128,1,64
T=2048,2048,2048,2048,0,64,64,1,0,26,38,10,13,2,2,4,512,1,512
V=2048,2048,2048,2048,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
for cfg in "auto auto" "16 1" "16 2" "16 3" "8 2" "8 3"; do
  set -- $cfg
  if [ $1 = auto ]; then unset LMT_FORCE_U LMT_FORCE_D; else export LMT_FORCE_U=$1 LMT_FORCE_D=$2; fi
  echo "== U=$1 D=$2" >> $OUT/ud.txt
  timeout 600 python tools/ncu_one.py $A $E $H $I $K $T $V >> $OUT/ud.txt 2>&1
done
cat $OUT/ud.txt | awk '/^==/{print; next} {print $3, $5, $9, $11}'
