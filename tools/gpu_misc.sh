#!/bin/bash
# (1) the ahead-of-time kernels (LMT_JIT=0) still agree bitwise on representative
#     shapes; (2) K2 slots vs work units on a tiny-workgroup xy_reuse launch.
OUT=gpurun_out/${1:-r01misc}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
B=2048,2048,2048,2048,0,16,16,2,1,6,44,13,0,2,4,256,2048,2,1
G=2048,2048,2048,2048,3,32,8,0,2,10,34,12,4,1,3,128,16,32,8
H=2048,2048,1024,1024,0,32,32,0,2,37,9,9,5,4,4,16,64,1,1
LMT_JIT=0 timeout 600 python tools/ncu_one.py $A $B $G $H > $OUT/aot.txt 2>&1
P404=2048,2048,2048,2048,0,64,64,2,1,6,44,13,0,2,4,256,2048,2,1
for cfg in "auto auto" "2 2" "2 3" "4 4" "4 5" "1 2" "1 1"; do
  set -- $cfg
  if [ $1 = auto ]; then unset LMT_FORCE_U LMT_FORCE_STAGES; else export LMT_FORCE_U=$1 LMT_FORCE_STAGES=$2; fi
  echo "== U=$1 S=$2 $(timeout 300 python tools/ncu_one.py $P404 2>&1 | tail -n 1)" >> $OUT/p404.txt
done
cat $OUT/aot.txt $OUT/p404.txt
