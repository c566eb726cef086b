#!/bin/bash
# JIT path: parity tests, representative-instance times (JIT vs AOT), bench sample.
TAG=${1:-r01d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
B=2048,2048,2048,2048,0,16,16,2,1,6,44,13,0,2,4,256,2048,2,1
C=1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,16,16
D=2048,2048,2048,2048,1,64,2,0,1,17,24,8,12,4,0,16,128,8,128
timeout 300 python tools/ncu_one.py $A $B $C $D > $OUT/times_jit.txt 2>&1
LMT_JIT=0 timeout 300 python tools/ncu_one.py $A $B $C $D > $OUT/times_aot.txt 2>&1
timeout 900 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu --dump $OUT/sample.npz > $OUT/bench.json 2> $OUT/bench.err
tail -2 $OUT/pytest_gpu.log; cat $OUT/times_jit.txt $OUT/times_aot.txt; tail -3 $OUT/bench.err; head -c 600 $OUT/bench.json
