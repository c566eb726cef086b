#!/bin/bash
# Quick GPU check after a kernel change: parity tests, representative shapes, bench sample.
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
A=2048,2048,512,512,0,64,64,1,0,25,47,5,12,1,4,32,16,16,1
B=2048,2048,2048,2048,0,16,16,2,1,6,44,13,0,2,4,256,2048,2,1
D=2048,2048,2048,2048,1,64,2,0,1,17,24,8,12,4,0,16,128,8,128
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
G=2048,2048,2048,2048,3,32,8,0,2,10,34,12,4,1,3,128,16,32,8
H=2048,2048,1024,1024,0,32,32,0,2,37,9,9,5,4,4,16,64,1,1
I=2048,2048,2048,2048,0,32,16,0,1,35,19,6,13,4,4,128,4,64,2
J=2048,2048,2048,2048,0,64,32,2,2,11,33,7,11,3,3,2048,2048,128,4
K=2048,2048,1024,1024,0,32,32,1,1,33,28,10,2,3,2,4,128,1,64
timeout 600 python tools/ncu_one.py $A $B $D $E $G $H $I $J $K > $OUT/times.txt 2>&1
if [ -n "$ALT" ]; then env $ALT timeout 600 python tools/ncu_one.py $A $B $D $E $G $H $I $J $K > $OUT/times_alt.txt 2>&1; fi
timeout 900 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu --no-rf --dump $OUT/sample.npz > $OUT/bench.json 2> $OUT/bench.err
tail -2 $OUT/pytest.log; cat $OUT/times.txt; [ -n "$ALT" ] && echo "== $ALT" && cat $OUT/times_alt.txt; tail -2 $OUT/bench.err; python -c "import json; d=json.load(open('$OUT/bench.json')); print('value', d['value'], 'floor', d['launch_floor']['frac'])"
