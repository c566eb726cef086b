#!/bin/bash
# default bench timed end to end; FFMA-chain register-parity probe
OUT=gpurun_out/r02s7; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chainp tools/probes/chain_probe.cu && /tmp/chainp > $OUT/chain_probe.txt 2>&1
S=$(date +%s); timeout 2400 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$? wall_s=$(( $(date +%s) - S ))" >> $OUT/bench.err
cat $OUT/chain_probe.txt; tail -2 $OUT/bench.err; head -c 400 $OUT/bench.json
