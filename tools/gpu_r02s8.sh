#!/bin/bash
OUT=gpurun_out/r02s8; mkdir -p $OUT
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I. -o /tmp/mvtp tools/probes/mvt_probe.cu -lcuda > $OUT/build.log 2>&1
timeout 300 /tmp/mvtp > $OUT/mvt_probe.txt 2>&1
cat $OUT/mvt_probe.txt
