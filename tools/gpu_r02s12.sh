#!/bin/bash
OUT=gpurun_out/r02s12; mkdir -p $OUT
nvcc -O3 -o /tmp/h2dp tools/probes/h2d_probe.cu && timeout 300 /tmp/h2dp > $OUT/h2d_probe.txt 2>&1
nvidia-smi -q | grep -iE "link gen|link width|Bus Id" | head > $OUT/pcie.txt
cat $OUT/h2d_probe.txt $OUT/pcie.txt
