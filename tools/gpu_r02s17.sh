#!/bin/bash
# ncu of the HBM legs with the final memory-bound launch policy
bash tools/ncu_hbm.sh r02s17_hbm > /dev/null 2>&1
bash tools/ncu_src.sh r02s17_H16 2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,2048,2048,32,8 > /dev/null 2>&1
cat gpurun_out/r02s17_hbm/times.txt
