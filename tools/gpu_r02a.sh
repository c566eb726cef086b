#!/bin/bash
# round 2 first look: green-context probe, cfg1 event time vs ncu kernel time
OUT=gpurun_out/r02a
mkdir -p $OUT
nvidia-smi -L > $OUT/smi.txt 2>&1
timeout 120 ./tools/probes/green_probe > $OUT/green.txt 2>&1; echo "rc=$?" >> $OUT/green.txt
CFG1=1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,16,16
timeout 300 python tools/ncu_one.py $CFG1 $CFG1 $CFG1 > $OUT/cfg1_events.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $OUT/cfg1_ncu.csv python tools/ncu_one.py $CFG1 > $OUT/cfg1_ncu.log 2>&1
cat $OUT/green.txt; cat $OUT/cfg1_events.txt; grep -E "lmt_kernel|k_" $OUT/cfg1_ncu.csv | head -40
