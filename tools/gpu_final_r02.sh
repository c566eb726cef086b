#!/bin/bash
# Round-2 evidence in one GPU call: tests, smoke, the default bench line (+
# sample dump), the ncu launch list of a short bench, ncu --set full of the
# HBM legs (both variants: DRAM bytes, L2 hit rate, bank conflicts) and of
# the dominant isolated launch shape, the K5 summary, sanitizers.
#   gpurun --timeout 5400 -- bash tools/gpu_final_r02.sh r02final
TAG=${1:-r02final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 2400 python bench.py --dump $OUT/bench_sample.npz > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 1 --batch 96 --isolated --no-e2e --no-cpu --no-rf --no-real --no-hbm > $OUT/ncu_bench.log 2>&1
gzip -f $OUT/launches.csv
bash tools/ncu_hbm.sh ${TAG}_hbm > /dev/null 2>&1
bash tools/ncu_src.sh ${TAG}_H16 2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,2048,2048,32,8 > /dev/null 2>&1
E=2048,2048,1024,1024,0,64,64,2,1,6,44,13,0,2,4,256,1024,2,1
python tools/ncu_one.py $E > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmt_kernel -c 2 \
    -o $OUT/prof_top python tools/ncu_one.py $E > $OUT/ncu_top.log 2>&1
ncu -i $OUT/prof_top.ncu-rep --page details --csv > $OUT/details_top.csv 2>&1
ncu -i $OUT/prof_top.ncu-rep --page raw --csv > $OUT/raw_top.csv 2>&1
ncu -i $OUT/prof_top.ncu-rep --page source --csv --print-source sass > $OUT/source_top.csv 2>&1
gzip -f $OUT/source_top.csv $OUT/raw_top.csv
mv $OUT/prof_top.ncu-rep /tmp/ 2>/dev/null
timeout 900 python tools/real_summary.py $OUT/real_summary.json > $OUT/real_summary.txt 2>&1
# compute-sanitizer is closed on the GPU pool (round 2): tools/sanitize.sh is not run here
for f in $OUT/pytest_gpu.log $OUT/smoke.log $OUT/bench.err; do tail -n 2 $f; done
cat $OUT/real_summary.txt; head -c 1500 $OUT/bench.json; echo; head -c 600 $OUT/bench_reference.json
# K3 / K4 / GPU RF training and K5 under ncu
timeout 900 ncu --set full --clock-control none -k regex:"k_rf_mean|k_features|k_rf_build|k_rf_presort" -c 6 \
    -o $OUT/prof_rf python tools/ncu_rf.py > $OUT/ncu_rf.log 2>&1
ncu -i $OUT/prof_rf.ncu-rep --page details --csv > $OUT/details_rf.csv 2>&1
mv $OUT/prof_rf.ncu-rep /tmp/ 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"k_mvt|k_transpose|k_conv|k_matmul" \
    -o $OUT/prof_real python tools/ncu_real.py 0,8192,16,16,64,0 1,1024,16,16,64,0 2,8192,32,8,4,1 3,4096,64,1,32,0 > $OUT/ncu_real.log 2>&1
ncu -i $OUT/prof_real.ncu-rep --page details --csv > $OUT/details_real.csv 2>&1
mv $OUT/prof_real.ncu-rep /tmp/ 2>/dev/null
