#!/bin/bash
# Round evidence in one GPU call: fp32 peak probe, pytest -m gpu, smoke, the
# default bench line, the ncu launch list of a short bench, and a full ncu
# capture (exported as text) of the dominant kernel on a proxy instance.
#   gpurun --timeout 2700 -- bash tools/gpu_round.sh r01k
TAG=${1:-r01k}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
(cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu && ./fp32_peak) > $OUT/fp32_peak.json 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
cp $OUT/fp32_peak.json profiles/fp32_peak.json 2>/dev/null
timeout 1200 python bench.py --dump $OUT/bench_sample.npz > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $OUT/ncu_bench.log 2>&1
E=2048,2048,1024,1024,0,64,64,1,0,26,38,10,13,2,2,4,256,1,256
python tools/ncu_one.py $E > /dev/null 2>&1   # fill the JIT disk cache first
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmt_kernel -c 2 \
    -o $OUT/prof_top python tools/ncu_one.py $E > $OUT/ncu_top.log 2>&1
ncu -i $OUT/prof_top.ncu-rep --page details --csv > $OUT/details_top.csv 2>&1
ncu -i $OUT/prof_top.ncu-rep --page raw --csv > $OUT/raw_top.csv 2>&1
ncu -i $OUT/prof_top.ncu-rep --page source --csv --print-source sass > $OUT/source_top.csv 2>&1
gzip -f $OUT/source_top.csv $OUT/raw_top.csv
mv $OUT/prof_top.ncu-rep /tmp/ 2>/dev/null
for f in $OUT/pytest_gpu.log $OUT/smoke.log $OUT/bench.err; do tail -n 2 $f; done; cat $OUT/fp32_peak.json $OUT/bench.json
