#!/bin/bash
# BASELINE configs[2] (+ the RF study of configs[3] on measured labels): the
# dense-linear-algebra family, 100k instances of the 1M sweep, measured on one
# B200 (SM-partition placement), 16 output cells per instance checked against
# the CPU oracle.
OUT=gpurun_out/${1:-r02_dla100k}
BIG=/tmp/${1:-r02_dla100k}
mkdir -p $OUT $BIG
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m paper_1412_6986_b200.run_sweep --out $BIG/small --family dla --sample 300 --concurrent --samples 16 --study > $OUT/small.json 2> $OUT/small.err; echo "small rc=$?"
tail -2 $OUT/small.err
python bench.py --verify-sweep $BIG/small > $OUT/small_verify.json; cat $OUT/small_verify.json
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/clocks_before.txt
timeout 5400 python -m paper_1412_6986_b200.run_sweep --out $BIG/run --family dla --sample 100000 --concurrent --samples 16 --study --chunk 1024 > $OUT/run.json 2> $OUT/run.err; echo "run rc=$?"
tail -3 $OUT/run.err
python bench.py --verify-sweep $BIG/run > $OUT/verify.json; cat $OUT/verify.json
cp $BIG/run/summary.json $BIG/run/study.json $BIG/run/labels.npz $OUT/ 2>/dev/null
head -c 2000 $OUT/run.json
