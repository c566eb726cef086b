#!/bin/bash
# A 50,000-instance random sample of the full 1M sweep (both families), the
# default placement (SM partitions), 16 output cells per instance checked
# against the CPU oracle, then the RF study on measured vs modelled labels.
OUT=gpurun_out/${1:-r02_sweep50k}
BIG=/tmp/${1:-r02_sweep50k}
mkdir -p $OUT $BIG
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout ${T:-3000} python -m paper_1412_6986_b200.run_sweep --out $BIG/run --sample ${N:-50000} --samples 16 --study > $OUT/run.json 2> $OUT/run.err; echo "run rc=$?"
tail -3 $OUT/run.err
python bench.py --verify-sweep $BIG/run > $OUT/verify.json; cat $OUT/verify.json
cp $BIG/run/summary.json $BIG/run/study.json $BIG/run/labels.npz $OUT/ 2>/dev/null
head -c 1500 $OUT/run.json
