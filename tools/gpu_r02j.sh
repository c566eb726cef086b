#!/bin/bash
OUT=gpurun_out/${1:-r02j}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
(cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o transpose_probe transpose_probe.cu && timeout 300 ./transpose_probe) > $OUT/transpose_probe.txt 2>&1
cat $OUT/transpose_probe.txt
timeout 900 python tools/real_summary.py $OUT/real_summary.json > $OUT/real_summary.txt 2>&1
cat $OUT/real_summary.txt
