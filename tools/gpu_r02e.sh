#!/bin/bash
# kernel change check: GPU parity tests, then the HBM-leg times + ncu
OUT=gpurun_out/${1:-r02e}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
bash tools/ncu_hbm.sh ${1:-r02e}_hbm
