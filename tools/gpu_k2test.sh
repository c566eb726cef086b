#!/bin/bash
OUT=gpurun_out/r01al
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -n 3 $OUT/pytest.log
bash tools/gpu_optu.sh r01al_optu 2>&1 | tail -40
