#!/bin/bash
OUT=gpurun_out/${1:-r02q}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_real.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
python tools/ncu_real.py 3,4096,32,1,32,0 3,4096,32,1,16,0 3,4096,64,1,32,0 3,4096,128,1,32,0
bash tools/gpu_contract.sh r02_contract 8000
