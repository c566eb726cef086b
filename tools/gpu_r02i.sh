#!/bin/bash
OUT=gpurun_out/${1:-r02i}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
C1=1024,1024,1024,1024,5,1,1,2,1,0,0,0,0,0,0,1024,1024,16,16
H16=2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,2048,2048,32,8
H64=2048,2048,8192,8192,5,1,1,2,1,0,0,0,0,0,0,1024,1024,32,8
P16=2048,2048,8192,8192,5,1,1,0,0,0,0,0,0,0,0,2048,2048,32,8
python tools/ncu_one.py $C1 $H16 $H64 $P16 $C1 $H16 $H64 $P16 > $OUT/hbm_times.txt 2>&1
cat $OUT/hbm_times.txt
timeout 1500 python bench.py --steps 3 --warmup 1 --batch 256 --no-rf --no-real --no-e2e --cpu-seconds 5 --dump $OUT/bench_dump.npz > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?"
tail -3 $OUT/bench.err; head -c 1500 $OUT/bench.json
