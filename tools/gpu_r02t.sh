#!/bin/bash
OUT=gpurun_out/${1:-r02t}
mkdir -p $OUT
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python tools/ncu_real.py 3,4096,32,1,32,0 3,4096,64,1,32,0 3,4096,128,1,32,0 3,4096,32,1,16,0
timeout 1500 python tools/tune_records.py $OUT/tune_top.json 2 \
  2048,2048,1024,1024,0,64,64,2,1,6,44,13,0,2,4,256,1024,2,1 \
  2048,2048,1024,1024,0,32,32,0,2,37,9,9,5,4,4,16,32,1,1 \
  2048,2048,1024,1024,0,64,64,1,1,32,34,12,1,0,1,128,32,4,2 \
  2048,2048,1024,1024,0,64,32,2,2,16,7,8,1,0,0,512,16,1,4 \
  2048,2048,1024,1024,3,32,8,0,2,10,34,12,4,1,3,128,8,32,8 > $OUT/tune_top.txt 2>&1
cat $OUT/tune_top.txt
LMT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 1 --batch 48 --no-rf --no-real --no-hbm --no-cpu > $OUT/bench_2ranks.json 2> $OUT/bench_2ranks.err; echo "2ranks rc=$?"
head -c 800 $OUT/bench_2ranks.json; tail -3 $OUT/bench_2ranks.err
