#!/bin/bash
# End-of-round evidence: the paper's RF study on the committed 40k measured
# labels, the round evidence run, and the 2-rank (gloo, one GPU) bench path.
TAG=${1:-r01final}
mkdir -p gpurun_out/${TAG}_study
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp profiles/r01_sweep40k_labels.npz gpurun_out/${TAG}_study/labels.npz
python -c "import json; json.dump({'max_instances': 1000000, 'seed': 0}, open('gpurun_out/${TAG}_study/summary.json', 'w'))"
timeout 900 python tools/measured_study.py gpurun_out/${TAG}_study > gpurun_out/${TAG}_study/study_stdout.json 2>&1
rm -f gpurun_out/${TAG}_study/labels.npz
bash tools/gpu_round.sh $TAG
LMT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --no-rf --no-real \
    > gpurun_out/$TAG/bench_2ranks.json 2> gpurun_out/$TAG/bench_2ranks.err
tail -n 3 gpurun_out/$TAG/bench_2ranks.json | cut -c1-400
