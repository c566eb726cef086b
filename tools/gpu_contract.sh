#!/bin/bash
# The measurement contract's effect on the labels: the same
# sweep sample measured literal vs register-blocked, L2-cold vs warm (all on
# the whole device, no partitions), each followed by the RF study.
OUT=gpurun_out/${1:-r02_contract}
N=${2:-8000}
BIG=/tmp/${1:-r02_contract}
mkdir -p $OUT $BIG
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for mode in "literal_cold:" "literal_warm:--warm-l2" "regblock_cold:--regblock" "regblock_warm:--regblock --warm-l2"; do
  name=${mode%%:*}; flags=${mode#*:}
  timeout 3000 python -m paper_1412_6986_b200.run_sweep --out $BIG/$name --sample $N --study --chunk 1024 --isolated $flags > $OUT/$name.json 2> $OUT/$name.err
  echo "$name rc=$?"; tail -1 $OUT/$name.err
  cp $BIG/$name/labels.npz $OUT/${name}_labels.npz 2>/dev/null
  cp $BIG/$name/study.json $OUT/${name}_study.json 2>/dev/null
done
