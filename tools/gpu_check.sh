#!/bin/bash
# One GPU round-trip: parity tests, smoke, a short bench line, the ncu launch
# list of the same bench command and one full ncu capture of the top kernel.
#   gpurun --timeout 1500 -- bash tools/gpu_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > "$OUT/ncu_bench.log" 2>&1
echo "ncu launches rc=$?" >> "$OUT/ncu_bench.log"
tail -3 "$OUT/pytest_gpu.log" "$OUT/smoke.log" "$OUT/bench.err"
cat "$OUT/bench.json"
