OUT=gpurun_out/r01as
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_real.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -n 2 $OUT/pytest.log
timeout 900 python bench.py --no-e2e --no-cpu --no-rf --steps 3 > $OUT/bench.json 2> $OUT/bench.err
python -c "import json; d=json.load(open('$OUT/bench.json')); print(json.dumps(d['real_kernels']['MVT'])); print(d['real_kernels']['instances'], d['real_kernels']['verified_bitwise'])"
