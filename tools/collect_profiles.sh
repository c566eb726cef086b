#!/bin/bash
# Copy the judged summaries of one tools/gpu_final_r02.sh run into profiles/.
#   bash tools/collect_profiles.sh r02final3
T=${1:-r02final3}; R=gpurun_out/$T; H=gpurun_out/${T}_hbm
cp $R/bench.json profiles/r02_bench.json
cp $R/bench_reference.json profiles/r02_bench_reference.json
cp $R/launches.csv.gz profiles/r02_launches.csv.gz
{ echo "# ncu --set full, HBM legs (tools/ncu_hbm.sh, gpurun $T): [0] = K1 baseline, [1] = K2 optimized"; echo "# times (CUDA events, L2 flushed):"; cat $H/times.txt; for c in C1 H16 P16; do echo; echo "## $c"; python tools/ncu_summary.py $H/details_$c.csv $H/raw_$c.csv.gz; done; } > profiles/r02_hbm_ncu.txt
{ echo "# ncu --set full of the dominant isolated launch shape (xy_reuse 64x64 star r=1, 2-thread workgroups, out 1024^2 proxy), gpurun $T: [0] K1, [1] K2"; python tools/ncu_summary.py $R/details_top.csv $R/raw_top.csv.gz; echo; echo "# hottest SASS (stall samples)"; python tools/src_hot.py $R/source_top.csv.gz 12; } > profiles/r02_ncu_top.txt
{ echo "# ncu --set full: K4 k_features, K3 k_rf_mean, GPU RF training (k_rf_presort, k_rf_build) on config 4 (tools/ncu_rf.py), gpurun $T"; python tools/ncu_summary.py $R/details_rf.csv; } > profiles/r02_ncu_rf.txt
{ echo "# ncu --set full: K5 best shapes (transpose 8192 T64 C4, matrixMul 1024 T64 4x4, convolution 8192 R1 W4, MVT 4096 wg64 T32: kernels 1 and 2 serialised by ncu), both variants, gpurun $T"; python tools/ncu_summary.py $R/details_real.csv; } > profiles/r02_ncu_real.txt
cp $R/real_summary.json profiles/r02_real_kernels.json; cp $R/real_summary.txt profiles/r02_real_kernels.txt
{ for f in gpurun_out/${T}_san/memcheck.log gpurun_out/${T}_san/racecheck.log gpurun_out/${T}_san/synccheck.log; do echo "== $f"; cat $f; done; } > profiles/r02_sanitizer.txt
python - "$T" <<'PY'
import csv, gzip, json, sys
T = sys.argv[1]
rr = list(csv.reader(gzip.open(f"gpurun_out/{T}_H16/raw.csv.gz", "rt"))); h = {n: i for i, n in enumerate(rr[0])}
b = [float(r[h["dram__bytes_read.sum"]]) * 1e6 + float(r[h["dram__bytes_write.sum"]]) * 1e6 for r in rr[2:4]]
alg = 537001984.0
json.dump({"source": f"ncu --set full (dram__bytes_read.sum + dram__bytes_write.sum per launch), gpurun {T}, tools/ncu_src.sh on the 8192^2 star r=1 HBM leg (2048x2048 grid, 32x8 workgroups, 16 work units per thread)",
           "kernel": "lmt_kernel", "algorithmic_bytes_per_launch": alg,
           "baseline": {"dram_bytes_per_launch": b[0], "ratio_to_algorithmic": b[0] / alg},
           "optimized": {"dram_bytes_per_launch": b[1], "ratio_to_algorithmic": b[1] / alg},
           "note": "reads equal the 268.5 MB of `in` (+halo rows); part of the 268 MB of outputs is still in L2 when the launch ends, so the write bytes per launch are below the algorithmic ones"},
          open("profiles/r02_hbm_traffic.json", "w"), indent=1)
PY
ls -la profiles/r02_*
