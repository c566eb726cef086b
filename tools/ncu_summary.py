"""Text summary of ncu `--page details --csv` and `--page raw --csv` exports:
per kernel launch the duration, DRAM throughput and bytes, L2 hit rate,
shared-memory bank conflicts, occupancy, registers, issue-slot use.
    python tools/ncu_summary.py DETAILS.csv [RAW.csv.gz] > OUT.txt"""
import csv
import gzip
import sys

want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Issue Slots Busy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Grid Size", "Block Size"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = {h: i for i, h in enumerate(rows[0])}
per = {}
for r in rows[1:]:
    if len(r) <= hdr["Metric Value"]:
        continue
    key = (int(r[hdr["ID"]]), r[hdr["Kernel Name"]])
    if r[hdr["Metric Name"]] in want:
        per.setdefault(key, {})[r[hdr["Metric Name"]]] = f'{r[hdr["Metric Value"]]} {r[hdr["Metric Unit"]]}'.strip()
    per.setdefault(key, {})["Grid Size"] = r[hdr["Grid Size"]]
    per[key]["Block Size"] = r[hdr["Block Size"]]
raw = {}
if len(sys.argv) > 2:
    f = gzip.open(sys.argv[2], "rt") if sys.argv[2].endswith(".gz") else open(sys.argv[2])
    rr = list(csv.reader(f))
    h = {n: i for i, n in enumerate(rr[0])}
    for k, r in enumerate(rr[2:]):
        g = lambda n: r[h[n]] if n in h else ""  # noqa: E731
        raw[k] = {"dram_read_MB": g("dram__bytes_read.sum"), "dram_write_MB": g("dram__bytes_write.sum"),
                  "smem_ld_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
                  "smem_st_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
                  "l2_sector_hit_pct": g("lts__t_sector_hit_rate.pct")}
for (i, name), m in sorted(per.items()):
    print(f"[{i}] {name[:90]}")
    for k in want:
        if k in m:
            print(f"    {k:34s} {m[k]}")
    if i in raw:
        for k, v in raw[i].items():
            print(f"    {k:34s} {v}")
