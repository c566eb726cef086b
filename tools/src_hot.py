"""Summarise an ncu `--page source --csv --print-source sass` export: per
kernel, executed warp instructions by opcode and the hottest instructions by
stall samples.   python tools/src_hot.py source.csv.gz [top]"""
import collections
import csv
import gzip
import re
import sys

top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
f = gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])
kern = []
hdr = None
for row in csv.reader(f):
    if row and row[0] == "Kernel Name":
        kern.append([])
        hdr = None
        continue
    if row and row[0] == "Address":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr and row:
        kern[-1].append((row, hdr))
for k, rows in enumerate(kern):
    ops = collections.Counter()
    total = samples = 0
    hot = []
    for row, h in rows:
        src = row[h["Source"]].strip()
        ex = int(row[h["Instructions Executed"]] or 0)
        st = int(row[h["Warp Stall Sampling (All Samples)"]] or 0)
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0].split(".")[0]
        ops[op] += ex
        total += ex
        samples += st
        hot.append((st, ex, src))
    print(f"== kernel {k}: {total:,} warp instructions executed, {samples} stall samples")
    print("   ", ", ".join(f"{o} {c / total:.1%}" for o, c in ops.most_common(16)))
    for st, ex, src in sorted(hot, reverse=True)[:top]:
        print(f"   {st:6d} {ex:12,d}  {src}")
