"""Summarise an `ncu --page source --csv --print-source sass` export: total
stall samples per reason and the hottest SASS instructions."""
import csv
import gzip
import sys
from collections import Counter


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as fh:
        lines = fh.read().splitlines()
    kernels, cur = [], None
    for line in lines:
        if line.startswith('"Kernel Name"'):
            cur = [line.split('","')[1].rstrip('",')]
            kernels.append(cur)
        elif cur is not None:
            cur.append(line)
    out = []
    for k in kernels:
        rows = list(csv.reader(k[1:]))
        out.append((k[0], rows[0], rows[1:]))
    return out


def main(path, top=25):
    for name, hdr, rows in load(path):
        ix = {h: i for i, h in enumerate(hdr)}
        stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot = Counter()
        for r in rows:
            for h in stall_cols:
                try:
                    tot[h] += int(r[ix[h]])
                except (ValueError, IndexError):
                    pass
        s = sum(tot.values()) or 1
        print("=" * 8, name[:90], "samples", s)
        print("  ", ", ".join(f"{k[6:]} {v / s * 100:.1f}%" for k, v in tot.most_common(8)))
        samp = ix.get("Warp Stall Sampling (All Samples)")
        hot = sorted(rows, key=lambda r: -int(r[samp] or 0))[:top]
        for r in hot:
            reasons = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
            print(f"   {int(r[samp]):7d}  {r[ix['Source']].strip()[:60]:60s} {reasons}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
