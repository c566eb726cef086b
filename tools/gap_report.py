"""Largest contributors to (measured - launch floor) in a bench --dump sample.

    python tools/gap_report.py SAMPLE.npz [N]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_6986_b200 import sweep  # noqa: E402

z = np.load(sys.argv[1])
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rec, res = z["rec"], z["res"]
ch, iss = sweep.floor_seconds(rec)
fl = np.maximum(ch, iss) * 1e3
tb, to = res["t_base_ms"], res["t_opt_ms"]
gb, go = tb - fl, np.where(to > 0, to - fl, 0)
print(f"measured base {tb.sum():.0f} opt {to[to > 0].sum():.0f} ms; gap base {gb.sum():.0f} opt {go.sum():.0f} ms")
items = sorted([(gb[i], "base", i) for i in range(len(rec))] + [(go[i], "opt", i) for i in range(len(rec))],
               reverse=True)
cum = 0.0
for g, v, i in items[:N]:
    cum += g
    r = rec[i]
    t = (tb if v == "base" else to)[i]
    print(f"{g:7.1f} cum {cum:7.1f} {v:4s} t={t:7.1f} fl={fl[i]:6.1f} #{i:<3d} kid {res['kernel_id'][i]} "
          f"S{res['nstages'][i]} pat={r[4]} n={r[5]} m={r[6]} sh={r[7]} r={r[8]} ci={r[9]} co={r[11]} "
          f"un={r[13]} g={r[15]}x{r[16]} wg={r[17]}x{r[18]}")
