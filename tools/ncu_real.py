"""Run a few K5 instances once (an ncu target).
    python tools/ncu_real.py kernel,n,wg_x,wg_y,tile,radius ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402

insts = [L.real.RealInstance(*[int(x) for x in a.split(",")]) for a in sys.argv[1:]]
ms = L.real.measure(insts)
for i, m in zip(insts, ms):
    print(i, "base", m["t_base_ms"], "opt", m["t_opt_ms"], "mism", m["mismatches"], flush=True)
