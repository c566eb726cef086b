"""K5 (configs[1]) on this GPU: every instance of real.instance_set in both
variants (L2 flushed before each), per kernel the best launch of each variant
on its roof.   python tools/real_summary.py [OUT.json]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6986_b200 as L  # noqa: E402

R = L.real
insts = R.instance_set()
R.measure(insts)
ms = R.measure(insts)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]
fp32 = json.load(open("profiles/fp32_peak.json"))["fp32_fma_tflops"]
rows = []
for i, m in zip(insts, ms):
    t_b, t_o = m["t_base_ms"] / 1e3, m["t_opt_ms"] / 1e3
    if i.kernel == 1:
        fb, fo = m["alg_flops"] / t_b / 1e12 / fp32, m["alg_flops"] / t_o / 1e12 / fp32
    else:
        fb, fo = m["alg_bytes"] / t_b / 1e9 / hbm, m["alg_bytes"] / t_o / 1e9 / hbm
    rows.append(dict(kernel=R.KERNELS[i.kernel], n=i.n, wg=[i.wg_x, i.wg_y], tile=i.tile, radius=i.radius,
                     base_ms=float(m["t_base_ms"]), opt_ms=float(m["t_opt_ms"]), base_frac=float(fb),
                     opt_frac=float(fo), mismatches=int(m["mismatches"])))
for k in R.KERNELS:
    sub = [r for r in rows if r["kernel"] == k]
    b = max(sub, key=lambda r: r["base_frac"])
    o = max(sub, key=lambda r: r["opt_frac"])
    print(f"{k:24s} base best {b['base_frac']:.3f} ({b['n']} wg {b['wg']} T {b['tile']} R {b['radius']})  "
          f"opt best {o['opt_frac']:.3f} ({o['n']} wg {o['wg']} T {o['tile']} R {o['radius']})  "
          f"mism {sum(r['mismatches'] for r in sub)}")
json.dump(rows, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/real_summary.json", "w"), indent=0)
