"""Per-instance report of a bench --dump sample against the floor model."""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1412_6986_b200 import sweep  # noqa: E402

NAMES = "in_h in_w out_h out_w pat n m shape r cilb cep coilb coep uilb uep gx gy wx wy".split()


def main(path, ref=None, top=15):
    d = np.load(path)
    rec, res = d["rec"], d["res"]
    tb, to = res["t_base_ms"], np.where(res["t_opt_ms"] > 0, res["t_opt_ms"], 0.0)
    ch, iss = sweep.floor_seconds(rec)
    fl = np.maximum(ch, iss) * 1e3
    ran = res["t_opt_ms"] > 0
    print(f"n={len(rec)} base {tb.sum():.0f} ms opt {to.sum():.0f} ms  floor(base+opt) {fl.sum() + fl[ran].sum():.0f} ms")
    if ref:
        r = np.load(ref)["res"]
        t0 = r["t_base_ms"] + np.where(r["t_opt_ms"] > 0, r["t_opt_ms"], 0.0)
        print(f"reference sample total {t0.sum():.0f} ms -> {tb.sum() + to.sum():.0f} ms")
    tot = tb + to
    o = np.argsort(-tot)
    for i in o[:top]:
        desc = " ".join(f"{k}={int(v)}" for k, v in zip(NAMES[4:], rec[i][4:]))
        print(f"{tot[i]:8.1f} ms  base {tb[i]:7.1f} opt {to[i]:7.1f} floor {fl[i]:6.1f} kid {res['kernel_id'][i]} "
              f"S {res['nstages'][i]} | {desc}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
