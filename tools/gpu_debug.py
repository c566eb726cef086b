"""GPU triage helper: per-variant parity on the golden cases and crash
bisection over sweep batches (each instance synchronised individually)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_1412_6986_b200 as L  # noqa: E402
from conftest import make_instance  # noqa: E402


def parity():
    g = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))
    nbad = 0
    for k, r in enumerate(g["interp"]):
        inst = make_instance(r)
        a, b = oracle.make_inputs(inst)
        want = oracle.execute(inst, 0, a, b)
        for v in (0, 1):
            got = L.execute(inst, L.Variant.BASELINE if v == 0 else L.Variant.OPTIMIZED, a, b)
            if not np.array_equal(got, want):
                nbad += 1
                diff = np.argwhere(~((got == want) | (np.isnan(got) & np.isnan(want))))
                geo = L.emit_geometry(inst)
                print(f"case {k} variant {v}: {r['pattern']} {r['shape']}{r['radius']} n={r['n']} m={r['m']} "
                      f"wg={r['wg_x']}x{r['wg_y']} grid={r['grid_x']}x{r['grid_y']} out={r['out_h']} in={r['in_h']}x{r['in_w']} "
                      f"counts={r['num_comp_ilb']},{r['num_comp_ep']},{r['num_coal_ilb']},{r['num_coal_ep']},"
                      f"{r['num_uncoal_ilb']},{r['num_uncoal_ep']} alloc={geo.alloc_h}x{geo.alloc_w} "
                      f"region={geo.r_rows}x{geo.r_cols} ndiff={len(diff)} first={diff[:3].tolist()} "
                      f"got={got[tuple(diff[0])]} want={want[tuple(diff[0])]}", flush=True)
    print("parity bad variants:", nbad, flush=True)


def crash(start=0, count=64, batch=16):
    import torch

    import bench

    _, table, perm = bench.workload(0)
    for s in range(start, start + count):
        rows = bench.step_rows(perm, s, 1, batch)
        for r in rows:
            rec = table.records([r])
            print("row", int(r), rec.tolist(), flush=True)
            res = L.measure_records(rec)
            torch.cuda.synchronize()
            print("  ok", res["t_base_ms"][0], res["t_opt_ms"][0], res["status"][0], res["mismatches"][0],
                  res["nstages"][0], res["kernel_id"][0], flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "parity":
        parity()
    elif what == "crash":
        crash(int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 6)
    elif what == "case":
        g = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))
        r = g["interp"][int(sys.argv[2])]
        inst = make_instance(r)
        a, b = oracle.make_inputs(inst)
        want = oracle.execute(inst, 0, a, b)
        got = L.execute(inst, L.Variant.OPTIMIZED, a, b)
        geo = L.emit_geometry(inst)
        print(r, geo)
        bad = np.argwhere(got != want)
        print("mismatches", len(bad), bad[:10].tolist())
        if len(bad):
            print(got[tuple(bad[0])], want[tuple(bad[0])])
    elif what == "one":
        rec = np.array([[int(x) for x in sys.argv[2].split(",")]], dtype=np.int32)
        res = L.measure_records(rec)
        print(res)
