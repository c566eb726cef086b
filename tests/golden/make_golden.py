"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (lmtune, read-only at /root/reference/pkg/src) in the build container.

    python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed here
and every parity test compares against them (or against the oracle, which is
itself pinned to them by tests/test_oracle.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("LMTUNE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))

from lmtune import access_analysis as aa  # noqa: E402
from lmtune import codegen, cost_model, dataset, forest, interp  # noqa: E402
from lmtune.kernel_model import (  # noqa: E402
    HomeAccessPattern,
    KernelInstance,
    LaunchConfig,
    StencilPattern,
    StencilShape,
    TemplateParams,
    validate_instance,
)

OUT = os.path.dirname(os.path.abspath(__file__))
P, S = HomeAccessPattern, StencilShape
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def digest(a: np.ndarray) -> int:
    """sum_i mix64(i * 0x9E3779B97F4A7C15 + bits_i) mod 2^64 (the product's
    k_digest / the oracle's ora_out_hash)."""
    bits = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).ravel().astype(np.uint64)
    with np.errstate(over="ignore"):
        z = np.arange(bits.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + bits
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return int(np.sum(z, dtype=np.uint64))


def rec(inst) -> dict:
    p, lc = inst.params, inst.launch
    return dict(in_h=p.in_h, in_w=p.in_w, out_h=p.out_h, out_w=p.out_w, pattern=p.pattern.value, n=p.n, m=p.m,
                shape=p.stencil.shape.value, radius=p.stencil.radius, num_comp_ilb=p.num_comp_ilb,
                num_comp_ep=p.num_comp_ep, num_coal_ilb=p.num_coal_ilb, num_coal_ep=p.num_coal_ep,
                num_uncoal_ilb=p.num_uncoal_ilb, num_uncoal_ep=p.num_uncoal_ep, grid_x=lc.grid_x,
                grid_y=lc.grid_y, wg_x=lc.wg_x, wg_y=lc.wg_y)


def small(pattern, n=2, m=2, shape=S.RECTANGULAR, radius=1, out=32, grid=32, wg=(8, 8), inh=64, **counts):
    base = dict(num_comp_ilb=3, num_comp_ep=2, num_coal_ilb=1, num_coal_ep=1, num_uncoal_ilb=1, num_uncoal_ep=1)
    base.update(counts)
    params = TemplateParams(in_h=inh, in_w=inh, out_h=out, out_w=out, pattern=pattern, n=n, m=m,
                            stencil=StencilPattern(shape, radius), **base)
    return KernelInstance(params, LaunchConfig(grid, grid, wg[0], wg[1]))


def interp_cases():
    """Reduced-geometry instances: the shapes of test_interp.py / test_c_emulation.py
    and a seeded random spread over patterns, stencils, launches and counts."""
    cases = []
    for pat in P:
        for shape in S:
            for r in (0, 1, 2):
                cases.append(small(pat, shape=shape, radius=r))
    for pat in (P.XY_REUSE, P.Y_REUSE_COL, P.NO_REUSE_ROW_MAJOR, P.NO_REUSE_COL_MAJOR):
        cases.append(small(pat, out=64, grid=32))
    for wg in ((32, 1), (1, 32), (16, 2), (4, 8), (1, 1), (32, 32), (2, 16)):
        cases.append(small(P.X_REUSE_COL, wg=wg))
        cases.append(small(P.Y_REUSE_ROW, wg=wg, m=8))
    for n, m in ((1, 8), (8, 1), (4, 2)):
        cases.append(small(P.XY_REUSE, n=n, m=m))
    cases.append(small(P.XY_REUSE, num_comp_ilb=0, num_comp_ep=0, num_coal_ilb=0, num_coal_ep=0,
                       num_uncoal_ilb=0, num_uncoal_ep=0))
    # +-inf producing chains (odd comp_ilb doubles acc per (i, j)) and wraps of in2
    cases.append(small(P.XY_REUSE, n=8, m=16, num_comp_ilb=41, num_comp_ep=7, out=32, grid=32, wg=(8, 4)))
    cases.append(small(P.NO_REUSE_ROW_MAJOR, n=4, m=4, num_comp_ilb=43, num_coal_ilb=13, num_uncoal_ilb=4,
                       num_coal_ep=13, num_uncoal_ep=4, inh=16))
    rng = np.random.default_rng(1234)
    for _ in range(70):
        pat = list(P)[rng.integers(7)]
        big_n = pat in (P.XY_REUSE, P.X_REUSE_ROW, P.Y_REUSE_ROW)
        big_m = pat in (P.XY_REUSE, P.X_REUSE_COL, P.Y_REUSE_COL)
        n = int(2 ** rng.integers(0, 5 if big_n else 3))
        m = int(2 ** rng.integers(0, 5 if big_m else 3))
        out = int(2 ** rng.integers(5, 7))
        gx = int(2 ** rng.integers(4, int(np.log2(out)) + 1))
        gy = max(512 // gx, int(2 ** rng.integers(4, int(np.log2(out)) + 1)))
        gy = min(gy, out)
        if gx * gy < 512:
            continue
        wx = int(2 ** rng.integers(0, int(np.log2(gx)) + 1))
        wy = int(2 ** rng.integers(0, int(np.log2(gy)) + 1))
        while wx * wy > 1024:
            wy //= 2
        inh = int(2 ** rng.integers(3, 8))
        params = TemplateParams(
            in_h=inh, in_w=int(2 ** rng.integers(3, 8)), out_h=out, out_w=out, pattern=pat, n=n, m=m,
            stencil=StencilPattern(list(S)[rng.integers(3)], int(rng.integers(0, 3))),
            num_comp_ilb=int(rng.integers(0, 45)), num_comp_ep=int(rng.integers(0, 49)),
            num_coal_ilb=int(rng.integers(0, 14)), num_coal_ep=int(rng.integers(0, 14)),
            num_uncoal_ilb=int(rng.integers(0, 5)), num_uncoal_ep=int(rng.integers(0, 5)))
        inst = KernelInstance(params, LaunchConfig(gx, gy, wx, wy))
        if validate_instance(inst):
            continue
        cases.append(inst)
    return cases


def _rec19(inst):
    p, lc = inst.params, inst.launch
    return [p.in_h, p.in_w, p.out_h, p.out_w, list(HomeAccessPattern).index(p.pattern), p.n, p.m,
            list(StencilShape).index(p.stencil.shape), p.stencil.radius, p.num_comp_ilb, p.num_comp_ep,
            p.num_coal_ilb, p.num_coal_ep, p.num_uncoal_ilb, p.num_uncoal_ep, lc.grid_x, lc.grid_y, lc.wg_x, lc.wg_y]


def feature_fixture():
    """features.npz: rec [n,19] int32, X [n,18] f64, label [n] f64 (label_speedup with the coalescing
    override, exactly build_dataset's label, dataset.py:264-271), dev [n,10] int32 device descriptor."""
    from lmtune.device import DeviceDescriptor

    insts = dataset._select_instances(dataset.SamplingSpec(max_instances=20000, seed=5))
    rng = np.random.default_rng(11)
    devs = [DeviceDescriptor()] * len(insts)
    # non-default devices: other warp / transaction sizes, capacities, latencies
    alt = [DeviceDescriptor(transaction_bytes=64, warp_size=16, lmem_capacity_bytes=16 * 1024),
           DeviceDescriptor(transaction_bytes=256, warp_size=64, max_regs_per_thread=255,
                            register_file_per_sm=65536, max_warps_per_sm=64, max_workgroups_per_sm=32,
                            dram_latency_cycles=600, issue_cycles_per_op=2, lmem_capacity_bytes=227 * 1024),
           DeviceDescriptor(transaction_bytes=32, warp_size=32, element_bytes=4)]
    extra = [insts[i] for i in rng.choice(len(insts), size=600, replace=False)]
    insts = insts + extra * len(alt)
    devs = devs + [d for d in alt for _ in extra]
    rec, X, lab, dv = [], [], [], []
    for inst, d in zip(insts, devs):
        fv = aa.extract_features(inst, d)
        rec.append(_rec19(inst))
        X.append(fv.to_array())
        lab.append(cost_model.label_speedup(inst, d, coalescing_override=fv.noncoalescing_degree))
        dv.append([getattr(d, f) for f in ("transaction_bytes", "warp_size", "element_bytes",
                                            "lmem_capacity_bytes", "register_file_per_sm", "max_regs_per_thread",
                                            "max_warps_per_sm", "max_workgroups_per_sm", "dram_latency_cycles",
                                            "issue_cycles_per_op")])
    np.savez_compressed(os.path.join(OUT, "features.npz"), rec=np.array(rec, dtype=np.int32),
                        X=np.array(X, dtype=np.float64), label=np.array(lab, dtype=np.float64),
                        dev=np.array(dv, dtype=np.int32))
    print("features:", len(rec), "rows")


def main():
    golden = {}
    # 1. hash KAT (interp.py:22-27)
    idx = [0, 1, 7, 100, 999, 12345, 2**20 + 3]
    golden["hash"] = {
        "salt0": [float(interp._hash_fill(i + 1, 0)[i]) for i in idx],
        "salt1": [float(interp._hash_fill(i + 1, 1)[i]) for i in idx],
        "idx": idx,
    }
    # 2. interp outputs on reduced geometry (both variants, bitwise)
    cases = interp_cases()
    recs = []
    keep = {}
    for k, inst in enumerate(cases):
        base, opt = interp.run_pair(inst)
        assert np.array_equal(base, opt)
        in_arr, in2 = interp.make_inputs(inst)
        r = rec(inst)
        r.update(digest=str(digest(base)), sha256=hashlib.sha256(base.tobytes()).hexdigest(),
                 in_digest=str(digest(in_arr)), in2_digest=str(digest(in2)),
                 n_inf=int(np.isinf(base).sum()))
        recs.append(r)
        if k % 9 == 0:
            keep[f"out{k}"] = base
    golden["interp"] = recs
    np.savez_compressed(os.path.join(OUT, "interp_outputs.npz"), **keep)
    # 3. cfg1 (BASELINE.json configs[0]): 1024^2, 5-point star, wg 16x16
    cfg1 = KernelInstance(
        TemplateParams(1024, 1024, 1024, 1024, P.NO_REUSE_ROW_MAJOR, 1, 1, StencilPattern(S.STAR, 1), 0, 0, 0, 0, 0, 0),
        LaunchConfig(1024, 1024, 16, 16))
    b, o = interp.run_pair(cfg1)
    assert np.array_equal(b, o)
    golden["cfg1"] = dict(rec(cfg1), digest=str(digest(b)), sha256=hashlib.sha256(b.tobytes()).hexdigest())
    # 4. geometry / footprint / validation over instances from the default sweep + invalid ones
    sweep = dataset._select_instances(dataset.SamplingSpec(max_instances=20000, seed=0))
    geo = []
    for inst in sweep[::50] + cases:
        g = codegen.emit_geometry(inst)
        fp = aa.footprint(inst)
        geo.append(dict(rec(inst), geometry=[getattr(g, f) for f in g.__dataclass_fields__],
                        footprint=[fp.row_span, fp.col_span, fp.padded_col_span, fp.bytes]))
    golden["geometry"] = geo
    bad = [small(P.XY_REUSE, grid=16), small(P.XY_REUSE, wg=(64, 32)), small(P.XY_REUSE, wg=(3, 8)),
           KernelInstance(TemplateParams(0, 64, 32, 32, P.XY_REUSE, 0, 2, StencilPattern(S.STAR, 1),
                                         -1, 0, 0, 0, 0, -2), LaunchConfig(32, 24, 64, 8))]
    golden["invalid"] = [dict(rec(i), violations=validate_instance(i)) for i in bad]
    # 5. selection pin (dataset.py:207-250)
    sel = {}
    for cap in (1000, 20000, 100000):
        lst = dataset._select_instances(dataset.SamplingSpec(max_instances=cap, seed=0))
        keys = "\n".join(dataset.instance_key(i) for i in lst)
        sel[str(cap)] = dict(n=len(lst), sha256=hashlib.sha256(keys.encode()).hexdigest(),
                             first=dataset.instance_key(lst[0]), last=dataset.instance_key(lst[-1]))
    golden["selection"] = sel
    # 6. random forest: reference train on a small labelled set, predict on held-out rows
    spec = dataset.SamplingSpec(max_instances=3000, seed=0)
    rows = dataset.build_dataset(spec, threads=1).rows
    rng = np.random.default_rng(7)
    perm = rng.permutation(len(rows))
    tr = [rows[i] for i in perm[:800]]
    ev = [rows[i] for i in perm[800:]]
    f = forest.train(tr, forest.Hyperparams(num_trees=20, features_per_node=4, seed=3))
    forest.save(f, os.path.join(OUT, "forest_small.txt"))
    X = np.stack([r.features.to_array() for r in ev])
    acc = np.zeros(len(X))
    for t in f.trees:
        acc += t.predict(X)
    mean = acc / len(f.trees)
    pred = forest.predict(f, X)
    assert np.array_equal(pred, 2.0 ** mean)
    np.savez_compressed(os.path.join(OUT, "forest_eval.npz"), X=X, mean=mean, pred=pred,
                        speedup=np.array([r.speedup for r in ev]))
    golden["forest"] = dict(rows=len(X), trees=len(f.trees), nodes=int(sum(len(t.feature) for t in f.trees)))
    # 7. cost-model label KAT + features for the same held-out rows (K4 next)
    golden["labels"] = [float(cost_model.label_speedup(r.instance)) for r in ev[:200]]
    # 8. features + modelled labels (K4, access_analysis.py:272-308, cost_model.py:94-158) for every
    #    instance of a 20k-instance selection plus non-default devices
    feature_fixture()
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(golden, fh, indent=0, sort_keys=True)
    print("wrote", len(recs), "interp cases,", len(geo), "geometry rows")


if __name__ == "__main__":
    main()
