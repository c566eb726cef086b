"""Host-side logic of the product (no GPU): geometry, validation, selection,
sharding and the model-file format, against the reference's golden vectors
and KATs."""

import hashlib

import numpy as np
import pytest

import paper_1412_6986_b200 as L
from conftest import GOLDEN_DIR, make_instance


def test_geometry_matches_reference(golden):
    for r in golden["geometry"]:
        inst = make_instance(r)
        g = L.emit_geometry(inst)
        assert [getattr(g, f) for f in g.__dataclass_fields__] == r["geometry"]
        fp = L.footprint(inst)
        assert [fp.row_span, fp.col_span, fp.padded_col_span, fp.bytes] == r["footprint"]


def test_validation_messages_match_reference(golden):
    for r in golden["invalid"]:
        assert L.validate_instance(make_instance(r)) == r["violations"]
    for r in golden["interp"][:20]:
        assert L.validate_instance(make_instance(r)) == []


def test_codegen_kats():
    P, S = L.HomeAccessPattern, L.StencilShape

    def inst(pattern=P.XY_REUSE, n=8, m=8, radius=1, launch=L.LaunchConfig(512, 512, 16, 16)):
        p = L.TemplateParams(2048, 2048, 2048, 2048, pattern, n, m, L.StencilPattern(S.RECTANGULAR, radius),
                             10, 10, 2, 2, 1, 1)
        return L.KernelInstance(p, launch)

    # test_codegen.py:112-127
    g = L.emit_geometry(inst(n=32, m=32, radius=0))
    assert (g.num_segs, g.num_warps, g.seg_elems, g.segs_per_row) == (32, 8, 32, 1)
    g = L.emit_geometry(inst(n=4, m=4, radius=0))
    assert (g.r_rows, g.r_cols_pad) == (4, 4)
    with pytest.raises(L.OptimizationInfeasible, match="exceeds capacity"):
        L.geometry.check_optimizable(inst(P.NO_REUSE_ROW_MAJOR, n=8, m=8, radius=0))
    # test_codegen.py:172-185 and copy_transaction_count KATs (150-160)
    assert L.mad_constants(0) == (2.0, 1 / 64)
    assert L.mad_constants(1) == (0.5, -2 / 64)
    assert L.mad_constants(3) == (0.5, -0.0625)
    assert L.mad_constants(5) == (0.5, -1 / 64)
    assert L.copy_transaction_count(L.Footprint(32, 32, 32, 4096)) == 32
    assert L.copy_transaction_count(L.Footprint(34, 34, 64, 8704)) == 68
    assert L.copy_transaction_count(L.Footprint(5, 3, 4, 80)) == 5


def test_work_unit_map_kat():
    # test_kernel_model.py:35-44 (wu_x = 99 example) and bijection
    p = L.TemplateParams(64, 64, 256, 256, L.HomeAccessPattern.XY_REUSE, 1, 1,
                         L.StencilPattern(L.StencilShape.STAR, 0), 0, 0, 0, 0, 0, 0)
    lc = L.LaunchConfig(64, 64, 16, 16)
    seen = set()
    for gy in range(4):
        for gx in range(4):
            for iy in range(4):
                for ix in range(4):
                    for wy in (0, 15):
                        for wx in (0, 3, 15):
                            c = L.work_unit_for(lc, p, L.Coord(gy, gx), L.Coord(wy, wx), L.Coord(iy, ix))
                            assert c not in seen
                            seen.add(c)
    c = L.work_unit_for(lc, p, L.Coord(0, 1), L.Coord(0, 3), L.Coord(0, 1))
    assert c.col == 1 * 16 * 4 + 1 * 16 + 3 == 83


def test_selection_matches_reference(golden):
    for cap, want in golden["selection"].items():
        tab = L.select_instance_table(L.SamplingSpec(max_instances=int(cap), seed=0))
        keys = "\n".join(L.instance_key(i) for i in tab.instances())
        assert len(tab) == want["n"]
        assert hashlib.sha256(keys.encode()).hexdigest() == want["sha256"]


def test_launch_sweep_size():
    # test_dataset.py:112-128: 4,224 launch configurations at out 2048^2
    assert len(L.sweep.launch_configs(2048, 2048)) == 4224


def test_records_roundtrip():
    tab = L.select_instance_table(L.SamplingSpec(max_instances=500, seed=3))
    rec = tab.records()
    arr = L.kernel_model.to_c_array(tab.instances())
    import ctypes

    raw = np.frombuffer(bytes(memoryview(arr))[: rec.nbytes], dtype=np.int32).reshape(rec.shape)
    assert np.array_equal(raw, rec)


def test_sharding_is_disjoint_and_balanced():
    tab = L.select_instance_table(L.SamplingSpec(max_instances=5000, seed=0))
    cost = L.sweep.estimated_cost(tab.records())
    for world in (1, 2, 4, 8):
        for shards in (L.sweep.shard_balanced(cost, world), L.sweep.shard_contiguous(cost, world)):
            allrows = np.concatenate(shards)
            assert len(allrows) == len(tab) and len(np.unique(allrows)) == len(tab)
        loads = [cost[s].sum() for s in L.sweep.shard_balanced(cost, world)]
        assert max(loads) <= 1.05 * cost.sum() / world + cost.max()


def test_model_file_roundtrip(tmp_path):
    f = L.load(f"{GOLDEN_DIR}/forest_small.txt")
    assert f.hyperparams == L.Hyperparams(num_trees=20, features_per_node=4, seed=3)
    p = tmp_path / "m.txt"
    L.save(f, p)
    assert p.read_text() == open(f"{GOLDEN_DIR}/forest_small.txt").read()


def test_model_file_errors_name_the_line(tmp_path):
    good = open(f"{GOLDEN_DIR}/forest_small.txt").read().splitlines()
    bad = tmp_path / "bad.txt"
    bad.write_text("not-a-model 9\n")
    with pytest.raises(L.ModelFormatError, match="line 1"):
        L.load(bad)
    bad.write_text("\n".join(good[:4]) + "\n")
    with pytest.raises(L.ModelFormatError, match="unexpected end of file"):
        L.load(bad)
    lines = list(good)
    lines[1] = "num_trees many"
    bad.write_text("\n".join(lines) + "\n")
    with pytest.raises(L.ModelFormatError, match="line 2"):
        L.load(bad)
    lines = list(good)
    lines[8] = "feature_names a,b,c"
    bad.write_text("\n".join(lines) + "\n")
    with pytest.raises(L.ModelFormatError, match="line 9"):
        L.load(bad)
    first = next(ln for ln in good if ln.startswith("node "))
    bad.write_text("\n".join(good).replace(first, "node 18" + first[len(first.split()[0]) + 1 + len(first.split()[1]):], 1) + "\n")
    with pytest.raises(L.ModelFormatError, match="feature index 18 out of range"):
        L.load(bad)


def test_reference_forest_load_agrees(lmtune_ref):
    from lmtune.forest import load as ref_load

    a = ref_load(f"{GOLDEN_DIR}/forest_small.txt")
    b = L.load(f"{GOLDEN_DIR}/forest_small.txt")
    for ta, tb in zip(a.trees, b.trees):
        for f in ("feature", "threshold", "left", "right", "value"):
            assert np.array_equal(getattr(ta, f), getattr(tb, f))


def test_speedup_to_target():
    assert L.speedup_to_target(1.0) == 0.0
    assert L.speedup_to_target(8.0) == 3.0
    assert L.speedup_to_target(0.0) == -10.0


def test_split_matches_reference_fixture():
    """cli.split_rows (cli.py:54-64) on the 100k selection: the reference's
    held-out indices of the config-4 fixture."""
    import numpy as np

    import paper_1412_6986_b200 as L
    from conftest import GOLDEN_DIR

    ev = np.load(f"{GOLDEN_DIR}/forest_sweep100k_eval.npz")
    tr, he = L.dataset.split_indices(100_000, 0.10, 0)
    assert np.array_equal(tr, ev["train_idx"]) and np.array_equal(he, ev["held_idx"])
    a, b = L.split_rows(list(range(10)), 0.3, 5)
    assert len(a) == 3 and len(b) == 7 and sorted(a + b) == list(range(10))


def test_split_against_reference(lmtune_ref):
    from lmtune.cli import split_rows as ref_split

    import paper_1412_6986_b200 as L

    rows = list(range(1234))
    for seed in (0, 1, 99):
        assert L.split_rows(rows, 0.1, seed) == ref_split(rows, 0.1, seed)


def test_dataset_csv_matches_reference_bytes(lmtune_ref, tmp_path):
    """write_rows is byte-identical to dataset.write_rows; read_rows parses the
    reference's file back losslessly (dataset.py:284-404)."""
    import numpy as np
    from lmtune import dataset as ref_ds

    import paper_1412_6986_b200 as L
    from conftest import make_instance

    res = ref_ds.build_dataset(ref_ds.SamplingSpec(max_instances=300, seed=4))
    ref_path, our_path = tmp_path / "ref.csv", tmp_path / "ours.csv"
    ref_ds.write_rows(ref_path, res.rows)
    ours = []
    for r in res.rows:
        p, lc = r.instance.params, r.instance.launch
        rec = dict(in_h=p.in_h, in_w=p.in_w, out_h=p.out_h, out_w=p.out_w, pattern=p.pattern.value, n=p.n, m=p.m,
                   shape=p.stencil.shape.value, radius=p.stencil.radius, num_comp_ilb=p.num_comp_ilb,
                   num_comp_ep=p.num_comp_ep, num_coal_ilb=p.num_coal_ilb, num_coal_ep=p.num_coal_ep,
                   num_uncoal_ilb=p.num_uncoal_ilb, num_uncoal_ep=p.num_uncoal_ep, grid_x=lc.grid_x,
                   grid_y=lc.grid_y, wg_x=lc.wg_x, wg_y=lc.wg_y)
        ours.append(L.LabeledInstance(make_instance(rec), L.FeatureVector.from_array(r.features.to_array()),
                                      r.speedup, r.beneficial))
    L.write_rows(our_path, ours)
    assert our_path.read_bytes() == ref_path.read_bytes()
    back = L.read_rows(ref_path)
    assert len(back) == len(res.rows)
    for a, b in zip(back, res.rows):
        assert np.array_equal(a.features.to_array(), b.features.to_array()) and a.speedup == b.speedup
        assert L.sweep.instance_key(a.instance) == ref_ds.instance_key(b.instance)
    assert L.CSV_HEADER == ref_ds.CSV_HEADER


def test_dataset_csv_errors_name_the_line(tmp_path):
    import pytest

    import paper_1412_6986_b200 as L

    p = tmp_path / "bad.csv"
    p.write_text(",".join(L.CSV_HEADER) + "\nxy_reuse,rect,1\n")
    with pytest.raises(L.DatasetFormatError, match="line 2"):
        L.read_rows(p)
    p.write_text("a,b\n")
    with pytest.raises(L.DatasetFormatError, match="line 1"):
        L.read_rows(p)


def test_train_matches_reference(lmtune_ref, tmp_path):
    """forest.train (forest.py:72-196): the native tree builder gives the
    reference's trees node for node and a byte-identical model file."""
    import numpy as np
    from lmtune import forest as ref_forest

    import paper_1412_6986_b200 as L
    from conftest import GOLDEN_DIR

    ev = np.load(f"{GOLDEN_DIR}/forest_eval.npz")
    X = ev["X"][:900]
    y = np.array([L.speedup_to_target(s) for s in ev["speedup"][:900]])
    for hp_args in (dict(num_trees=4, features_per_node=4, seed=3),
                    dict(num_trees=3, features_per_node=6, seed=1, max_depth=7, min_samples_leaf=3),
                    dict(num_trees=2, features_per_node=18, seed=9, bootstrap=False)):
        ref = ref_forest.train_arrays(X, y, ref_forest.Hyperparams(**hp_args))
        ours = L.train_arrays(X, y, L.Hyperparams(**hp_args), threads=2)
        assert len(ref.trees) == len(ours.trees)
        for a, b in zip(ref.trees, ours.trees):
            for f in ("feature", "threshold", "left", "right", "value"):
                assert np.array_equal(getattr(a, f), getattr(b, f)), f
            if a.oob_indices is None:
                assert b.oob_indices is None
            else:
                assert np.array_equal(a.oob_indices, b.oob_indices)
        ref_forest.save(ref, tmp_path / "r.txt")
        L.save(ours, tmp_path / "o.txt")
        assert (tmp_path / "r.txt").read_bytes() == (tmp_path / "o.txt").read_bytes()


def test_launch_plans_fit_the_device():
    """Every launch plan of a sweep sample (lmt_plan_info, no GPU): the
    optimized variant's ring fits shared memory whenever it can run, work
    units per thread stay within the kernels' limits."""
    import ctypes

    from paper_1412_6986_b200._lib import CInstance, lib

    t = L.select_instance_table(L.SamplingSpec(max_instances=1_000_000, seed=0))
    rows = np.random.default_rng(5).choice(len(t), size=3000, replace=False)
    out = (ctypes.c_int64 * 16)()
    cap = 227 * 1024
    for flags in (0x8, 0x18):
        for r in t.records(rows):
            ci = CInstance(*[int(v) for v in r[:19]])
            assert lib().lmt_plan_info(ctypes.byref(ci), None, flags, out) == 0
            v = list(out)
            assert 1 <= v[0] <= 16 and 1 <= v[1] <= 3 and 1 <= v[5] <= 8 and 1 <= v[9] <= 16, (r.tolist(), v)
            if v[12] * 4 <= cap:  # one region fits: the ring must too
                assert v[10] <= cap, (r.tolist(), v)


def test_memory_bound_and_single_warp_plans():
    """The launch policy's measured choices (lmt_plan_info, no GPU): on the
    HBM legs a multi-tap stencil runs K1 at 48 warps/SM with U = 4 and K2 at
    2-CTA launch bounds, a one-tap stencil keeps 32 warps and U = 8
    (profiles/r02_tune_hbm_deep.json); single-warp CTAs in two waves of 4
    per SM run without a prefetch ring (profiles/r02_tune_iso.json)."""
    import ctypes

    from bench import hbm_records
    from paper_1412_6986_b200._lib import CInstance, lib

    out = (ctypes.c_int64 * 16)()

    def plan(r):
        assert lib().lmt_plan_info(ctypes.byref(CInstance(*[int(v) for v in r[:19]])), None, 0x8, out) == 0
        return list(out)

    legs = hbm_records()
    for r in legs[1:3]:  # 8192^2 star r=1
        v = plan(r)
        assert (v[0], v[2], v[7]) == (4, 6, 2), v
    v = plan(legs[3])  # 8192^2 point
    assert (v[0], v[2]) == (8, 4), v
    v = plan([2048, 2048, 2048, 2048, 0, 64, 64, 2, 0, 28, 35, 11, 7, 1, 1, 2, 2048, 2, 1])  # 2,048 CTAs of 2 threads
    assert v[1] == 1 and v[14] == 2048, v


def test_native_feature_draws():
    """lmt_rf_feature_draws continues a numpy Generator(PCG64) stream with
    Generator.choice's own algorithm: draw for draw equal to numpy's, after a
    bootstrap `integers` call has left a buffered 32-bit half or not."""
    import ctypes

    from paper_1412_6986_b200._lib import lib

    mask = (1 << 64) - 1
    for seed, n, nfeat, k in ((0, 10000, 18, 4), (7, 37, 18, 6), (3, 500, 18, 18), (11, 9, 5, 2)):
        rng = np.random.Generator(np.random.PCG64(seed))
        rng.integers(0, n, size=n)
        st = rng.bit_generator.state
        s4 = np.array([st["state"]["state"] >> 64, st["state"]["state"] & mask, st["state"]["inc"] >> 64,
                       st["state"]["inc"] & mask], dtype=np.uint64)
        got = np.empty((500, k), dtype=np.int32)
        assert lib().lmt_rf_feature_draws(ctypes.c_void_p(s4.ctypes.data), int(st["has_uint32"]),
                                          int(st["uinteger"]), nfeat, k, 500, ctypes.c_void_p(got.ctypes.data)) == 0
        want = np.stack([np.sort(rng.choice(nfeat, size=k, replace=False)) for _ in range(500)])
        assert np.array_equal(got, want), (seed, nfeat, k)
