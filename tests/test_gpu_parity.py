"""GPU parity: the CUDA path (through the C ABI) against the golden vectors
of the reference and against the CPU oracle. Bit-exact for every fp32 output
(+-inf included), bit-exact fp64 RF means, bit-identical predictions."""

import os

import numpy as np
import pytest

import oracle
import paper_1412_6986_b200 as L
from conftest import GOLDEN_DIR, ROOT, make_instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda(golden):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    # compile every specialised kernel the module launches up front, in
    # parallel host threads (the reference's per-kernel compile step)
    insts = [make_instance(r) for r in golden["interp"]] + [make_instance(golden["cfg1"])]
    L.prepare_instances(insts)


def test_fill_matches_hash_kat(golden):
    h = golden["hash"]
    for salt, key in ((0, "salt0"), (1, "salt1")):
        n = max(h["idx"]) + 1
        t = L.interp.device_fill(1, n, salt)[0, :n].cpu().numpy()
        for i, v in zip(h["idx"], h[key]):
            assert t[i] == np.float32(v)
        assert np.array_equal(t, oracle.hash_fill(n, salt))


def test_make_inputs_match_reference(golden):
    for r in golden["interp"][:40]:
        a, b = L.make_inputs(make_instance(r))
        assert oracle.out_hash(a) == int(r["in_digest"]) and oracle.out_hash(b) == int(r["in2_digest"])


def test_run_pair_matches_reference_all_cases(golden):
    keep = np.load(f"{GOLDEN_DIR}/interp_outputs.npz")
    bad = []
    for k, r in enumerate(golden["interp"]):
        base, opt = L.run_pair(make_instance(r))
        if oracle.out_hash(base) != int(r["digest"]) or not np.array_equal(base, opt):
            bad.append((k, r["pattern"], r["shape"], r["radius"], oracle.out_hash(base) == int(r["digest"])))
        if f"out{k}" in keep:
            assert np.array_equal(base, keep[f"out{k}"])
    assert not bad, bad


def test_measure_host_buffers_match_reference(golden):
    """lmt_measure_batch_host (the e2e path: host inputs, double-buffered
    device slots, copies on their own streams): per-instance outputs read
    back bit-identical to the reference's, digests equal to the device-input
    path's, across more instances than slots and with growing sizes."""
    recs = golden["interp"][:12]
    insts = [make_instance(r) for r in recs]
    ins = [L.make_inputs(k) for k in insts]
    ob = [np.full((k.params.out_h, k.params.out_w), np.nan, np.float32) for k in insts]
    oo = [np.full_like(o, np.nan) for o in ob]
    got = L.measure_instances_host(insts, [a for a, _ in ins], [b for _, b in ins], out_base=ob, out_opt=oo)
    dev = L.measure_instances(insts)
    for r, m, d, b, o in zip(recs, got, dev, ob, oo):
        assert m.status in (0, 2) and m.digest_base == d.digest_base
        assert oracle.out_hash(b) == int(r["digest"])
        if m.t_opt_ms is not None:
            assert m.mismatches == 0 and np.array_equal(b, o) and m.digest_opt == d.digest_opt


def test_inf_cases_present_and_exact(golden):
    inf_cases = [r for r in golden["interp"] if r["n_inf"] > 0]
    assert inf_cases, "golden set must include +-inf producing chains"
    for r in inf_cases:
        base, opt = L.run_pair(make_instance(r))
        assert oracle.out_hash(base) == int(r["digest"])
        assert np.isinf(base).sum() == r["n_inf"]


def test_execute_accepts_reference_inputs(golden):
    # execute with inputs of a *different* (larger) instance, like
    # test_interp.py:121-130 does
    r = golden["interp"][5]
    inst = make_instance(r)
    in_arr, in2 = oracle.make_inputs(inst)
    big = np.pad(in_arr, ((0, 3), (0, 5)))
    for v in (L.Variant.BASELINE, L.Variant.OPTIMIZED):
        got = L.execute(inst, v, big, in2)
        want = oracle.execute(inst, 0, big, in2)
        assert np.array_equal(got, want)


def test_cfg1_matches_reference(golden):
    r = golden["cfg1"]
    base, opt = L.run_pair(make_instance(r))
    assert oracle.out_hash(base) == int(r["digest"])
    assert np.array_equal(base, opt)


def test_measure_digests_match_oracle(golden):
    cases = [make_instance(r) for r in golden["interp"][::3]]
    ms = L.measure_instances(cases)
    for m, r in zip(ms, golden["interp"][::3]):
        assert m.status == 0, (m.status, L.measure.last_error())
        assert m.verified and m.mismatches == 0
        assert m.digest_base == int(r["digest"]) == m.digest_opt
        assert m.t_base_ms > 0 and m.t_opt_ms > 0


def test_invalid_and_infeasible_are_reported():
    P, S = L.HomeAccessPattern, L.StencilShape
    good = L.TemplateParams(2048, 2048, 2048, 2048, P.NO_REUSE_ROW_MAJOR, 8, 8, L.StencilPattern(S.STAR, 0),
                            5, 1, 0, 0, 0, 0)
    infeasible = L.KernelInstance(good, L.LaunchConfig(2048, 2048, 32, 32))
    invalid = L.KernelInstance(good, L.LaunchConfig(16, 16, 8, 8))
    ms = L.measure_instances([invalid, infeasible])
    assert ms[0].status == 1 and ms[0].t_opt_ms is None
    assert ms[1].status == 2 and ms[1].t_opt_ms is None and ms[1].t_base_ms > 0 and ms[1].speedup == 0.0
    with pytest.raises(L.InvalidInstance):
        L.run_pair(invalid)


def _sample_check(inst, wg_count=3):
    """Full-size instance: base == opt bitwise everywhere, and the first
    workgroups match the oracle (size-independent spot check)."""
    import torch

    geo = L.emit_geometry(inst)
    p = inst.params
    a = L.interp.device_fill(geo.alloc_h, geo.alloc_w, 0)
    b = L.interp.device_fill(p.in_h, p.in_w, 1)
    base = L.interp.execute_device(inst, L.Variant.BASELINE, a[:, : geo.alloc_w], b[:, : p.in_w])
    opt = L.interp.execute_device(inst, L.Variant.OPTIMIZED, a[:, : geo.alloc_w], b[:, : p.in_w])
    assert torch.equal(base.view(torch.int32), opt.view(torch.int32))
    in_h = a[:, : geo.alloc_w].cpu().numpy()
    want = oracle.execute(inst, 0, in_h, b[:, : p.in_w].cpu().numpy(), wg_range=(0, wg_count))
    done = ~np.isnan(want)
    got = base.cpu().numpy()
    assert np.array_equal(got[done], want[done])


def test_full_size_sweep_instances():
    tab = L.select_instance_table(L.SamplingSpec(max_instances=20000, seed=0))
    rng = np.random.default_rng(5)
    rows = rng.choice(len(tab), size=40, replace=False)
    cost = L.sweep.estimated_cost(tab.records(rows))
    L.prepare_records(tab.records(rows))
    for r, c in zip(rows, cost):
        inst = tab.instance(int(r))
        if c > 0.5 or L.footprint(inst).bytes > 48 * 1024:
            continue
        _sample_check(inst)


def test_forest_mean_bitwise():
    f = L.load(f"{GOLDEN_DIR}/forest_small.txt")
    ev = np.load(f"{GOLDEN_DIR}/forest_eval.npz")
    mean = L.forest.predict_mean(f, ev["X"])
    assert np.array_equal(mean, ev["mean"])
    pred = L.predict(f, ev["X"])
    assert np.array_equal(pred, ev["pred"])
    assert list(L.predict(f, ev["X"][:10])) == [L.predict(f, ev["X"][i]) for i in range(10)]
    assert np.array_equal(L.decide(f, ev["X"]), ev["pred"] > 1.0)


def test_tree_predict_and_votes():
    f = L.forest.synthetic_forest(ntrees=37, nodes_per_tree=2001, seed=4)  # > 32 trees: two lane chunks
    X = np.random.default_rng(1).normal(0, 1000, size=(3001, 18))
    g = L.forest.gpu_forest(f)
    mean, votes = g.mean(X, votes=True)
    assert np.array_equal(mean, oracle.forest_mean(f.trees, X))
    leaves = np.stack([f.trees[t].predict(X) for t in range(3)])
    for t in range(3):
        assert np.array_equal(leaves[t], oracle.forest_mean([f.trees[t]], X))
    want_votes = sum((oracle.forest_mean([t], X) > 0).astype(int) for t in f.trees)
    assert np.array_equal(votes, want_votes)


def test_reference_objects_accepted(lmtune_ref):
    from lmtune.interp import run_pair as ref_run_pair
    from lmtune.kernel_model import (HomeAccessPattern, KernelInstance, LaunchConfig, StencilPattern,
                                     StencilShape, TemplateParams)

    p = TemplateParams(64, 64, 32, 32, HomeAccessPattern.Y_REUSE_COL, 2, 4, StencilPattern(StencilShape.DIAMOND, 2),
                       3, 2, 1, 1, 1, 1)
    k = KernelInstance(p, LaunchConfig(32, 32, 4, 8))
    b, o = L.run_pair(k)
    rb, ro = ref_run_pair(k)
    assert np.array_equal(b, rb) and np.array_equal(o, ro)


def _golden_devices(dv):
    return [L.DeviceDescriptor(*[int(x) for x in row]) for row in dv]


def test_features_and_labels_bitwise():
    """K4 against the reference's extract_features + label_speedup on 21.8k
    rows (20k sweep instances at the default device, 600 x 3 other devices)."""
    g = np.load(f"{GOLDEN_DIR}/features.npz")
    rec, X, lab, dv = g["rec"], g["X"], g["label"], g["dev"]
    default = (dv == dv[0]).all(axis=1)
    b = L.features_records(rec[default], L.DEFAULT_DEVICE)
    assert (b.status[default[default]] != 1).all()
    assert np.array_equal(b.X, X[default])
    assert np.array_equal(b.label, lab[default])
    other = ~default
    b2 = L.features_records(rec[other], _golden_devices(dv[other]))
    assert np.array_equal(b2.X, X[other])
    assert np.array_equal(b2.label, lab[other])


def test_feature_api_single_instance(golden):
    r = golden["interp"][3]
    inst = make_instance(r)
    fv = L.extract_features(inst)
    b = L.features_instances([inst]) if hasattr(L, "features_instances") else L.access_analysis.features_instances([inst])
    assert np.array_equal(fv.to_array(), b.X[0])
    assert L.label_speedup(inst) == b.label[0]
    tb = L.kernel_time(inst, L.Variant.BASELINE)
    assert tb.total_cycles == b.times[0, 3]
    bad = L.KernelInstance(inst.params, L.LaunchConfig(16, 16, 8, 8))
    with pytest.raises(L.InvalidInstance):
        L.extract_features(bad)


def test_config4_forest_on_gpu_features_matches_reference():
    """BASELINE config 4: the reference model trained on 10% of a 100k sweep;
    features of the held-out 90% rebuilt on the GPU (K4) and predictions (K3)
    must be bit-identical to the reference's forest.predict."""
    import gzip
    import hashlib
    import tempfile

    ev = np.load(f"{GOLDEN_DIR}/forest_sweep100k_eval.npz")
    with gzip.open(f"{GOLDEN_DIR}/forest_sweep100k.txt.gz", "rb") as fh, \
            tempfile.NamedTemporaryFile(suffix=".txt", delete=False) as out:
        out.write(fh.read())
    f = L.load(out.name)
    table = L.select_instance_table(L.SamplingSpec(max_instances=100_000, seed=0))
    held = ev["held_idx"]
    fb = L.features_records(table.records(held))
    assert hashlib.sha256(fb.X.tobytes()).digest() == ev["X_sha256"].tobytes()
    pred = L.predict(f, fb.X)
    assert np.array_equal(pred[::8], ev["pred_every8"])
    assert hashlib.sha256(pred.tobytes()).digest() == ev["pred_sha256"].tobytes()
    assert np.array_equal(fb.label[::8], ev["speedup_every8"])
    # and the forest itself, trained natively on the GPU-featurised 10%
    tr = L.features_records(table.records(ev["train_idx"]))
    y = np.array([L.speedup_to_target(s) for s in tr.label])
    ours = L.train_arrays(tr.X, y, L.Hyperparams(num_trees=20, features_per_node=4, seed=0),
                          feature_names=f.feature_names, threads=8)
    # node numbering differs between a trained (creation order) and a loaded
    # (pre-order) forest; the model file is the canonical form
    L.save(ours, out.name + ".ours")
    with gzip.open(f"{GOLDEN_DIR}/forest_sweep100k.txt.gz", "rb") as fh:
        golden = fh.read()
    assert open(out.name + ".ours", "rb").read() == golden
    # and trained on the GPU (lmt_rf_train_gpu, one CTA per tree)
    gpu = L.train_arrays_gpu(tr.X, y, L.Hyperparams(num_trees=20, features_per_node=4, seed=0),
                             feature_names=f.feature_names)
    L.save(gpu, out.name + ".gpu")
    assert open(out.name + ".gpu", "rb").read() == golden


def test_gpu_training_matches_native_trainer():
    """forest.train on the GPU node for node against the
    native trainer, which tests/test_host.py pins to the reference: default
    hyperparameters, depth / leaf-size limits, no bootstrap, many features
    per node."""
    ev = np.load(f"{GOLDEN_DIR}/forest_eval.npz")
    X = ev["X"][:1500]
    y = np.array([L.speedup_to_target(s) for s in ev["speedup"][:1500]])
    for hp_args in (dict(num_trees=6, features_per_node=4, seed=3),
                    dict(num_trees=3, features_per_node=6, seed=1, max_depth=7, min_samples_leaf=3),
                    dict(num_trees=2, features_per_node=18, seed=9, bootstrap=False)):
        hp = L.Hyperparams(**hp_args)
        cpu = L.train_arrays(X, y, hp, threads=2)
        gpu = L.train_arrays_gpu(X, y, hp)
        assert len(cpu.trees) == len(gpu.trees)
        for a, b in zip(cpu.trees, gpu.trees):
            for fld in ("feature", "threshold", "left", "right", "value"):
                assert np.array_equal(getattr(a, fld), getattr(b, fld)), (hp_args, fld)


def test_run_sweep_checkpoint_resume_and_dataset(tmp_path):
    """The sweep job on one GPU: chunks checkpointed, a second run resumes
    every chunk, labels + the 39-column dataset written (rows = the K4 rows
    of this rank's share)."""
    import json

    from paper_1412_6986_b200 import run_sweep

    out = str(tmp_path / "sweep")
    argv = ["--out", out, "--max-instances", "3000", "--seed", "2", "--chunk", "8", "--limit", "24"]
    s1 = run_sweep.run(argv)
    assert s1["rows"] == 24 and s1["chunks_resumed"] == 0 and s1["mismatched"] == 0
    s2 = run_sweep.run(argv)
    assert s2["chunks_resumed"] == 3
    lab = np.load(f"{out}/labels.npz")
    assert len(lab["row"]) == 24 and (lab["t_base_ms"] > 0).all()
    rows = L.read_rows(f"{out}/dataset.csv")
    assert len(rows) == 24
    table = L.select_instance_table(L.SamplingSpec(max_instances=3000, seed=2))
    fb = L.features_records(table.records(lab["row"]))
    assert np.array_equal(np.stack([r.features.to_array() for r in rows]), fb.X)
    assert json.load(open(f"{out}/summary.json"))["total_rows"] == 24


def test_run_sweep_study_two_ranks_match_one(tmp_path):
    """run_sweep --study (SURVEY 8(e) after the gather): one rank, then two
    ranks on this GPU over gloo (torchrun), on the same 32-instance sample --
    the same study.json; every held-out row predicted by exactly one rank."""
    import json
    import subprocess
    import sys

    common = ["--max-instances", "3000", "--seed", "2", "--sample", "32", "--chunk", "8", "--study"]
    one, two = str(tmp_path / "one"), str(tmp_path / "two")
    env = dict(os.environ, PYTHONPATH=ROOT)
    subprocess.run([sys.executable, "-m", "paper_1412_6986_b200.run_sweep", "--out", one] + common,
                   check=True, cwd=ROOT, env=env, timeout=900)
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                    "--master-addr", "127.0.0.1", "--master-port", "29533", "-m", "paper_1412_6986_b200.run_sweep",
                    "--out", two, "--backend", "gloo"] + common, check=True, cwd=ROOT, env=env, timeout=900)
    a, b = json.load(open(f"{one}/study.json")), json.load(open(f"{two}/study.json"))
    assert (a.pop("ranks"), b.pop("ranks")) == (1, 2)
    # modelled labels are deterministic: identical across world sizes; measured
    # ones are timings (they differ run to run), so the 2-rank study is compared
    # with a one-process study over the same gathered labels
    assert a["modelled_labels"] == b["modelled_labels"] and a["rows"] == b["rows"] >= 24
    assert a["train"] + a["held_out"] == a["rows"]
    idx = [np.load(f"{two}/rank{r:03d}/study_pred.npz")["idx"] for r in range(2)]
    assert len(np.intersect1d(*idx)) == 0 and len(idx[0]) + len(idx[1]) == b["held_out"]
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "measured_study.py"), two], check=True, cwd=ROOT,
                   env=env, timeout=600, capture_output=True)
    c = json.load(open(f"{two}/study.json"))
    assert c.pop("ranks") == 1 and c == b


def _small(pat, n, m, shape, r, counts, out, grid, wg, inh=64):
    params = L.TemplateParams(inh, inh, out[0], out[1], pat, n, m, L.StencilPattern(shape, r), **counts)
    return L.KernelInstance(params, L.LaunchConfig(grid[0], grid[1], wg[0], wg[1]))


def test_edge_paths_against_oracle():
    """Kernel paths the golden set does not reach: context counts beyond the
    in2 halo (ctx-wrap), regions wider than one 256-column TMA box (wide),
    radius 3 stencils, in2 smaller than the halo, 1024-thread workgroups."""
    P, S = L.HomeAccessPattern, L.StencilShape
    base = dict(num_comp_ilb=3, num_comp_ep=2, num_coal_ilb=1, num_coal_ep=1, num_uncoal_ilb=1, num_uncoal_ep=1)
    wrap = dict(num_comp_ilb=5, num_comp_ep=3, num_coal_ilb=20, num_coal_ep=18, num_uncoal_ilb=11, num_uncoal_ep=9)
    cases = [
        _small(P.XY_REUSE, 4, 4, S.RECTANGULAR, 1, wrap, (64, 64), (32, 32), (8, 8)),
        _small(P.NO_REUSE_ROW_MAJOR, 2, 2, S.STAR, 2, wrap, (32, 32), (32, 32), (4, 8), inh=16),
        _small(P.Y_REUSE_COL, 2, 4, S.RECTANGULAR, 1, base, (32, 512), (512, 2), (512, 1), inh=64),
        _small(P.X_REUSE_COL, 4, 2, S.DIAMOND, 2, base, (512, 32), (2, 512), (1, 512), inh=64),
        _small(P.NO_REUSE_COL_MAJOR, 2, 3, S.RECTANGULAR, 3, base, (32, 32), (32, 32), (8, 4)),
        _small(P.Y_REUSE_ROW, 3, 2, S.STAR, 3, base, (64, 64), (32, 32), (32, 32)),
        _small(P.XY_REUSE, 8, 8, S.DIAMOND, 0, base, (64, 64), (64, 16), (32, 16), inh=4),
    ]
    L.prepare_instances(cases)
    for inst in cases:
        base_out, opt_out = L.run_pair(inst)
        want_b, _ = oracle.run_pair(inst)
        assert np.array_equal(base_out, want_b), inst
        assert np.array_equal(opt_out, want_b), inst
        m = L.measure_instances([inst])[0]
        assert m.verified and m.digest_base == oracle.out_hash(want_b)


def test_measure_modes_bitwise(golden):
    """The measurement modes (SM partitions, register-blocked variants, warm
    L2) change where and how the kernels run, never their outputs: every
    golden instance's digests match the reference's in every mode, and the
    few-CTA instances really ran inside partitions."""
    recs = golden["interp"][::2]
    cases = [make_instance(r) for r in recs]
    for kw in (dict(concurrent=True), dict(regblock=True), dict(concurrent=True, regblock=True, warm_l2=True)):
        L.prepare_instances(cases, **kw)
        ms = L.measure_instances(cases, **kw)
        for m, r in zip(ms, recs):
            assert m.status == 0, (kw, m.status, L.measure.last_error())
            assert m.verified and m.digest_base == int(r["digest"]) == m.digest_opt, (kw, r)
        if kw.get("concurrent") and L._lib.partitions():
            biggest = max(L._lib.partitions())
            assert all((m.lane_sms > 0) == (m.ctas <= biggest) for m in ms)
            assert all(m.lane_sms >= m.ctas for m in ms if m.lane_sms > 0)
            assert any(m.lane_sms > 0 for m in ms)


def test_sampled_cells_match_oracle_at_full_size():
    """Paper-geometry instances of the 1M sweep (2048^2 outputs, `in` up to
    ~1 GiB), both variants, measured in SM partitions: the cells gathered by
    the measurement equal the CPU oracle's point evaluation of
    interp.execute bit for bit -- an independent check of K1 and K2 (not
    just K1 == K2)."""
    sys_path_bench()
    import bench

    tab = L.select_instance_table(L.SamplingSpec(max_instances=1_000_000, seed=0))
    rng = np.random.default_rng(11)
    rows = np.sort(rng.choice(len(tab), size=400, replace=False))
    rec = tab.records(rows)
    keep = L.sweep.launch_cost(rec) < 0.4
    rec = rec[keep][:48]
    idx = bench.sample_cells(rec, 24, 3)
    L.prepare_records(rec, concurrent=True)
    res, vals = L.measure_records(rec, samples=idx, concurrent=True)
    assert (res["status"] != 1).all() and (res["t_base_ms"] > 0).all()
    orc = bench.oracle_check(rec, res, idx, vals)
    assert orc["instances"] == len(rec) and orc["mismatched"] == 0, orc
    assert (res["mismatches"][res["t_opt_ms"] > 0] == 0).all()


def test_vec_baseline_charges_its_layout():
    """A radius-2 instance whose baseline reads 128-bit shifted copies of
    `in`: the copy is built inside the baseline's timed window
    (in_copies == 4) and the output is still the reference's."""
    P, S = L.HomeAccessPattern, L.StencilShape
    params = L.TemplateParams(2048, 2048, 2048, 2048, P.Y_REUSE_ROW, 32, 8, L.StencilPattern(S.RECTANGULAR, 2),
                              num_comp_ilb=10, num_comp_ep=3, num_coal_ilb=2, num_coal_ep=1, num_uncoal_ilb=1,
                              num_uncoal_ep=2)
    inst = L.KernelInstance(params, L.LaunchConfig(128, 16, 32, 8))
    rec = L.sweep.instances_to_records([inst])
    idx = np.array([[0, 1, 2047, 2048 * 2048 - 1, 12345, 777777]], dtype=np.int64)
    res, vals = L.measure_records(rec, samples=idx)
    assert res["in_copies"][0] == 4 and res["mismatches"][0] == 0
    for v in (0, 1):
        assert np.array_equal(vals[0, :, v].view(np.uint32), oracle.eval_units(rec[0], v, idx[0]).view(np.uint32))


def sys_path_bench():
    import sys

    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
