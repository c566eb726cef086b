"""The rest of the reference's public API (lmtune/__init__.py:9-84) on the
drop-in: every name exists, metrics and the cost-model helpers agree with the
reference, and the emitted kernel sources are what NVRTC compiles."""

import ctypes
import os

import numpy as np
import pytest

import paper_1412_6986_b200 as L
from conftest import make_instance


def test_every_reference_export_exists(lmtune_ref):
    names = getattr(lmtune_ref, "__all__", None) or [n for n in dir(lmtune_ref) if not n.startswith("_")]
    mods = {"access_analysis", "codegen", "cost_model", "dataset", "device", "errors", "forest", "interp",
            "kernel_model", "metrics", "seeding", "enumeration", "cli", "config"}
    # the CLI's config plumbing (config.py: RunConfig, Paths, load_config) is out of scope (DESIGN 8)
    out_of_scope = {"RunConfig", "Paths", "load_config"}
    missing = [n for n in names if n not in mods and n not in out_of_scope and not hasattr(L, n)]
    assert not missing, missing


def test_metrics_match_reference(lmtune_ref):
    from lmtune import metrics as M

    rng = np.random.default_rng(3)
    s = np.exp(rng.normal(0, 1.5, size=5000))
    s[::17] = 0.0
    s[::31] = 1.0
    d = rng.random(5000) < 0.5
    assert L.evaluate(d, s) == M.evaluate(d, s) or L.evaluate(d, s).as_kv() == M.evaluate(d, s).as_kv()
    assert L.count_accuracy(d, s) == M.count_accuracy(d, s)
    assert L.penalty_weighted_accuracy(d, s) == M.penalty_weighted_accuracy(d, s)
    assert L.speedup_histogram(s) == M.speedup_histogram(s)
    with pytest.raises(ValueError):
        L.evaluate([], [])


def test_cost_model_helpers_match_reference(lmtune_ref, golden):
    from lmtune import cost_model as C
    from lmtune.codegen import Variant as RV
    from lmtune.kernel_model import (HomeAccessPattern, KernelInstance, LaunchConfig, StencilPattern,
                                     StencilShape, TemplateParams)

    for r in golden["interp"][:60]:
        ours = make_instance(r)
        p = TemplateParams(r["in_h"], r["in_w"], r["out_h"], r["out_w"], HomeAccessPattern(r["pattern"]), r["n"],
                           r["m"], StencilPattern(StencilShape(r["shape"]), r["radius"]), r["num_comp_ilb"],
                           r["num_comp_ep"], r["num_coal_ilb"], r["num_coal_ep"], r["num_uncoal_ilb"],
                           r["num_uncoal_ep"])
        ref = KernelInstance(p, LaunchConfig(r["grid_x"], r["grid_y"], r["wg_x"], r["wg_y"]))
        for ov, rv in ((L.Variant.BASELINE, RV.BASELINE), (L.Variant.OPTIMIZED, RV.OPTIMIZED)):
            assert L.estimate_registers(ours.params, ov) == C.estimate_registers(p, rv)
            u, ru = L.resource_usage(ours, ov), C.resource_usage(ref, rv)
            assert (u.regs_per_thread, u.lmem_per_wg, u.wg_size, u.warps_per_wg) == \
                (ru.regs_per_thread, ru.lmem_per_wg, ru.wg_size, ru.warps_per_wg)
            assert L.occupancy(u) == C.occupancy(ru)


def test_emitted_source_is_what_nvrtc_compiles(golden):
    r = golden["interp"][7]
    inst = make_instance(r)
    src = L.emit_baseline(inst)
    d = dict(src.compile_defines)
    assert d["LMT_CI"] == r["num_comp_ilb"] and d["LMT_NC"] == r["num_coal_ilb"] and d["LMT_OPT"] == 0
    assert src.entry_name == "lmt_kernel" and "extern \"C\" __global__" in src.source_text
    assert L.defines_manifest(src).startswith("-D LMT_SHAPE=")
    assert L.kernel_filename(inst.params, L.Variant.OPTIMIZED).endswith("_optimized.cu")
    opt = L.emit_optimized(inst)
    assert dict(opt.compile_defines)["LMT_OPT"] == 1
    nvrtc = "/usr/local/cuda/lib64/libnvrtc.so"
    if not os.path.exists(nvrtc):
        pytest.skip("no NVRTC")
    nv = ctypes.CDLL(nvrtc)
    for s in (src, opt):
        prog = ctypes.c_void_p()
        assert nv.nvrtcCreateProgram(ctypes.byref(prog), s.source_text.encode(), b"k.cu", 0, None, None) == 0
        opts = (ctypes.c_char_p * 2)(b"-arch=sm_100a", b"-std=c++17")
        assert nv.nvrtcCompileProgram(prog, 2, opts) == 0
        nv.nvrtcDestroyProgram(ctypes.byref(prog))


def test_emit_optimized_infeasible(golden):
    P, S = L.HomeAccessPattern, L.StencilShape
    p = L.TemplateParams(2048, 2048, 2048, 2048, P.NO_REUSE_ROW_MAJOR, 8, 8, L.StencilPattern(S.STAR, 0),
                         5, 1, 0, 0, 0, 0)
    with pytest.raises(L.OptimizationInfeasible):
        L.emit_optimized(L.KernelInstance(p, L.LaunchConfig(2048, 2048, 32, 32)))


def test_shared_load_paths_are_exercised_by_the_goldens(golden):
    """LMT_SHARE (one load per tap for a group of work units with the same
    home coordinate) is off in the literal kernels (the measurement
    contract), only ever enabled for xy_reuse / x_reuse_* in the register-
    blocked ones, and the golden parity set (run bitwise on the GPU in both
    modes) reaches it for both kinds, in both variants."""
    seen = {}
    for r in golden["interp"]:
        inst = make_instance(r)
        assert dict(L.emit_baseline(inst).compile_defines)["LMT_SHARE"] == 0
        for variant, src in (("base", L.emit_baseline(inst, regblock=True)), ("opt", None)):
            if variant == "opt":
                try:
                    src = L.emit_optimized(inst, regblock=True)
                    assert dict(L.emit_optimized(inst).compile_defines)["LMT_SHARE"] == 0
                except L.OptimizationInfeasible:
                    continue
            d = dict(src.compile_defines)
            if d["LMT_SHARE"]:
                assert r["pattern"] in ("xy_reuse", "x_reuse_row", "x_reuse_col"), r
                assert d["LMT_U"] > 1
                seen.setdefault((variant, r["pattern"] == "xy_reuse"), 0)
                seen[(variant, r["pattern"] == "xy_reuse")] += 1
    assert set(seen) == {("base", True), ("base", False), ("opt", True), ("opt", False)}, seen
