"""Benchmark: synthetic instances timed per second (both variants) on the
full synthetic sweep (BASELINE.json configs[4]; the single-GPU line is the
same sweep at N=1), plus the HBM roofline of the synthetic-kernel launches.

A *step* is one batch of sweep instances per rank: for each instance the
inputs are generated on the device (K0), the baseline (K1) and the
local-memory variant (K2) are each run once and timed with CUDA events, and
the two outputs are digested and compared bit for bit on the device.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): each step's global batch of N*B
instances is split across ranks by estimated cost (no data-path
collective); the per-instance labels (t_base, t_opt) are all-gathered over
NCCL after the timed region, as SURVEY 8(e) prescribes.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SWEEP_CAP = 1_000_000
# collectives: NCCL over NVLink between GPUs; LMT_DIST_BACKEND=gloo runs the
# same multi-rank code with host tensors (e.g. several ranks on one GPU)
BACKEND = os.environ.get("LMT_DIST_BACKEND", "nccl")
COLL = "cuda" if BACKEND == "nccl" else "cpu"
METRIC = "synthetic instances timed/sec (both variants)"
UNIT = "instances/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=96, help="instances per rank per step")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-rf", action="store_true")
    ap.add_argument("--no-real", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dump", default=None, help="save per-instance records and measurements (npz)")
    return ap.parse_args()


# ---------------------------------------------------------------- workload

def workload(seed: int):
    import paper_1412_6986_b200 as L

    spec = L.SamplingSpec(max_instances=SWEEP_CAP, seed=seed)
    table = L.select_instance_table(spec)
    perm = np.random.default_rng(seed ^ 0x5EED).permutation(len(table))
    return L, table, perm


def step_rows(perm, step: int, world: int, batch: int):
    g = perm[(step * world * batch) % len(perm):][: world * batch]
    return g


_SHARES = {}


def shard_for_rank(L, table, perm, step: int, world: int, rank: int, batch: int):
    """This rank's share of step `step`'s global batch. Steps are assigned in
    order with the predicted per-rank load carried over (longest-processing-
    time on the launch-floor cost), identically on every rank, so the ranks
    stay balanced over the whole run; memoised so every pass over a step
    (compile, warm-up, timed, e2e) sees the same share."""
    key = (world, rank, batch)
    if key not in _SHARES:
        _SHARES[key] = ([], np.zeros(world))
    shares, loads = _SHARES[key]
    while len(shares) <= step:
        s = len(shares)
        shares.append(L.dist.rank_rows(table, step_rows(perm, s, world, batch), world, rank, loads))
    return shares[step]


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i", str(self.index),
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:6]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------- CPU legs

def cpu_sample(L, table, rows, budget_s: float):
    """The reference's CPU path (the oracle's plain-C restatement of
    interp.execute, both variants) timed on a bounded sample of every
    instance of the batch: the first `units` work units of workgroup 0 per
    variant on one thread, extrapolated linearly to all out_h * out_w work
    units and then divided by the host's core count (perfect parallel
    scaling over workgroups -- optimistic for the CPU). Returns
    (instances/s, cores, description)."""
    import oracle

    cores = os.cpu_count() or 1
    total_s, n_inst, spent, units_done = 0.0, 0, 0.0, 0
    t_start = time.perf_counter()
    for r in rows:
        inst = table.instance(int(r))
        geo = L.emit_geometry(inst)
        p = inst.params
        a = np.zeros((geo.alloc_h, geo.alloc_w), dtype=np.float32)  # calloc'd: only touched pages exist
        b = oracle.hash_fill(p.in_h * p.in_w, 1).reshape(p.in_h, p.in_w)
        feasible = L.footprint(inst).bytes <= 48 * 1024
        units = 64
        t_inst = 0.0
        for variant in ((0, 1) if feasible else (0,)):
            t0 = time.perf_counter()
            done = oracle.execute_sample(inst, variant, a, b, max_units=units)
            dt = time.perf_counter() - t0
            t_inst += dt * (p.out_h * p.out_w) / max(done, 1)
            units_done += done
        total_s += t_inst
        n_inst += 1
        if time.perf_counter() - t_start > budget_s:
            break
    spent = time.perf_counter() - t_start
    rate = n_inst / (total_s / cores) if total_s > 0 else 0.0
    desc = (f"oracle C port of interp.execute: {n_inst} instances of the timed batch, both variants, the first 64 "
            f"work units of workgroup 0 each ({units_done} units, {spent:.1f} s), extrapolated to all work units "
            f"and divided by {cores} cores (perfect scaling assumed)")
    return rate, cores, desc


def bench_config(args, world: int) -> dict:
    """The workload both arms report (BASELINE.json configs[4] at N ranks)."""
    return {
        "workload": f"full synthetic sweep SamplingSpec(max_instances={SWEEP_CAP}, seed={args.seed}); "
                    f"each step a seeded-random batch of {args.batch} instances per rank (both variants each)",
        "batch_per_rank": args.batch, "out": "2048x2048", "parallelism": f"dp{world} (cost-balanced shards)",
        "l2": "per-step working set >> 126 MB L2 (each instance writes 2x16 MB outputs plus its inputs)",
    }


def fp32_peak_tflops():
    """fp32 FMA peak: measured by tools/probes/fp32_peak.cu on this pool's
    B200 (profiles/fp32_peak.json), else the nominal 148 SMs x 128 lanes x 2
    flops x 1.965 GHz."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp32_peak.json")))
        return float(d["fp32_fma_tflops"]), "measured (profiles/fp32_peak.json)"
    except (OSError, ValueError, KeyError):
        return 148 * 128 * 2 * 1.965e9 / 1e12, "nominal (148 SMs x 128 lanes x 2 x 1.965 GHz)"


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    L, table, perm = workload(args.seed)
    rates = []
    for s in range(args.warmup + args.steps):
        rows = step_rows(perm, s, 1, args.batch)
        rate, cores, desc = cpu_sample(L, table, rows, budget_s=max(2.0, args.cpu_seconds / max(1, args.steps)))
        if s >= args.warmup:
            rates.append(rate)
    value = float(np.mean(rates)) if rates else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": (args.batch / value * 1e3) if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU leg

def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    L, table, perm = workload(args.seed)
    from paper_1412_6986_b200 import _lib

    lib_stream = torch.cuda.ExternalStream(_lib.library_stream())

    def barrier():
        if world > 1:
            dist.barrier()

    # compile + load every specialised kernel the run will launch (NVRTC,
    # sm_100a; the reference's per-kernel compile step), before any timing
    t_prep = time.perf_counter()
    all_rows = np.concatenate([shard_for_rank(L, table, perm, s, world, rank, args.batch)
                               for s in range(args.warmup + args.steps)])
    n_kernels = L.prepare_records(table.records(all_rows))
    t_prep = time.perf_counter() - t_prep
    jit_compiled, jit_seconds = _lib.jit_stats()

    for s in range(args.warmup):
        rows = shard_for_rank(L, table, perm, s, world, rank, args.batch)
        L.measure_records(table.records(rows))

    # ---- timed region: device-resident inputs (generated by K0 inside the step)
    results = []
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        ev0.record(lib_stream)
        for s in range(args.warmup, args.warmup + args.steps):
            rows = shard_for_rank(L, table, perm, s, world, rank, args.batch)
            res = L.measure_records(table.records(rows))
            results.append((rows, res))
        ev1.record(lib_stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([elapsed_ms], device=COLL, dtype=torch.float64)
    n_local = sum(len(r) for r, _ in results)
    cnt = torch.tensor([n_local], device=COLL, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    max_ms = float(t.item())
    n_total = int(cnt.item())
    value = n_total / (max_ms / 1e3)

    # ---- labels: NCCL all-gather of (row, t_base, t_opt) -- the only collective
    rows_all = np.concatenate([r for r, _ in results])
    res_all = np.concatenate([x for _, x in results])
    labels = L.dist.all_gather_labels(L.dist.label_matrix(rows_all, res_all), device=COLL)
    n_labels = int(labels.shape[0])

    # ---- per-kernel accounting (the synthetic kernels are the dominant launches)
    ok = res_all["t_base_ms"] > 0
    ran_opt = res_all["t_opt_ms"] > 0
    k_ms = float(res_all["t_base_ms"][ok].sum() + res_all["t_opt_ms"][ran_opt].sum())
    k_bytes = float(res_all["alg_bytes"][ok].sum() + res_all["alg_bytes"][ran_opt].sum())
    k_flops = float(res_all["alg_flops"][ok].sum() + res_all["alg_flops"][ran_opt].sum())
    n_launch_kernels = int(ok.sum() + ran_opt.sum())
    fill_ms = float(res_all["t_fill_ms"].sum())
    counts = torch.tensor([((res_all["mismatches"] == 0) & ran_opt).sum(), ((res_all["mismatches"] > 0) & ran_opt).sum(),
                           (~ok).sum(), int(res_all["launches"].sum())], device=COLL, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    verified, mismatched, failed, launches_all = (int(v) for v in counts.tolist())
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    fp32_peak, fp32_src = fp32_peak_tflops()
    roof = L.measure.roofline(res_all, hbm_peak, fp32_peak)
    floor = L.measure.launch_floor(table.records(rows_all), res_all, hbm_peak)
    gpu_launches = launches_all
    if args.dump:
        np.savez(args.dump if world == 1 else f"{args.dump}.rank{rank}", rows=rows_all,
                 rec=table.records(rows_all), res=res_all)

    # ---- end to end: host (pinned) inputs -> H2D -> K1, K2, digest -> D2H outputs
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, L, table, perm, world, rank, barrier)
    rf = None if args.no_rf else run_rf(args, L, world, rank, barrier)
    real = None if (args.no_real or rank != 0) else run_real(args, L, hbm_peak, fp32_peak)

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu:
        rows0 = step_rows(perm, args.warmup, world, args.batch)
        rate, cores, desc = cpu_sample(L, table, rows0, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args, world),
        "instances_timed": n_total, "labels_gathered": n_labels, "verified_bitwise": verified,
        "mismatched": mismatched, "failed": failed,
        "kernel_ms": k_ms, "fill_ms": fill_ms, "step_ms_total": max_ms,
        "roofline": dict(roof, traffic=None, peak_source={"hbm": hbm_src, "fp32": fp32_src},
                         kernel="lmt_kernel (K1 baseline + K2 optimized, NVRTC-specialised), all launches of the "
                                "timed steps",
                         note="per launch: algorithmic bytes 4*(|U_in|+|U_in2|+out) at the HBM peak vs algorithmic "
                              "flops (MAD=2) at the fp32 peak, SURVEY 8(d); achieved/frac on the dominant roof, "
                              "frac_of_binding = sum of per-launch roof times / sum of measured times"),
        "launch_floor": dict(floor, note="per launch max(HBM bytes/peak, per-thread chain floor, per-SM issue "
                                         "floor) with the workgroup->CTA mapping fixed (sweep.floor_seconds); frac "
                                         "= sum of floors / sum of measured kernel times"),
        "gpu_launches": gpu_launches,
        "jit": {"kernels": n_kernels, "compiled": jit_compiled, "compile_s": round(jit_seconds, 2),
                "prepare_wall_s": round(t_prep, 2),
                "note": "NVRTC sm_100a specialisation per compile tuple, done before the timed region"},
        "clocks": clocks.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if rf:
        line["rf"] = rf
    if real:
        line["real_kernels"] = real
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_real(args, L, hbm_peak: float, fp32_peak: float):
    """BASELINE config 2: the real-kernel set (transpose, matrixMul,
    convolution-separable, MVT; K5) in both variants on this GPU, one warm-up
    pass then one measured pass; per kernel the best launch of each variant on
    its roof (transpose/convolution/MVT: HBM bytes; matrixMul: fp32 flops)."""
    R = L.real
    insts = R.instance_set()
    R.measure(insts)  # warm-up
    ms = R.measure(insts)
    out = {"instances": len(insts), "verified_bitwise": int((ms["mismatches"] == 0).sum()),
           "sizes": {"transpose": 2048, "matrixMul": 1024, "convolution-separable": 2048, "MVT": 4096}}
    for k, name in enumerate(R.KERNELS):
        sel = np.array([i.kernel == k and i.n <= 4096 for i in insts])
        m = ms[sel]
        sub = [i for i in insts if i.kernel == k]
        entry = {"instances": int(sel.sum())}
        for col, var in (("t_base_ms", "baseline"), ("t_opt_ms", "optimized")):
            j = int(np.argmin(m[col]))
            t = float(m[col][j]) / 1e3
            i = sub[j]
            if k == 1:
                entry[var] = {"best_ms": t * 1e3, "tflops": m["alg_flops"][j] / t / 1e12,
                              "frac": m["alg_flops"][j] / t / 1e12 / fp32_peak,
                              "config": f"tile {i.tile} wg {i.wg_x}x{i.wg_y}"}
            else:
                entry[var] = {"best_ms": t * 1e3, "gbs": m["alg_bytes"][j] / t / 1e9,
                              "frac": m["alg_bytes"][j] / t / 1e9 / hbm_peak,
                              "config": f"wg {i.wg_x}x{i.wg_y}" + (f" tile {i.tile}" if i.tile else "")
                                        + (f" radius {i.radius}" if i.radius else "")}
        big = [(i, mm) for i, mm in zip(insts, ms) if i.kernel == k and i.n > 4096]
        if big:  # the HBM-scale instances on their own
            for col, var in (("t_base_ms", "baseline"), ("t_opt_ms", "optimized")):
                i, mm = min(big, key=lambda x: x[1][col])
                t = float(mm[col]) / 1e3
                entry[f"{var}_8192"] = {"best_ms": t * 1e3, "gbs": mm["alg_bytes"] / t / 1e9,
                                        "frac": mm["alg_bytes"] / t / 1e9 / hbm_peak,
                                        "config": f"wg {i.wg_x}x{i.wg_y}" + (f" radius {i.radius}" if i.radius else "")}
        sp = m["t_base_ms"] / m["t_opt_ms"]
        entry["speedup_opt_over_base"] = {"min": float(sp.min()), "median": float(np.median(sp)),
                                          "max": float(sp.max())}
        out[name] = entry
    return out


def run_rf(args, L, world, rank, barrier):
    """BASELINE config 4 beside the sweep: the reference model trained on 10%
    of a 100k sweep (tests/golden/forest_sweep100k.txt.gz, made by the
    reference), the held-out 90% featurised on the GPU (K4) and predicted (K3);
    predictions checked bitwise against the reference's. Rows shard
    contiguously across ranks; times are max over ranks."""
    import gzip
    import hashlib
    import tempfile

    import torch
    import torch.distributed as dist

    gdir = os.path.join(ROOT, "tests", "golden")
    ev = np.load(os.path.join(gdir, "forest_sweep100k_eval.npz"))
    with gzip.open(os.path.join(gdir, "forest_sweep100k.txt.gz"), "rb") as fh, \
            tempfile.NamedTemporaryFile(suffix=".txt", delete=False) as out:
        out.write(fh.read())
    forest = L.load(out.name)
    os.unlink(out.name)
    table = L.select_instance_table(L.SamplingSpec(max_instances=100_000, seed=0))
    held = ev["held_idx"]
    mine = np.array_split(held, world)[rank]
    rec = table.records(mine)
    L.features_records(rec[:64])  # warm-up
    barrier()
    t0 = time.perf_counter()
    fb = L.features_records(rec)
    t_feat = time.perf_counter() - t0
    g = L.forest.gpu_forest(forest)
    X_t = torch.tensor(fb.X, device="cuda")
    out_t = torch.empty(len(mine), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(3):
        g.mean_device(X_t, out_t, stream=stream.cuda_stream)
    reps = max(3, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    for _ in range(reps):
        g.mean_device(X_t, out_t, stream=stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t_k3 = e0.elapsed_time(e1) / 1e3 / reps
    t0 = time.perf_counter()
    pred = L.predict(forest, fb.X)  # host X in, host predictions out (2 ** mean in numpy)
    t_e2e = time.perf_counter() - t0
    train_info = {}
    if rank == 0:  # the native trainer on the GPU-featurised 10% (forest.train, bit-exact)
        tr = L.features_records(table.records(ev["train_idx"]))
        y = np.array([L.speedup_to_target(v) for v in tr.label])
        t0 = time.perf_counter()
        trained = L.train_arrays(tr.X, y, L.Hyperparams(num_trees=20, features_per_node=4, seed=0),
                                 threads=min(20, os.cpu_count() or 1))
        t_train = time.perf_counter() - t0
        trained = L.Forest(trained.hyperparams, forest.feature_names, trained.trees)
        with tempfile.NamedTemporaryFile(suffix=".txt", delete=False) as tmpf:
            pass
        L.save(trained, tmpf.name)
        with gzip.open(os.path.join(gdir, "forest_sweep100k.txt.gz"), "rb") as fh:
            same = open(tmpf.name, "rb").read() == fh.read()
        os.unlink(tmpf.name)
        train_info = {"train_s": t_train, "train_rows": int(len(y)), "train_threads": min(20, os.cpu_count() or 1),
                      "trained_model_file_bitwise_reference": same}
    t = torch.tensor([t_feat, t_k3, t_e2e], dtype=torch.float64, device=COLL)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_feat, t_k3, t_e2e = (float(v) for v in t.tolist())
    out = {"workload": "config 4: reference forest (20 trees, 4 features/node, trained on 10% of "
                       "SamplingSpec(100k, seed=0)), held-out 90% = 90,000 rows",
           "trees": len(forest.trees), "nodes": int(sum(len(tr.feature) for tr in forest.trees)),
           "rows": int(len(held)), "k3_rows_per_s": len(held) / t_k3,
           "predict_e2e_rows_per_s": len(held) / t_e2e, "k4_features_rows_per_s": len(held) / t_feat,
           **train_info}
    if world == 1:
        out["features_bitwise_reference"] = hashlib.sha256(fb.X.tobytes()).digest() == ev["X_sha256"].tobytes()
        out["predictions_bitwise_reference"] = bool(
            hashlib.sha256(pred.tobytes()).digest() == ev["pred_sha256"].tobytes()
            and np.array_equal(pred[::8], ev["pred_every8"]))
        if not args.no_cpu and rank == 0:
            import oracle

            n = min(len(held), 20000)
            t0 = time.perf_counter()
            oracle.forest_mean(forest.trees, fb.X[:n], nthreads=1)
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": n / dt, "unit": "rows/s", "cores": 1, "kind": "port",
                                   "sample": f"oracle C port of forest.predict's tree walk on {n} held-out rows"}
    return out


def run_e2e(args, L, table, perm, world, rank, barrier):
    """Same metric through the public host-buffer API: each instance's `in`
    and `in2` come from pinned host memory and both outputs go back to pinned
    host memory inside the timed region."""
    import torch

    steps = range(args.warmup, args.warmup + args.steps)  # the same steps as the device-timed region
    plan = []
    host_in = {}
    in2_host = None
    pinned_bytes = 0
    for s in steps:
        rows = shard_for_rank(L, table, perm, s, world, rank, args.batch)
        insts = table.instances(rows)
        keep = []
        for inst in insts:
            g = L.emit_geometry(inst)
            if g.alloc_h * g.alloc_w * 4 > 2**30 + 2**28:
                continue
            key = (g.alloc_h, g.alloc_w)
            if key not in host_in:
                dev = L.interp.device_fill(g.alloc_h, g.alloc_w, 0)[:, : g.alloc_w]
                h = torch.empty((g.alloc_h, g.alloc_w), dtype=torch.float32, pin_memory=True)
                h.copy_(dev)
                host_in[key] = h
                pinned_bytes += h.numel() * 4
            keep.append((inst, host_in[key]))
        plan.append(keep)
    p0 = plan[0][0][0].params
    in2_host = torch.empty((p0.in_h, p0.in_w), dtype=torch.float32, pin_memory=True)
    in2_host.copy_(L.interp.device_fill(p0.in_h, p0.in_w, 1)[:, : p0.in_w])
    out_b = torch.empty((p0.out_h, p0.out_w), dtype=torch.float32, pin_memory=True)
    out_o = torch.empty_like(out_b)
    torch.cuda.synchronize()
    barrier()
    h2d = d2h = n = 0
    t0 = time.perf_counter()
    for keep in plan:
        insts = [i for i, _ in keep]
        ins = [h for _, h in keep]
        ms = L.measure_instances_host(insts, ins, [in2_host] * len(insts), out_base=[out_b] * len(insts),
                                      out_opt=[out_o] * len(insts))
        for m, h in zip(ms, ins):
            h2d += h.numel() * 4 + in2_host.numel() * 4
            d2h += out_b.numel() * 4 * (2 if m.t_opt_ms is not None else 1)
        n += len(insts)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    import torch.distributed as dist

    t = torch.tensor([el, float(n)], device=COLL, dtype=torch.float64)
    if world > 1:
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        el, n_all = float(mx.item()), float(t[1].item())
    else:
        n_all = float(n)
    return {"value": n_all / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d / len(plan)),
            "d2h_bytes_per_step": int(d2h / len(plan)), "steps": len(plan),
            "note": "wall clock around synchronous C-ABI calls (lmt_measure_batch_host) with pinned host buffers"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank % max(1, torch.cuda.device_count()))
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # LMT_DIST_BACKEND=gloo: exercise the multi-rank path with several ranks on one GPU
            dist.init_process_group(BACKEND)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
