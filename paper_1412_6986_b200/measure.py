"""Measured labels: run and time both variants of many instances on the GPU.

This is the B200 counterpart of the reference's *modelled* label
(cost_model.kernel_time / label_speedup, cost_model.py:94-158): instead of
estimating T_baseline / T_optimized it executes both kernels, times each with
CUDA events, and verifies that the two outputs are bitwise identical (the
reference's own invariant, test_interp.py:70-110) through on-device digests.

Failures are per instance, as in build_dataset's skip log
(dataset.py:264-281): a failing instance gets ``status != 0`` and an error
string; the batch carries on.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import (
    LMT_ERR_INFEASIBLE,
    LMT_OK,
    MEASURE_ALLOW_LARGE_LMEM,
    MEASURE_CONCURRENT,
    MEASURE_REGBLOCK,
    MEASURE_SKIP_OPT,
    MEASURE_WARM_L2,
    CMeasureOpts,
    CMeasurement,
    check,
    last_error,
    lib,
)
from .device import DEFAULT_DEVICE
from .geometry import c_device
from .kernel_model import to_c_array

STATUS_NAMES = {0: "ok", 1: "InvalidInstance", 2: "OptimizationInfeasible", 3: "CudaError",
                4: "BadArgument", 5: "TooLarge"}


@dataclass(frozen=True)
class Measurement:
    instance: object
    t_base_ms: float
    t_opt_ms: float | None          # None: optimized variant infeasible / not run
    digest_base: int
    digest_opt: int | None
    mismatches: int                 # -1 when the optimized variant did not run
    alg_bytes: float                # algorithmic bytes per variant
    alg_flops: float                # algorithmic fp32 ops per variant
    t_fill_ms: float
    status: int
    kernel_id: int
    launches: int
    nstages: int
    lane_sms: int = 0               # SM partition it ran in (0 = the whole device, L2 flushed per variant)
    order: int = 0                  # 1: the optimized variant was timed first
    in_copies: int = 1              # 4: the baseline built and read 128-bit shifted copies (inside t_base)
    ctas: int = 0

    @property
    def ok(self) -> bool:
        return self.status in (LMT_OK, LMT_ERR_INFEASIBLE) and self.t_base_ms > 0

    @property
    def verified(self) -> bool:
        """Both variants ran and agree bit for bit."""
        return self.t_opt_ms is not None and self.mismatches == 0

    @property
    def speedup(self) -> float:
        """Measured T_baseline / T_optimized; 0.0 when the optimized variant is
        infeasible, matching label_speedup's convention (cost_model.py:154-157)."""
        if self.t_opt_ms is None or self.t_opt_ms <= 0:
            return 0.0
        return self.t_base_ms / self.t_opt_ms

    @property
    def beneficial(self) -> bool:
        return self.speedup > 1.0


def _convert(instances, raw) -> list[Measurement]:
    out = []
    for inst, m in zip(instances, raw):
        ran_opt = m.t_opt_ms >= 0
        out.append(Measurement(
            instance=inst, t_base_ms=m.t_base_ms, t_opt_ms=m.t_opt_ms if ran_opt else None,
            digest_base=int(m.digest_base), digest_opt=int(m.digest_opt) if ran_opt else None,
            mismatches=int(m.mismatches), alg_bytes=m.alg_bytes, alg_flops=m.alg_flops,
            t_fill_ms=m.t_fill_ms, status=int(m.status), kernel_id=int(m.kernel_id),
            launches=int(m.launches), nstages=int(m.nstages), lane_sms=int(m.lane_sms), order=int(m.order),
            in_copies=int(m.in_copies), ctas=int(m.ctas),
        ))
    return out


def measure_flags(*, skip_opt: bool = False, allow_large_lmem: bool = False, concurrent: bool = False,
                  regblock: bool = False, warm_l2: bool = False) -> int:
    """lmt_measure_batch flags (include/lmt_b200.h). Defaults are the
    measurement contract: every instance on the whole device, L2 flushed
    before each variant, each work unit issuing its own loads."""
    return ((MEASURE_SKIP_OPT if skip_opt else 0) | (MEASURE_ALLOW_LARGE_LMEM if allow_large_lmem else 0)
            | (MEASURE_CONCURRENT if concurrent else 0) | (MEASURE_REGBLOCK if regblock else 0)
            | (MEASURE_WARM_L2 if warm_l2 else 0))


def measure_raw(instances, dev=DEFAULT_DEVICE, *, chunk: int = 4096, **kw):
    """lmt_measure_batch over ``instances``; returns the raw ctypes records."""
    flags = measure_flags(**kw)
    cdev = c_device(dev)
    res = []
    for s in range(0, len(instances), chunk):
        part = instances[s: s + chunk]
        arr = to_c_array(part)
        out = (CMeasurement * max(len(part), 1))()
        check(lib().lmt_measure_batch(arr, len(part), ctypes.byref(cdev), flags, out), what="measure_batch")
        res.extend(out[: len(part)])
    return res


def measure_records(records, dev=DEFAULT_DEVICE, *, samples: np.ndarray | None = None, tune=None, **kw):
    """Measure an int32 [n, 19] record table (sweep.InstanceTable.records);
    returns a numpy structured view of the lmt_measurement records. With
    ``samples`` (int64 [n, S] linear output indices) returns
    ``(records, values)``, values float32 [n, S, 2] = the baseline and
    optimized output at those cells, for an independent (oracle) check.
    ``tune``: kernel-shape overrides for tuning studies (lmt_measure_opts.tune:
    baseline U, D, min CTAs/SM, optimized U, slots, min CTAs/SM; 0 = auto)."""
    from .sweep import records_to_c

    n = len(records)
    arr = records_to_c(records)
    out = (CMeasurement * max(n, 1))()
    opts = CMeasureOpts(measure_flags(**kw), 0, None, None)
    if tune is not None:
        for k, v in enumerate(list(tune)[:6]):
            opts.tune[k] = int(v)
    vals = None
    if samples is not None:
        samples = np.ascontiguousarray(samples, dtype=np.int64).reshape(n, -1)
        vals = np.zeros((n, samples.shape[1], 2), dtype=np.float32)
        opts.samples = samples.shape[1]
        opts.sample_idx = samples.ctypes.data
        opts.h_sample_vals = vals.ctypes.data
    check(lib().lmt_measure_batch_ex(arr, n, ctypes.byref(c_device(dev)), ctypes.byref(opts), None, None, None,
                                     None, None, None, out), what="measure_batch")
    res = np.frombuffer(out, dtype=MEASUREMENT_DTYPE, count=n).copy()
    return res if samples is None else (res, vals)


def prepare_records(records, dev=DEFAULT_DEVICE, *, nthreads: int = 0, **kw) -> int:
    """Compile (NVRTC, sm_100a) and load every specialised kernel that
    measuring ``records`` will launch -- the reference's per-kernel compile
    step (codegen.py:150-182) -- in parallel host threads. Returns the number
    of distinct kernels the batch needs."""
    from .sweep import records_to_c

    flags = measure_flags(**kw)
    n = len(records)
    arr = records_to_c(records)
    out = ctypes.c_int64()
    check(lib().lmt_prepare(arr, n, ctypes.byref(c_device(dev)), flags, nthreads, ctypes.byref(out)),
          what="prepare")
    return int(out.value)


def prepare_instances(instances, dev=DEFAULT_DEVICE, *, nthreads: int = 0, **kw) -> int:
    """prepare_records for KernelInstance objects."""
    flags = measure_flags(**kw)
    instances = list(instances)
    out = ctypes.c_int64()
    check(lib().lmt_prepare(to_c_array(instances), len(instances), ctypes.byref(c_device(dev)), flags, nthreads,
                            ctypes.byref(out)), what="prepare")
    return int(out.value)


MEASUREMENT_DTYPE = np.dtype([
    ("t_base_ms", "f8"), ("t_opt_ms", "f8"), ("digest_base", "u8"), ("digest_opt", "u8"),
    ("mismatches", "i8"), ("alg_bytes", "f8"), ("alg_flops", "f8"), ("t_fill_ms", "f8"),
    ("status", "i4"), ("kernel_id", "i4"), ("launches", "i4"), ("nstages", "i4"),
    ("lane_sms", "i4"), ("order", "i4"), ("in_copies", "i4"), ("ctas", "i4"),
])


def measure_instances(instances, dev=DEFAULT_DEVICE, **kw) -> list[Measurement]:
    """Run, time and verify both variants of every instance on the current GPU."""
    return _convert(instances, measure_raw(list(instances), dev, **kw))


def measure_instances_host(instances, in_arrays, in2_arrays, dev=DEFAULT_DEVICE, *, out_base=None,
                           out_opt=None, samples: np.ndarray | None = None, **kw):
    """End-to-end variant: instance i's inputs come from host arrays (ideally
    pinned) and are copied to the device inside the timed batch; outputs are
    optionally copied back into ``out_base[i]`` / ``out_opt[i]``."""
    n = len(instances)
    vp = ctypes.c_void_p
    keep = []

    def ptrs(arrs, writable=False):
        if arrs is None:
            return None
        a = (vp * max(n, 1))()
        for k, x in enumerate(arrs):
            if x is None:
                a[k] = None
                continue
            if hasattr(x, "data_ptr"):
                a[k] = x.data_ptr()
            else:
                x = np.ascontiguousarray(x, dtype=np.float32) if not writable else x
                keep.append(x)
                a[k] = x.ctypes.data
        return a

    rows = (ctypes.c_int64 * max(n, 1))(*[int(x.shape[0]) for x in in_arrays])
    cols = (ctypes.c_int64 * max(n, 1))(*[int(x.shape[1]) for x in in_arrays])
    arr = to_c_array(instances)
    out = (CMeasurement * max(n, 1))()
    opts = CMeasureOpts(measure_flags(**kw), 0, None, None)
    vals = None
    if samples is not None:
        samples = np.ascontiguousarray(samples, dtype=np.int64).reshape(n, -1)
        vals = np.zeros((n, samples.shape[1], 2), dtype=np.float32)
        opts.samples = samples.shape[1]
        opts.sample_idx = samples.ctypes.data
        opts.h_sample_vals = vals.ctypes.data
    rc = lib().lmt_measure_batch_ex(arr, n, ctypes.byref(c_device(dev)), ctypes.byref(opts), ptrs(in_arrays), rows,
                                    cols, ptrs(in2_arrays), ptrs(out_base, True), ptrs(out_opt, True), out)
    check(rc, what="measure_batch_host")
    ms = _convert(instances, out[:n])
    return ms if samples is None else (ms, vals)


def launch_floor(records: np.ndarray, res: np.ndarray, hbm_gbs: float) -> dict:
    """How close the measured launches are to what their own launch shape
    allows: per launch max(HBM bytes / peak, chain floor, per-SM issue floor)
    (sweep.floor_seconds), summed over both variants, over summed measured
    time."""
    from .sweep import floor_seconds

    ch, iss = floor_seconds(records)
    fl, t, kind = [], [], []
    for col in ("t_base_ms", "t_opt_ms"):
        ran = res[col] > 0
        parts = np.stack([res["alg_bytes"][ran] / (hbm_gbs * 1e9), ch[ran], iss[ran]])
        fl.append(parts.max(0))
        kind.append(parts.argmax(0))
        t.append(res[col][ran] / 1e3)
    fl, t, kind = np.concatenate(fl), np.concatenate(t), np.concatenate(kind)
    out = {"frac": float(fl.sum() / t.sum()) if t.sum() > 0 else 0.0, "floor_s": float(fl.sum()),
           "kernel_s": float(t.sum()), "by_binding_floor": {}}
    # which floor binds each launch: HBM bytes, the per-thread chain (few
    # threads: the launch shape), or the per-SM fp32 issue
    for k, name in enumerate(("hbm", "thread_chain", "sm_issue")):
        m = kind == k
        if m.any():
            out["by_binding_floor"][name] = {"launches": int(m.sum()), "floor_s": float(fl[m].sum()),
                                             "kernel_s": float(t[m].sum()), "frac": float(fl[m].sum() / t[m].sum())}
    return out


def roofline(res: np.ndarray, hbm_gbs: float, fp32_tflops: float) -> dict:
    """Roofline accounting of measured launches (a MEASUREMENT_DTYPE array,
    both variants): each launch is bound by the slower of its
    algorithmic HBM bytes at ``hbm_gbs`` and its algorithmic fp32 flops (MAD =
    2) at ``fp32_tflops``.

    Returns the dominant roof over the set (the one that carries more of the
    summed roof time), achieved = algorithmic bytes (or flops) / summed
    kernel time against that peak, and ``frac_of_binding`` = summed per-launch
    roof time / summed measured time, i.e. how close the launches are to
    their own binding roofs."""
    t, b, f, c = [], [], [], []
    for col in ("t_base_ms", "t_opt_ms"):
        ran = res[col] > 0
        t.append(res[col][ran] / 1e3)
        b.append(res["alg_bytes"][ran])
        f.append(res["alg_flops"][ran])
        c.append(res["ctas"][ran])
    t, b, f, c = np.concatenate(t), np.concatenate(b), np.concatenate(f), np.concatenate(c)
    if t.size == 0 or t.sum() <= 0:
        return {}
    t_hbm = b / (hbm_gbs * 1e9)
    t_fp = f / (fp32_tflops * 1e12)
    roof = np.maximum(t_hbm, t_fp)
    hbm_bound = t_hbm >= t_fp
    dominant = "hbm" if roof[hbm_bound].sum() >= roof[~hbm_bound].sum() else "fp32"
    T = float(t.sum())
    out = {"bound": dominant, "launches": int(t.size), "kernel_s": T,
           "frac_of_binding": float(roof.sum() / T),
           "hbm_bound_launches": int(hbm_bound.sum()), "fp32_bound_launches": int((~hbm_bound).sum())}
    if dominant == "hbm":
        ach = float(b.sum() / T / 1e9)
        out.update(achieved=ach, peak=hbm_gbs, unit="GB/s", frac=ach / hbm_gbs)
    else:
        ach = float(f.sum() / T / 1e12)
        out.update(achieved=ach, peak=fp32_tflops, unit="TFLOP/s", frac=ach / fp32_tflops)
    if hbm_bound.any():  # the memory-bound subset on its own roof, split by whether a launch can fill the chip
        def sub(m):
            tb = float(t[m].sum())
            return {"launches": int(m.sum()), "achieved": float(b[m].sum() / tb / 1e9), "peak": hbm_gbs,
                    "unit": "GB/s", "frac": float(b[m].sum() / tb / 1e9 / hbm_gbs), "kernel_s": tb}

        out["hbm_subset"] = sub(hbm_bound)
        full = c >= 2 * 148  # at least two CTAs per SM
        for name, m in (("fills_chip", hbm_bound & full), ("cannot_fill_chip", hbm_bound & ~full)):
            if m.any():
                out["hbm_subset"][name] = sub(m)
    return out


def error_of(m: Measurement) -> str:
    return STATUS_NAMES.get(m.status, f"status {m.status}")


__all__ = ["Measurement", "roofline", "measure_instances", "measure_instances_host", "measure_raw", "prepare_records",
           "prepare_instances", "last_error"]
