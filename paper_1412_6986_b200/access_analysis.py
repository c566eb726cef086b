"""Per-instance feature vector and modelled label, computed on the GPU (K4)
behind the reference's ``access_analysis`` / ``cost_model`` signatures
(access_analysis.py:216-308, cost_model.py:28-158).

``features_records`` is the batched entry point the sweep uses: one warp per
instance (``lmt_features`` in liblmt_b200.so) produces the 18 features in
``FEATURE_NAMES`` order and ``label_speedup`` with the coalescing override
``build_dataset`` passes (dataset.py:264-271), bit-identical to the
reference. The single-instance functions below run the same kernel on a batch
of one.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields

import numpy as np

from ._lib import CDevice, check, lib
from .device import DEFAULT_DEVICE, device_tuple
from .errors import InvalidInstance, OptimizationInfeasible
from .kernel_model import validate_instance

FEATURE_NAMES = (
    "reuse_degree",
    "lmem_bytes",
    "noncoalescing_degree",
    "num_target_accesses",
    "offset_min_row",
    "offset_max_row",
    "offset_min_col",
    "offset_max_col",
    "comp_ilb",
    "comp_ep",
    "ctx_coal_ilb",
    "ctx_uncoal_ilb",
    "ctx_coal_ep",
    "ctx_uncoal_ep",
    "regs_per_thread",
    "grid_size",
    "wg_size",
    "wus_per_workitem",
)

STATUS_OK, STATUS_INVALID, STATUS_INFEASIBLE, STATUS_UNSUPPORTED = 0, 1, 2, 5


@dataclass(frozen=True)
class FeatureVector:
    """The 18 features of one instance, in FEATURE_NAMES order (access_analysis.py:238-269)."""

    reuse_degree: float
    lmem_bytes: float
    noncoalescing_degree: float
    num_target_accesses: float
    offset_min_row: float
    offset_max_row: float
    offset_min_col: float
    offset_max_col: float
    comp_ilb: float
    comp_ep: float
    ctx_coal_ilb: float
    ctx_uncoal_ilb: float
    ctx_coal_ep: float
    ctx_uncoal_ep: float
    regs_per_thread: float
    grid_size: float
    wg_size: float
    wus_per_workitem: float

    def to_array(self) -> np.ndarray:
        return np.array([getattr(self, f.name) for f in fields(self)], dtype=np.float64)

    @classmethod
    def from_array(cls, arr) -> "FeatureVector":
        vals = [float(x) for x in arr]
        if len(vals) != len(FEATURE_NAMES):
            raise ValueError(f"expected {len(FEATURE_NAMES)} features, got {len(vals)}")
        return cls(*vals)


@dataclass(frozen=True)
class TimeEstimate:
    """cost_model.py:34-38."""

    compute_cycles: float
    mem_transactions: float
    active_warps: float
    total_cycles: float


@dataclass
class FeatureBatch:
    X: np.ndarray        # float64 [n, 18]
    label: np.ndarray    # float64 [n] (0.0 infeasible, NaN invalid)
    times: np.ndarray    # float64 [n, 8]: baseline then optimized TimeEstimate fields
    status: np.ndarray   # int32 [n]


def _c_devices(dev, n: int):
    if isinstance(dev, (list, tuple)) and dev and not isinstance(dev[0], int):
        if len(dev) != n:
            raise ValueError("one device per instance expected")
        arr = (CDevice * n)(*[CDevice(*device_tuple(d)) for d in dev])
        return arr, n
    arr = (CDevice * 1)(CDevice(*device_tuple(dev)))
    return arr, 1


def features_records(records: np.ndarray, dev=DEFAULT_DEVICE, *, coalescing_override=None,
                     lmem_override=None) -> FeatureBatch:
    """K4 over an int32 [n, 19] record table (sweep.InstanceTable.records).
    ``dev`` is one descriptor or a list with one per instance."""
    from .sweep import records_to_c

    rec = np.ascontiguousarray(records, dtype=np.int32)
    n = len(rec)
    X = np.empty((n, 18), dtype=np.float64)
    label = np.empty(n, dtype=np.float64)
    times = np.empty((n, 8), dtype=np.float64)
    status = np.empty(n, dtype=np.int32)
    if n == 0:
        return FeatureBatch(X, label, times, status)
    devs, ndev = _c_devices(dev, n)
    co = None if coalescing_override is None else np.ascontiguousarray(coalescing_override, dtype=np.float64)
    lo = None if lmem_override is None else np.ascontiguousarray(lmem_override, dtype=np.int64)
    vp = lambda a: None if a is None else ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    check(lib().lmt_features(records_to_c(rec), n, devs, ndev, vp(co), vp(lo), vp(X), vp(label), vp(times),
                             vp(status)), what="features")
    return FeatureBatch(X, label, times, status)


def features_instances(instances, dev=DEFAULT_DEVICE, **kw) -> FeatureBatch:
    from .sweep import instances_to_records

    return features_records(instances_to_records(instances), dev, **kw)


def _one(instance, dev, **kw) -> FeatureBatch:
    v = validate_instance(instance)
    if v:
        raise InvalidInstance(v)
    b = features_instances([instance], dev, **kw)
    if b.status[0] == STATUS_UNSUPPORTED:
        from .errors import LmtuneError

        raise LmtuneError("device descriptor not supported by the feature kernel")
    return b


def extract_features(instance, dev=DEFAULT_DEVICE) -> FeatureVector:
    """access_analysis.extract_features (access_analysis.py:272-308), on the GPU."""
    return FeatureVector.from_array(_one(instance, dev).X[0])


def coalescing_degree(instance, dev=DEFAULT_DEVICE) -> float:
    """Mean DRAM transactions per warp for the home access (access_analysis.py:119-155)."""
    return float(_one(instance, dev).X[0, 2])


def reuse_degree(instance) -> float:
    """access_analysis.py:74-88."""
    return float(_one(instance, DEFAULT_DEVICE).X[0, 0])


def kernel_time(instance, variant, dev=DEFAULT_DEVICE, *, coalescing_override=None, lmem_override=None) -> TimeEstimate:
    """cost_model.kernel_time (cost_model.py:94-141); raises
    OptimizationInfeasible for an optimized variant that cannot stage."""
    from .geometry import variant_id

    b = _one(instance, dev, coalescing_override=None if coalescing_override is None else [coalescing_override],
             lmem_override=None if lmem_override is None else [lmem_override])
    if variant_id(variant) == 0:
        return TimeEstimate(*[float(x) for x in b.times[0, :4]])
    if b.status[0] == STATUS_INFEASIBLE:
        from .geometry import footprint

        cap = dev.lmem_capacity_bytes
        need = footprint(instance, dev).bytes if lmem_override is None else lmem_override
        raise OptimizationInfeasible(need, cap)
    return TimeEstimate(*[float(x) for x in b.times[0, 4:]])


def label_speedup(instance, dev=DEFAULT_DEVICE, *, coalescing_override=None, lmem_override=None) -> float:
    """cost_model.label_speedup (cost_model.py:144-158): modelled T_base / T_opt, 0.0 if infeasible."""
    b = _one(instance, dev, coalescing_override=None if coalescing_override is None else [coalescing_override],
             lmem_override=None if lmem_override is None else [lmem_override])
    return float(b.label[0])


__all__ = ["FEATURE_NAMES", "FeatureVector", "TimeEstimate", "FeatureBatch", "features_records",
           "features_instances", "extract_features", "coalescing_degree", "reuse_degree", "kernel_time",
           "label_speedup"]
