"""The labelled dataset of the instance sweep (mirrors lmtune/dataset.py:97-281
and the seeded split of cli.py:54-64).

``build_dataset`` keeps the reference's signature and result type: every
selected instance gets its 18 features and the modelled speedup label,
computed on the GPU by K4 (``lmt_features``, bit-identical to
``extract_features`` + ``label_speedup``), per-instance failures go to the
skip log. ``build_arrays`` is the same without per-row Python objects, for
million-instance sweeps.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .access_analysis import STATUS_INVALID, STATUS_UNSUPPORTED, FeatureVector, features_records
from .device import DEFAULT_DEVICE
from .errors import DatasetFormatError
from .seeding import mix_seed
from .sweep import SamplingSpec, instance_key, select_instance_table

_SPLIT_STREAM = 0x53504C49  # cli.py:51


@dataclass(frozen=True)
class LabeledInstance:
    """dataset.py:97-106."""

    instance: object
    features: FeatureVector
    speedup: float
    beneficial: bool

    def __post_init__(self):
        if self.beneficial != (self.speedup > 1.0):
            raise ValueError(f"beneficial={self.beneficial} inconsistent with speedup {self.speedup}")


@dataclass
class BuildResult:
    rows: list
    skips: list  # (instance key, reason)


@dataclass
class DatasetArrays:
    table: object          # sweep.InstanceTable
    records: np.ndarray    # int32 [n, 19]
    X: np.ndarray          # float64 [n, 18]
    speedup: np.ndarray    # float64 [n], the modelled label
    status: np.ndarray     # int32 [n]: 0 ok, 2 infeasible (label 0.0), 1 invalid, 5 unsupported

    @property
    def ok(self) -> np.ndarray:
        return (self.status != STATUS_INVALID) & (self.status != STATUS_UNSUPPORTED)


def build_arrays(spec: SamplingSpec, dev=DEFAULT_DEVICE) -> DatasetArrays:
    table = select_instance_table(spec)
    rec = table.records()
    fb = features_records(rec, dev)
    return DatasetArrays(table, rec, fb.X, fb.label, fb.status)


def build_dataset(spec: SamplingSpec, dev=DEFAULT_DEVICE, threads: int = 1) -> BuildResult:
    """dataset.build_dataset (dataset.py:253-281) with K4 on the GPU. ``threads``
    is accepted for signature compatibility; results never depend on it."""
    from ._lib import lib
    from .kernel_model import to_c

    a = build_arrays(spec, dev)
    rows, skips = [], []
    for i in range(len(a.records)):
        inst = a.table.instance(i)
        if a.status[i] == STATUS_INVALID:
            import ctypes

            buf = ctypes.create_string_buffer(4096)
            lib().lmt_validate(ctypes.byref(to_c(inst)), buf, len(buf))
            skips.append((instance_key(inst), f"InvalidInstance: {buf.value.decode()}"))
            continue
        if a.status[i] == STATUS_UNSUPPORTED:
            skips.append((instance_key(inst), "LmtuneError: device descriptor not supported"))
            continue
        sp = float(a.speedup[i])
        rows.append(LabeledInstance(inst, FeatureVector.from_array(a.X[i]), sp, sp > 1.0))
    return BuildResult(rows=rows, skips=skips)


def split_rows(rows, fraction: float, seed: int):
    """cli.split_rows (cli.py:54-64): seeded (train, held_out) partition, the
    train side gets round(fraction * n) rows clamped so both are non-empty."""
    n = len(rows)
    if n < 2:
        raise DatasetFormatError(f"need at least 2 rows to split, got {n}")
    size = max(1, min(n - 1, round(fraction * n)))
    perm = np.random.default_rng(mix_seed(seed, _SPLIT_STREAM)).permutation(n)
    train_idx = np.sort(perm[:size])
    held_idx = np.sort(perm[size:])
    return [rows[i] for i in train_idx], [rows[i] for i in held_idx]


def split_indices(n: int, fraction: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """split_rows on row indices (no per-row objects)."""
    tr, he = split_rows(np.arange(n), fraction, seed)
    return np.array(tr, dtype=np.int64), np.array(he, dtype=np.int64)
