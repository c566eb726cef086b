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

import csv
from dataclasses import dataclass

import numpy as np

from .access_analysis import FEATURE_NAMES, STATUS_INVALID, STATUS_UNSUPPORTED, FeatureVector, features_records
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


# ------------------------------------------------------------ dataset files (dataset.py:284-410)

KEY_COLUMNS = (
    "pattern", "stencil_shape", "stencil_radius", "n", "m", "in_h", "in_w", "out_h", "out_w",
    "num_comp_ilb", "num_comp_ep", "num_coal_ilb", "num_coal_ep", "num_uncoal_ilb", "num_uncoal_ep",
    "grid_x", "grid_y", "wg_x", "wg_y",
)
CSV_HEADER = KEY_COLUMNS + FEATURE_NAMES + ("speedup", "beneficial")


def _key_fields(p, lc) -> list:
    return [getattr(p.pattern, "value", p.pattern), getattr(p.stencil.shape, "value", p.stencil.shape),
            str(p.stencil.radius), str(p.n), str(p.m), str(p.in_h), str(p.in_w), str(p.out_h), str(p.out_w),
            str(p.num_comp_ilb), str(p.num_comp_ep), str(p.num_coal_ilb), str(p.num_coal_ep),
            str(p.num_uncoal_ilb), str(p.num_uncoal_ep), str(lc.grid_x), str(lc.grid_y), str(lc.wg_x), str(lc.wg_y)]


def write_rows(path, rows) -> None:
    """The 39-column CSV (header, then one row per labelled instance; floats
    as repr, so the file round-trips bit-exactly), byte-identical to
    dataset.write_rows (dataset.py:308-341)."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for row in rows:
            inst = row.instance
            feats = [repr(float(v)) for v in row.features.to_array()]
            w.writerow(_key_fields(inst.params, inst.launch) + feats +
                       [repr(float(row.speedup)), "1" if row.beneficial else "0"])


def write_arrays(path, a: DatasetArrays, rows=None) -> int:
    """write_rows for a DatasetArrays (no per-row objects): the ok rows, or
    the given row indices, in table order. Returns the number of rows."""
    from .kernel_model import PATTERN_ORDER, SHAPE_ORDER

    idx = np.nonzero(a.ok)[0] if rows is None else np.asarray(rows)
    rec = a.records[idx].tolist()
    X = a.X[idx].tolist()
    sp = a.speedup[idx].tolist()
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for r, x, y in zip(rec, X, sp):
            key = [PATTERN_ORDER[r[4]], SHAPE_ORDER[r[7]], str(r[8]), str(r[5]), str(r[6]), str(r[0]), str(r[1]),
                   str(r[2]), str(r[3])] + [str(v) for v in r[9:19]]
            w.writerow(key + [repr(v) for v in x] + [repr(y), "1" if y > 1.0 else "0"])
    return len(idx)


def _parse_row(fields):
    from .kernel_model import (HomeAccessPattern, KernelInstance, LaunchConfig, StencilPattern, StencilShape,
                               TemplateParams)

    it = iter(fields)
    nxt = it.__next__
    pattern = HomeAccessPattern(nxt())
    shape = StencilShape(nxt())
    radius = int(nxt())
    n, m = int(nxt()), int(nxt())
    in_h, in_w, out_h, out_w = int(nxt()), int(nxt()), int(nxt()), int(nxt())
    counts = [int(nxt()) for _ in range(6)]
    launch = LaunchConfig(int(nxt()), int(nxt()), int(nxt()), int(nxt()))
    params = TemplateParams(in_h, in_w, out_h, out_w, pattern, n, m, StencilPattern(shape, radius), *counts)
    features = FeatureVector.from_array([float(nxt()) for _ in range(len(FEATURE_NAMES))])
    speedup = float(nxt())
    flag = nxt()
    if flag not in ("0", "1"):
        raise ValueError(f"beneficial flag {flag!r} is not 0 or 1")
    return LabeledInstance(KernelInstance(params, launch), features, speedup, flag == "1")


def read_rows(path) -> list:
    """dataset.read_rows (dataset.py:381-404): malformed content raises
    DatasetFormatError naming the line."""
    rows = []
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        try:
            header = next(reader)
        except StopIteration:
            raise DatasetFormatError("line 1: missing header") from None
        if tuple(header) != CSV_HEADER:
            raise DatasetFormatError(f"line 1: header {header[:3]}... does not match schema")
        for lineno, fields in enumerate(reader, start=2):
            if not fields:
                continue
            if len(fields) != len(CSV_HEADER):
                raise DatasetFormatError(f"line {lineno}: expected {len(CSV_HEADER)} fields, got {len(fields)}")
            try:
                rows.append(_parse_row(fields))
            except ValueError as exc:
                raise DatasetFormatError(f"line {lineno}: {exc}") from None
    return rows


def write_skip_log(path, skips) -> None:
    """dataset.py:407-410."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        for key, reason in skips:
            fh.write(f"{key}\t{reason}\n")


# ------------------------------------------------------------ sharded sweeps

def shard_path(path_prefix: str, rank: int, world: int) -> str:
    return f"{path_prefix}.shard{rank:03d}-of-{world:03d}.csv"


def write_shard(path_prefix: str, a: DatasetArrays, rows, rank: int, world: int) -> str:
    """One rank's rows of a sharded sweep, in the reference's CSV schema. A
    rank that crashes loses only its own file; `merge_shards` restores the
    table order."""
    path = shard_path(path_prefix, rank, world)
    tmp = path + ".tmp"
    write_arrays(tmp, a, rows)
    import os

    os.replace(tmp, path)
    return path


def merge_shards(path_prefix: str, world: int, out_path: str, table) -> int:
    """Concatenate the per-rank CSVs into one file ordered like the selection
    (dataset.py's canonical instance-key order); returns the row count."""
    from .kernel_model import PATTERN_ORDER, SHAPE_ORDER

    order = {}
    rec = table.records()
    for i, r in enumerate(rec.tolist()):
        order[tuple(r)] = i
    lines = []
    for rank in range(world):
        with open(shard_path(path_prefix, rank, world), encoding="utf-8", newline="") as fh:
            rd = csv.reader(fh)
            header = next(rd)
            if tuple(header) != CSV_HEADER:
                raise DatasetFormatError(f"shard {rank}: header does not match schema")
            for f in rd:
                if not f:
                    continue
                key = (int(f[5]), int(f[6]), int(f[7]), int(f[8]), PATTERN_ORDER.index(f[0]), int(f[3]), int(f[4]),
                       SHAPE_ORDER.index(f[1]), int(f[2])) + tuple(int(x) for x in f[9:19])
                lines.append((order[key], f))
    lines.sort(key=lambda x: x[0])
    with open(out_path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for _, f in lines:
            w.writerow(f)
    return len(lines)
