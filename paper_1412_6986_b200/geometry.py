"""Geometry of the two kernel variants: the affine access table, the staging
footprint and the emitted-kernel geometry (mirrors access_analysis.py:32-62,
158-213 and codegen.py:33-139).

The integer arithmetic is done once, natively, by ``lmt_emit_geometry`` in
liblmt_b200.so -- the same routine the GPU path plans its launches with --
and is exposed here with the reference's dataclasses.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

from ._lib import CDevice, CGeometry, check, lib
from .device import DEFAULT_DEVICE, device_tuple
from .errors import InvalidInstance, OptimizationInfeasible
from .kernel_model import to_c, validate_instance


class Variant(enum.Enum):
    BASELINE = "baseline"
    OPTIMIZED = "optimized"


def variant_id(variant) -> int:
    v = getattr(variant, "value", variant)
    if v in ("baseline", 0):
        return 0
    if v in ("optimized", 1):
        return 1
    raise ValueError(f"unknown variant {variant!r}")


@dataclass(frozen=True)
class AffineAccess:
    row_wu_x: int
    row_wu_y: int
    row_i: int
    row_j: int
    col_wu_x: int
    col_wu_y: int
    col_i: int
    col_j: int


# access_analysis.py:51-62, columns: row_wu_x row_wu_y row_i row_j col_wu_x col_wu_y col_i col_j
_AFFINE = {
    "xy_reuse": lambda n, m: (0, 0, 1, 0, 0, 0, 0, 1),
    "x_reuse_row": lambda n, m: (0, 1, 0, 0, 0, 0, 0, 1),
    "x_reuse_col": lambda n, m: (0, 0, 0, 1, 0, 1, 0, 0),
    "y_reuse_row": lambda n, m: (1, 0, 0, 0, 0, 0, 0, 1),
    "y_reuse_col": lambda n, m: (0, 0, 0, 1, 1, 0, 0, 0),
    "no_reuse_row_major": lambda n, m: (0, n, 1, 0, m, 0, 0, 1),
    "no_reuse_col_major": lambda n, m: (0, m, 0, 1, n, 0, 1, 0),
}


def pattern_affine(pattern, n: int, m: int) -> AffineAccess:
    return AffineAccess(*_AFFINE[getattr(pattern, "value", pattern)](n, m))


@dataclass(frozen=True)
class Footprint:
    row_span: int
    col_span: int
    padded_col_span: int
    bytes: int


@dataclass(frozen=True)
class EmitGeometry:
    pad: int
    off_min_row: int
    off_min_col: int
    r_rows: int
    r_cols: int
    r_cols_pad: int
    seg_elems: int
    segs_per_row: int
    num_segs: int
    num_warps: int
    lanes_per_warp: int
    alloc_h: int
    alloc_w: int
    org_row_wu_x: int
    org_row_wu_y: int
    org_col_wu_x: int
    org_col_wu_y: int


def c_device(dev=DEFAULT_DEVICE) -> CDevice:
    return CDevice(*device_tuple(dev))


def raw_geometry(instance, dev=DEFAULT_DEVICE) -> CGeometry:
    g = CGeometry()
    check(lib().lmt_emit_geometry(ctypes.byref(to_c(instance)), ctypes.byref(c_device(dev)), ctypes.byref(g)),
          what="emit_geometry")
    return g


def pad_col_span(col_span: int, dev=DEFAULT_DEVICE) -> int:
    """access_analysis.py:169-181."""
    tx = dev.transaction_bytes // dev.element_bytes
    if col_span % tx == 0:
        return col_span
    if col_span > tx:
        return (col_span // tx + 1) * tx
    return 1 << (col_span - 1).bit_length()


def footprint(instance, dev=DEFAULT_DEVICE) -> Footprint:
    """Staging region of one workgroup (access_analysis.py:184-213)."""
    g = raw_geometry(instance, dev)
    return Footprint(g.r_rows, g.r_cols, g.r_cols_pad, g.footprint_bytes)


def emit_geometry(instance, dev=DEFAULT_DEVICE, fp: Footprint | None = None) -> EmitGeometry:
    """codegen.py:94-132. ``fp`` is accepted for signature parity; the region
    is always recomputed from the instance (as the reference does when None)."""
    g = raw_geometry(instance, dev)
    return EmitGeometry(**{f: getattr(g, f) for f in EmitGeometry.__dataclass_fields__})


def mad_constants(k: int) -> tuple[float, float]:
    """codegen.py:58-66: (c1, c2) of the k-th multiply-add."""
    sign = -1.0 if k & 1 else 1.0
    return (0.5 if k & 1 else 2.0), sign * (1 + k % 5) / 64.0


def copy_transaction_count(fp: Footprint, dev=DEFAULT_DEVICE) -> int:
    """codegen.py:135-139."""
    return fp.row_span * -(-fp.padded_col_span * dev.element_bytes // dev.transaction_bytes)


def check_optimizable(instance, dev=DEFAULT_DEVICE) -> Footprint:
    """The gate of emit_optimized (codegen.py:343-354): raises
    InvalidInstance / OptimizationInfeasible like the reference."""
    v = validate_instance(instance)
    if v:
        raise InvalidInstance(v)
    fp = footprint(instance, dev)
    if fp.bytes > dev.lmem_capacity_bytes:
        raise OptimizationInfeasible(fp.bytes, dev.lmem_capacity_bytes)
    return fp
