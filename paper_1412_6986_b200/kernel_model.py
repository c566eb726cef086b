"""Domain types of the synthetic kernel family (mirrors lmtune/kernel_model.py).

Same names, fields and enum values as the reference (kernel_model.py:15-108),
so instances built against either package are interchangeable: every
function here and in the GPU path accepts any object with ``.params`` /
``.launch`` shaped like the reference's ``KernelInstance``.

Validation is delegated to the C ABI (``lmt_validate``), which is the
implementation the GPU measurement path uses as well.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class HomeAccessPattern(enum.Enum):
    XY_REUSE = "xy_reuse"
    X_REUSE_ROW = "x_reuse_row"
    X_REUSE_COL = "x_reuse_col"
    Y_REUSE_ROW = "y_reuse_row"
    Y_REUSE_COL = "y_reuse_col"
    NO_REUSE_ROW_MAJOR = "no_reuse_row_major"
    NO_REUSE_COL_MAJOR = "no_reuse_col_major"


class StencilShape(enum.Enum):
    RECTANGULAR = "rect"
    DIAMOND = "diamond"
    STAR = "star"


PATTERN_ORDER = tuple(p.value for p in HomeAccessPattern)
SHAPE_ORDER = tuple(s.value for s in StencilShape)


@dataclass(frozen=True)
class StencilPattern:
    shape: StencilShape
    radius: int

    def __post_init__(self):
        if self.radius < 0:
            raise ValueError(f"stencil radius {self.radius} < 0")


@dataclass(frozen=True)
class Coord:
    row: int
    col: int


@dataclass(frozen=True)
class TemplateParams:
    in_h: int
    in_w: int
    out_h: int
    out_w: int
    pattern: HomeAccessPattern
    n: int
    m: int
    stencil: StencilPattern
    num_comp_ilb: int
    num_comp_ep: int
    num_coal_ilb: int
    num_coal_ep: int
    num_uncoal_ilb: int
    num_uncoal_ep: int


@dataclass(frozen=True)
class LaunchConfig:
    grid_x: int
    grid_y: int
    wg_x: int
    wg_y: int

    @property
    def wg_size(self) -> int:
        return self.wg_x * self.wg_y

    @property
    def grid_size(self) -> int:
        return self.grid_x * self.grid_y


@dataclass(frozen=True)
class KernelInstance:
    params: TemplateParams
    launch: LaunchConfig

    @property
    def num_wus_x(self) -> int:
        return self.params.out_w // self.launch.grid_x

    @property
    def num_wus_y(self) -> int:
        return self.params.out_h // self.launch.grid_y

    @property
    def wus_per_workitem(self) -> int:
        return self.num_wus_x * self.num_wus_y


def is_power_of_two(v: int) -> bool:
    return v > 0 and not (v & (v - 1))


def _shape_name(s) -> str:
    return getattr(s, "value", s)


def stencil_offsets(stencil) -> list[tuple[int, int]]:
    """Row-major (d_row, d_col) offsets (kernel_model.py:115-130)."""
    r, shape = stencil.radius, _shape_name(stencil.shape)
    span = range(-r, r + 1)
    keep = {
        "rect": lambda a, b: True,
        "diamond": lambda a, b: abs(a) + abs(b) <= r,
        "star": lambda a, b: a == 0 or b == 0,
    }[shape]
    return [(a, b) for a in span for b in span if keep(a, b)]


def home_coordinate(pattern, wu: Coord, i: int, j: int, params) -> Coord:
    """Home coordinate of work unit ``wu`` at loop iteration (i, j)
    (kernel_model.py:133-155), via the affine table."""
    from .geometry import pattern_affine

    a = pattern_affine(pattern, params.n, params.m)
    return Coord(
        a.row_wu_x * wu.col + a.row_wu_y * wu.row + a.row_i * i + a.row_j * j,
        a.col_wu_x * wu.col + a.col_wu_y * wu.row + a.col_i * i + a.col_j * j,
    )


def work_unit_for(launch, params, wg: Coord, wi: Coord, it: Coord) -> Coord:
    """Blocked across workgroups, cyclic across workitems (kernel_model.py:158-170)."""
    nx, ny = params.out_w // launch.grid_x, params.out_h // launch.grid_y
    return Coord(
        row=(wg.row * ny + it.row) * launch.wg_y + wi.row,
        col=(wg.col * nx + it.col) * launch.wg_x + wi.col,
    )


def to_c(instance):
    """Flatten an instance into the C ABI record (include/lmt_b200.h)."""
    from ._lib import CInstance

    p, lc = instance.params, instance.launch
    return CInstance(
        int(p.in_h), int(p.in_w), int(p.out_h), int(p.out_w),
        PATTERN_ORDER.index(getattr(p.pattern, "value", p.pattern)), int(p.n), int(p.m),
        SHAPE_ORDER.index(_shape_name(p.stencil.shape)), int(p.stencil.radius),
        int(p.num_comp_ilb), int(p.num_comp_ep), int(p.num_coal_ilb), int(p.num_coal_ep),
        int(p.num_uncoal_ilb), int(p.num_uncoal_ep),
        int(lc.grid_x), int(lc.grid_y), int(lc.wg_x), int(lc.wg_y),
    )


def to_c_array(instances):
    """Contiguous lmt_instance[] for a batch (numpy-built, no per-field ctypes)."""
    from ._lib import CInstance

    n = len(instances)
    rec = np.empty((n, 19), dtype=np.int32)
    for k, inst in enumerate(instances):
        p, lc = inst.params, inst.launch
        rec[k] = (
            p.in_h, p.in_w, p.out_h, p.out_w,
            PATTERN_ORDER.index(getattr(p.pattern, "value", p.pattern)), p.n, p.m,
            SHAPE_ORDER.index(_shape_name(p.stencil.shape)), p.stencil.radius,
            p.num_comp_ilb, p.num_comp_ep, p.num_coal_ilb, p.num_coal_ep,
            p.num_uncoal_ilb, p.num_uncoal_ep, lc.grid_x, lc.grid_y, lc.wg_x, lc.wg_y,
        )
    arr = (CInstance * max(n, 1))()
    if n:
        import ctypes

        ctypes.memmove(arr, rec.ctypes.data, rec.nbytes)
    return arr


def validate_params(params) -> list[str]:
    """Template-parameter violations only (kernel_model.py:173-193)."""
    msgs = []
    for name in ("in_h", "in_w", "out_h", "out_w", "n", "m"):
        if getattr(params, name) < 1:
            msgs.append(f"{name} {getattr(params, name)} < 1")
    for name in ("num_comp_ilb", "num_comp_ep", "num_coal_ilb", "num_coal_ep",
                 "num_uncoal_ilb", "num_uncoal_ep"):
        if getattr(params, name) < 0:
            msgs.append(f"{name} {getattr(params, name)} < 0")
    if params.stencil.radius < 0:
        msgs.append(f"stencil radius {params.stencil.radius} < 0")
    return msgs


def validate_instance(instance) -> list[str]:
    """All violations, reference wording and order (kernel_model.py:196-219).
    Computed by the C ABI's ``lmt_validate``."""
    import ctypes

    from ._lib import lib

    buf = ctypes.create_string_buffer(4096)
    count = lib().lmt_validate(ctypes.byref(to_c(instance)), buf, len(buf))
    if count == 0:
        return []
    return buf.value.decode().split("; ")
