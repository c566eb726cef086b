"""The instance sweep: the deterministic instance list of the reference's
dataset builder, its cost-balanced sharding across ranks, and the measured
sweep driver (mirrors dataset.py:44-281; GPU measurement takes the place of
the per-instance ``label`` closure at dataset.py:264-271).

Selection reproduces ``lmtune.dataset._select_instances`` exactly (same numpy
PCG64 draws in the same order); tests/test_sweep.py pins it against the
reference. For million-instance sweeps the list is also available as a
compact integer table (kernels x launches x picked pairs) that converts to
the C ABI's ``lmt_instance[]`` without building Python objects.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .kernel_model import (
    PATTERN_ORDER,
    SHAPE_ORDER,
    HomeAccessPattern,
    KernelInstance,
    LaunchConfig,
    StencilPattern,
    StencilShape,
    TemplateParams,
)
from .seeding import mix_seed

_LARGE_N = {"xy_reuse", "x_reuse_row", "y_reuse_row"}
_LARGE_M = {"xy_reuse", "x_reuse_col", "y_reuse_col"}

DLA_FAMILY = ("xy_reuse", "x_reuse_row", "x_reuse_col", "y_reuse_row", "y_reuse_col")
GRID_FAMILY = ("no_reuse_row_major", "no_reuse_col_major")


@dataclass(frozen=True)
class SamplingSpec:
    """dataset.py:44-80 (same fields and defaults)."""

    num_tuples: int = 100
    radius_range: tuple[int, int] = (0, 2)
    comp_ilb_range: tuple[int, int] = (5, 44)
    comp_ep_range: tuple[int, int] = (1, 48)
    coal_range: tuple[int, int] = (0, 13)
    uncoal_range: tuple[int, int] = (0, 4)
    large_values: tuple[int, ...] = (8, 16, 32, 64)
    small_values: tuple[int, ...] = (1, 2, 4, 8)
    in_h: int = 2048
    in_w: int = 2048
    out_h: int = 2048
    out_w: int = 2048
    max_instances: int = 50_000
    seed: int = 0

    def __post_init__(self):
        if self.num_tuples < 1:
            raise ValueError(f"num_tuples {self.num_tuples} < 1")
        if self.max_instances < 1:
            raise ValueError(f"max_instances {self.max_instances} < 1")
        for name in ("radius_range", "comp_ilb_range", "comp_ep_range", "coal_range", "uncoal_range"):
            lo, hi = getattr(self, name)
            if lo > hi:
                raise ValueError(f"{name} ({lo}, {hi}) is empty")
        if not self.large_values or not self.small_values:
            raise ValueError("value sets must be non-empty")

    def n_values(self, pattern) -> tuple[int, ...]:
        return self.large_values if getattr(pattern, "value", pattern) in _LARGE_N else self.small_values

    def m_values(self, pattern) -> tuple[int, ...]:
        return self.large_values if getattr(pattern, "value", pattern) in _LARGE_M else self.small_values


@dataclass(frozen=True)
class CompileTuple:
    stencil: StencilPattern
    num_comp_ilb: int
    num_comp_ep: int
    num_coal_ilb: int
    num_coal_ep: int
    num_uncoal_ilb: int
    num_uncoal_ep: int


def sample_compile_tuples(spec: SamplingSpec) -> list[CompileTuple]:
    """dataset.py:109-134: shape, radius, then the six counts, per tuple."""
    rng = np.random.default_rng(spec.seed)
    shapes = list(StencilShape)
    out = []
    for _ in range(spec.num_tuples):
        shape = shapes[int(rng.integers(0, len(shapes)))]
        draws = [int(rng.integers(lo, hi + 1)) for lo, hi in (
            spec.radius_range, spec.comp_ilb_range, spec.comp_ep_range, spec.coal_range, spec.coal_range,
            spec.uncoal_range, spec.uncoal_range)]
        out.append(CompileTuple(StencilPattern(shape, draws[0]), *draws[1:]))
    return out


def expand_patterns(tup: CompileTuple, spec: SamplingSpec) -> list[TemplateParams]:
    """dataset.py:137-161: 7 patterns x |N values| x |M values|."""
    return [
        TemplateParams(spec.in_h, spec.in_w, spec.out_h, spec.out_w, pat, n, m, tup.stencil,
                       tup.num_comp_ilb, tup.num_comp_ep, tup.num_coal_ilb, tup.num_coal_ep,
                       tup.num_uncoal_ilb, tup.num_uncoal_ep)
        for pat in HomeAccessPattern
        for n in spec.n_values(pat)
        for m in spec.m_values(pat)
    ]


@lru_cache(maxsize=8)
def launch_configs(out_h: int, out_w: int, min_grid_size: int = 512, max_wg_size: int = 1024):
    """dataset.py:164-188, ordered by (grid_x, grid_y, wg_x, wg_y)."""

    def divisors(v):
        return [1 << k for k in range(v.bit_length()) if v % (1 << k) == 0]

    return tuple(
        LaunchConfig(gx, gy, wx, wy)
        for gx in divisors(out_w)
        for gy in divisors(out_h)
        if gx * gy >= min_grid_size
        for wx in divisors(gx)
        for wy in divisors(gy)
        if wx * wy <= max_wg_size
    )


def enumerate_launch_configs(params, min_grid_size: int = 512, max_wg_size: int = 1024) -> list[LaunchConfig]:
    return list(launch_configs(params.out_h, params.out_w, min_grid_size, max_wg_size))


def instance_key(instance) -> str:
    """dataset.py:191-198."""
    p, lc = instance.params, instance.launch
    pat = getattr(p.pattern, "value", p.pattern)
    shape = getattr(p.stencil.shape, "value", p.stencil.shape)
    return (f"{pat} n={p.n} m={p.m} {shape} r={p.stencil.radius} "
            f"comp={p.num_comp_ilb}/{p.num_comp_ep} coal={p.num_coal_ilb}/{p.num_coal_ep} "
            f"uncoal={p.num_uncoal_ilb}/{p.num_uncoal_ep} "
            f"grid={lc.grid_x}x{lc.grid_y} wg={lc.wg_x}x{lc.wg_y}")


@dataclass
class InstanceTable:
    """Compact sweep: instance r is (kernels[picked[r, 0]], launches[picked[r, 1]])."""

    kernels: list          # TemplateParams, dedup order
    launches: tuple        # LaunchConfig sweep
    picked: np.ndarray     # int64 [n, 2] (kernel index, launch index), sorted

    def __len__(self) -> int:
        return len(self.picked)

    def instance(self, r: int) -> KernelInstance:
        k, lidx = self.picked[r]
        return KernelInstance(self.kernels[int(k)], self.launches[int(lidx)])

    def instances(self, rows=None) -> list[KernelInstance]:
        rows = range(len(self)) if rows is None else rows
        return [self.instance(int(r)) for r in rows]

    @property
    def kernel_matrix(self) -> np.ndarray:
        if getattr(self, "_km", None) is None:
            km = np.empty((len(self.kernels), 15), dtype=np.int32)
            for i, p in enumerate(self.kernels):
                km[i] = (p.in_h, p.in_w, p.out_h, p.out_w, PATTERN_ORDER.index(p.pattern.value), p.n, p.m,
                         SHAPE_ORDER.index(p.stencil.shape.value), p.stencil.radius, p.num_comp_ilb,
                         p.num_comp_ep, p.num_coal_ilb, p.num_coal_ep, p.num_uncoal_ilb, p.num_uncoal_ep)
            self._km = km
        return self._km

    @property
    def launch_matrix(self) -> np.ndarray:
        return np.array([(lc.grid_x, lc.grid_y, lc.wg_x, lc.wg_y) for lc in self.launches], dtype=np.int32)

    def records(self, rows=None) -> np.ndarray:
        """int32 [n, 19] rows laid out like the C ``lmt_instance``."""
        pk = self.picked if rows is None else self.picked[np.asarray(rows, dtype=np.int64)]
        return np.ascontiguousarray(
            np.concatenate([self.kernel_matrix[pk[:, 0]], self.launch_matrix[pk[:, 1]]], axis=1), dtype=np.int32)


def select_instance_table(spec: SamplingSpec) -> InstanceTable:
    """dataset.py:207-250 (_select_instances): kernels deduplicated in sampling
    order, a seeded shuffle of the launch sweep per kernel, round-robin picks
    under the cap, then sorted by (kernel, launch)."""
    kernels, seen = [], set()
    for tup in sample_compile_tuples(spec):
        for p in expand_patterns(tup, spec):
            if p not in seen:
                seen.add(p)
                kernels.append(p)
    launches = launch_configs(kernels[0].out_h, kernels[0].out_w) if kernels else ()
    lcount = len(launches)
    # fewest round-robin passes that can reach the cap
    rounds, reachable = 0, 0
    while reachable < spec.max_instances and rounds < lcount:
        rounds += 1
        reachable = len(kernels) * min(lcount, rounds)
    take = min(lcount, rounds)
    orders = np.empty((len(kernels), take), dtype=np.int64)
    for k in range(len(kernels)):
        orders[k] = np.random.default_rng(mix_seed(spec.seed, k)).choice(lcount, size=take, replace=False)
    # round r visits kernels 0..K-1 in order; the cap truncates mid-round
    total = min(spec.max_instances, len(kernels) * take)
    r_idx = np.arange(total) // max(len(kernels), 1)
    k_idx = np.arange(total) % max(len(kernels), 1)
    picked = np.stack([k_idx, orders[k_idx, r_idx]], axis=1) if total else np.zeros((0, 2), np.int64)
    order = np.lexsort((picked[:, 1], picked[:, 0]))
    return InstanceTable(kernels, launches, picked[order])


def select_instances(spec: SamplingSpec) -> list[KernelInstance]:
    return select_instance_table(spec).instances()


def family_rows(table: InstanceTable, patterns) -> np.ndarray:
    """Rows whose pattern is in ``patterns`` (e.g. DLA_FAMILY / GRID_FAMILY)."""
    want = {PATTERN_ORDER.index(p) for p in patterns}
    pat = table.kernel_matrix[table.picked[:, 0], 4]
    return np.nonzero(np.isin(pat, list(want)))[0]


# ------------------------------------------------------------ cost and sharding

_K_BY_SHAPE_R = {}


def _num_offsets(shape: int, r: int) -> int:
    key = (shape, r)
    if key not in _K_BY_SHAPE_R:
        rng = range(-r, r + 1)
        _K_BY_SHAPE_R[key] = sum(
            1 for a in rng for b in rng
            if not (shape == 1 and abs(a) + abs(b) > r) and not (shape == 2 and a and b))
    return _K_BY_SHAPE_R[key]


def estimated_cost(records: np.ndarray, fp32_lane_ops_per_s: float = 6.0e13, clock_hz: float = 1.9e9,
                   sms: int = 148) -> np.ndarray:
    """Rough per-instance GPU seconds (both variants) for load balancing:
    the larger of the issue-bound time and the per-thread dependence chain
    (each work unit is a serial fp32 chain, kernels launch one thread per
    workitem)."""
    rec = np.asarray(records, dtype=np.int64)
    n_, m_ = rec[:, 5], rec[:, 6]
    K = np.array([_num_offsets(int(s), int(r)) for s, r in zip(rec[:, 7], rec[:, 8])], dtype=np.float64)
    chain = (n_ * m_) * (K + rec[:, 9] + rec[:, 11] + rec[:, 13]) + rec[:, 10] + rec[:, 12] + rec[:, 14]
    out = rec[:, 2] * rec[:, 3]
    grid = rec[:, 15] * rec[:, 16]
    wus = out // np.maximum(grid, 1)
    issue = 2.0 * chain * out / fp32_lane_ops_per_s
    threads_per_sm = np.minimum(grid / sms, 2048.0)
    lat = wus * chain * 4.0 / clock_hz / np.maximum(1.0, threads_per_sm / 512.0)
    return 2.0 * (np.maximum(issue, lat) + 4e-6)


def chain_ops(records: np.ndarray) -> np.ndarray:
    """Dependent fp32 operations in one work unit's accumulator chain:
    N*M*(K + comp_ilb + coal_ilb + uncoal_ilb) + comp_ep + coal_ep + uncoal_ep
    (codegen.py:207-237; a MAD is one instruction)."""
    rec = np.asarray(records, dtype=np.int64)
    K = np.array([_num_offsets(int(s), int(r)) for s, r in zip(rec[:, 7], rec[:, 8])], dtype=np.int64)
    return rec[:, 5] * rec[:, 6] * (K + rec[:, 9] + rec[:, 11] + rec[:, 13]) + rec[:, 10] + rec[:, 12] + rec[:, 14]


def floor_seconds(records: np.ndarray, clock_hz: float = 1.965e9, sms: int = 148) -> tuple[np.ndarray, np.ndarray]:
    """Per-variant lower bounds on one launch of each instance with the
    reference's mapping fixed (workgroup -> CTA on one SM, workitem -> thread):

    - chain: a workitem's work units are independent but each is a serial
      chain of fp32 ops in a fixed order (bit-exact), and a warp issues at
      most one instruction per cycle, so a thread needs >= wus * chain cycles
      however its work units are interleaved;
    - issue: a CTA's warps share one SM's four schedulers, and the CTAs are
      spread over at most 148 SMs: ceil(ctas / 148) * warps_per_cta * wus *
      chain / 4 cycles (partial warps pay for 32 lanes).

    Returns (chain_floor_s, issue_floor_s); the HBM floor is alg_bytes /
    peak (see measure.roofline)."""
    rec = np.asarray(records, dtype=np.int64)
    chain = chain_ops(rec).astype(np.float64)
    grid = rec[:, 15] * rec[:, 16]
    wg = np.maximum(rec[:, 17] * rec[:, 18], 1)
    wus = rec[:, 2] * rec[:, 3] // np.maximum(grid, 1)
    ctas = grid // wg
    warps = (wg + 31) // 32
    chain_s = wus * chain / clock_hz
    issue_s = np.ceil(ctas / sms) * warps * wus * chain / 4.0 / clock_hz
    return chain_s, issue_s


def launch_cost(records: np.ndarray) -> np.ndarray:
    """Balancing cost of an instance (both variants): its launch floor,
    2 * max(chain, per-SM issue) seconds (floor_seconds). Correlates with the
    measured time better than estimated_cost (log-correlation 0.96 vs 0.91 on
    the round-1 bench sample)."""
    ch, iss = floor_seconds(records)
    return 2.0 * np.maximum(ch, iss) + 4e-6


def shard_balanced(costs: np.ndarray, world: int, loads: np.ndarray | None = None) -> list[np.ndarray]:
    """Disjoint shards of equal estimated cost (greedy longest-processing-time);
    each shard keeps ascending index order. ``loads`` (per rank, updated in
    place) carries the cost already assigned by earlier batches, so balance
    holds over a run of batches, not just within each."""
    costs = np.asarray(costs, dtype=np.float64)
    order = np.argsort(-costs, kind="stable")
    if loads is None:
        loads = np.zeros(world)
    owner = np.empty(len(costs), dtype=np.int64)
    for i in order:
        w = int(np.argmin(loads))
        owner[i] = w
        loads[w] += costs[i]
    return [np.nonzero(owner == w)[0] for w in range(world)]


def shard_contiguous(costs: np.ndarray, world: int) -> list[np.ndarray]:
    """Contiguous ranges split on the prefix sum of estimated cost."""
    c = np.cumsum(np.asarray(costs, dtype=np.float64))
    total = c[-1] if len(c) else 0.0
    cuts = [0] + [int(np.searchsorted(c, total * w / world, side="left")) for w in range(1, world)] + [len(c)]
    return [np.arange(cuts[w], cuts[w + 1]) for w in range(world)]


def instances_to_records(instances) -> np.ndarray:
    """int32 [n, 19] records of KernelInstance-shaped objects (ours or the reference's)."""
    rows = []
    for inst in instances:
        p, lc = inst.params, inst.launch
        rows.append((p.in_h, p.in_w, p.out_h, p.out_w, PATTERN_ORDER.index(getattr(p.pattern, "value", p.pattern)),
                     p.n, p.m, SHAPE_ORDER.index(getattr(p.stencil.shape, "value", p.stencil.shape)),
                     p.stencil.radius, p.num_comp_ilb, p.num_comp_ep, p.num_coal_ilb, p.num_coal_ep,
                     p.num_uncoal_ilb, p.num_uncoal_ep, lc.grid_x, lc.grid_y, lc.wg_x, lc.wg_y))
    return np.array(rows, dtype=np.int32).reshape(-1, 19)


def records_to_c(records: np.ndarray):
    from ._lib import CInstance

    rec = np.ascontiguousarray(records, dtype=np.int32)
    arr = (CInstance * max(len(rec), 1))()
    if len(rec):
        ctypes.memmove(arr, rec.ctypes.data, rec.nbytes)
    return arr


def sample_cells(rec: np.ndarray, S: int, seed: int) -> np.ndarray:
    """int64 [n, S] output cells per instance to read back for an
    independent check against the CPU reference: four cells of workgroup 0's
    first work-unit iteration, four of its last, the last cell of the output,
    and the rest uniform over the output."""
    rng = np.random.default_rng(seed)
    out = np.empty((len(rec), S), dtype=np.int64)
    for i, r in enumerate(np.asarray(rec, dtype=np.int64)):
        oh, ow, gx, gy, wx, wy = r[2], r[3], r[15], r[16], r[17], r[18]
        nwx, nwy = ow // gx, oh // gy
        first = [(0, 0), (0, wx - 1), (wy - 1, 0), (wy - 1, wx - 1)]
        ly, lx = (nwy - 1) * wy, (nwx - 1) * wx
        last = [(ly, lx), (ly, lx + wx - 1), (ly + wy - 1, lx), (ly + wy - 1, lx + wx - 1)]
        fixed = [y * ow + x for y, x in first + last] + [oh * ow - 1]
        k = min(len(fixed), S)
        out[i, :k] = fixed[:k]
        if S > k:
            out[i, k:] = rng.integers(0, oh * ow, size=S - k)
    return out
