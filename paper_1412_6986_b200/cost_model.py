"""The reference's resource model helpers (mirrors lmtune/cost_model.py:28-91).

``kernel_time`` / ``label_speedup`` -- the per-instance model the dataset
labels come from -- run on the GPU (K4, access_analysis.py here); these are
the small integer helpers around them, for callers that use them directly.
"""

from __future__ import annotations

from dataclasses import dataclass

from .access_analysis import TimeEstimate, kernel_time, label_speedup  # noqa: F401
from .device import DEFAULT_DEVICE
from .geometry import Variant, footprint, variant_id
from .kernel_model import stencil_offsets


@dataclass(frozen=True)
class ResourceUsage:
    regs_per_thread: int
    lmem_per_wg: int
    wg_size: int
    warps_per_wg: int


def estimate_registers(params, variant, dev=DEFAULT_DEVICE) -> int:
    """cost_model.py:41-60 (the optimized variant costs 4 more, past the clamp)."""
    ctx = params.num_coal_ilb + params.num_coal_ep + params.num_uncoal_ilb + params.num_uncoal_ep
    raw = 10 + len(stencil_offsets(params.stencil)) + -(-params.num_comp_ilb // 4) + -(-params.num_comp_ep // 8) + 2 * ctx
    base = min(max(raw, 10), dev.max_regs_per_thread)
    return base + 4 if variant_id(variant) == 1 else base


def resource_usage(instance, variant, dev=DEFAULT_DEVICE, lmem_bytes: int | None = None) -> ResourceUsage:
    """cost_model.py:63-79."""
    if lmem_bytes is None:
        lmem_bytes = 0 if variant_id(variant) == 0 else footprint(instance, dev).bytes
    wg = instance.launch.wg_x * instance.launch.wg_y
    return ResourceUsage(estimate_registers(instance.params, variant, dev), lmem_bytes, wg,
                         (wg + dev.warp_size - 1) // dev.warp_size)


def occupancy(usage: ResourceUsage, dev=DEFAULT_DEVICE) -> float:
    """cost_model.py:82-91: active warps per SM, floored at one warp."""
    limits = [dev.max_workgroups_per_sm]
    if usage.lmem_per_wg > 0:
        limits.append(dev.lmem_capacity_bytes // usage.lmem_per_wg)
    limits.append(dev.register_file_per_sm // (usage.regs_per_thread * usage.wg_size))
    limits.append(dev.max_warps_per_sm // usage.warps_per_wg)
    return float(max(1, min(limits) * usage.warps_per_wg))


__all__ = ["ResourceUsage", "TimeEstimate", "Variant", "estimate_registers", "resource_usage", "occupancy",
           "kernel_time", "label_speedup"]
