"""Kernel sources of the two variants (mirrors the lmtune/codegen.py API:
KernelSource, emit_baseline, emit_optimized, defines_manifest,
kernel_filename, codegen.py:33-359).

The reference emits OpenCL C text for each instance with its geometry and
counts as #defines; the B200 path compiles CUDA C++ (csrc/lmt_jit.cuh) with
NVRTC for sm_100a, specialised by a block of LMT_* #defines (stencil, the six
counts, in2 shape, variant, work units per thread, prefetch depth). These
functions return exactly the text that gets compiled for an instance, and its
defines.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from ._lib import MEASURE_REGBLOCK, check, lib
from .device import DEFAULT_DEVICE
from .errors import OptimizationInfeasible
from .geometry import Variant, c_device, footprint
from .kernel_model import to_c


@dataclass(frozen=True)
class KernelSource:
    variant: Variant
    entry_name: str
    source_text: str
    compile_defines: tuple


def _source(instance, variant: Variant, dev, regblock: bool) -> KernelSource:
    L = lib()
    n = ctypes.c_int64()
    vid = 0 if variant is Variant.BASELINE else 1
    flags = MEASURE_REGBLOCK if regblock else 0
    check(L.lmt_kernel_source(ctypes.byref(to_c(instance)), ctypes.byref(c_device(dev)), vid, flags, None, 0,
                              ctypes.byref(n)), what="kernel_source")
    buf = ctypes.create_string_buffer(n.value + 1)
    check(L.lmt_kernel_source(ctypes.byref(to_c(instance)), ctypes.byref(c_device(dev)), vid, flags, buf, len(buf),
                              ctypes.byref(n)), what="kernel_source")
    text = buf.value.decode()
    defines = []
    for line in text.splitlines():
        if not line.startswith("#define LMT_"):
            break
        _, name, value = line.split(maxsplit=2)
        defines.append((name, int(value)))
    return KernelSource(variant, "lmt_kernel", text, tuple(defines))


def emit_baseline(instance, dev=DEFAULT_DEVICE, *, regblock: bool = False) -> KernelSource:
    """codegen.py:336-340; raises InvalidInstance on constraint violations.
    ``regblock``: the register-blocked kernel (LMT_MEASURE_REGBLOCK) instead
    of the literal one."""
    return _source(instance, Variant.BASELINE, dev, regblock)


def emit_optimized(instance, fp=None, dev=DEFAULT_DEVICE, *, regblock: bool = False) -> KernelSource:
    """codegen.py:343-354; raises OptimizationInfeasible when the staging
    region exceeds the device's local-memory capacity."""
    if fp is None:
        fp = footprint(instance, dev)
    if fp.bytes > dev.lmem_capacity_bytes:
        raise OptimizationInfeasible(fp.bytes, dev.lmem_capacity_bytes)
    return _source(instance, Variant.OPTIMIZED, dev, regblock)


def defines_manifest(source: KernelSource) -> str:
    """One -D binding per line (codegen.py:357-359)."""
    return "".join(f"-D {name}={value}\n" for name, value in source.compile_defines)


def kernel_filename(params, variant) -> str:
    """codegen.py:142-146, with the CUDA extension."""
    s = params.stencil
    pat = getattr(params.pattern, "value", params.pattern)
    shape = getattr(s.shape, "value", s.shape)
    v = getattr(variant, "value", variant)
    return f"{pat}_{params.n}x{params.m}_{shape}{s.radius}_{v}.cu"
