"""ctypes binding of liblmt_b200.so (the C ABI in include/lmt_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``) into
``paper_1412_6986_b200/lib/liblmt_b200.so``. There is no CPU fallback: if
the library is missing every entry point raises ``LmtuneError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import InvalidInstance, LmtuneError, OptimizationInfeasible

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liblmt_b200.so")

LMT_OK = 0
LMT_ERR_INVALID_INSTANCE = 1
LMT_ERR_INFEASIBLE = 2
LMT_ERR_CUDA = 3
LMT_ERR_ARG = 4
LMT_ERR_TOO_LARGE = 5

MEASURE_SKIP_OPT = 0x1
MEASURE_ALLOW_LARGE_LMEM = 0x4
MEASURE_CONCURRENT = 0x8
MEASURE_REGBLOCK = 0x10
MEASURE_WARM_L2 = 0x20

INSTANCE_FIELDS = (
    "in_h", "in_w", "out_h", "out_w", "pattern", "n", "m", "stencil_shape",
    "stencil_radius", "num_comp_ilb", "num_comp_ep", "num_coal_ilb", "num_coal_ep",
    "num_uncoal_ilb", "num_uncoal_ep", "grid_x", "grid_y", "wg_x", "wg_y",
)
DEVICE_FIELDS = (
    "transaction_bytes", "warp_size", "element_bytes", "lmem_capacity_bytes",
    "register_file_per_sm", "max_regs_per_thread", "max_warps_per_sm",
    "max_workgroups_per_sm", "dram_latency_cycles", "issue_cycles_per_op",
)


class CInstance(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in INSTANCE_FIELDS]


class CDevice(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in DEVICE_FIELDS]


class CGeometry(ctypes.Structure):
    _fields_ = [
        ("pad", ctypes.c_int32), ("off_min_row", ctypes.c_int32), ("off_min_col", ctypes.c_int32),
        ("r_rows", ctypes.c_int32), ("r_cols", ctypes.c_int32), ("r_cols_pad", ctypes.c_int32),
        ("seg_elems", ctypes.c_int32), ("segs_per_row", ctypes.c_int32), ("num_segs", ctypes.c_int32),
        ("num_warps", ctypes.c_int32), ("lanes_per_warp", ctypes.c_int32),
        ("alloc_h", ctypes.c_int64), ("alloc_w", ctypes.c_int64),
        ("org_row_wu_x", ctypes.c_int32), ("org_row_wu_y", ctypes.c_int32),
        ("org_col_wu_x", ctypes.c_int32), ("org_col_wu_y", ctypes.c_int32),
        ("row_i", ctypes.c_int32), ("row_j", ctypes.c_int32),
        ("col_i", ctypes.c_int32), ("col_j", ctypes.c_int32),
        ("footprint_bytes", ctypes.c_int64), ("num_offsets", ctypes.c_int32),
    ]


class CRealInstance(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("kernel", "n", "wg_x", "wg_y", "tile", "radius")]


class CMeasurement(ctypes.Structure):
    _fields_ = [
        ("t_base_ms", ctypes.c_double), ("t_opt_ms", ctypes.c_double),
        ("digest_base", ctypes.c_uint64), ("digest_opt", ctypes.c_uint64),
        ("mismatches", ctypes.c_int64), ("alg_bytes", ctypes.c_double),
        ("alg_flops", ctypes.c_double), ("t_fill_ms", ctypes.c_double),
        ("status", ctypes.c_int32), ("kernel_id", ctypes.c_int32),
        ("launches", ctypes.c_int32), ("nstages", ctypes.c_int32),
        ("lane_sms", ctypes.c_int32), ("order", ctypes.c_int32),
        ("in_copies", ctypes.c_int32), ("ctas", ctypes.c_int32),
    ]


class CMeasureOpts(ctypes.Structure):
    _fields_ = [
        ("flags", ctypes.c_int32), ("samples", ctypes.c_int32),
        ("sample_idx", ctypes.c_void_p), ("h_sample_vals", ctypes.c_void_p),
        ("tune", ctypes.c_int32 * 6),
    ]


# every symbol include/lmt_b200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "lmt_version", "lmt_last_error", "lmt_validate", "lmt_emit_geometry", "lmt_fill",
    "lmt_execute", "lmt_measure_batch", "lmt_measure_batch_host", "lmt_digest",
    "lmt_rf_create", "lmt_rf_mean", "lmt_rf_mean_host", "lmt_rf_destroy", "lmt_sync",
    "lmt_get_stream", "lmt_prepare", "lmt_jit_stats", "lmt_features", "lmt_real_validate",
    "lmt_real_execute", "lmt_real_measure", "lmt_rf_train_tree", "lmt_kernel_source",
    "lmt_measure_batch_ex", "lmt_partitions", "lmt_current_device", "lmt_plan_info", "lmt_rf_train_gpu", "lmt_rf_feature_draws",
)

_lib = None
_lock = threading.Lock()


def _declare(L):
    P = ctypes.POINTER
    c_i64, c_i32, c_u32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p
    L.lmt_version.restype = ctypes.c_char_p
    L.lmt_version.argtypes = []
    L.lmt_last_error.restype = ctypes.c_char_p
    L.lmt_last_error.argtypes = []
    L.lmt_validate.argtypes = [P(CInstance), ctypes.c_char_p, c_i64]
    L.lmt_emit_geometry.argtypes = [P(CInstance), P(CDevice), P(CGeometry)]
    L.lmt_fill.argtypes = [vp, c_i64, c_i64, c_i64, c_u32, vp]
    L.lmt_execute.argtypes = [P(CInstance), P(CDevice), ctypes.c_int, vp, c_i64, c_i64, c_i64, vp, vp, vp]
    L.lmt_measure_batch.argtypes = [P(CInstance), c_i64, P(CDevice), c_i32, P(CMeasurement)]
    L.lmt_measure_batch_host.argtypes = [
        P(CInstance), c_i64, P(CDevice), c_i32, P(vp), P(c_i64), P(c_i64), P(vp), P(vp), P(vp),
        P(CMeasurement),
    ]
    L.lmt_measure_batch_ex.argtypes = [
        P(CInstance), c_i64, P(CDevice), P(CMeasureOpts), P(vp), P(c_i64), P(c_i64), P(vp), P(vp), P(vp),
        P(CMeasurement),
    ]
    L.lmt_partitions.argtypes = [P(c_i32), c_i32, P(c_i32)]
    L.lmt_digest.argtypes = [vp, c_i64, P(ctypes.c_uint64), vp]
    L.lmt_rf_create.argtypes = [vp, vp, vp, vp, vp, vp, c_i32, c_i32, P(vp)]
    L.lmt_rf_mean.argtypes = [vp, vp, c_i64, vp, vp, vp]
    L.lmt_rf_mean_host.argtypes = [vp, vp, c_i64, vp, vp]
    L.lmt_rf_destroy.argtypes = [vp]
    L.lmt_rf_destroy.restype = None
    L.lmt_current_device.argtypes = [P(c_i32)]
    L.lmt_plan_info.argtypes = [P(CInstance), P(CDevice), c_i32, P(c_i64)]
    L.lmt_rf_feature_draws.argtypes = [vp, c_i32, c_u32, c_i32, c_i32, c_i64, vp]
    L.lmt_rf_train_gpu.argtypes = [vp, vp, c_i64, c_i32, c_i32, vp, vp, c_i64, c_i32, c_i32, c_i32, vp, vp, vp, vp,
                                   vp, c_i64, vp, vp]
    L.lmt_sync.argtypes = []
    L.lmt_get_stream.argtypes = [P(vp)]
    L.lmt_prepare.argtypes = [P(CInstance), c_i64, P(CDevice), c_i32, c_i32, P(c_i64)]
    L.lmt_jit_stats.argtypes = [P(c_i64), P(ctypes.c_double)]
    L.lmt_real_validate.argtypes = [P(CRealInstance), ctypes.c_char_p, c_i64]
    L.lmt_real_execute.argtypes = [P(CRealInstance), ctypes.c_int, P(vp), vp, vp]
    L.lmt_real_measure.argtypes = [P(CRealInstance), c_i64, c_i32, P(CMeasurement)]
    L.lmt_rf_train_tree.argtypes = [vp, vp, c_i64, c_i32, vp, c_i64, vp, c_i64, c_i32, c_i32, c_i32, vp, vp, vp,
                                    vp, vp, c_i64, P(c_i64), P(c_i64)]
    L.lmt_kernel_source.argtypes = [P(CInstance), P(CDevice), ctypes.c_int, c_i32, ctypes.c_char_p, c_i64, P(c_i64)]
    L.lmt_features.argtypes = [P(CInstance), c_i64, P(CDevice), c_i64, vp, vp, vp, vp, vp, vp]
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in ("lmt_version", "lmt_last_error", "lmt_rf_destroy"):
            fn.restype = ctypes.c_int


def lib():
    """The loaded library; raises LmtuneError (no fallback) when it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise LmtuneError(
                        f"CUDA library {LIB_PATH} is missing; run __graft_entry__.build() "
                        "(there is no CPU fallback for the lmtune B200 path)"
                    )
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def last_error() -> str:
    return lib().lmt_last_error().decode("utf-8", "replace")


def check(rc: int, *, what: str = "") -> None:
    """Map an LMT_ERR_* code onto the reference exception hierarchy
    (errors.py:6-36)."""
    if rc == LMT_OK:
        return
    msg = last_error()
    if rc == LMT_ERR_INVALID_INSTANCE:
        raise InvalidInstance(msg.split("; ") if msg else [what or "invalid instance"])
    if rc == LMT_ERR_INFEASIBLE:
        raise OptimizationInfeasible(*_parse_infeasible(msg))
    raise LmtuneError(f"{what + ': ' if what else ''}{msg or f'lmt error {rc}'}")


def _parse_infeasible(msg: str) -> tuple[int, int]:
    # "local-memory footprint <b> bytes exceeds capacity <c>"
    try:
        words = msg.split()
        return int(words[2]), int(words[-1])
    except (IndexError, ValueError):
        return -1, -1


def library_stream() -> int:
    """cudaStream_t (as int) the library launches measurement batches on."""
    s = ctypes.c_void_p()
    check(lib().lmt_get_stream(ctypes.byref(s)), what="get_stream")
    return int(s.value or 0)


def partitions() -> list[int]:
    """SM counts of the partitions MEASURE_CONCURRENT runs in on the current
    device (empty: no green contexts, every instance runs on the whole device)."""
    sizes = (ctypes.c_int32 * 64)()
    n = ctypes.c_int32()
    check(lib().lmt_partitions(sizes, 64, ctypes.byref(n)), what="partitions")
    return [int(sizes[k]) for k in range(n.value)]


def jit_stats() -> tuple[int, float]:
    """(kernels compiled by NVRTC in this process, host seconds spent compiling)."""
    n, t = ctypes.c_int64(), ctypes.c_double()
    check(lib().lmt_jit_stats(ctypes.byref(n), ctypes.byref(t)), what="jit_stats")
    return int(n.value), float(t.value)
