"""GPU execution of the two kernel variants behind the reference's
``lmtune.interp`` signatures (interp.py:30-124).

``make_inputs`` generates the inputs on the device (K0, the hash fill of
interp.py:22-27) and returns host arrays; ``execute`` runs one variant on the
B200 (K1 plain global loads / K2 TMA-staged shared memory) and returns the
host ``out`` array; ``run_pair`` runs both on identical inputs. Inputs may
also be torch CUDA tensors, in which case no host copy of them is made.

Device memory and streams come from torch (plumbing only); every kernel is
in liblmt_b200.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from ._lib import check, lib
from .device import DEFAULT_DEVICE
from .errors import InvalidInstance
from .geometry import c_device, emit_geometry, variant_id
from .kernel_model import to_c, validate_instance


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .errors import LmtuneError

        raise LmtuneError("no CUDA device: the lmtune B200 path has no CPU fallback")
    return torch


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _pitch(cols: int) -> int:
    return (cols + 3) // 4 * 4


def device_fill(rows: int, cols: int, salt: int):
    """Hash-filled [rows, cols] array on the device, physical pitch
    round_up(cols, 4); returns the padded torch tensor."""
    torch = _torch()
    t = torch.empty((rows, _pitch(cols)), dtype=torch.float32, device="cuda")
    check(lib().lmt_fill(ctypes.c_void_p(t.data_ptr()), rows, cols, t.shape[1], salt, _stream(torch)),
          what="fill")
    return t


def make_inputs(instance, dev=DEFAULT_DEVICE) -> tuple[np.ndarray, np.ndarray]:
    """Allocate and fill ``in`` (with apron margins) and ``in2``
    (interp.py:30-38), generated on the GPU."""
    geo = emit_geometry(instance, dev)
    p = instance.params
    a = device_fill(geo.alloc_h, geo.alloc_w, 0)
    b = device_fill(p.in_h, p.in_w, 1)
    in_arr = a[:, : geo.alloc_w].cpu().numpy()
    in2 = b[:, : p.in_w].cpu().numpy()
    return np.ascontiguousarray(in_arr), np.ascontiguousarray(in2)


def _as_device_in(torch, arr):
    """Device copy of `in` with a 16-byte-multiple pitch: (tensor, rows, cols, pitch)."""
    if torch.is_tensor(arr) and arr.is_cuda:
        t = arr.to(torch.float32)
        rows, cols = t.shape
        if t.stride(1) == 1 and t.stride(0) % 4 == 0 and t.data_ptr() % 16 == 0:
            return t, rows, cols, t.stride(0)
        padded = torch.zeros((rows, _pitch(cols)), dtype=torch.float32, device="cuda")
        padded[:, :cols] = t
        return padded, rows, cols, padded.shape[1]
    a = np.asarray(arr, dtype=np.float32)
    if a.ndim != 2:
        raise ValueError(f"in must be 2-D, got shape {a.shape}")
    rows, cols = a.shape
    padded = torch.zeros((rows, _pitch(cols)), dtype=torch.float32, device="cuda")
    padded[:, :cols] = torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=False)
    return padded, rows, cols, padded.shape[1]


def _as_device_in2(torch, arr, p):
    if torch.is_tensor(arr) and arr.is_cuda:
        t = arr.to(torch.float32).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(arr, dtype=np.float32))).to("cuda")
    if tuple(t.shape) != (p.in_h, p.in_w):
        raise ValueError(f"in2 must be {(p.in_h, p.in_w)}, got {tuple(t.shape)}")
    return t


def execute_device(instance, variant, in_t, in2_t, dev=DEFAULT_DEVICE, out=None):
    """Run one variant on device tensors; returns the device ``out`` tensor
    (asynchronous on torch's current stream)."""
    torch = _torch()
    v = validate_instance(instance)
    if v:
        raise InvalidInstance(v)
    p = instance.params
    d_in, rows, cols, pitch = _as_device_in(torch, in_t)
    d_in2 = _as_device_in2(torch, in2_t, p)
    if out is None:
        out = torch.empty((p.out_h, p.out_w), dtype=torch.float32, device="cuda")
    rc = lib().lmt_execute(
        ctypes.byref(to_c(instance)), ctypes.byref(c_device(dev)), variant_id(variant),
        ctypes.c_void_p(d_in.data_ptr()), rows, cols, pitch, ctypes.c_void_p(d_in2.data_ptr()),
        ctypes.c_void_p(out.data_ptr()), _stream(torch),
    )
    check(rc, what="execute")
    return out


def execute(instance, variant, in_arr, in2, dev=DEFAULT_DEVICE) -> np.ndarray:
    """Run one variant over the full launch and return ``out``
    (interp.py:41-114), on the GPU."""
    out = execute_device(instance, variant, in_arr, in2, dev)
    return out.cpu().numpy()


def run_pair(instance, dev=DEFAULT_DEVICE) -> tuple[np.ndarray, np.ndarray]:
    """Both variants on identical device-generated inputs (interp.py:117-124)."""
    from .geometry import Variant

    geo = emit_geometry(instance, dev)
    p = instance.params
    a = device_fill(geo.alloc_h, geo.alloc_w, 0)
    b = device_fill(p.in_h, p.in_w, 1)
    in_view = a[:, : geo.alloc_w]
    in2_view = b[:, : p.in_w]
    base = execute_device(instance, Variant.BASELINE, in_view, in2_view, dev)
    opt = execute_device(instance, Variant.OPTIMIZED, in_view, in2_view, dev)
    return base.cpu().numpy(), opt.cpu().numpy()
