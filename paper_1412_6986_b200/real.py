"""The real-world kernel set of the paper (BASELINE.json
configs[1]): transpose, matrixMul, convolution-separable and MVT, each run and
timed with and without staging the reused tile in shared memory (K5,
csrc/lmt_real.cuh).

The reference does not implement these; the instance sets below
vary launch shape and tiling factor the way the paper describes ("we vary
kernel parameters such as launch configurations and tiling factors"), at the
sizes BASELINE names (2048 x 2048 target arrays; matrixMul at 1024, MVT at
4096).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import CMeasurement, CRealInstance, check, lib

KERNELS = ("transpose", "matrixMul", "convolution-separable", "MVT")


@dataclass(frozen=True)
class RealInstance:
    kernel: int      # index into KERNELS
    n: int           # square problem size
    wg_x: int
    wg_y: int
    tile: int = 0    # transpose tile (wg_x * columns per thread) / matrixMul tile (== wg_x), MVT j-tile,
    #                  convolution outputs per thread
    radius: int = 0  # convolution radius

    @property
    def name(self) -> str:
        return KERNELS[self.kernel]

    def to_c(self) -> CRealInstance:
        return CRealInstance(self.kernel, self.n, self.wg_x, self.wg_y, self.tile, self.radius)


def validate(inst: RealInstance) -> str:
    buf = ctypes.create_string_buffer(256)
    lib().lmt_real_validate(ctypes.byref(inst.to_c()), buf, len(buf))
    return buf.value.decode()


def instance_set(n_transpose: int = 2048, n_matmul: int = 1024, n_conv: int = 2048, n_mvt: int = 4096) -> list:
    """The configs[1] instance set: 18 transpose (tile T in {8,16,32} x rows
    per CTA step, and 64 x 64 tiles with two columns per thread), 20 matrixMul (T in {4..64} x rows x columns per thread, up to 8 x 8 register tiles), 24
    convolution (radius in {1,2,4,8} x 6 workgroups), 10 MVT (workgroup x
    j-tile), plus 9 transpose and 8 convolution instances at 8192 x 8192
    (arrays well beyond L2) for the HBM roof."""
    out = []
    for T in (8, 16, 32):
        for wy in (1, 2, 4, 8, 16, 32):
            if wy <= T:
                out.append(RealInstance(0, n_transpose, T, wy, tile=T))
    for wy in (4, 8, 16):  # 64 x 64 tiles, two columns per thread
        out.append(RealInstance(0, n_transpose, 32, wy, tile=64))
    for T in (4, 8, 16, 32):
        for W in (1, 2, 4, 8):
            if W <= T and T // W >= 1 and W in (1, 2, 4) + ((8,) if T >= 16 else ()):
                out.append(RealInstance(1, n_matmul, T, T // W, tile=T))
    for T, CC, W in ((32, 2, 8), (32, 4, 4), (32, 4, 8), (64, 4, 8), (64, 4, 4), (64, 8, 8)):  # register tiles W x CC
        out.append(RealInstance(1, n_matmul, T // CC, T // W, tile=T))
    for R in (1, 2, 4, 8):
        for wx, wy in ((16, 4), (32, 4), (32, 8), (64, 4), (128, 1), (16, 16)):
            out.append(RealInstance(2, n_conv, wx, wy, tile=1, radius=R))
    for wg in (32, 64, 128, 256, 512):
        for T in (16, 32):
            out.append(RealInstance(3, n_mvt, wg, 1, tile=T))
    # HBM-scale instances (8192^2: 256 MB per array, beyond L2) for the bandwidth roof
    for wy in (1, 2, 4, 8):  # 32 .. 4 elements per thread in flight
        out.append(RealInstance(0, 8192, 32, wy, tile=32))
    out.append(RealInstance(0, 8192, 16, 16, tile=16))
    for wy in (4, 8):
        out.append(RealInstance(0, 8192, 32, wy, tile=64))
    for wy in (8, 16):  # four columns per thread (128-bit loads and stores)
        out.append(RealInstance(0, 8192, 16, wy, tile=64))
    for R in (1, 2, 4, 8):
        for W in (1, 4):  # outputs per thread
            out.append(RealInstance(2, 8192, 32, 8, tile=W, radius=R))
    return out


def measure(instances, *, skip_opt: bool = False) -> np.ndarray:
    """Both variants of every instance on the current GPU (hash-filled inputs,
    CUDA-event times, outputs digested and compared bitwise); returns a
    measure.MEASUREMENT_DTYPE array."""
    from .measure import MEASUREMENT_DTYPE

    n = len(instances)
    arr = (CRealInstance * max(n, 1))(*[i.to_c() for i in instances])
    out = (CMeasurement * max(n, 1))()
    check(lib().lmt_real_measure(arr, n, 1 if skip_opt else 0, out), what="real_measure")
    return np.frombuffer(out, dtype=MEASUREMENT_DTYPE, count=n).copy()


def execute_device(inst: RealInstance, variant: int, inputs, out=None):
    """One variant on torch CUDA tensors: inputs transpose [A], matrixMul [A, B],
    convolution [in], MVT [A, y1, y2, x1_0, x2_0]; returns the output tensor
    (MVT: x1 then x2)."""
    import torch

    err = validate(inst)
    if err:
        from .errors import InvalidInstance

        raise InvalidInstance([err])
    ins = [t.to(torch.float32).contiguous() for t in inputs]
    size = 2 * inst.n if inst.kernel == 3 else inst.n * inst.n
    if out is None:
        out = torch.empty(size, dtype=torch.float32, device="cuda")
    ptrs = (ctypes.c_void_p * len(ins))(*[t.data_ptr() for t in ins])
    check(lib().lmt_real_execute(ctypes.byref(inst.to_c()), int(variant), ptrs, ctypes.c_void_p(out.data_ptr()),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), what="real_execute")
    return out


def execute(inst: RealInstance, variant: int, inputs) -> np.ndarray:
    """Host arrays in, host output out (n*n or 2n floats)."""
    import torch

    ts = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda() for a in inputs]
    return execute_device(inst, variant, ts).cpu().numpy()


__all__ = ["KERNELS", "RealInstance", "instance_set", "measure", "execute", "execute_device", "validate"]
