"""Compile the NVRTC kernel source (lmt_args.h + lmt_jit.cuh) for a few keys
here (no GPU needed) and report registers/spills via cuobjdump, so the
(U, D) register model can be checked before spending GPU time.

    python tools/jit_check.py "shape r ci ce nc nce nu nue U D opt wide wrap maxt" ...
"""
import ctypes
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = os.path.join(ROOT, "paper_1412_6986_b200", "csrc")
NAMES = "SHAPE R CI CE NC NCE NU NUE U D OPT WIDE CTXWRAP MAXT H2 W2 P2 PF VEC MINB SHARE NM1".split()


def source(vals):
    text = open(os.path.join(CS, "lmt_args.h")).read() + "\n" + open(os.path.join(CS, "lmt_jit.cuh")).read()
    text = text.replace('#include "lmt_args.h"', "")
    vals = list(vals) + [1, 0, 0][len(vals) - 19:] if len(vals) < len(NAMES) else list(vals)  # MINB 1, SHARE 0, NM1 0
    return "".join(f"#define LMT_{n} {v}\n" for n, v in zip(NAMES, vals)) + text


def compile_cubin(src):
    nv = ctypes.CDLL("/usr/local/cuda/lib64/libnvrtc.so")
    prog = ctypes.c_void_p()
    assert nv.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"lmt_jit.cu", 0, None, None) == 0
    opts = [b"-arch=sm_100a", b"-std=c++17", b"-default-device", b"-lineinfo", b"-Xptxas=-v"]
    arr = (ctypes.c_char_p * len(opts))(*opts)
    rc = nv.nvrtcCompileProgram(prog, len(opts), arr)
    n = ctypes.c_size_t()
    nv.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value)
    nv.nvrtcGetProgramLog(prog, log)
    if rc != 0:
        raise SystemExit(log.value.decode())
    nv.nvrtcGetCUBINSize(prog, ctypes.byref(n))
    buf = ctypes.create_string_buffer(n.value)
    nv.nvrtcGetCUBIN(prog, buf)
    return buf.raw, log.value.decode()


if __name__ == "__main__":
    import time
    for arg in sys.argv[1:]:
        vals = [int(x) for x in arg.split()]
        t0 = time.time()
        cub, log = compile_cubin(source(vals))
        dt = time.time() - t0
        with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as f:
            f.write(cub)
        res = subprocess.run(["cuobjdump", "-res-usage", f.name], capture_output=True, text=True).stdout
        line = [l.strip() for l in res.splitlines() if "REG" in l]
        print(arg, f"{dt:.2f}s", line, [l for l in log.splitlines() if "spill" in l][:2])
        if os.environ.get("SASS"):
            print(subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout)
        os.unlink(f.name)
