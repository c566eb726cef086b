"""Opcode mix of the specialised kernel of one instance, compiled here (NVRTC,
no GPU): the source lmt_kernel_source returns, the cubin's SASS, and the
opcode histogram of the hottest loop (the largest backward-branch body).

    python tools/sass_mix.py SAMPLE.npz IDX [base|opt]     # a bench-sample row
"""
import collections
import ctypes
import os
import re
import subprocess
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_6986_b200._lib import CInstance, lib  # noqa: E402
from tools.jit_check import compile_cubin  # noqa: E402


def source_of(rec, variant):
    L = lib()
    inst = CInstance(*[int(v) for v in rec[:19]])
    n = ctypes.c_int64()
    assert L.lmt_kernel_source(ctypes.byref(inst), None, variant, None, 0, ctypes.byref(n)) == 0, L.lmt_last_error()
    buf = ctypes.create_string_buffer(n.value + 1)
    assert L.lmt_kernel_source(ctypes.byref(inst), None, variant, buf, len(buf), ctypes.byref(n)) == 0
    return buf.value.decode()


def loops(sass):
    """[(start, end)] instruction-index ranges of backward branches."""
    ins = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    out = []
    for i, (a, txt) in enumerate(ins):
        m = re.search(r"\bBRA(?:\.\w+)*\s+[^;]*?0x([0-9a-f]+)", txt)
        if m:
            t = int(m.group(1), 16)
            if t < a and t in addr:
                out.append((addr[t], i))
    return ins, out


def opcode(txt):
    t = re.sub(r"^@!?U?P\w+\s+", "", txt.strip())
    return t.split()[0]


if __name__ == "__main__":
    z = np.load(sys.argv[1])
    idx = int(sys.argv[2])
    variant = 1 if len(sys.argv) > 3 and sys.argv[3] == "opt" else 0
    rec = z["rec"][idx]
    src = source_of(rec, variant)
    for kv in sys.argv[4:]:  # NAME=VALUE overrides of the LMT_* defines (e.g. U=8 D=2)
        k, v = kv.split("=")
        src = re.sub(rf"#define LMT_{k} \S+", f"#define LMT_{k} {v}", src)
    print("\n".join(l for l in src.splitlines() if l.startswith("#define LMT_")))
    cub, log = compile_cubin(src)
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as f:
        f.write(cub)
    sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
    os.unlink(f.name)
    ins, lps = loops(sass)
    print("instructions", len(ins), [l for l in log.splitlines() if "registers" in l or "spill" in l][:2])
    if lps:
        inner = [p for p in lps if not any(q != p and p[0] <= q[0] and q[1] <= p[1] for q in lps)]
        s, e = max(inner, key=lambda p: p[1] - p[0])
        body = [opcode(t) for _, t in ins[s:e + 1]]
        c = collections.Counter(body)
        fp = sum(v for k, v in c.items() if k.split(".")[0] in ("FFMA", "FADD", "FMUL"))
        print(f"hottest loop: {len(body)} instructions, fp32 {fp} ({fp / len(body):.2f})")
        for k, v in c.most_common(20):
            print(f"  {k:24s} {v}")
    if os.environ.get("DUMP"):
        open(os.environ["DUMP"], "w").write(sass)
