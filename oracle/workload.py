"""The sweep's instance list for the CPU reference arm -- TEST / BENCH
INFRASTRUCTURE ONLY (see oracle/__init__.py).

``bench.py --impl reference`` must not import the product package, yet it
has to time the same instances as the GPU arm. This is a standalone
restatement of the reference's ``dataset._select_instances``
(dataset.py:207-250) with ``sample_compile_tuples`` (109-134),
``expand_patterns`` (137-161), ``enumerate_launch_configs`` (164-188) and
``seeding.mix_seed`` (seeding.py:11-17), producing the flat 19-int records
of the C oracle (oracle.FIELDS order) sorted exactly like the reference's
``picked.sort()``. tests/test_oracle.py pins it record for record against
the product's table, which tests/test_host.py pins against the reference.
"""

from __future__ import annotations

import numpy as np

PATTERNS = ("xy_reuse", "x_reuse_row", "x_reuse_col", "y_reuse_row", "y_reuse_col",
            "no_reuse_row_major", "no_reuse_col_major")
_LARGE_N = {"xy_reuse", "x_reuse_row", "y_reuse_row"}
_LARGE_M = {"xy_reuse", "x_reuse_col", "y_reuse_col"}
_M64 = 0xFFFFFFFFFFFFFFFF


def mix_seed(seed: int, k: int) -> int:
    """seeding.py:11-17 (SplitMix64 finaliser)."""
    x = (seed + (k + 1) * 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def sweep_records(max_instances: int, seed: int = 0, num_tuples: int = 100, size: int = 2048) -> np.ndarray:
    """int32 [n, 19] records of SamplingSpec(max_instances, seed) with the
    default ranges (dataset.py:44-80)."""
    rng = np.random.default_rng(seed)
    kernels, seen = [], set()
    for _ in range(num_tuples):
        shape = int(rng.integers(0, 3))  # StencilShape order: rect, diamond, star
        radius, ci, ce, nc, nce, nu, nue = (int(rng.integers(lo, hi + 1)) for lo, hi in (
            (0, 2), (5, 44), (1, 48), (0, 13), (0, 13), (0, 4), (0, 4)))
        for pi, pat in enumerate(PATTERNS):
            for n in ((8, 16, 32, 64) if pat in _LARGE_N else (1, 2, 4, 8)):
                for m in ((8, 16, 32, 64) if pat in _LARGE_M else (1, 2, 4, 8)):
                    k = (size, size, size, size, pi, n, m, shape, radius, ci, ce, nc, nce, nu, nue)
                    if k not in seen:
                        seen.add(k)
                        kernels.append(k)
    divs = [1 << k for k in range(size.bit_length()) if size % (1 << k) == 0]
    launches = [(gx, gy, wx, wy) for gx in divs for gy in divs if gx * gy >= 512
                for wx in divs if gx % wx == 0 for wy in divs if gy % wy == 0 and wx * wy <= 1024]
    lcount = len(launches)
    rounds, reachable = 0, 0
    while reachable < max_instances and rounds < lcount:
        rounds += 1
        reachable = len(kernels) * min(lcount, rounds)
    take = min(lcount, rounds)
    orders = np.stack([np.random.default_rng(mix_seed(seed, k)).choice(lcount, size=take, replace=False)
                       for k in range(len(kernels))])
    total = min(max_instances, len(kernels) * take)
    k_idx = np.arange(total) % len(kernels)
    l_idx = orders[k_idx, np.arange(total) // len(kernels)]
    order = np.lexsort((l_idx, k_idx))
    km = np.array(kernels, dtype=np.int32)
    lm = np.array(launches, dtype=np.int32)
    return np.ascontiguousarray(np.concatenate([km[k_idx[order]], lm[l_idx[order]]], axis=1))
