"""Seed fan-out (mirrors lmtune/seeding.py:11-17): SplitMix64 finaliser of
seed + (k + 1) * golden-ratio increment, so per-item RNG streams do not depend
on scheduling."""

from __future__ import annotations

_M64 = 0xFFFFFFFFFFFFFFFF


def mix_seed(seed: int, k: int) -> int:
    x = (seed + (k + 1) * 0x9E3779B97F4A7C15) & _M64
    for shift, mul in ((30, 0xBF58476D1CE4E5B9), (27, 0x94D049BB133111EB)):
        x = ((x ^ (x >> shift)) * mul) & _M64
    return x ^ (x >> 31)
