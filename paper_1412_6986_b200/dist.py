"""Data-parallel sweep over ranks.

One process per GPU. Every rank regenerates the same deterministic instance
list (dataset.py:207-250 is a pure function of the SamplingSpec), takes a
disjoint, cost-balanced share of each batch -- no collective on the data
path -- measures it, and the per-instance labels are all-gathered once at the
end: the only collective, NCCL on GPUs (any torch.distributed backend works;
the tests use gloo on CPU).
"""

from __future__ import annotations

import numpy as np

from . import sweep

LABEL_COLUMNS = ("row", "t_base_ms", "t_opt_ms")


def rank_rows(table, rows: np.ndarray, world: int, rank: int, loads: np.ndarray | None = None) -> np.ndarray:
    """This rank's share of `rows` (greedy longest-processing-time on the
    launch-floor cost, sweep.launch_cost; shares are disjoint and cover
    `rows`). Pass the same `loads` array (length world) for consecutive
    batches on every rank to balance across batches too."""
    rows = np.asarray(rows)
    if world == 1:
        return rows
    cost = sweep.launch_cost(table.records(rows))
    return rows[sweep.shard_balanced(cost, world, loads)[rank]]


def label_matrix(rows: np.ndarray, res: np.ndarray) -> np.ndarray:
    """float64 [n, 3]: (row, t_base_ms, t_opt_ms) per measured instance
    (t_opt_ms < 0 when the optimized variant did not run)."""
    return np.stack([np.asarray(rows, dtype=np.float64), res["t_base_ms"].astype(np.float64),
                     res["t_opt_ms"].astype(np.float64)], axis=1)


def all_gather_labels(labels: np.ndarray, device=None, group=None, sizes=None) -> np.ndarray:
    """All-gather variable-length [n_r, k] label blocks from every rank and
    return them sorted by row: one all-gather of blocks padded to the
    largest. ``sizes`` (rows per rank) is known to every rank when the
    sharding is deterministic; without it the sizes are exchanged first."""
    import torch
    import torch.distributed as dist

    lab = torch.as_tensor(np.ascontiguousarray(labels, dtype=np.float64), device=device)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        out = lab.cpu().numpy()
        return out[np.argsort(out[:, 0], kind="stable")]
    world = dist.get_world_size(group)
    if sizes is None:
        n = torch.tensor([lab.shape[0]], dtype=torch.int64, device=device)
        got = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(got, n, group=group)
        sizes = [int(s.item()) for s in got]
    sizes = [int(s) for s in sizes]
    if len(sizes) != world or sizes[dist.get_rank(group)] != lab.shape[0]:
        raise ValueError(f"label block sizes {sizes} do not match this rank's {lab.shape[0]} rows")
    mx = max(sizes)
    pad = torch.zeros((mx, lab.shape[1]), dtype=torch.float64, device=device)
    pad[: lab.shape[0]] = lab
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    out = torch.cat([b[:s] for b, s in zip(bufs, sizes)]).cpu().numpy()
    return out[np.argsort(out[:, 0], kind="stable")]
