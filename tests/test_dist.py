"""The N>1 host path on CPU: world-size-2 gloo processes shard a sweep batch
disjointly by cost and all-gather the label blocks (the only collective;
NCCL on the GPU box)."""

import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1412_6986_b200 as L

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        table = L.select_instance_table(L.SamplingSpec(max_instances=5000, seed=3))
        rows = np.random.default_rng(7).permutation(len(table))[:97]
        mine = L.dist.rank_rows(table, rows, world, rank)
        # stand-in measurements (the GPU fills these): deterministic per row
        res = np.zeros(len(mine), dtype=L.measure.MEASUREMENT_DTYPE)
        res["t_base_ms"] = mine * 0.5 + 1.0
        res["t_opt_ms"] = np.where(mine % 3 == 0, -1.0, mine * 0.25 + 2.0)
        labels = L.dist.all_gather_labels(L.dist.label_matrix(mine, res))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), mine=mine, labels=labels, rows=rows)
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_and_label_gather(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    rows = got[0]["rows"]
    mine = [g["mine"] for g in got]
    # disjoint and complete
    assert len(np.intersect1d(mine[0], mine[1])) == 0
    assert np.array_equal(np.sort(np.concatenate(mine)), np.sort(rows))
    # every rank holds every label, sorted by row, values intact
    for g in got:
        lab = g["labels"]
        assert np.array_equal(lab[:, 0], np.sort(rows).astype(np.float64))
        r = lab[:, 0]
        assert np.array_equal(lab[:, 1], r * 0.5 + 1.0)
        assert np.array_equal(lab[:, 2], np.where(r % 3 == 0, -1.0, r * 0.25 + 2.0))
    assert np.array_equal(got[0]["labels"], got[1]["labels"])
    # cost balance: neither shard carries much more than half of the estimate
    import paper_1412_6986_b200 as L

    table = L.select_instance_table(L.SamplingSpec(max_instances=5000, seed=3))
    per = L.sweep.launch_cost(table.records(rows))
    cost = [L.sweep.launch_cost(table.records(m)).sum() for m in mine]
    # LPT bound: no share exceeds the mean by more than the largest single instance
    assert max(cost) <= sum(cost) / 2 + per.max() + 1e-12
    del torch


def _fake_study_set(table, labels):
    """Stand-in for study.study_set (K4 needs the GPU): deterministic rows,
    features and both label kinds from the gathered rows."""
    rows = np.sort(labels[:, 0].astype(np.int64))
    rng = np.random.default_rng(11)
    X = np.round(rng.uniform(0, 64, size=(len(rows), 18)))
    modelled = 2.0 ** (X[:, 0] / 16 - 2 + (X[:, 3] > 32))
    measured = np.where(rows % 7 == 0, 0.0, 2.0 ** (X[:, 1] / 32 - 1))
    return rows, X, modelled, measured


def _cpu_predict(forest, X):
    import oracle

    return 2.0 ** oracle.forest_mean(forest.trees, np.asarray(X, dtype=np.float64), nthreads=1)


def _study_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1412_6986_b200 as L

    L.study.study_set = _fake_study_set
    L.forest.predict = _cpu_predict
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = np.arange(400)
        mine = rows[rank::world]  # any disjoint cover
        labels = np.stack([rows.astype(np.float64)] + [np.zeros(400)] * 4, 1)
        L.study.run_rank(out_dir, None, labels, mine, rank, seed=5, threads=2)
        if world > 1:
            dist.barrier()
        if rank == 0:
            L.study.merge(out_dir, None, labels, world, seed=5)
    finally:
        if world > 1:
            dist.destroy_process_group()


def test_two_rank_study_matches_one_rank(tmp_path):
    """study.py's distributed form (SURVEY 8(e) "after the gather"): two gloo
    ranks each predict their own held-out rows; rank 0's merged scores equal
    a one-rank run's."""
    pytest.importorskip("torch")
    import json

    import torch.multiprocessing as mp

    one, two = tmp_path / "one", tmp_path / "two"
    one.mkdir()
    two.mkdir()
    mp.start_processes(_study_worker, args=(1, 0, str(one)), nprocs=1, join=True, start_method="spawn")
    mp.start_processes(_study_worker, args=(2, _free_port(), str(two)), nprocs=2, join=True, start_method="spawn")
    a = json.load(open(one / "study.json"))
    b = json.load(open(two / "study.json"))
    assert a["ranks"] == 1 and b["ranks"] == 2
    a.pop("ranks"), b.pop("ranks")
    assert a == b
    assert a["held_out"] == 360 and a["train"] == 40
    for k in ("modelled_labels", "measured_labels"):
        assert 0.0 <= a[k]["count_accuracy"] <= 1.0 and sum(a[k]["confusion"]) == 360


def _bench_worker(rank, world, port, out_dir):
    """bench.py's multi-rank plumbing with stand-in measurements: per step
    the contiguous cost-prefix share (bench.step_rows), the label all-gather
    with locally known sizes (the only data collective; gloo here, NCCL on
    GPUs) and timers/counters through a separate gloo group."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    import paper_1412_6986_b200 as L

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    meta = dist.new_group(backend="gloo")
    try:
        table = L.select_instance_table(L.SamplingSpec(max_instances=20_000, seed=0))
        steps, batch = range(1, 3), 24
        mine = np.concatenate([bench.step_rows(table, 0, s, world, rank, batch) for s in steps])
        sizes = [sum(len(bench.step_rows(table, 0, s, world, r, batch)) for s in steps) for r in range(world)]
        res = np.zeros(len(mine), dtype=L.measure.MEASUREMENT_DTYPE)
        res["t_base_ms"] = mine * 0.5 + 1.0
        res["t_opt_ms"] = np.where(mine % 3 == 0, -1.0, mine * 0.25 + 2.0)
        labels = L.dist.all_gather_labels(L.dist.label_matrix(mine, res), sizes=sizes)
        (mx,), (n,) = bench.max_sum_over_ranks([float(rank)], [len(mine)], world, meta)
        glob = np.concatenate([bench.global_rows(0, len(table), s, world, batch) for s in steps])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), mine=mine, labels=labels, mx=mx, n=n, glob=glob)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bench_sharding_and_gather(tmp_path, world):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp

    mp.start_processes(_bench_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    mine = [g["mine"] for g in got]
    glob = got[0]["glob"]
    allm = np.concatenate(mine)
    assert len(np.unique(allm)) == len(allm) == len(glob)  # disjoint
    assert np.array_equal(np.sort(allm), np.sort(glob))    # complete
    for g in got:
        lab = g["labels"]
        r = lab[:, 0]
        assert np.array_equal(r, np.sort(glob).astype(np.float64))
        assert np.array_equal(lab[:, 1], r * 0.5 + 1.0)
        assert np.array_equal(lab[:, 2], np.where(r % 3 == 0, -1.0, r * 0.25 + 2.0))
        assert g["mx"] == world - 1 and g["n"] == len(glob)
