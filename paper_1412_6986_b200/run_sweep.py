"""The measured instance sweep as a job: every selected instance of a
SamplingSpec is featurised (K4), run and timed in both variants (K1/K2) and
verified on the GPU, sharded over the ranks of one node, checkpointed per
chunk, and written in the reference's dataset schema plus a measured-label
file.

    python -m paper_1412_6986_b200.run_sweep --out DIR [--max-instances 1000000] [--seed 0]
    torchrun --nproc-per-node 8 -m paper_1412_6986_b200.run_sweep --out DIR     # one rank per GPU

Per rank: a cost-balanced disjoint share of the selection (no data-path
collective), chunk files DIR/rank{r:03d}/chunk{k:06d}.npz written atomically
(a restarted job skips the chunks it already has), then the per-instance
labels are all-gathered (NCCL on GPUs, the only collective) and rank 0 writes
DIR/labels.npz; every rank writes its rows of the 39-column dataset CSV
(DIR/dataset.shardRRR-of-WWW.csv, dataset.py:284-341), and rank 0 merges them
into DIR/dataset.csv in the reference's row order. With --study, the
paper's random-forest study follows on the gathered labels (study.py: every
rank trains the same forests, predicts its own held-out rows, rank 0 scores
them into DIR/study.json).
"""

from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np


def _args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--out", required=True)
    ap.add_argument("--max-instances", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=1024,
                    help="instances per checkpoint, measured as one batch (small launches packed into SM partitions)")
    ap.add_argument("--limit", type=int, default=0, help="only the first N rows of this rank's share (testing)")
    ap.add_argument("--sample", type=int, default=0, help="a seeded random subset of N rows of the selection")
    ap.add_argument("--backend", default=None, help="torch.distributed backend (default nccl with a GPU, else gloo)")
    ap.add_argument("--study", action="store_true",
                    help="after the gather: the paper's RF study on modelled and measured labels (study.py)")
    ap.add_argument("--family", default="all", choices=("all", "dla", "grid"),
                    help="restrict to the dense-linear-algebra or structured-grid patterns (sweep.DLA_FAMILY / "
                         "GRID_FAMILY)")
    ap.add_argument("--concurrent", action="store_true", default=True,
                    help="launches of <= 74 CTAs in disjoint SM partitions (the default: the bench's placement)")
    ap.add_argument("--isolated", dest="concurrent", action="store_false",
                    help="every launch alone on the whole device")
    ap.add_argument("--regblock", action="store_true",
                    help="register-blocked variants (units sharing home coordinates load once) instead of the "
                         "literal ones (DESIGN.md 5, the measurement contract)")
    ap.add_argument("--warm-l2", action="store_true", help="no L2 flush before each whole-device variant")
    ap.add_argument("--samples", type=int, default=0,
                    help="output cells per instance read back into the chunk files (sweep.sample_cells), so an "
                         "independent checker can compare them with the CPU reference")
    return ap.parse_args(argv)


def rank_share(table, world: int, rank: int, sample: int = 0, seed: int = 0, family: str = "all") -> np.ndarray:
    """Cost-balanced disjoint share of the whole selection (or of one pattern
    family), or of a seeded random subset of `sample` rows (sorted rows)."""
    from . import sweep

    rows = np.arange(len(table))
    if family != "all":
        rows = sweep.family_rows(table, sweep.DLA_FAMILY if family == "dla" else sweep.GRID_FAMILY)
    if sample and sample < len(rows):
        rows = np.sort(np.random.default_rng(seed ^ 0x5A3B1E).choice(rows, size=sample, replace=False))
    if world == 1:
        return rows
    cost = sweep.launch_cost(table.records(rows))
    return np.sort(rows[sweep.shard_balanced(cost, world)[rank]])


def run(argv=None) -> dict:
    import torch
    import torch.distributed as dist

    from . import dataset, dist as ldist, measure, study, sweep
    from .access_analysis import features_records

    args = _args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cuda = torch.cuda.is_available()
    if cuda:
        torch.cuda.set_device(local % torch.cuda.device_count())  # ranks may share a GPU (tests)
    backend = args.backend or ("nccl" if cuda else "gloo")
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend)
    device = "cuda" if cuda and backend == "nccl" else None  # where the label gather's buffers live

    spec = sweep.SamplingSpec(max_instances=args.max_instances, seed=args.seed)
    table = sweep.select_instance_table(spec)
    mine = rank_share(table, world, rank, args.sample, args.seed, args.family)
    if args.limit:
        mine = mine[: args.limit]
    rdir = os.path.join(args.out, f"rank{rank:03d}")
    os.makedirs(rdir, exist_ok=True)
    t0 = time.time()
    rec = table.records(mine)
    fb = features_records(rec)
    mode = dict(concurrent=args.concurrent, regblock=args.regblock, warm_l2=args.warm_l2)
    measure.prepare_records(rec, **mode)
    t_prep = time.time() - t0

    # ---- chunks with checkpoint/resume
    done_rows, done_res, resumed = [], [], 0
    t_meas = 0.0
    for k, s in enumerate(range(0, len(mine), args.chunk)):
        path = os.path.join(rdir, f"chunk{k:06d}.npz")
        rows = mine[s: s + args.chunk]
        if os.path.exists(path):
            z = np.load(path)
            if np.array_equal(z["rows"], rows):
                done_rows.append(z["rows"])
                done_res.append(z["res"])
                resumed += 1
                continue
        crec = table.records(rows)
        extra = {}
        t1 = time.time()
        if args.samples:
            idx = sweep.sample_cells(crec, args.samples, args.seed * 1_000_003 + k)
            res, vals = measure.measure_records(crec, samples=idx, **mode)
            extra = dict(sample_idx=idx, sample_vals=vals)
        else:
            res = measure.measure_records(crec, **mode)
        t_meas += time.time() - t1
        tmp = path + ".tmp.npz"
        np.savez(tmp, rows=rows, res=res, rec=crec, **extra)
        os.replace(tmp, path)
        done_rows.append(rows)
        done_res.append(res)
    rows_all = np.concatenate(done_rows) if done_rows else np.zeros(0, np.int64)
    res_all = np.concatenate(done_res) if done_res else np.zeros(0, measure.MEASUREMENT_DTYPE)

    # ---- dataset rows (reference schema, modelled labels) per rank
    a = dataset.DatasetArrays(table, table.records(), np.full((len(table), 18), np.nan), np.full(len(table), np.nan),
                              np.full(len(table), -1, np.int32))
    a.X[mine], a.speedup[mine], a.status[mine] = fb.X, fb.label, fb.status
    ok_mine = mine[a.ok[mine]]
    dataset.write_shard(os.path.join(args.out, "dataset"), a, ok_mine, rank, world)

    # ---- the only collective: measured labels
    lab = ldist.label_matrix(rows_all, res_all)
    extra = np.stack([res_all["mismatches"].astype(np.float64), res_all["status"].astype(np.float64)], 1)
    # every rank's share is a deterministic function of the selection: sizes need no exchange
    sizes = [len(rank_share(table, world, r, args.sample, args.seed, args.family)[: args.limit or None])
             for r in range(world)]
    labels = ldist.all_gather_labels(np.concatenate([lab, extra], 1), device=device, sizes=sizes)
    summary = {"rank": rank, "world": world, "max_instances": args.max_instances, "seed": args.seed,
               "family": args.family, "sample": args.sample, "concurrent": args.concurrent,
               "regblock": args.regblock, "warm_l2": args.warm_l2,
               "rows": int(len(mine)), "chunks_resumed": resumed,
               "prepare_s": t_prep, "measure_s": t_meas,
               "instances_per_s": (len(mine) - resumed * args.chunk) / t_meas if t_meas > 0 else None,
               "mismatched": int((res_all["mismatches"] > 0).sum()),
               "verified": int((res_all["mismatches"] == 0).sum())}
    if args.study:  # every rank trains the same forests, predicts the held-out rows it measured
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        threads = max(1, (os.cpu_count() or 1) // max(1, local_world))
        summary["study"] = study.run_rank(args.out, table, labels, rows_all, rank, args.seed, threads)
    if rank == 0:
        if world > 1:
            dist.barrier()
        n = dataset.merge_shards(os.path.join(args.out, "dataset"), world, os.path.join(args.out, "dataset.csv"),
                                 table)
        row = labels[:, 0].astype(np.int64)
        tb, to = labels[:, 1], labels[:, 2]
        measured = np.where(to > 0, tb / np.where(to > 0, to, 1.0), 0.0)
        np.savez(os.path.join(args.out, "labels.npz"), row=row, t_base_ms=tb, t_opt_ms=to,
                 measured_speedup=measured, mismatches=labels[:, 3], status=labels[:, 4])
        summary.update(total_rows=int(len(row)), dataset_rows=n)
        if args.study:
            summary["study_result"] = study.merge(args.out, table, labels, world, args.seed)
        with open(os.path.join(args.out, "summary.json"), "w") as fh:
            json.dump(summary, fh, indent=1)
    elif world > 1:
        dist.barrier()
    if world > 1:
        dist.destroy_process_group()
    return summary


if __name__ == "__main__":
    print(json.dumps(run()))
