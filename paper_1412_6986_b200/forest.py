"""Random-forest inference on the GPU behind the reference's forest API
(lmtune/forest.py:38-69, 199-380).

``predict(forest, X)`` uploads the forest once (breadth-first node layout,
16-byte nodes, the top levels of each tree staged in shared memory) and runs
K3 (``k_rf_mean``): one warp per sample, one lane per tree, the leaf values
summed in tree order in fp64 -- bit-identical to the reference's
``acc += tree.predict(X)`` loop and ``acc / len(trees)`` (forest.py:215-218).
The final ``2.0 ** mean`` is evaluated by numpy on the host exactly as the
reference does, because numpy's SIMD ``pow`` is not reproducible by any CUDA
``pow`` (hard part 7).

Training is not on this path: forests come from the reference's CPU
``lmtune.forest.train`` (or any object with the same ``trees`` arrays), or
from a model file through ``load`` (the ``lmforest 1`` text format,
forest.py:227-380).
"""

from __future__ import annotations

import ctypes
import functools
import math
import threading
import zlib
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib
from .errors import ModelFormatError

FORMAT_NAME = "lmforest"
FORMAT_VERSION = 1
TARGET_FLOOR = -10.0


@dataclass(frozen=True)
class Hyperparams:
    num_trees: int = 20
    features_per_node: int = 4
    max_depth: int | None = None
    min_samples_leaf: int = 1
    bootstrap: bool = True
    seed: int = 0


@dataclass
class Tree:
    """Node arrays of one regression tree; feature -1 marks a leaf."""

    feature: np.ndarray
    threshold: np.ndarray
    left: np.ndarray
    right: np.ndarray
    value: np.ndarray
    oob_indices: np.ndarray | None = None

    def predict(self, X: np.ndarray) -> np.ndarray:
        """Leaf value per row (forest.py:49-58), on the GPU (a one-tree forest:
        value / 1.0 is exact)."""
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        if X.ndim == 1:
            X = X[None, :]
        g = GpuForest([self], X.shape[1])
        try:
            return g.mean(X)
        finally:
            g.close()


@dataclass
class Forest:
    hyperparams: Hyperparams
    feature_names: tuple[str, ...]
    trees: list[Tree] = field(default_factory=list)


def _tree_draws(seed: int, n: int, nfeat: int, hp: Hyperparams, ndraws: int):
    """The tree's numpy draws in the reference's order (forest.py:117-122, 77):
    bootstrap rows, then one sorted feature subset per split attempt."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if hp.bootstrap:
        sample = rng.integers(0, n, size=n)
        oob = np.setdiff1d(np.arange(n), sample)
    else:
        sample = np.arange(n)
        oob = None
    k = min(hp.features_per_node, nfeat)
    draws = np.empty((ndraws, k), dtype=np.int32)
    if nfeat <= 10000 and k <= 64:
        # the same numpy stream continued natively (lmt_rf_feature_draws:
        # PCG64 + Generator.choice's algorithm, bit-identical): a Python loop
        # of rng.choice calls costs ~12 us per draw
        st = rng.bit_generator.state
        mask = (1 << 64) - 1
        s4 = np.array([st["state"]["state"] >> 64, st["state"]["state"] & mask, st["state"]["inc"] >> 64,
                       st["state"]["inc"] & mask], dtype=np.uint64)
        check(lib().lmt_rf_feature_draws(ctypes.c_void_p(s4.ctypes.data), int(st["has_uint32"]),
                                         int(st["uinteger"]), nfeat, k, ndraws, ctypes.c_void_p(draws.ctypes.data)),
              what="rf_feature_draws")
    else:
        for i in range(ndraws):
            draws[i] = np.sort(rng.choice(nfeat, size=k, replace=False))
    return np.ascontiguousarray(sample, dtype=np.int64), oob, draws


def _build_tree(X: np.ndarray, y: np.ndarray, hp: Hyperparams, tree_seed: int) -> Tree:
    """forest.py:117-163 in native code (lmt_rf_train_tree), bit-identical."""
    n, nfeat = X.shape
    ndraws = min(2 * n, 4096)
    while True:
        sample, oob, draws = _tree_draws(tree_seed, n, nfeat, hp, ndraws)
        cap = 2 * n + 1
        feat = np.empty(cap, dtype=np.int32)
        thr = np.empty(cap, dtype=np.float64)
        left = np.empty(cap, dtype=np.int32)
        right = np.empty(cap, dtype=np.int32)
        val = np.empty(cap, dtype=np.float64)
        nodes, used = ctypes.c_int64(), ctypes.c_int64()
        vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        rc = lib().lmt_rf_train_tree(vp(X), vp(y), n, nfeat, vp(sample), len(sample), vp(draws), len(draws),
                                     draws.shape[1], -1 if hp.max_depth is None else hp.max_depth,
                                     hp.min_samples_leaf, vp(feat), vp(thr), vp(left), vp(right), vp(val), cap,
                                     ctypes.byref(nodes), ctypes.byref(used))
        if rc != 0 and used.value == -1 and ndraws < 2 * n + 1:
            ndraws = min(2 * n + 1, ndraws * 4)  # more split attempts than drawn: draw more
            continue
        check(rc, what="rf_train_tree")
        m = nodes.value
        return Tree(feat[:m].copy(), thr[:m].copy(), left[:m].copy(), right[:m].copy(), val[:m].copy(),
                    oob_indices=oob)


def _training_set(X, y, feature_names):
    """Contiguous float64 copies of the training arrays, checked as
    forest.train_arrays checks them (same ValueError messages), and the
    feature names (f0, f1, ... by default); plus one seed per tree."""
    Xc = np.ascontiguousarray(X, dtype=np.float64)
    yc = np.ascontiguousarray(y, dtype=np.float64)
    if Xc.ndim != 2 or Xc.shape[0] != yc.shape[0]:
        raise ValueError(f"bad training shapes {Xc.shape} vs {yc.shape}")
    if yc.shape[0] == 0:
        raise ValueError("empty training set")
    names = tuple(feature_names) if feature_names is not None else tuple(f"f{i}" for i in range(Xc.shape[1]))
    return Xc, yc, names


def _tree_seeds(hp: Hyperparams) -> list:
    from .seeding import mix_seed

    return [mix_seed(hp.seed, t) for t in range(hp.num_trees)]


def train_arrays(X, y, hp: Hyperparams, feature_names=None, threads: int = 1) -> Forest:
    """forest.train_arrays (forest.py:166-188): fit on a feature matrix and
    log2-speedup targets. Each tree is built natively from its own seed
    (no shared state), so host threads change nothing but the wall time."""
    Xc, yc, names = _training_set(X, y, feature_names)
    build = functools.partial(_build_tree, Xc, yc, hp)
    seeds = _tree_seeds(hp)
    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=threads) as pool:
            trees = list(pool.map(build, seeds))
    else:
        trees = list(map(build, seeds))
    return Forest(hyperparams=hp, feature_names=names, trees=trees)


def train_arrays_gpu(X, y, hp: Hyperparams, feature_names=None) -> Forest:
    """train_arrays with every tree built on the GPU in one call
    (lmt_rf_train_gpu, one CTA per tree; csrc/lmt_train_gpu.cuh), bit-identical
    to the reference's forest.train_arrays (forest.py:166-188). The bootstrap
    rows and per-node feature subsets are numpy's draws, made here in the
    reference's order."""
    X, y, feature_names = _training_set(X, y, feature_names)
    n, nfeat = X.shape
    T = hp.num_trees
    seeds = _tree_seeds(hp)
    ndraws = min(2 * n + 1, 4096)
    cap = 2 * n + 1
    vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    while True:
        drawn = [_tree_draws(sd, n, nfeat, hp, ndraws) for sd in seeds]
        samples = np.ascontiguousarray(np.stack([d[0] for d in drawn]), dtype=np.int64)
        draws = np.ascontiguousarray(np.stack([d[2] for d in drawn]), dtype=np.int32)
        k = draws.shape[2]
        feat = np.empty((T, cap), dtype=np.int32)
        thr = np.empty((T, cap), dtype=np.float64)
        left = np.empty((T, cap), dtype=np.int32)
        right = np.empty((T, cap), dtype=np.int32)
        val = np.empty((T, cap), dtype=np.float64)
        nodes = np.zeros(T, dtype=np.int64)
        used = np.zeros(T, dtype=np.int64)
        rc = lib().lmt_rf_train_gpu(vp(X), vp(y), n, nfeat, T, vp(samples), vp(draws), ndraws, k,
                                    -1 if hp.max_depth is None else hp.max_depth, hp.min_samples_leaf, vp(feat),
                                    vp(thr), vp(left), vp(right), vp(val), cap, vp(nodes), vp(used))
        if rc != 0 and (used == -1).any() and ndraws < 2 * n + 1:
            ndraws = min(2 * n + 1, ndraws * 4)  # more split attempts than drawn: draw more
            continue
        check(rc, what="rf_train_gpu")
        trees = [Tree(feat[t, :m].copy(), thr[t, :m].copy(), left[t, :m].copy(), right[t, :m].copy(),
                      val[t, :m].copy(), oob_indices=drawn[t][1]) for t, m in enumerate(nodes)]
        return Forest(hyperparams=hp, feature_names=tuple(feature_names), trees=trees)


def train(rows, hp: Hyperparams = Hyperparams(), threads: int = 1) -> Forest:
    """forest.train (forest.py:191-196): rows with .features and .speedup;
    target log2(speedup), infeasible floored at -10."""
    from .access_analysis import FEATURE_NAMES

    X = np.stack([r.features.to_array() for r in rows])
    y = np.array([speedup_to_target(r.speedup) for r in rows], dtype=np.float64)
    return train_arrays(X, y, hp, feature_names=FEATURE_NAMES, threads=threads)


def speedup_to_target(speedup: float) -> float:
    """log2 target with the infeasible floor (forest.py:68-69)."""
    return math.log2(speedup) if speedup > 0 else TARGET_FLOOR


class GpuForest:
    """A forest uploaded to the current GPU (lmt_rf_create)."""

    def __init__(self, trees, nfeat: int):
        feats = [np.ascontiguousarray(np.asarray(t.feature, dtype=np.int32)) for t in trees]
        self.feature = np.concatenate(feats)
        self.threshold = np.ascontiguousarray(np.concatenate([np.asarray(t.threshold, dtype=np.float64) for t in trees]))
        self.left = np.ascontiguousarray(np.concatenate([np.asarray(t.left, dtype=np.int32) for t in trees]))
        self.right = np.ascontiguousarray(np.concatenate([np.asarray(t.right, dtype=np.int32) for t in trees]))
        self.value = np.ascontiguousarray(np.concatenate([np.asarray(t.value, dtype=np.float64) for t in trees]))
        self.offsets = np.zeros(len(trees) + 1, dtype=np.int64)
        self.offsets[1:] = np.cumsum([len(f) for f in feats])
        self.ntrees, self.nfeat = len(trees), int(nfeat)
        h = ctypes.c_void_p()
        vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        check(lib().lmt_rf_create(vp(self.feature), vp(self.threshold), vp(self.left), vp(self.right),
                                  vp(self.value), vp(self.offsets), self.ntrees, self.nfeat, ctypes.byref(h)),
              what="rf_create")
        self.handle = h

    def mean(self, X: np.ndarray, votes: bool = False):
        """acc / T per row; with ``votes`` also the per-row count of trees
        whose leaf (log2 speedup) is > 0."""
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        if X.ndim != 2 or X.shape[1] != self.nfeat:
            raise ValueError(f"expected [n, {self.nfeat}] features, got {X.shape}")
        n = X.shape[0]
        out = np.empty(n, dtype=np.float64)
        v = np.empty(n, dtype=np.int32) if votes else None
        if n:
            check(lib().lmt_rf_mean_host(self.handle, ctypes.c_void_p(X.ctypes.data), n,
                                         ctypes.c_void_p(out.ctypes.data),
                                         ctypes.c_void_p(v.ctypes.data) if votes else None), what="rf_mean")
        return (out, v) if votes else out

    def mean_device(self, X_t, out_t, votes_t=None, stream=None):
        """Device-resident variant on torch tensors (no host copies)."""
        check(lib().lmt_rf_mean(self.handle, ctypes.c_void_p(X_t.data_ptr()), X_t.shape[0],
                                ctypes.c_void_p(out_t.data_ptr()),
                                ctypes.c_void_p(votes_t.data_ptr()) if votes_t is not None else None,
                                ctypes.c_void_p(stream) if stream else None), what="rf_mean")

    def close(self):
        if self.handle:
            lib().lmt_rf_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache_lock = threading.Lock()
_cache: dict[tuple, tuple[object, tuple, GpuForest]] = {}


def _fingerprint(forest) -> tuple:
    """Content of every tree (crc32 of its arrays, cheap next to a predict),
    so trees edited in place are re-uploaded like the reference re-reads them."""
    fp = []
    for t in forest.trees:
        h = 0
        for a in (t.feature, t.threshold, t.left, t.right, t.value):
            h = zlib.crc32(np.ascontiguousarray(a).tobytes(), h)
        fp.append((len(t.feature), h))
    return tuple(fp)


def _current_device() -> int:
    d = ctypes.c_int32(0)
    check(lib().lmt_current_device(ctypes.byref(d)), what="current_device")
    return int(d.value)


def gpu_forest(forest) -> GpuForest:
    """Upload once per (forest object, CUDA device), re-uploaded when the
    trees' contents change."""
    key = (id(forest), _current_device())
    fp = _fingerprint(forest)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0] is forest and hit[1] == fp:
            return hit[2]
        g = GpuForest(forest.trees, len(forest.feature_names))
        if len(_cache) > 8:
            _cache.clear()
        _cache[key] = (forest, fp, g)
        return g


def _as_matrix(features) -> tuple[np.ndarray, bool]:
    if hasattr(features, "to_array"):
        return np.asarray(features.to_array(), dtype=np.float64)[None, :], True
    arr = np.asarray(features, dtype=np.float64)
    if arr.ndim == 1:
        return arr[None, :], True
    return arr, False


def predict_mean(forest, features) -> np.ndarray:
    """The fp64 mean of per-tree leaf values (before 2 ** .), on the GPU."""
    X, _ = _as_matrix(features)
    if X.shape[1] != len(forest.feature_names):
        raise ValueError(f"feature count {X.shape[1]} does not match model ({len(forest.feature_names)})")
    return gpu_forest(forest).mean(X)


def predict(forest, features):
    """Predicted speedup(s) = 2 ** mean(leaf values) (forest.py:208-219)."""
    X, single = _as_matrix(features)
    if X.shape[1] != len(forest.feature_names):
        raise ValueError(f"feature count {X.shape[1]} does not match model ({len(forest.feature_names)})")
    mean = gpu_forest(forest).mean(X)
    pred = 2.0 ** mean
    return float(pred[0]) if single else pred


def decide(forest, features):
    """True = apply the local-memory optimization (forest.py:222-224)."""
    return predict(forest, features) > 1.0


# ------------------------------------------------------------ model file I/O


def save(forest, path) -> None:
    """``lmforest 1`` text dump, pre-order nodes (forest.py:231-258)."""
    hp = forest.hyperparams
    out = [
        f"{FORMAT_NAME} {FORMAT_VERSION}",
        f"num_trees {hp.num_trees}",
        f"features_per_node {hp.features_per_node}",
        "max_depth " + ("none" if hp.max_depth is None else str(hp.max_depth)),
        f"min_samples_leaf {hp.min_samples_leaf}",
        "bootstrap " + ("true" if hp.bootstrap else "false"),
        f"seed {hp.seed}",
        f"num_features {len(forest.feature_names)}",
        "feature_names " + ",".join(forest.feature_names),
    ]
    for t, tree in enumerate(forest.trees):
        out.append(f"tree {t}")
        todo = [0]
        while todo:
            k = todo.pop()
            if tree.feature[k] < 0:
                out.append(f"leaf {float(tree.value[k])!r}")
            else:
                out.append(f"node {tree.feature[k]} {float(tree.threshold[k])!r}")
                todo += [int(tree.right[k]), int(tree.left[k])]
    out.append("end")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(out) + "\n")


class _Lines:
    def __init__(self, path):
        with open(path, encoding="utf-8") as fh:
            self.lines = fh.read().splitlines()
        self.i = 0

    def take(self) -> tuple[int, str]:
        if self.i >= len(self.lines):
            raise ModelFormatError(f"line {self.i + 1}: unexpected end of file")
        self.i += 1
        return self.i, self.lines[self.i - 1]

    def keyed_int(self, key: str) -> int:
        ln, line = self.take()
        parts = line.split()
        if len(parts) != 2 or parts[0] != key:
            raise ModelFormatError(f"line {ln}: expected '{key} <value>', got {line!r}")
        try:
            return int(parts[1])
        except ValueError as exc:
            raise ModelFormatError(f"line {ln}: bad integer for {key}: {parts[1]!r}") from exc


def _read_tree(rd: _Lines, nfeat: int) -> Tree:
    feature, threshold, left, right, value = [], [], [], [], []

    def node() -> int:
        ln, line = rd.take()
        parts = line.split()
        k = len(feature)
        if len(parts) == 2 and parts[0] == "leaf":
            try:
                v = float(parts[1])
            except ValueError as exc:
                raise ModelFormatError(f"line {ln}: bad leaf value {parts[1]!r}") from exc
            feature.append(-1)
            threshold.append(0.0)
            value.append(v)
        elif len(parts) == 3 and parts[0] == "node":
            try:
                f, thr = int(parts[1]), float(parts[2])
            except ValueError as exc:
                raise ModelFormatError(f"line {ln}: bad node line {line!r}") from exc
            if not 0 <= f < nfeat:
                raise ModelFormatError(f"line {ln}: feature index {f} out of range")
            feature.append(f)
            threshold.append(thr)
            value.append(0.0)
        else:
            raise ModelFormatError(f"line {ln}: expected node or leaf, got {line!r}")
        left.append(-1)
        right.append(-1)
        return k

    # pre-order: each node hangs under the deepest internal node still missing a child
    pending = [node()]
    if feature[pending[0]] < 0:
        pending = []
    while pending:
        k = node()
        parent = pending[-1]
        if left[parent] < 0:
            left[parent] = k
        else:
            right[parent] = k
            pending.pop()
        if feature[k] >= 0:
            pending.append(k)
    return Tree(np.array(feature, dtype=np.int32), np.array(threshold, dtype=np.float64),
                np.array(left, dtype=np.int32), np.array(right, dtype=np.int32),
                np.array(value, dtype=np.float64))


def load(path) -> Forest:
    """Parse an ``lmforest 1`` file; malformed input raises ModelFormatError
    naming the line (forest.py:285-380)."""
    rd = _Lines(path)
    ln, line = rd.take()
    if line.split() != [FORMAT_NAME, str(FORMAT_VERSION)]:
        raise ModelFormatError(f"line {ln}: unsupported format header {line!r}")
    num_trees = rd.keyed_int("num_trees")
    if num_trees < 1:
        raise ModelFormatError(f"line 2: num_trees {num_trees} < 1")
    fpn = rd.keyed_int("features_per_node")
    ln, line = rd.take()
    if not line.startswith("max_depth "):
        raise ModelFormatError(f"line {ln}: expected max_depth, got {line!r}")
    raw = line.split(maxsplit=1)[1]
    max_depth = None if raw == "none" else int(raw)
    msl = rd.keyed_int("min_samples_leaf")
    ln, line = rd.take()
    if line not in ("bootstrap true", "bootstrap false"):
        raise ModelFormatError(f"line {ln}: expected bootstrap true|false, got {line!r}")
    bootstrap = line == "bootstrap true"
    seed = rd.keyed_int("seed")
    nfeat = rd.keyed_int("num_features")
    ln, line = rd.take()
    if not line.startswith("feature_names "):
        raise ModelFormatError(f"line {ln}: expected feature_names, got {line!r}")
    names = tuple(line.split(maxsplit=1)[1].split(","))
    if len(names) != nfeat:
        raise ModelFormatError(f"line {ln}: {len(names)} names for {nfeat} features")
    trees = []
    for t in range(num_trees):
        ln, line = rd.take()
        if line != f"tree {t}":
            raise ModelFormatError(f"line {ln}: expected 'tree {t}', got {line!r}")
        trees.append(_read_tree(rd, nfeat))
    ln, line = rd.take()
    if line != "end":
        raise ModelFormatError(f"line {ln}: expected 'end', got {line!r}")
    return Forest(Hyperparams(num_trees, fpn, max_depth, msl, bootstrap, seed), names, trees)


def synthetic_forest(ntrees: int = 20, nfeat: int = 18, nodes_per_tree: int = 8501, max_depth: int = 31,
                     seed: int = 0) -> Forest:
    """A deterministic random forest of the reference's shape (20 trees of
    ~8.5k nodes, depth <= 31) for benchmarking without a trained
    model. Thresholds/values are random fp64; structure is a random binary
    tree grown breadth-first to ``nodes_per_tree`` (odd) nodes."""
    rng = np.random.default_rng(seed)
    trees = []
    for _ in range(ntrees):
        n = nodes_per_tree | 1
        feature = np.full(n, -1, dtype=np.int32)
        left = np.full(n, -1, dtype=np.int32)
        right = np.full(n, -1, dtype=np.int32)
        depth = np.zeros(n, dtype=np.int32)
        frontier = [0]
        nxt = 1
        while nxt + 1 < n and frontier:
            k = frontier.pop(int(rng.integers(len(frontier))))
            if depth[k] >= max_depth:
                continue
            feature[k] = rng.integers(nfeat)
            left[k], right[k] = nxt, nxt + 1
            depth[nxt] = depth[nxt + 1] = depth[k] + 1
            frontier += [nxt, nxt + 1]
            nxt += 2
        n = nxt
        thr = rng.normal(0, 1000, size=n)
        val = rng.normal(0, 2, size=n)
        trees.append(Tree(feature[:n].copy(), np.where(feature[:n] >= 0, thr, 0.0), left[:n].copy(),
                          right[:n].copy(), np.where(feature[:n] < 0, val, 0.0)))
    return Forest(Hyperparams(num_trees=ntrees, seed=seed), tuple(f"f{i}" for i in range(nfeat)), trees)
