// lmt_train_gpu.cuh -- random-forest training on the GPU,
// bit-identical to the reference's numpy trainer (forest.py:72-163,
// _best_split / _build_tree) and to the host restatement in lmt_train.h.
//
// One CTA per tree. The tree is built in the reference's DFS order (the
// node numbering and the per-split-attempt feature draws depend on it), but
// all the data-parallel work of a node runs across the CTA:
//
//  * presort (k_rf_presort): for every feature, the bootstrap positions
//    p = 0..n-1 sorted by (X[sample[p]][f], p) -- numpy's stable argsort of
//    the node's rows, whose order is always a subsequence of the sample
//    order, so position breaks ties exactly as stability does. One more
//    array holds the positions in natural order. Bitonic sort per (tree,
//    feature) in global memory.
//  * every node owns the same contiguous segment [begin, begin + nr) of all
//    nfeat + 1 arrays; a split stably partitions each segment (left rows
//    first, order kept), so the children's segments are again sorted and
//    contiguous: no per-node sort.
//  * _best_split per drawn feature: gather xs / ys in sorted order
//    (parallel), the two cumsums sequentially (one thread per feature, as
//    numpy's cumsum associates), the SSE of every candidate in parallel with
//    one IEEE op per numpy op (__dmul_rn / __ddiv_rn / __dsub_rn /
//    __dadd_rn, nothing fused), first-minimum argmin by a (sse, index)
//    reduction, then the midpoint threshold exactly as forest.py:100-103.
//  * leaf value: numpy's pairwise sum of the node's y in row order / nr.
//
// The feature subsets and the bootstrap sample are numpy's draws, generated
// on the host in the reference's order (they do not depend on the data).
#pragma once

#include <cuda_runtime.h>

namespace lmt {

constexpr int kRfTrainThreads = 256;
constexpr int kRfMaxK = 32;  // features drawn per node (features_per_node)

// (key, position) order of numpy's stable argsort
__device__ __forceinline__ bool rf_less(double ka, int pa, double kb, int pb) {
    return ka < kb || (ka == kb && pa < pb);
}

// Bitonic sort of the positions of one (tree, feature) by (X[sample[p]][f], p).
// keys/pos: [N2] scratch (N2 = next power of two >= n; padding sorts last);
// out: [n] sorted positions. f == nfeat: natural order.
__global__ void __launch_bounds__(kRfTrainThreads) k_rf_presort(const double *__restrict__ X, const int32_t *__restrict__ samples,
                                                                int n, int nfeat, int N2, double *__restrict__ keys_all,
                                                                int32_t *__restrict__ pos_all, int32_t *__restrict__ sorted_all) {
    const int tree = blockIdx.y, f = blockIdx.x;  // f in [0, nfeat]
    const int32_t *sample = samples + (size_t)tree * n;
    int32_t *out = sorted_all + ((size_t)tree * (nfeat + 1) + f) * n;
    if (f == nfeat) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = i;
        return;
    }
    double *keys = keys_all + ((size_t)tree * nfeat + f) * N2;
    int32_t *pos = pos_all + ((size_t)tree * nfeat + f) * N2;
    for (int i = threadIdx.x; i < N2; i += blockDim.x) {
        if (i < n) {
            keys[i] = X[(size_t)sample[i] * nfeat + f];
            pos[i] = i;
        } else {
            keys[i] = __longlong_as_double(0x7ff0000000000000ll);  // +inf, position beyond n: last
            pos[i] = i;
        }
    }
    __syncthreads();
    for (int k = 2; k <= N2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < N2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const double ki = keys[i], kl = keys[l];
                    const int pi = pos[i], pl = pos[l];
                    const bool up = (i & k) == 0;
                    const bool swap = up ? rf_less(kl, pl, ki, pi) : rf_less(ki, pi, kl, pl);
                    if (swap) {
                        keys[i] = kl;
                        keys[l] = ki;
                        pos[i] = pl;
                        pos[l] = pi;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = pos[i];
}

// numpy's pairwise_sum for float64 (lmt_train.h np_pairwise_sum)
__device__ double rf_pairwise_sum(const double *a, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(rf_pairwise_sum(a, n2), rf_pairwise_sum(a + n2, n - n2));
}

struct RfTrainArgs {
    const double *X, *y;
    const int32_t *samples;  // [T][n] bootstrap rows
    const int32_t *draws;    // [T][ndraws][k]
    int32_t *sorted;         // [T][nfeat + 1][n]
    int32_t *tmp;            // [T][n]
    uint8_t *flag;           // [T][n]
    double *xs, *ys, *s1, *s2;  // [T][k][n]
    int32_t *stack;          // [T][n + 1][4]
    int32_t *feature, *left, *right;  // [T][cap]
    double *threshold, *value;        // [T][cap]
    int64_t *nodes_out, *draws_used;  // [T]; draws_used -1: more draws needed
    int n, nfeat, k, ndraws, max_depth, msl;
    int64_t cap;
};

// Block-wide helpers over kRfTrainThreads threads
__device__ __forceinline__ int rf_block_sum(int v, int *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    int t = 0;
    for (int i = 0; i < kRfTrainThreads / 32; i++) t += sh[i];
    __syncthreads();
    return t;
}

// exclusive scan of one flag per thread; returns the prefix, *total the sum
__device__ __forceinline__ int rf_block_scan(int v, int *sh, int *total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    __syncthreads();
    if (l == 31) sh[w] = x;
    __syncthreads();
    int base = 0, t = 0;
    for (int i = 0; i < kRfTrainThreads / 32; i++) {
        if (i < w) base += sh[i];
        t += sh[i];
    }
    __syncthreads();
    *total = t;
    return base + x - v;
}

__global__ void __launch_bounds__(kRfTrainThreads) k_rf_build(const RfTrainArgs a) {
    const int tree = blockIdx.x, tid = threadIdx.x;
    const int n = a.n, F = a.nfeat, K = a.k;
    const int32_t *sample = a.samples + (size_t)tree * n;
    const int32_t *draws = a.draws + (size_t)tree * a.ndraws * K;
    int32_t *sorted = a.sorted + (size_t)tree * (F + 1) * n;
    int32_t *tmp = a.tmp + (size_t)tree * n;
    uint8_t *flag = a.flag + (size_t)tree * n;
    double *xs = a.xs + (size_t)tree * K * n, *ys = a.ys + (size_t)tree * K * n;
    double *s1 = a.s1 + (size_t)tree * K * n, *s2 = a.s2 + (size_t)tree * K * n;
    int32_t *stack = a.stack + (size_t)tree * (n + 1) * 4;
    int32_t *feature = a.feature + (size_t)tree * a.cap, *left = a.left + (size_t)tree * a.cap;
    int32_t *right = a.right + (size_t)tree * a.cap;
    double *threshold = a.threshold + (size_t)tree * a.cap, *value = a.value + (size_t)tree * a.cap;
    const int32_t *natural = sorted + (size_t)F * n;

    __shared__ int sh_int[32];
    __shared__ int s_begin, s_len, s_depth, s_slot, s_top, s_nodes, s_draw, s_done, s_stop, s_split, s_f, s_err;
    __shared__ double s_thr, s_best;
    __shared__ double r_sse[kRfTrainThreads / 32];
    __shared__ int r_idx[kRfTrainThreads / 32];
    __shared__ int s_feats[kRfMaxK];

    if (tid == 0) {
        s_nodes = 1;  // the root, slot 0
        feature[0] = -1;
        threshold[0] = 0.0;
        left[0] = right[0] = -1;
        value[0] = 0.0;
        stack[0] = 0;
        stack[1] = n;
        stack[2] = 0;
        stack[3] = 0;
        s_top = 1;
        s_draw = 0;
        s_err = 0;
    }
    __syncthreads();
    for (;;) {
        if (tid == 0) {
            s_done = s_top == 0 || s_err;
            if (!s_done) {
                const int t = --s_top;
                s_begin = stack[t * 4 + 0];
                s_len = stack[t * 4 + 1];
                s_depth = stack[t * 4 + 2];
                s_slot = stack[t * 4 + 3];
            }
        }
        __syncthreads();
        if (s_done) break;
        const int begin = s_begin, nr = s_len, depth = s_depth, slot = s_slot;
        const int32_t *nat = natural + begin;
        // stop rules (forest.py:138-143): depth, size, all targets equal
        const double y0 = a.y[sample[nat[0]]];
        int ne = 0;
        for (int i = tid; i < nr; i += kRfTrainThreads) ne |= a.y[sample[nat[i]]] != y0;
        const int anyne = rf_block_sum(ne, sh_int);
        if (tid == 0) s_stop = (a.max_depth >= 0 && depth >= a.max_depth) || nr < 2 * a.msl || anyne == 0;
        __syncthreads();
        bool split = false;
        if (!s_stop) {
            if (tid == 0) {
                if (s_draw >= a.ndraws) s_err = 1;
                else
                    for (int q = 0; q < K; q++) s_feats[q] = draws[(size_t)s_draw * K + q];
                s_draw++;
                s_split = 0;
            }
            __syncthreads();
            if (s_err) break;
            // gather xs / ys of every drawn feature in its sorted order
            for (int q = 0; q < K; q++) {
                const int32_t *seg = sorted + (size_t)s_feats[q] * n + begin;
                const int f = s_feats[q];
                for (int i = tid; i < nr; i += kRfTrainThreads) {
                    const int r = sample[seg[i]];
                    xs[(size_t)q * n + i] = a.X[(size_t)r * F + f];
                    ys[(size_t)q * n + i] = a.y[r];
                }
            }
            __syncthreads();
            // cumsum(ys), cumsum(ys * ys): sequential, one thread per feature
            if ((tid & 31) == 0 && (tid >> 5) < K) {
                for (int q = tid >> 5; q < K; q += kRfTrainThreads / 32) {
                    const double *yq = ys + (size_t)q * n;
                    double *a1 = s1 + (size_t)q * n, *a2 = s2 + (size_t)q * n;
                    double c1 = 0.0, c2 = 0.0;
                    for (int i = 0; i < nr; i++) {
                        const double v = yq[i];
                        c1 = __dadd_rn(c1, v);
                        c2 = __dadd_rn(c2, __dmul_rn(v, v));
                        a1[i] = c1;
                        a2[i] = c2;
                    }
                }
            }
            __syncthreads();
            for (int q = 0; q < K; q++) {
                const double *x = xs + (size_t)q * n;
                if (x[0] == x[nr - 1]) continue;  // constant feature
                const double *a1 = s1 + (size_t)q * n, *a2 = s2 + (size_t)q * n;
                const double S1 = a1[nr - 1], S2 = a2[nr - 1];
                double best = 0.0;
                int bi = -1;
                for (int kk = tid; kk + 1 < nr; kk += kRfTrainThreads) {
                    if (!(x[kk] < x[kk + 1])) continue;
                    if (a.msl > 1 && !((kk + 1 >= a.msl) && (nr - kk - 1 >= a.msl))) continue;
                    const double nl = (double)(kk + 1);
                    const double nrr = __dsub_rn((double)nr, nl);
                    const double t1 = __dsub_rn(a2[kk], __ddiv_rn(__dmul_rn(a1[kk], a1[kk]), nl));
                    const double c = __dsub_rn(S1, a1[kk]);
                    const double t2 = __dsub_rn(__dsub_rn(S2, a2[kk]), __ddiv_rn(__dmul_rn(c, c), nrr));
                    const double sse = __dadd_rn(t1, t2);
                    if (bi < 0 || sse < best) {  // each thread walks kk ascending: first minimum
                        best = sse;
                        bi = kk;
                    }
                }
                // (sse, index) minimum across the CTA: the first minimum of numpy's argmin
                for (int o = 16; o > 0; o >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (oi >= 0 && (bi < 0 || ob < best || (ob == best && oi < bi))) {
                        best = ob;
                        bi = oi;
                    }
                }
                if ((tid & 31) == 0) {
                    r_sse[tid >> 5] = best;
                    r_idx[tid >> 5] = bi;
                }
                __syncthreads();
                if (tid == 0) {
                    double b = 0.0;
                    int ix = -1;
                    for (int w = 0; w < kRfTrainThreads / 32; w++) {
                        const int oi = r_idx[w];
                        if (oi >= 0 && (ix < 0 || r_sse[w] < b || (r_sse[w] == b && oi < ix))) {
                            b = r_sse[w];
                            ix = oi;
                        }
                    }
                    if (ix >= 0 && (!s_split || b < s_best)) {  // strictly better than the earlier features
                        const double lo = x[ix], hi = x[ix + 1];
                        double thr = __dadd_rn(lo, __ddiv_rn(__dsub_rn(hi, lo), 2.0));
                        if (thr >= hi) thr = lo;  // midpoint rounded up between adjacent floats
                        s_best = b;
                        s_f = s_feats[q];
                        s_thr = thr;
                        s_split = 1;
                    }
                }
                __syncthreads();
            }
            split = s_split != 0;
        }
        if (!split) {
            // leaf: numpy's pairwise mean of the node's targets in row order
            for (int i = tid; i < nr; i += kRfTrainThreads) ys[i] = a.y[sample[nat[i]]];
            __syncthreads();
            if (tid == 0) value[slot] = __ddiv_rn(rf_pairwise_sum(ys, nr), (double)nr);
            __syncthreads();
            continue;
        }
        // split: X[row, f] <= thr goes left; stable partition of every array's segment
        const int f = s_f;
        const double thr = s_thr;
        for (int i = tid; i < nr; i += kRfTrainThreads) {
            const int p = nat[i];
            flag[p] = a.X[(size_t)sample[p] * F + f] <= thr ? 1 : 0;
        }
        __syncthreads();
        int nl = 0;
        for (int arr = 0; arr <= F; arr++) {
            int32_t *seg = sorted + (size_t)arr * n + begin;
            int lbase = 0, rbase = 0, tot = 0;
            // left count first (the right part starts after it)
            if (arr == 0) {
                int c = 0;
                for (int i = tid; i < nr; i += kRfTrainThreads) c += flag[seg[i]];
                nl = rf_block_sum(c, sh_int);
            }
            for (int t0 = 0; t0 < nr; t0 += kRfTrainThreads) {
                const int i = t0 + tid;
                const int p = i < nr ? seg[i] : 0;
                const int fl = i < nr ? flag[p] : 0;
                const int pre = rf_block_scan(fl, sh_int, &tot);
                const int cnt = min(kRfTrainThreads, nr - t0);
                if (i < nr) {
                    if (fl) tmp[lbase + pre] = p;
                    else tmp[nl + rbase + (i - t0 - pre)] = p;
                }
                lbase += tot;
                rbase += cnt - tot;
            }
            __syncthreads();
            for (int i = tid; i < nr; i += kRfTrainThreads) seg[i] = tmp[i];
            __syncthreads();
        }
        if (tid == 0) {
            const int l = s_nodes, r = s_nodes + 1;
            s_nodes += 2;
            if (r >= a.cap) {
                s_err = 2;
            } else {
                feature[slot] = f;
                threshold[slot] = thr;
                left[slot] = l;
                right[slot] = r;
                for (int c : {l, r}) {
                    feature[c] = -1;
                    threshold[c] = 0.0;
                    left[c] = right[c] = -1;
                    value[c] = 0.0;
                }
                int t = s_top;
                stack[t * 4 + 0] = begin + nl;  // right child: pushed first, popped last
                stack[t * 4 + 1] = nr - nl;
                stack[t * 4 + 2] = depth + 1;
                stack[t * 4 + 3] = r;
                t++;
                stack[t * 4 + 0] = begin;
                stack[t * 4 + 1] = nl;
                stack[t * 4 + 2] = depth + 1;
                stack[t * 4 + 3] = l;
                s_top = t + 1;
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.nodes_out[tree] = s_nodes;
        a.draws_used[tree] = s_err == 1 ? -1 : (s_err == 2 ? -2 : s_draw);
    }
}

}  // namespace lmt
