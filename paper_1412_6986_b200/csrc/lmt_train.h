// lmt_train.h -- host (C++) random-forest tree builder, bit-identical to the
// reference's numpy trainer (forest.py:72-163: _best_split, _build_tree).
//
// The reference keeps training on the CPU and puts inference on the GPU
// (north_star: "model train/predict" API unchanged); this is the native
// equivalent of its trainer so the drop-in package can train without the
// reference installed. The random draws stay numpy's: the caller passes the
// bootstrap rows and the per-node feature subsets drawn from the tree's
// PCG64 stream in the reference's order (the bootstrap first, then one
// `sort(choice(n_features, k, replace=False))` per split attempt, in the
// reference's DFS order -- the draws do not depend on the data, so they can
// be generated up front). Every floating-point operation mirrors one numpy
// operation: stable argsort, sequential cumsum, the elementwise SSE
// expression, first-minimum argmin, the midpoint threshold, and numpy's
// pairwise summation for the leaf mean. Compiled with -ffp-contract=off.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

namespace lmt {

// numpy's pairwise_sum for float64 (umath/loops_utils.h.src): blocks of 8
// partial sums up to 128 elements, recursive halving above
inline double np_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// numpy's Generator(PCG64) stream from a given state, and its
// choice(pop, k, replace=False) for pop <= 10000 (Floyd's algorithm over a
// hash set, then a Fisher-Yates shuffle of the k picks; every bounded draw
// is Lemire's method on the buffered 32-bit output). Verified draw for draw
// against numpy 2.3 (tests/test_host.py::test_native_feature_draws).
struct NpPcg64 {
    unsigned __int128 state, inc;
    bool has32;
    uint32_t u32;
    uint64_t next64() {
        const unsigned __int128 mult = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
        state = state * mult + inc;
        const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        const uint64_t x = hi ^ lo;
        return rot ? (x >> rot) | (x << (64 - rot)) : x;
    }
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return u32;
        }
        const uint64_t v = next64();
        has32 = true;
        u32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // random_bounded_uint64(off = 0, rng, use_masked = false) for rng < 2^32
    uint64_t bounded(uint64_t rng) {
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        const uint32_t ex = (uint32_t)rng + 1;
        uint64_t m = (uint64_t)next32() * ex;
        uint32_t left = (uint32_t)m;
        if (left < ex) {
            const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % ex);
            while (left < thr) {
                m = (uint64_t)next32() * ex;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
    // sort(choice(pop, k, replace=False)) into out[k]
    void choice_sorted(int pop, int k, int32_t *out) {
        int64_t idx[64];
        for (int j = pop - k; j < pop; j++) {
            const int64_t val = (int64_t)bounded((uint64_t)j);
            bool seen = false;
            for (int q = 0; q < j - (pop - k); q++) seen |= idx[q] == val;
            idx[j - pop + k] = seen ? j : val;
        }
        for (int i = k - 1; i > 0; i--) {
            const int64_t jj = (int64_t)bounded((uint64_t)i);
            std::swap(idx[i], idx[jj]);
        }
        std::sort(idx, idx + k);
        for (int q = 0; q < k; q++) out[q] = (int32_t)idx[q];
    }
};

struct TreeOut {
    std::vector<int32_t> feature, left, right;
    std::vector<double> threshold, value;
    int64_t draws_used = 0;
};

// Returns 0, or 1 when more feature draws are needed than `ndraws`.
inline int build_tree(const double *X, const double *y, int64_t nfeat, const int64_t *sample, int64_t nsample,
                      const int32_t *draws, int64_t ndraws, int k, int max_depth, int msl, TreeOut *out) {
    struct Item {
        std::vector<int64_t> rows;
        int depth;
        int64_t slot;
    };
    auto new_node = [&]() {
        out->feature.push_back(-1);
        out->threshold.push_back(0.0);
        out->left.push_back(-1);
        out->right.push_back(-1);
        out->value.push_back(0.0);
        return (int64_t)out->feature.size() - 1;
    };
    std::vector<Item> stack;
    stack.push_back({std::vector<int64_t>(sample, sample + nsample), 0, new_node()});
    int64_t next_draw = 0;
    std::vector<double> yv, x, xs, ys, s1, s2;
    std::vector<int64_t> order;
    while (!stack.empty()) {
        Item it = std::move(stack.back());
        stack.pop_back();
        const int64_t nr = (int64_t)it.rows.size();
        yv.resize(nr);
        for (int64_t i = 0; i < nr; i++) yv[i] = y[it.rows[i]];
        bool all_eq = true;
        for (int64_t i = 1; i < nr && all_eq; i++) all_eq = yv[i] == yv[0];
        const bool stop = (max_depth >= 0 && it.depth >= max_depth) || nr < 2 * (int64_t)msl || all_eq;
        bool split = false;
        int best_f = -1;
        double best_thr = 0.0, best_sse = 0.0;
        if (!stop) {
            if (next_draw >= ndraws) return 1;
            const int32_t *feats = draws + next_draw * k;
            next_draw++;
            // _best_split (forest.py:72-114)
            x.resize(nr);
            order.resize(nr);
            xs.resize(nr);
            ys.resize(nr);
            s1.resize(nr);
            s2.resize(nr);
            for (int q = 0; q < k; q++) {
                const int f = feats[q];
                for (int64_t i = 0; i < nr; i++) x[i] = X[it.rows[i] * nfeat + f];
                std::iota(order.begin(), order.end(), 0);
                std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return x[a] < x[b]; });
                for (int64_t i = 0; i < nr; i++) xs[i] = x[order[i]];
                if (xs[0] == xs[nr - 1]) continue;
                double c1 = 0.0, c2 = 0.0;
                for (int64_t i = 0; i < nr; i++) {
                    ys[i] = yv[order[i]];
                    c1 += ys[i];
                    const double sq = ys[i] * ys[i];
                    c2 += sq;
                    s1[i] = c1;
                    s2[i] = c2;
                }
                const double S1 = s1[nr - 1], S2 = s2[nr - 1];
                bool any = false;
                int64_t pos = -1;
                double pos_sse = 0.0;
                for (int64_t kk = 0; kk + 1 < nr; kk++) {
                    if (!(xs[kk] < xs[kk + 1])) continue;
                    if (msl > 1 && !((kk + 1 >= msl) && (nr - kk - 1 >= msl))) continue;
                    const double nl = (double)(kk + 1);
                    const double nrr = (double)nr - nl;
                    const double a = s2[kk] - (s1[kk] * s1[kk]) / nl;
                    const double c = S1 - s1[kk];
                    const double b = (S2 - s2[kk]) - (c * c) / nrr;
                    const double sse = a + b;
                    if (!any || sse < pos_sse) {  // argmin: the first minimum
                        any = true;
                        pos = kk;
                        pos_sse = sse;
                    }
                }
                if (!any) continue;
                if (!split || pos_sse < best_sse) {
                    const double a = xs[pos], b = xs[pos + 1];
                    double thr = a + (b - a) / 2;
                    if (thr >= b) thr = a;  // midpoint rounded up between adjacent floats
                    best_sse = pos_sse;
                    best_f = f;
                    best_thr = thr;
                    split = true;
                }
            }
        }
        if (!split) {
            out->value[it.slot] = np_pairwise_sum(yv.data(), nr) / (double)nr;
            continue;
        }
        std::vector<int64_t> lrows, rrows;
        for (int64_t i = 0; i < nr; i++) {
            const int64_t r = it.rows[i];
            (X[r * nfeat + best_f] <= best_thr ? lrows : rrows).push_back(r);
        }
        out->feature[it.slot] = best_f;
        out->threshold[it.slot] = best_thr;
        const int64_t l = new_node(), rr = new_node();
        out->left[it.slot] = (int32_t)l;
        out->right[it.slot] = (int32_t)rr;
        stack.push_back({std::move(rrows), it.depth + 1, rr});
        stack.push_back({std::move(lrows), it.depth + 1, l});
    }
    out->draws_used = next_draw;
    return 0;
}

}  // namespace lmt
