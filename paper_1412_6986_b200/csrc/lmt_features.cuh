// lmt_features.cuh -- K4: per-instance feature vector and modelled label on
// the GPU, one warp per instance.
//
//   access_analysis.extract_features  (access_analysis.py:272-308)
//     reuse_degree 74-88, footprint 184-213, coalescing_degree 119-155,
//     estimate_registers (cost_model.py:41-60)
//   cost_model.kernel_time / label_speedup with the coalescing override the
//     dataset builder passes (cost_model.py:63-158, dataset.py:264-271)
//
// Bit-exactness: every feature is an integer converted to double except
// noncoalescing_degree = total / (nwarps * n * m), an int / int true division
// that __ddiv_rn rounds exactly like Python; the label arithmetic is the
// reference's expression tree, one IEEE double operation per Python
// operator in Python's left-to-right order (__dmul_rn / __dadd_rn /
// __ddiv_rn, so nothing is contracted into an FMA).
#pragma once

#include "lmt_args.h"

namespace lmt {

constexpr int kFeatMaxTx = 4096;  // transaction_bytes supported by the phase table

struct FeatInst {  // lmt_instance, as plain ints
    int in_h, in_w, out_h, out_w, pattern, n, m, shape, r;
    int ci, ce, nc, nce, nu, nue, gx, gy, wx, wy;
};
struct FeatDev {  // lmt_device
    int tx, warp, eb, lmem_cap, regfile, max_regs, max_warps, max_wgs, lat, issue;
};

__device__ __forceinline__ bool fpow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

// kernel_model.py:173-219 -- the number of violations (messages are built on
// the host for the rare failing instance).
__device__ int feat_violations(const FeatInst &p) {
    int v = 0;
    v += p.in_h < 1; v += p.in_w < 1; v += p.out_h < 1; v += p.out_w < 1; v += p.n < 1; v += p.m < 1;
    v += p.ci < 0; v += p.ce < 0; v += p.nc < 0; v += p.nce < 0; v += p.nu < 0; v += p.nue < 0;
    v += p.r < 0;
    v += !fpow2(p.gx); v += !fpow2(p.gy); v += !fpow2(p.wx); v += !fpow2(p.wy);
    v += p.wx > p.gx; v += p.wy > p.gy;
    v += (long long)p.wx * p.wy > 1024;
    v += (long long)p.gx * p.gy < 512;
    v += p.gx > 0 && p.out_w % p.gx != 0;
    v += p.gy > 0 && p.out_h % p.gy != 0;
    return v;
}

// access_analysis.py:51-62
__device__ void feat_affine(int pattern, int n, int m, int c[8]) {
    const int t[7][8] = {{0, 0, 1, 0, 0, 0, 0, 1}, {0, 1, 0, 0, 0, 0, 0, 1}, {0, 0, 0, 1, 0, 1, 0, 0},
                         {1, 0, 0, 0, 0, 0, 0, 1}, {0, 0, 0, 1, 1, 0, 0, 0}, {0, n, 1, 0, m, 0, 0, 1},
                         {0, m, 0, 1, n, 0, 1, 0}};
    for (int k = 0; k < 8; ++k) c[k] = t[pattern][k];
}

// access_analysis.py:169-181
__device__ long long feat_pad_col_span(long long span, long long tx_elems) {
    if (span % tx_elems == 0) return span;
    if (span > tx_elems) return (span / tx_elems + 1) * tx_elems;
    long long b = 1;
    while (b < span) b <<= 1;
    return b;
}

// cost_model.py:41-60 (BASELINE; OPTIMIZED is +4 past the clamp)
__device__ long long feat_regs(const FeatInst &p, int K, const FeatDev &d) {
    const long long ctx = (long long)p.nc + p.nce + p.nu + p.nue;
    const long long raw = 10 + K + (p.ci + 3) / 4 + (p.ce + 7) / 8 + 2 * ctx;
    long long b = raw < 10 ? 10 : raw;
    return b < d.max_regs ? b : d.max_regs;
}

// cost_model.py:82-91
__device__ double feat_occupancy(long long regs, long long lmem, long long wg_size, long long warps_per_wg,
                                 const FeatDev &d) {
    long long w = d.max_wgs;
    if (lmem > 0) w = min(w, (long long)d.lmem_cap / lmem);
    w = min(w, (long long)d.regfile / (regs * wg_size));
    w = min(w, (long long)d.max_warps / warps_per_wg);
    const long long a = w * warps_per_wg;
    return (double)(a > 1 ? a : 1);
}

// cost_model.py:94-141; returns total_cycles and fills the TimeEstimate fields
__device__ void feat_time(double compute, double mem_tx, double active, long long wus, const FeatDev &d,
                          double out[4]) {
    const double a = __dmul_rn(mem_tx, (double)d.issue);
    const double mx = compute >= a ? compute : a;  // Python max(): first on ties, same value
    const double per_wu = __dadd_rn(mx, __ddiv_rn(__dmul_rn(mem_tx, (double)d.lat), active));
    out[0] = compute;
    out[1] = mem_tx;
    out[2] = active;
    out[3] = __dmul_rn((double)wus, per_wu);
}

// (access_analysis.py:103-116) weights of the address residues one loop of
// `trips` iterations shifting by `step` bytes produces, added into w[0..tx)
__device__ void feat_phase_weights(long long step, long long trips, int tx, long long *w, int lane) {
    const long long sm = step % tx;
    long long g = tx, a = sm;
    while (a) { const long long t = g % a; g = a; a = t; }
    const long long period = sm ? tx / g : 1;
    const long long lim = trips < period ? trips : period;
    for (long long k = lane; k < lim; k += 32) {
        const long long cnt = (trips - k - 1) / period + 1;
        atomicAdd(reinterpret_cast<unsigned long long *>(&w[(k * step) % tx]), (unsigned long long)cnt);
    }
}

// One warp per instance. Shared memory per warp: wi[tx], wj[tx], ph[tx]
// (int64) plus, for warp_size > 32, the segment scratch.
__global__ void __launch_bounds__(128) k_features(const FeatInst *__restrict__ insts, long long n,
                                                  const FeatDev *__restrict__ devs, int ndev,
                                                  const double *__restrict__ coal_ov,
                                                  const long long *__restrict__ lmem_ov, double *__restrict__ X,
                                                  double *__restrict__ label, double *__restrict__ times,
                                                  int *__restrict__ status, int smem_longs) {
    extern __shared__ long long fsm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    long long *wi = fsm + (size_t)wib * smem_longs;
    const long long nwarps_total = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps_total) {
        const FeatInst p = insts[i];
        const FeatDev d = devs[ndev == 1 ? 0 : i];
        double *x = X + i * 18;
        if (feat_violations(p) || p.pattern < 0 || p.pattern > 6 || p.shape < 0 || p.shape > 2) {
            if (lane < 18) x[lane] = __longlong_as_double(0x7ff8000000000000ll);
            if (lane == 0) { label[i] = __longlong_as_double(0x7ff8000000000000ll); status[i] = 1; }
            continue;
        }
        const int tx = d.tx, eb = d.eb, W = d.warp;
        if (tx > kFeatMaxTx || tx <= 0 || eb <= 0 || W <= 0 || W > 1024) {
            if (lane == 0) status[i] = 5;
            continue;
        }
        int c[8];
        feat_affine(p.pattern, p.n, p.m, c);
        // stencil offsets (kernel_model.py:115-130): extremes are +-r for all shapes
        const int r = p.r;
        const int K = p.shape == 0 ? (2 * r + 1) * (2 * r + 1) : (p.shape == 1 ? 2 * r * r + 2 * r + 1 : 4 * r + 1);
        // footprint (access_analysis.py:184-213)
        const long long hrm = (long long)c[0] * (p.wx - 1) + (long long)c[1] * (p.wy - 1) +
                              (long long)c[2] * (p.n - 1) + (long long)c[3] * (p.m - 1);
        const long long hcm = (long long)c[4] * (p.wx - 1) + (long long)c[5] * (p.wy - 1) +
                              (long long)c[6] * (p.n - 1) + (long long)c[7] * (p.m - 1);
        const long long row_span = hrm + 1 + 2 * r, col_span = hcm + 1 + 2 * r;
        const long long padded = feat_pad_col_span(col_span, tx / eb);
        const long long fp_bytes = row_span * padded * eb;
        // reuse_degree (access_analysis.py:74-88)
        long long share = 1;
        if (c[0] == 0 && c[4] == 0) share *= p.wx;
        if (c[1] == 0 && c[5] == 0) share *= p.wy;
        const long long wg_size = (long long)p.wx * p.wy;
        const long long nwarps = (wg_size + W - 1) / W;
        // ---- coalescing_degree (access_analysis.py:119-155)
        long long *wj = wi + tx, *ph = wj + tx, *seg = ph + tx;
        for (int k = lane; k < 3 * tx; k += 32) wi[k] = 0;
        __syncwarp();
        const long long step_i = ((long long)c[2] * p.in_w + c[6]) * eb;
        const long long step_j = ((long long)c[3] * p.in_w + c[7]) * eb;
        feat_phase_weights(step_i, p.n, tx, wi, lane);
        feat_phase_weights(step_j, p.m, tx, wj, lane);
        __syncwarp();
        // phases[(pa + pb) % tx] += wa * wb
        for (int a = 0; a < tx; ++a) {
            const long long wa = wi[a];
            if (!wa) continue;
            for (int b = lane; b < tx; b += 32)
                if (wj[b]) ph[(a + b) % tx] += wa * wj[b];
            __syncwarp();
        }
        __syncwarp();
        unsigned long long total = 0;
        for (long long w = 0; w < nwarps; ++w) {
            const long long l0 = w * W;
            const long long nl = (l0 + W <= wg_size ? W : wg_size - l0);
            if (W <= 32) {
                const bool act = lane < nl;
                long long base = 0;
                if (act) {
                    const long long l = l0 + lane;
                    const long long wx_ = l % p.wx, wy_ = l / p.wx;
                    base = (((long long)c[0] * wx_ + (long long)c[1] * wy_) * p.in_w + (long long)c[4] * wx_ +
                            (long long)c[5] * wy_) * eb;
                }
                for (int q = 0; q < tx; ++q) {
                    const long long wq = ph[q];
                    if (!wq) continue;
                    const long long s = act ? (base + q) / tx : -1 - lane;
                    const unsigned grp = __match_any_sync(0xffffffffu, s);
                    const bool leader = act && (__ffs(grp) - 1 == lane);
                    total += (unsigned long long)__popc(__ballot_sync(0xffffffffu, leader)) * (unsigned long long)wq;
                }
            } else {  // logical warps wider than the hardware warp: count first occurrences
                for (int q = 0; q < tx; ++q) {
                    const long long wq = ph[q];
                    if (!wq) continue;
                    for (long long k = lane; k < nl; k += 32) {
                        const long long l = l0 + k;
                        const long long wx_ = l % p.wx, wy_ = l / p.wx;
                        seg[k] = ((((long long)c[0] * wx_ + (long long)c[1] * wy_) * p.in_w + (long long)c[4] * wx_ +
                                   (long long)c[5] * wy_) * eb + q) / tx;
                    }
                    __syncwarp();
                    unsigned long long cnt = 0;
                    for (long long k = lane; k < nl; k += 32) {
                        bool first = true;
                        for (long long j = 0; j < k && first; ++j) first = seg[j] != seg[k];
                        cnt += first;
                    }
                    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                    total += cnt * (unsigned long long)wq;
                    __syncwarp();
                }
            }
        }
        const double coal = __ddiv_rn((double)total, (double)(nwarps * p.n * p.m));
        // ---- feature vector (FEATURE_NAMES order, access_analysis.py:216-235)
        const long long regs_b = feat_regs(p, K, d);
        const long long wus = (long long)(p.out_w / p.gx) * (p.out_h / p.gy);
        if (lane == 0) {
            x[0] = (double)share;
            x[1] = (double)fp_bytes;
            x[2] = coal;
            x[3] = (double)K;
            x[4] = (double)-r;
            x[5] = (double)r;
            x[6] = (double)-r;
            x[7] = (double)r;
            x[8] = (double)p.ci;
            x[9] = (double)p.ce;
            x[10] = (double)p.nc;
            x[11] = (double)p.nu;
            x[12] = (double)p.nce;
            x[13] = (double)p.nue;
            x[14] = (double)regs_b;
            x[15] = (double)((long long)p.gx * p.gy);
            x[16] = (double)wg_size;
            x[17] = (double)wus;
            // ---- kernel_time x 2 and the label (cost_model.py:94-158)
            const double cov = coal_ov ? coal_ov[i] : coal;
            const double coal_used = cov == cov ? cov : coal;  // NaN: no override
            const long long nm = (long long)p.n * p.m;
            const long long ctx_inner_tx = p.nc + (long long)p.nu * W;
            const long long ctx_ep_tx = p.nce + (long long)p.nue * W;
            long long compute = (long long)d.issue * (p.ci * nm + p.ce);
            double tb[4], to[4];
            double mem_b = __dmul_rn((double)K, coal_used);
            mem_b = __dadd_rn(mem_b, (double)ctx_inner_tx);
            mem_b = __dmul_rn((double)nm, mem_b);
            mem_b = __dadd_rn(mem_b, (double)ctx_ep_tx);
            const double act_b = feat_occupancy(regs_b, 0, wg_size, nwarps, d);
            feat_time((double)compute, mem_b, act_b, wus, d, tb);
            const long long lmem = (lmem_ov && lmem_ov[i] >= 0) ? lmem_ov[i] : fp_bytes;
            double *tt = times ? times + i * 8 : nullptr;
            if (lmem > d.lmem_cap) {
                label[i] = 0.0;
                status[i] = 2;
                for (int k = 0; k < 4; ++k) to[k] = __longlong_as_double(0x7ff8000000000000ll);
            } else {
                const long long segs_per_row = (padded * eb + tx - 1) / tx;
                const long long ctc = row_span * segs_per_row;  // codegen.py:135-139
                double mem_o = __ddiv_rn((double)ctc, (double)nwarps);
                mem_o = __dadd_rn(mem_o, (double)(nm * ctx_inner_tx));
                mem_o = __dadd_rn(mem_o, (double)ctx_ep_tx);
                compute += (long long)K * nm;
                const double act_o = feat_occupancy(regs_b + 4, lmem, wg_size, nwarps, d);
                feat_time((double)compute, mem_o, act_o, wus, d, to);
                label[i] = __ddiv_rn(tb[3], to[3]);
                status[i] = 0;
            }
            if (tt)
                for (int k = 0; k < 4; ++k) { tt[k] = tb[k]; tt[4 + k] = to[k]; }
        }
        __syncwarp();
    }
}

}  // namespace lmt
