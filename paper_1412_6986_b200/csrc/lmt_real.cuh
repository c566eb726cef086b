// lmt_real.cuh -- K5: the real-world kernel set of the paper's Table 3
// that BASELINE.json configs[1] times on one GPU:
// transpose, matrixMul (NVIDIA SDK), convolution-separable (SDK) and MVT
// (Polybench), each as a baseline (plain global loads) and an optimized
// variant (the reused tile staged in shared memory), as in the paper's study.
// The reference has no implementation of these; the semantics
// below are this repository's and are pinned by the C oracle
// (oracle/lmt_oracle.c ora_real_*), bit for bit.
//
// Numerics: every multiply-add is one fmaf (FFMA) and both variants
// accumulate in the same order (k / j / tap ascending), so baseline,
// optimized and oracle agree bitwise. Convolution taps outside the image
// read 0 in all three (the optimized variant's apron is zero-filled).
// No tensor cores (north_star): these are fp32 CUDA-core kernels.
#pragma once

#include <cuda_runtime.h>

namespace lmt {

constexpr int kConvMaxRadius = 16;

struct RealConv {
    float w[2 * kConvMaxRadius + 1];
};

// ------------------------------------------------------------ transpose
// B[x][y] = A[y][x], n x n. CTA = one T x T tile, blockDim (T / C, wy): each
// thread owns C adjacent columns of the tile (C-wide vector loads and
// stores, C = T / wg_x in {1, 2, 4}) and walks T / wy rows
// (SDK transposeNaive / transposeCoalesced; C > 1 puts more bytes in flight
// per thread: measured on B200, tools/probes/transpose_probe.cu, a 64 x 64
// tile with 2 columns per thread reaches 0.8 of the copy bandwidth where the
// 32 x 32 one-column form stops at 0.55).
template <int C>
struct VecOf;
template <>
struct VecOf<1> { using T = float; };
template <>
struct VecOf<2> { using T = float2; };
template <>
struct VecOf<4> { using T = float4; };
struct float8v {
    float4 lo, hi;
};
template <>
struct VecOf<8> { using T = float8v; };
template <int C>
__device__ __forceinline__ float vget(const typename VecOf<C>::T &v, int q) {
    if constexpr (C == 1) return v;
    else if constexpr (C == 2) return q == 0 ? v.x : v.y;
    else if constexpr (C == 4) return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
    else return vget<4>(q < 4 ? v.lo : v.hi, q & 3);
}
template <int C>
__device__ __forceinline__ void vset(typename VecOf<C>::T &v, int q, float x) {
    if constexpr (C == 1) v = x;
    else if constexpr (C == 2) (q == 0 ? v.x : v.y) = x;
    else if constexpr (C == 4) (q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w) = x;
    else vset<4>(q < 4 ? v.lo : v.hi, q & 3, x);
}
// read-only vector load (two 128-bit loads for 8 floats)
template <int C>
__device__ __forceinline__ typename VecOf<C>::T ldv(const float *p) {
    if constexpr (C == 8) return float8v{__ldg(reinterpret_cast<const float4 *>(p)), __ldg(reinterpret_cast<const float4 *>(p) + 1)};
    else return __ldg(reinterpret_cast<const typename VecOf<C>::T *>(p));
}

template <int C>
__global__ void k_transpose_base(const float *__restrict__ A, float *__restrict__ B, int n, int T) {
    using V = typename VecOf<C>::T;
    const int x = blockIdx.x * T + C * threadIdx.x;
    for (int j = threadIdx.y; j < T; j += blockDim.y) {
        const int y = blockIdx.y * T + j;
        const V v = *reinterpret_cast<const V *>(A + (size_t)y * n + x);  // coalesced read
#pragma unroll
        for (int q = 0; q < C; ++q) B[(size_t)(x + q) * n + y] = vget<C>(v, q);  // strided writes
    }
}

template <int C>
__global__ void k_transpose_opt(const float *__restrict__ A, float *__restrict__ B, int n, int T) {
    using V = typename VecOf<C>::T;
    extern __shared__ float tile[];  // [T][T + 1]: the +1 keeps the column reads (nearly) bank-conflict free
    const int P = T + 1;
    const int cx = C * threadIdx.x;
    for (int j = threadIdx.y; j < T; j += blockDim.y) {
        const V v = *reinterpret_cast<const V *>(A + (size_t)(blockIdx.y * T + j) * n + blockIdx.x * T + cx);
#pragma unroll
        for (int q = 0; q < C; ++q) tile[j * P + cx + q] = vget<C>(v, q);
    }
    __syncthreads();
    for (int j = threadIdx.y; j < T; j += blockDim.y) {
        V v;
#pragma unroll
        for (int q = 0; q < C; ++q) vset<C>(v, q, tile[(cx + q) * P + j]);
        *reinterpret_cast<V *>(B + (size_t)(blockIdx.x * T + j) * n + blockIdx.y * T + cx) = v;  // coalesced write
    }
}

// ------------------------------------------------------------ matrixMul
// C = A x B, n x n. CTA = T x T outputs, blockDim (T / CC, T / W): thread
// (tx, ty) computes rows ty + r * (T / W), r < W, and columns CC * tx + q,
// q < CC (CC = 1: the SDK form, one column per thread; the tiling factors W
// and CC are the instance's). acc = fmaf(A[i][k], B[k][j], acc), k ascending.
// Both variants take k four at a time: one 128-bit read of A[row][k .. k+3]
// per row (the same address across the lanes of a row: a broadcast) and one
// CC-wide read of B[k][cols] per k feed 4 * W * CC FMAs, so a thread's
// register tile costs W + 4 loads per 4 k instead of 2 per FMA.
template <int CC>
__global__ void __launch_bounds__(1024) k_matmul_base(const float *__restrict__ A, const float *__restrict__ B,
                                                      float *__restrict__ C,
                              int n, int T, int W) {
    using V = typename VecOf<CC>::T;
    const int h = T / W;
    const int col = blockIdx.x * T + CC * threadIdx.x;
    for (int r = 0; r < W; ++r) {
        const int row = blockIdx.y * T + threadIdx.y + r * h;
        const float *ar = A + (size_t)row * n;
        float acc[CC];
#pragma unroll
        for (int q = 0; q < CC; ++q) acc[q] = 0.0f;
        if ((n & 3) == 0) {
            for (int k = 0; k < n; k += 4) {
                const float4 a = __ldg(reinterpret_cast<const float4 *>(ar + k));
                const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const V bv = ldv<CC>(B + (size_t)(k + kk) * n + col);
#pragma unroll
                    for (int q = 0; q < CC; ++q) acc[q] = __fmaf_rn(av[kk], vget<CC>(bv, q), acc[q]);
                }
            }
        } else {
            for (int k = 0; k < n; ++k)
#pragma unroll
                for (int q = 0; q < CC; ++q) acc[q] = __fmaf_rn(ar[k], B[(size_t)k * n + col + q], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < CC; ++q) C[(size_t)row * n + col + q] = acc[q];
    }
}

// optimized: A and B tiles staged in shared memory (rows padded to T + 4
// floats: 16-byte aligned for the 128-bit reads), the next tiles' elements
// loaded into registers while the current tiles are consumed.
// launch bounds: the most threads a tile of <= 64 x 64 needs at this W x CC
template <int W, int CC>
__global__ void __launch_bounds__(4096 / (W * CC) < 1024 ? 4096 / (W * CC) : 1024)
    k_matmul_opt(const float *__restrict__ A, const float *__restrict__ B, float *__restrict__ C, int n, int T) {
    using V = typename VecOf<CC>::T;
    extern __shared__ __align__(16) float sm[];  // As[T][T + 4], Bs[T][T + 4]
    const int P = T + 4, h = T / W;
    float *As = sm, *Bs = sm + T * P;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int nthr = blockDim.x * blockDim.y, tid = ty * blockDim.x + tx;
    const int col0 = blockIdx.x * T, row0 = blockIdx.y * T;
    // tile copy: each thread moves (T * T) / nthr = W * CC elements of A and
    // of B per k-tile, four at a time (T % 4 == 0): element e = 4 * (tid + i * nthr)
    constexpr int NF = (W * CC + 3) / 4;  // float4 per thread per tile
    const int per4 = (T * T / 4 + nthr - 1) / nthr;
    float acc[W][CC];
#pragma unroll
    for (int r = 0; r < W; ++r)
#pragma unroll
        for (int q = 0; q < CC; ++q) acc[r][q] = 0.0f;
    float4 ra[NF], rb[NF];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < NF; ++i)
            if (i < per4) {
                const int e = 4 * (tid + i * nthr);
                if (e < T * T) {
                    const int rr = e / T, cc = e - rr * T;
                    ra[i] = __ldg(reinterpret_cast<const float4 *>(A + (size_t)(row0 + rr) * n + k0 + cc));
                    rb[i] = __ldg(reinterpret_cast<const float4 *>(B + (size_t)(k0 + rr) * n + col0 + cc));
                }
            }
    };
    fetch(0);
    for (int k0 = 0; k0 < n; k0 += T) {
#pragma unroll
        for (int i = 0; i < NF; ++i)
            if (i < per4) {
                const int e = 4 * (tid + i * nthr);
                if (e < T * T) {
                    const int rr = e / T, cc = e - rr * T;
                    *reinterpret_cast<float4 *>(As + rr * P + cc) = ra[i];
                    *reinterpret_cast<float4 *>(Bs + rr * P + cc) = rb[i];
                }
            }
        __syncthreads();
        if (k0 + T < n) fetch(k0 + T);
        for (int kk = 0; kk < T; kk += 4) {
            V b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) b[u] = *reinterpret_cast<const V *>(Bs + (kk + u) * P + CC * tx);
#pragma unroll
            for (int r = 0; r < W; ++r) {
                const float4 a = *reinterpret_cast<const float4 *>(As + (ty + r * h) * P + kk);
                const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int q = 0; q < CC; ++q) acc[r][q] = __fmaf_rn(av[u], vget<CC>(b[u], q), acc[r][q]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < W; ++r)
#pragma unroll
        for (int q = 0; q < CC; ++q) C[(size_t)(row0 + ty + r * h) * n + col0 + CC * tx + q] = acc[r][q];
}

// optimized, tile shape compile-time (T, W, CC of the instance set): the tile
// copy's index math folds to shifts, the k loop over a tile unrolls fully,
// and two shared-memory buffers take one barrier per k-tile (the next
// tiles go from registers into the other buffer while this one is read).
// Same per-output order as k_matmul_opt (k ascending, one fmaf each).
template <int T, int W, int CC>
__global__ void __launch_bounds__((T / CC) * (T / W)) k_matmul_opt_t(const float *__restrict__ A,
                                                                    const float *__restrict__ B,
                                                                    float *__restrict__ C, int n) {
    using V = typename VecOf<CC>::T;
    constexpr int TX = T / CC, TY = T / W, NT = TX * TY, P = T + 4;
    constexpr int E4 = T * T / 4;             // float4 per tile
    constexpr int NF = (E4 + NT - 1) / NT;    // float4 per thread per tile
    extern __shared__ __align__(16) float sm[];  // [2][As[T][P], Bs[T][P]]
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int col0 = blockIdx.x * T, row0 = blockIdx.y * T;
    float acc[W][CC];
#pragma unroll
    for (int r = 0; r < W; ++r)
#pragma unroll
        for (int q = 0; q < CC; ++q) acc[r][q] = 0.0f;
    float4 ra[NF], rb[NF];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int e = tid + i * NT;
            if (E4 % NT == 0 || e < E4) {
                const int rr = e / (T / 4), cc = (e % (T / 4)) * 4;
                ra[i] = __ldg(reinterpret_cast<const float4 *>(A + (size_t)(row0 + rr) * n + k0 + cc));
                rb[i] = __ldg(reinterpret_cast<const float4 *>(B + (size_t)(k0 + rr) * n + col0 + cc));
            }
        }
    };
    auto store = [&](int b) {
        float *As = sm + b * 2 * T * P, *Bs = As + T * P;
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int e = tid + i * NT;
            if (E4 % NT == 0 || e < E4) {
                const int rr = e / (T / 4), cc = (e % (T / 4)) * 4;
                *reinterpret_cast<float4 *>(As + rr * P + cc) = ra[i];
                *reinterpret_cast<float4 *>(Bs + rr * P + cc) = rb[i];
            }
        }
    };
    const int nt = n / T;
    fetch(0);
    store(0);
    __syncthreads();
    for (int t = 0; t < nt; ++t) {
        if (t + 1 < nt) fetch((t + 1) * T);
        const float *As = sm + (t & 1) * 2 * T * P, *Bs = As + T * P;
        // the fragments of k-step kk + 4 are read from shared memory while
        // the FMAs of kk run (ncu: short_scoreboard was half the stalls)
        V bq[2][4];
        float4 aq[2][W];
        auto frag = [&](int b, int kk) {
#pragma unroll
            for (int u = 0; u < 4; ++u) bq[b][u] = *reinterpret_cast<const V *>(Bs + (kk + u) * P + CC * tx);
#pragma unroll
            for (int r = 0; r < W; ++r) aq[b][r] = *reinterpret_cast<const float4 *>(As + (ty + r * TY) * P + kk);
        };
        frag(0, 0);
#pragma unroll
        for (int kk = 0; kk < T; kk += 4) {
            const int cb = (kk >> 2) & 1;
            if (kk + 4 < T) frag(cb ^ 1, kk + 4);
#pragma unroll
            for (int r = 0; r < W; ++r) {
                const float av[4] = {aq[cb][r].x, aq[cb][r].y, aq[cb][r].z, aq[cb][r].w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int q = 0; q < CC; ++q) acc[r][q] = __fmaf_rn(av[u], vget<CC>(bq[cb][u], q), acc[r][q]);
            }
        }
        if (t + 1 < nt) store((t + 1) & 1);
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < W; ++r) {
        V v;
#pragma unroll
        for (int q = 0; q < CC; ++q) vset<CC>(v, q, acc[r][q]);
        *reinterpret_cast<V *>(C + (size_t)(row0 + ty + r * TY) * n + col0 + CC * tx) = v;
    }
}

// optimized, 64 x 64 tile with an 8 x 8 register tile per thread (blockDim
// 8 x 8, the instance (T 64, wg 8 x 8)): thread (tx, ty) owns rows
// {4ty .. 4ty+3, 32+4ty .. 32+4ty+3} and columns {4tx .. 4tx+3, 32+4tx ..
// 32+4tx+3}, so a k-step's fragments are four 128-bit reads (two of A, two
// of B) for 64 FMAs -- half the shared-memory reads per FMA of the 4 x 4
// tile, whose LSU pipe was the limit. A is staged k-major (As[k][m]: one
// thread's rows are contiguous at each k), transposed through registers on
// its way in; B goes global -> shared by cp.async. Per output the order is
// k ascending, one fmaf each, as in every matrixMul variant.
__device__ __forceinline__ void rk_cp16(float *dst, const float *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__global__ void __launch_bounds__(64) k_matmul_opt88(const float *__restrict__ A, const float *__restrict__ B,
                                                     float *__restrict__ C, int n) {
    constexpr int T = 64, P = T + 4, NF = T * T / 4 / 64;  // 16 float4 per thread per tile
    extern __shared__ __align__(16) float sm[];           // [2][As[T][P] (k-major), Bs[T][P]]
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 8 + tx;
    const int col0 = blockIdx.x * T, row0 = blockIdx.y * T;
    float acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[r][q] = 0.0f;
    float4 ra[NF];
    // A: lane-consecutive rows (the transposed shared stores hit distinct banks)
    auto fetch_a = [&](int k0) {
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int e = tid + i * 64, rr = e & 63, cc = (e >> 6) * 4;
            ra[i] = __ldg(reinterpret_cast<const float4 *>(A + (size_t)(row0 + rr) * n + k0 + cc));
        }
    };
    auto store_a = [&](int b) {
        float *As = sm + b * 2 * T * P;
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int e = tid + i * 64, rr = e & 63, cc = (e >> 6) * 4;
            As[(cc + 0) * P + rr] = ra[i].x;
            As[(cc + 1) * P + rr] = ra[i].y;
            As[(cc + 2) * P + rr] = ra[i].z;
            As[(cc + 3) * P + rr] = ra[i].w;
        }
    };
    auto copy_b = [&](int b, int k0) {
        float *Bs = sm + b * 2 * T * P + T * P;
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int e = tid + i * 64, rr = e >> 4, cc = (e & 15) * 4;
            rk_cp16(Bs + rr * P + cc, B + (size_t)(k0 + rr) * n + col0 + cc);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int nt = n / T;
    fetch_a(0);
    copy_b(0, 0);
    store_a(0);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int t = 0; t < nt; ++t) {
        if (t + 1 < nt) {
            fetch_a((t + 1) * T);
            copy_b((t + 1) & 1, (t + 1) * T);
        }
        const float *As = sm + (t & 1) * 2 * T * P, *Bs = As + T * P;
        float4 fa[2][2], fb[2][2];
        auto frag = [&](int b, int k) {
            fa[b][0] = *reinterpret_cast<const float4 *>(As + k * P + 4 * ty);
            fa[b][1] = *reinterpret_cast<const float4 *>(As + k * P + 32 + 4 * ty);
            fb[b][0] = *reinterpret_cast<const float4 *>(Bs + k * P + 4 * tx);
            fb[b][1] = *reinterpret_cast<const float4 *>(Bs + k * P + 32 + 4 * tx);
        };
        frag(0, 0);
#pragma unroll 8
        for (int k = 0; k < T; ++k) {
            const int cb = k & 1;
            if (k + 1 < T) frag(cb ^ 1, k + 1);
            const float av[8] = {fa[cb][0].x, fa[cb][0].y, fa[cb][0].z, fa[cb][0].w,
                                 fa[cb][1].x, fa[cb][1].y, fa[cb][1].z, fa[cb][1].w};
            const float bv[8] = {fb[cb][0].x, fb[cb][0].y, fb[cb][0].z, fb[cb][0].w,
                                 fb[cb][1].x, fb[cb][1].y, fb[cb][1].z, fb[cb][1].w};
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[r][q] = __fmaf_rn(av[r], bv[q], acc[r][q]);
        }
        if (t + 1 < nt) {
            store_a((t + 1) & 1);
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float *crow = C + (size_t)(row0 + (r < 4 ? 4 * ty + r : 32 + 4 * ty + r - 4)) * n + col0;
        *reinterpret_cast<float4 *>(crow + 4 * tx) = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
        *reinterpret_cast<float4 *>(crow + 32 + 4 * tx) = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
    }
}

// ------------------------------------------------------------ convolution-separable
// rows: out[y][x] = sum_{k=-R..R} in[y][x+k] * w[R-k]; cols: out[y][x] = sum_k in[y+k][x] * w[R-k];
// taps outside the image read 0. blockDim (wx, wy); each thread computes W
// outputs, blockDim apart along the pass direction (the tiling factor: W
// independent chains). RR is the radius when it is a compile-time constant
// (the instance set's 1, 2, 4, 8: the taps unroll, every load of a thread is
// issued before its FMA chains), 0 for the generic run-time radius.
template <int RR>
__global__ void k_conv_rows_base(const float *__restrict__ in, float *__restrict__ out, int n, int Rr, int W,
                                 RealConv c) {
    const int R = RR ? RR : Rr;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int x0 = blockIdx.x * blockDim.x * W + threadIdx.x;
    const float *row = in + (size_t)y * n;
    const int xb = blockIdx.x * blockDim.x * W;
    if (xb >= R && xb + (int)blockDim.x * W + R <= n) {  // CTA-uniform: every tap inside the image
        for (int q = 0; q < W; ++q) {
            const int x = x0 + q * blockDim.x;
            float acc = 0.0f;
#pragma unroll
            for (int k = -R; k <= R; ++k) acc = __fmaf_rn(__ldg(row + x + k), c.w[R - k], acc);
            out[(size_t)y * n + x] = acc;
        }
        return;
    }
    for (int q = 0; q < W; ++q) {
        const int x = x0 + q * blockDim.x;
        float acc = 0.0f;
#pragma unroll
        for (int k = -R; k <= R; ++k) {
            const int xx = x + k;
            const float v = (xx >= 0 && xx < n) ? __ldg(row + xx) : 0.0f;
            acc = __fmaf_rn(v, c.w[R - k], acc);
        }
        out[(size_t)y * n + x] = acc;
    }
}

template <int RR>
__global__ void k_conv_cols_base(const float *__restrict__ in, float *__restrict__ out, int n, int Rr, int W,
                                 RealConv c) {
    const int R = RR ? RR : Rr;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y0 = blockIdx.y * blockDim.y * W + threadIdx.y;
    const int yb = blockIdx.y * blockDim.y * W;
    if (yb >= R && yb + (int)blockDim.y * W + R <= n) {  // CTA-uniform: every tap inside the image
        for (int q = 0; q < W; ++q) {
            const int y = y0 + q * blockDim.y;
            const float *col = in + (size_t)y * n + x;
            float acc = 0.0f;
#pragma unroll
            for (int k = -R; k <= R; ++k) acc = __fmaf_rn(__ldg(col + (ptrdiff_t)k * n), c.w[R - k], acc);
            out[(size_t)y * n + x] = acc;
        }
        return;
    }
    for (int q = 0; q < W; ++q) {
        const int y = y0 + q * blockDim.y;
        float acc = 0.0f;
#pragma unroll
        for (int k = -R; k <= R; ++k) {
            const int yy = y + k;
            const float v = (yy >= 0 && yy < n) ? __ldg(in + (size_t)yy * n + x) : 0.0f;
            acc = __fmaf_rn(v, c.w[R - k], acc);
        }
        out[(size_t)y * n + x] = acc;
    }
}

// optimized: the CTA's rows (its W * wx columns plus the apron) staged once in
// shared memory; the interior sits at a 16-byte aligned offset (R rounded
// up to 4: R4) so it is copied with 128-bit loads and stores when aligned
template <int RR>
__global__ void k_conv_rows_opt(const float *__restrict__ in, float *__restrict__ out, int n, int Rr, int W,
                                RealConv c) {
    const int R = RR ? RR : Rr;
    const int R4 = (R + 3) & ~3;
    extern __shared__ __align__(16) float s[];  // [wy][R4 + W * wx + R4]: row data at [R4 - R, R4 + span + R)
    const int wx = blockDim.x, wy = blockDim.y, span = W * wx, P = span + 2 * R4;
    const int xb = blockIdx.x * span, y = blockIdx.y * wy + threadIdx.y;
    const float *row = in + (size_t)y * n;
    float *srow = s + threadIdx.y * P;
    if ((span & 3) == 0 && (n & 3) == 0) {
        for (int t = threadIdx.x; t < span / 4; t += wx)
            reinterpret_cast<float4 *>(srow + R4)[t] = __ldg(reinterpret_cast<const float4 *>(row + xb) + t);
        for (int t = threadIdx.x; t < 2 * R; t += wx) {  // the two aprons
            const int xx = t < R ? xb - R + t : xb + span + (t - R);
            srow[t < R ? R4 - R + t : R4 + span + (t - R)] = (xx >= 0 && xx < n) ? row[xx] : 0.0f;
        }
    } else {
        for (int t = threadIdx.x; t < span + 2 * R; t += wx) {
            const int xx = xb - R + t;
            srow[R4 - R + t] = (xx >= 0 && xx < n) ? row[xx] : 0.0f;
        }
    }
    // a row's staging and its outputs belong to the threads of that row: with
    // 32-wide workgroups that is one warp, which need not wait for the others
    if (wx == 32) __syncwarp();
    else __syncthreads();
    for (int q = 0; q < W; ++q) {
        const int lx = threadIdx.x + q * wx;
        float acc = 0.0f;
#pragma unroll
        for (int k = -R; k <= R; ++k) acc = __fmaf_rn(srow[lx + R4 + k], c.w[R - k], acc);
        out[(size_t)y * n + xb + lx] = acc;
    }
}

template <int RR>
__global__ void k_conv_cols_opt(const float *__restrict__ in, float *__restrict__ out, int n, int Rr, int W,
                                RealConv c) {
    const int R = RR ? RR : Rr;
    extern __shared__ float s[];  // [W * wy + 2R][wx]
    const int wx = blockDim.x, wy = blockDim.y, H = W * wy + 2 * R;
    const int x = blockIdx.x * wx + threadIdx.x, y0 = blockIdx.y * wy * W - R;
    // all of a thread's staging loads are issued before its shared-memory
    // stores (eight per pass): one memory latency per pass, not per row
    for (int t0 = threadIdx.y; t0 < H; t0 += 8 * wy) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int yy = y0 + t0 + i * wy;
            v[i] = (t0 + i * wy < H && yy >= 0 && yy < n) ? __ldg(in + (size_t)yy * n + x) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (t0 + i * wy < H) s[(t0 + i * wy) * wx + threadIdx.x] = v[i];
    }
    __syncthreads();
    for (int q = 0; q < W; ++q) {
        const int ly = threadIdx.y + q * wy;
        float acc = 0.0f;
#pragma unroll
        for (int k = -R; k <= R; ++k) acc = __fmaf_rn(s[(ly + R + k) * wx + threadIdx.x], c.w[R - k], acc);
        out[(size_t)(blockIdx.y * wy * W + ly) * n + x] = acc;
    }
}

// ------------------------------------------------------------ MVT (Polybench)
// x1[i] = x1_0[i] + sum_j A[i][j] * y1[j];  x2[i] = x2_0[i] + sum_j A[j][i] * y2[j]  (j ascending)
//
// n x n A is 64 MB at n = 4096 while only n threads carry a chain each, so
// what bounds both kernels is the bytes in flight per thread, not the
// arithmetic: the baselines read 128-bit (row walk) or coalesced (column
// walk) with the next loads issued before the current chain step; the
// optimized variants stream A through a TMA ring in shared memory.

// baseline kernel 1: thread i walks row i, four j per 128-bit load, eight loads in flight
__global__ void __launch_bounds__(512) k_mvt1_base(const float *__restrict__ A, const float *__restrict__ y1,
                                                   const float *__restrict__ x1_0, float *__restrict__ x1, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = x1_0[i];
    const float *row = A + (size_t)i * n;
    if ((n & 3) == 0) {
        const float4 *a4 = reinterpret_cast<const float4 *>(row);
        const float4 *y4 = reinterpret_cast<const float4 *>(y1);
        const int n4 = n >> 2;
        int q = 0;
        for (; q + 8 <= n4; q += 8) {
            float4 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldg(a4 + q + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float4 y = __ldg(y4 + q + u);
                acc = __fmaf_rn(a[u].x, y.x, acc);
                acc = __fmaf_rn(a[u].y, y.y, acc);
                acc = __fmaf_rn(a[u].z, y.z, acc);
                acc = __fmaf_rn(a[u].w, y.w, acc);
            }
        }
        for (int j = q * 4; j < n; ++j) acc = __fmaf_rn(row[j], y1[j], acc);
    } else {
        for (int j = 0; j < n; ++j) acc = __fmaf_rn(row[j], y1[j], acc);
    }
    x1[i] = acc;
}

// baseline kernel 2: thread i walks column i (coalesced across the warp), 16 rows in flight
__global__ void __launch_bounds__(512) k_mvt2_base(const float *__restrict__ A, const float *__restrict__ y2,
                                                   const float *__restrict__ x2_0, float *__restrict__ x2, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = x2_0[i];
    int j = 0;
    for (; j + 16 <= n; j += 16) {
        float a[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = __ldg(A + (size_t)(j + u) * n + i);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = __fmaf_rn(a[u], __ldg(y2 + j + u), acc);
    }
    for (; j < n; ++j) acc = __fmaf_rn(A[(size_t)j * n + i], y2[j], acc);
    x2[i] = acc;
}

// ---- TMA ring helpers (the optimized MVT kernels)
struct alignas(64) RealTmap {
    unsigned long long opaque[16];
};
__device__ __forceinline__ unsigned rk_smem(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void rk_bar_init(unsigned long long *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rk_smem(b)), "r"(c));
}
__device__ __forceinline__ void rk_expect(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rk_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void rk_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rk_smem(b)) : "memory");
}
__device__ __forceinline__ void rk_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "RK_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra RK_DONE;\n\t"
        "bra RK_WAIT;\n"
        "RK_DONE:\n\t}" ::"r"(rk_smem(b)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void rk_tma2d(void *dst, const RealTmap *m, unsigned long long *bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            rk_smem(dst)),
        "l"(reinterpret_cast<unsigned long long>(m)), "r"(rk_smem(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ float4 rk_lds4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float rk_lds(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
constexpr int kMvtMaxStages = 16;

// Copy a vector of n floats (n % 4 == 0, both 16-byte aligned) to shared
// memory: 128-bit loads, eight in flight per thread (a serial load -> store
// loop would pay one global latency per element of the thread).
__device__ __forceinline__ void rk_stage_vec(float *dst, const float *src, int n, int tid, int nthreads) {
    const float4 *s4 = reinterpret_cast<const float4 *>(src);
    const unsigned d = rk_smem(dst);
    const int n4 = n >> 2;
    for (int q0 = tid; q0 < n4; q0 += 8 * nthreads) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (q0 + u * nthreads < n4) v[u] = __ldg(s4 + q0 + u * nthreads);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (q0 + u * nthreads < n4)
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(d + (unsigned)((q0 + u * nthreads) * 16)),
                             "f"(v[u].x), "f"(v[u].y), "f"(v[u].z), "f"(v[u].w)
                             : "memory");
    }
}

// Kernel 1 (row dots): a ring of S stages, each 256 columns of the CTA's wg
// rows as two 2D TMA boxes of 128 + 4 columns: the 4 extra columns (3 %
// more bytes; zero-filled past the matrix) make the staged row pitch 528
// bytes = 33 x 16, so a quarter-warp's 128-bit reads of 8 rows hit 8
// distinct bank groups without swizzling, and each box row is a 528-byte
// request (2D boxes with the 128B swizzle are limited to 128-byte rows;
// one cp.async.bulk per row costs one issue per row in the only warp).
// Kernel 2 (column dots): stages of T rows x wg columns by 2D TMA boxes,
// read one float per lane (consecutive). Thread 0 issues the loads and
// refills a stage once every warp released it; each thread's registers hold
// the next sub-step while the current FMAs run: one warp per SM carries the
// serial chains, so latency is the limit.
constexpr int kMvtBoxCols = 128;  // useful columns per box (+4 padding columns)
constexpr int kMvtStageCols = 2 * kMvtBoxCols;
// (T = 32 needs ~150 registers for its two buffers of row values and y:
// launch bounds of 256 threads; wider workgroups use the T = 16 kernel, whose
// results are the same -- T only sets the staging granularity, the chain is
// j ascending either way)
template <int T>
__global__ void __launch_bounds__(T == 32 ? 256 : 512) k_mvt1_tma(const __grid_constant__ RealTmap tm,
                                                                 const float *__restrict__ y1,
                                                                 const float *__restrict__ x1_0,
                                                                 float *__restrict__ x1, int n, int S, int bwl,
                                                                 int NB) {
    const int bwu = 1 << bwl;
    // NB boxes of bwu useful columns per stage (2 x 128; fewer / narrower for wide workgroups)
    const int BW = bwu + 4;        // floats per staged row of a box: pitch = 16 x odd bytes
    const int SC = NB * bwu;       // columns per stage
    const int KB = SC / T;         // sub-steps per stage
    extern __shared__ unsigned char rk_raw[];
    __shared__ __align__(8) unsigned long long full[kMvtMaxStages], empty[kMvtMaxStages];
    float *st = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(rk_raw) + 127) & ~uintptr_t(127));
    const int wg = blockDim.x, tid = threadIdx.x, lane = tid & 31;
    const int i0 = blockIdx.x * wg, steps = n / SC;
    const int boxes = (wg + 255) / 256, brows = wg < 256 ? wg : 256;
    const int bf = wg * BW;       // floats per box (all rows)
    const int sf = NB * bf;       // floats per stage
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            rk_bar_init(&full[s], 1);
            rk_bar_init(&empty[s], wg / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int slot, int step) {
        rk_expect(&full[slot], (unsigned)(sf * 4));
        for (int nb = 0; nb < NB; ++nb)
            for (int b = 0; b < boxes; ++b)
                rk_tma2d(st + slot * sf + nb * bf + b * 256 * BW, &tm, &full[slot], step * SC + nb * bwu,
                         i0 + b * brows);
    };
    if (tid == 0)
        for (int s = 0; s < S && s < steps; ++s) issue(s, s);
    float *ys = st + (size_t)S * sf;  // y, whole, after the ring: LDS broadcasts
    rk_stage_vec(ys, y1, n, tid, wg);
    __syncthreads();
    const unsigned ybase = rk_smem(ys);
    float acc = x1_0[i0 + tid];
    const unsigned base = rk_smem(st) + (unsigned)(tid * BW * 4);
    // two register buffers, ping-pong: sub-step k = (stage k / KB, T-column
    // slice kb = k % KB) computes from one while the other receives k + 1
    float4 a0[T / 4], a1[T / 4], y0[T / 4], y1v[T / 4];
    const int total = steps * KB;
    int slot = 0, kb = 0, step = 0;
    unsigned phase = 0;
#define MVT1_NEXT(ns, nph, nkb, last) \
    const bool last = kb == KB - 1;   \
    int ns = slot;                    \
    unsigned nph = phase;             \
    if (last && ++ns == S) {          \
        ns = 0;                       \
        nph ^= 1;                     \
    }                                 \
    const int nkb = last ? 0 : kb + 1;
#define MVT1_LOAD(A_, Y_, sl, bk, kk)                                                                  \
    {                                                                                                  \
        const int col = (bk) * T;                                                                      \
        const unsigned bx = base + (unsigned)(((sl) * sf + (col >> bwl) * bf + (col & (bwu - 1))) * 4); \
        _Pragma("unroll") for (int c = 0; c < T / 4; ++c) {                                           \
            A_[c] = rk_lds4(bx + (unsigned)(c << 4));                                                  \
            Y_[c] = rk_lds4(ybase + (unsigned)(((kk) * T + 4 * c) * 4));                               \
        }                                                                                              \
    }
#define MVT1_FMA(A_, Y_)                                    \
    _Pragma("unroll") for (int c = 0; c < T / 4; ++c) {     \
        acc = __fmaf_rn(A_[c].x, Y_[c].x, acc);             \
        acc = __fmaf_rn(A_[c].y, Y_[c].y, acc);             \
        acc = __fmaf_rn(A_[c].z, Y_[c].z, acc);             \
        acc = __fmaf_rn(A_[c].w, Y_[c].w, acc);             \
    }
#define MVT1_RELEASE(last)                      \
    if (last) {                                 \
        __syncwarp();                           \
        if (lane == 0) rk_arrive(&empty[slot]); \
        if (tid == 0 && step + S < steps) {     \
            rk_wait(&empty[slot], phase);       \
            issue(slot, step + S);              \
        }                                       \
        ++step;                                 \
    }
    rk_wait(&full[0], 0);
    MVT1_LOAD(a0, y0, 0, 0, 0)
    for (int k = 0; k < total; k += 2) {
        {  // sub-step k from buffer 0, k + 1 into buffer 1
            MVT1_NEXT(ns, nph, nkb, last)
            if (k + 1 < total) {
                if (last) rk_wait(&full[ns], nph);
                MVT1_LOAD(a1, y1v, ns, nkb, k + 1)
            }
            MVT1_FMA(a0, y0)
            MVT1_RELEASE(last)
            slot = ns;
            phase = nph;
            kb = nkb;
        }
        if (k + 1 < total) {  // sub-step k + 1 from buffer 1, k + 2 into buffer 0
            MVT1_NEXT(ns, nph, nkb, last)
            if (k + 2 < total) {
                if (last) rk_wait(&full[ns], nph);
                MVT1_LOAD(a0, y0, ns, nkb, k + 2)
            }
            MVT1_FMA(a1, y1v)
            MVT1_RELEASE(last)
            slot = ns;
            phase = nph;
            kb = nkb;
        }
    }
#undef MVT1_NEXT
#undef MVT1_LOAD
#undef MVT1_FMA
#undef MVT1_RELEASE
    x1[i0 + tid] = acc;
}

template <int T>
__global__ void __launch_bounds__(T == 32 ? 256 : 512) k_mvt2_tma(const __grid_constant__ RealTmap tm, const float *__restrict__ y2,
                                                  const float *__restrict__ x2_0, float *__restrict__ x2, int n,
                                                  int S) {
    extern __shared__ unsigned char rk_raw[];
    __shared__ __align__(8) unsigned long long full[kMvtMaxStages], empty[kMvtMaxStages];
    float *st = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(rk_raw) + 127) & ~uintptr_t(127));
    const int wg = blockDim.x, tid = threadIdx.x, lane = tid & 31;
    const int i0 = blockIdx.x * wg, steps = n / T, sf = wg * T;
    const int boxes = (wg + 255) / 256, bcols = wg < 256 ? wg : 256;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            rk_bar_init(&full[s], 1);
            rk_bar_init(&empty[s], wg / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int slot, int step) {
        rk_expect(&full[slot], (unsigned)(sf * 4));
        for (int b = 0; b < boxes; ++b)
            rk_tma2d(st + slot * sf + b * T * bcols, &tm, &full[slot], i0 + b * bcols, step * T);
    };
    if (tid == 0)
        for (int s = 0; s < S && s < steps; ++s) issue(s, s);
    const int b = tid / bcols, c = tid - b * bcols;
    float acc = x2_0[i0 + tid];
    const unsigned base = rk_smem(st) + (unsigned)((b * T * bcols + c) * 4);
    float *ysm = st + (size_t)S * sf;  // y, whole, after the ring (LDS broadcasts)
    rk_stage_vec(ysm, y2, n, tid, wg);
    __syncthreads();
    const unsigned ybase = rk_smem(ysm);
    float a0[T], a1[T];
    float4 y0[T / 4], y1v[T / 4];
    int slot = 0;
    unsigned phase = 0;
#define MVT2_LOAD(A_, Y_, sl, stp)                                                                            \
    {                                                                                                         \
        _Pragma("unroll") for (int jj = 0; jj < T; ++jj) A_[jj] = rk_lds(base + (unsigned)(((sl) * sf + jj * bcols) * 4)); \
        _Pragma("unroll") for (int q = 0; q < T / 4; ++q) Y_[q] = rk_lds4(ybase + (unsigned)(((stp) * T + 4 * q) * 4)); \
    }
#define MVT2_FMA(A_, Y_)                                      \
    _Pragma("unroll") for (int q = 0; q < T / 4; ++q) {       \
        acc = __fmaf_rn(A_[4 * q + 0], Y_[q].x, acc);         \
        acc = __fmaf_rn(A_[4 * q + 1], Y_[q].y, acc);         \
        acc = __fmaf_rn(A_[4 * q + 2], Y_[q].z, acc);         \
        acc = __fmaf_rn(A_[4 * q + 3], Y_[q].w, acc);         \
    }
#define MVT2_STEP(CUR, CY, NXT, NY, stp)                 \
    {                                                    \
        int ns = slot + 1;                               \
        unsigned nph = phase;                            \
        if (ns == S) {                                   \
            ns = 0;                                      \
            nph ^= 1;                                    \
        }                                                \
        if ((stp) + 1 < steps) {                         \
            rk_wait(&full[ns], nph);                     \
            MVT2_LOAD(NXT, NY, ns, (stp) + 1)            \
        }                                                \
        MVT2_FMA(CUR, CY)                                \
        __syncwarp();                                    \
        if (lane == 0) rk_arrive(&empty[slot]);          \
        if (tid == 0 && (stp) + S < steps) {             \
            rk_wait(&empty[slot], phase);                \
            issue(slot, (stp) + S);                      \
        }                                                \
        slot = ns;                                       \
        phase = nph;                                     \
    }
    rk_wait(&full[0], 0);
    MVT2_LOAD(a0, y0, 0, 0)
    for (int step = 0; step < steps; step += 2) {
        MVT2_STEP(a0, y0, a1, y1v, step)
        if (step + 1 < steps) MVT2_STEP(a1, y1v, a0, y0, step + 1)
    }
#undef MVT2_LOAD
#undef MVT2_FMA
#undef MVT2_STEP
    x2[i0 + tid] = acc;
}

// ---- MVT ring kernels with compile-time stages (workgroups of <= 128 rows /
// columns; the kernels above stay for the wider ones). ncu on the kernels
// above: the only warp of an SM spent ~18 cycles per element, 15.6k
// instructions for 4,096 FMAs -- per-sub-step bookkeeping (which slot,
// which phase, is this the last sub-step) issued between the chain's FFMAs.
// Here a stage is a compile-time number of T-wide sub-steps, unrolled: the
// next sub-step's shared-memory loads are issued between the current FFMAs
// and the ring bookkeeping runs once per stage.
// one 1D bulk copy global -> shared (bytes % 16 == 0, both 16-byte aligned)
__device__ __forceinline__ void rk_bulk(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     rk_smem(dst)),
                 "l"(reinterpret_cast<unsigned long long>(src)), "r"(bytes), "r"(rk_smem(bar))
                 : "memory");
}
constexpr int kMvtRingCols = 128;  // kernel 1: columns per stage (one TMA box of 128 + 4 columns)
constexpr int kMvtRingRows = 128;  // kernel 2: rows per stage (one TMA box of 128 rows x wg columns)

template <int T>
__global__ void __launch_bounds__(128) k_mvt1_ring(const __grid_constant__ RealTmap tm, const float *__restrict__ y1,
                                                  const float *__restrict__ x1_0, float *__restrict__ x1, int n,
                                                  int S) {
    constexpr int BW = kMvtRingCols + 4;  // staged row pitch: 528 bytes = 33 x 16 (conflict-free 128-bit reads)
    constexpr int KB = kMvtRingCols / T;  // sub-steps per stage
    static_assert(KB % 2 == 0, "stages start on register buffer 0");
    extern __shared__ unsigned char rk_raw[];
    __shared__ __align__(8) unsigned long long full[kMvtMaxStages], empty[kMvtMaxStages], ybar;
    float *st = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(rk_raw) + 127) & ~uintptr_t(127));
    const int wg = blockDim.x, tid = threadIdx.x, lane = tid & 31;
    const int i0 = blockIdx.x * wg, steps = n / kMvtRingCols;
    const int sf = wg * BW;  // floats per stage
    float *ys = st + (size_t)S * sf;  // y, whole, after the ring (one bulk copy, in flight with the ring's first stages)
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            rk_bar_init(&full[s], 1);
            rk_bar_init(&empty[s], wg / 32);
        }
        rk_bar_init(&ybar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int slot, int step) {
        rk_expect(&full[slot], (unsigned)(sf * 4));
        rk_tma2d(st + slot * sf, &tm, &full[slot], step * kMvtRingCols, i0);
    };
    if (tid == 0) {
        rk_expect(&ybar, (unsigned)(n * 4));
        rk_bulk(ys, y1, (unsigned)(n * 4), &ybar);
        for (int s = 0; s < S && s < steps; ++s) issue(s, s);
    }
    rk_wait(&ybar, 0);
    const unsigned yb = rk_smem(ys);
    const unsigned rowb = rk_smem(st) + (unsigned)(tid * BW * 4);
    float acc = x1_0[i0 + tid];
    float4 a[2][T / 4], y[2][T / 4];
    auto load = [&](int b, unsigned pa, unsigned py) {
#pragma unroll
        for (int c = 0; c < T / 4; ++c) {
            a[b][c] = rk_lds4(pa + (unsigned)(c << 4));
            y[b][c] = rk_lds4(py + (unsigned)(c << 4));
        }
    };
    int slot = 0;
    unsigned phase = 0;
    rk_wait(&full[0], 0);
    load(0, rowb, yb);
    for (int step = 0; step < steps; ++step) {
        const unsigned sb = rowb + (unsigned)(slot * sf * 4);
        const unsigned ysb = yb + (unsigned)(step * kMvtRingCols * 4);
        int ns = slot + 1;
        unsigned nph = phase;
        if (ns == S) {
            ns = 0;
            nph ^= 1;
        }
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            if (kb + 1 < KB) {
                load((kb + 1) & 1, sb + (unsigned)((kb + 1) * T * 4), ysb + (unsigned)((kb + 1) * T * 4));
            } else if (step + 1 < steps) {  // the next stage's first sub-step
                rk_wait(&full[ns], nph);
                load(0, rowb + (unsigned)(ns * sf * 4), ysb + (unsigned)(kMvtRingCols * 4));
            }
#pragma unroll
            for (int c = 0; c < T / 4; ++c) {
                acc = __fmaf_rn(a[kb & 1][c].x, y[kb & 1][c].x, acc);
                acc = __fmaf_rn(a[kb & 1][c].y, y[kb & 1][c].y, acc);
                acc = __fmaf_rn(a[kb & 1][c].z, y[kb & 1][c].z, acc);
                acc = __fmaf_rn(a[kb & 1][c].w, y[kb & 1][c].w, acc);
            }
        }
        __syncwarp();
        if (lane == 0) rk_arrive(&empty[slot]);
        if (tid == 0 && step + S < steps) {
            rk_wait(&empty[slot], phase);
            issue(slot, step + S);
        }
        slot = ns;
        phase = nph;
    }
    x1[i0 + tid] = acc;
}

template <int T, int WG>
__global__ void __launch_bounds__(WG) k_mvt2_ring(const __grid_constant__ RealTmap tm, const float *__restrict__ y2,
                                                 const float *__restrict__ x2_0, float *__restrict__ x2, int n, int S) {
    constexpr int KB = kMvtRingRows / T;
    constexpr int sf = WG * kMvtRingRows;  // floats per stage: [128 rows][WG columns]
    static_assert(KB % 2 == 0, "stages start on register buffer 0");
    extern __shared__ unsigned char rk_raw[];
    __shared__ __align__(8) unsigned long long full[kMvtMaxStages], empty[kMvtMaxStages], ybar;
    float *st = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(rk_raw) + 127) & ~uintptr_t(127));
    const int tid = threadIdx.x, lane = tid & 31;
    const int i0 = blockIdx.x * WG, steps = n / kMvtRingRows;
    float *ys = st + (size_t)S * sf;  // y, whole, after the ring (one bulk copy)
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            rk_bar_init(&full[s], 1);
            rk_bar_init(&empty[s], WG / 32);
        }
        rk_bar_init(&ybar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int slot, int step) {
        rk_expect(&full[slot], (unsigned)(sf * 4));
        rk_tma2d(st + slot * sf, &tm, &full[slot], i0, step * kMvtRingRows);
    };
    if (tid == 0) {
        rk_expect(&ybar, (unsigned)(n * 4));
        rk_bulk(ys, y2, (unsigned)(n * 4), &ybar);
        for (int s = 0; s < S && s < steps; ++s) issue(s, s);
    }
    rk_wait(&ybar, 0);
    const unsigned yb = rk_smem(ys);
    const unsigned colb = rk_smem(st) + (unsigned)(tid * 4);
    float acc = x2_0[i0 + tid];
    float a[2][T];
    float4 y[2][T / 4];
    auto load = [&](int b, unsigned pa, unsigned py) {
#pragma unroll
        for (int jj = 0; jj < T; ++jj) a[b][jj] = rk_lds(pa + (unsigned)(jj * WG * 4));
#pragma unroll
        for (int q = 0; q < T / 4; ++q) y[b][q] = rk_lds4(py + (unsigned)(q << 4));
    };
    int slot = 0;
    unsigned phase = 0;
    rk_wait(&full[0], 0);
    load(0, colb, yb);
    for (int step = 0; step < steps; ++step) {
        const unsigned sb = colb + (unsigned)(slot * sf * 4);
        const unsigned ysb = yb + (unsigned)(step * kMvtRingRows * 4);
        int ns = slot + 1;
        unsigned nph = phase;
        if (ns == S) {
            ns = 0;
            nph ^= 1;
        }
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            if (kb + 1 < KB) {
                load((kb + 1) & 1, sb + (unsigned)((kb + 1) * T * WG * 4), ysb + (unsigned)((kb + 1) * T * 4));
            } else if (step + 1 < steps) {
                rk_wait(&full[ns], nph);
                load(0, colb + (unsigned)(ns * sf * 4), ysb + (unsigned)(kMvtRingRows * 4));
            }
#pragma unroll
            for (int q = 0; q < T / 4; ++q) {
                acc = __fmaf_rn(a[kb & 1][4 * q + 0], y[kb & 1][q].x, acc);
                acc = __fmaf_rn(a[kb & 1][4 * q + 1], y[kb & 1][q].y, acc);
                acc = __fmaf_rn(a[kb & 1][4 * q + 2], y[kb & 1][q].z, acc);
                acc = __fmaf_rn(a[kb & 1][4 * q + 3], y[kb & 1][q].w, acc);
            }
        }
        __syncwarp();
        if (lane == 0) rk_arrive(&empty[slot]);
        if (tid == 0 && step + S < steps) {
            rk_wait(&empty[slot], phase);
            issue(slot, step + S);
        }
        slot = ns;
        phase = nph;
    }
    x2[i0 + tid] = acc;
}

}  // namespace lmt
