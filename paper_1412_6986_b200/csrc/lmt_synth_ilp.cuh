// lmt_synth_ilp.cuh -- K1/K2 with per-thread instruction-level parallelism.
//
// Why: most sweep instances launch few workitems (median grid 16k threads,
// i.e. about one warp per SM sub-partition), so a thread's serial fp32 chain
// (every `acc += x` / MAD depends on the previous one) and its load latency
// set the time. A workitem's work units are independent
// (kernel_model.py:158-170: each writes its own out element), so a thread
// runs U of them in lockstep: U independent accumulators per step, all of a
// step's loads issued before the dependent chain consumes them.
//
// Per work unit the operation order is untouched (stencil offsets
// row-major, comp_ilb MADs, coal_ilb reads, uncoal_ilb reads, epilogue), so
// every output is bit-identical to the U = 1 kernels and to the reference.
//
// The in2 context reads of a step have the same address for all U work units
// of a thread (they depend on glin and i*M+j only, codegen.py:220-235), so a
// step loads each once and adds it to the U accumulators; the target-array
// (`in`) reads -- the accesses the local-memory study is about -- are issued
// per work unit: from global memory in K1, from the TMA-staged region in K2.
//
// Runtime counts (coal_ilb <= 16, uncoal_ilb <= 8 on the fast path) are
// handled by entering a fixed straight-line sequence at slot CAP - count
// (Duff-style), so no predicated-off slots are issued.
#pragma once

#include "lmt_kernels.cuh"

namespace lmt {

constexpr int kMaxStagesG = 8;
constexpr int kCoalCap = 16;
constexpr int kUncoalCap = 8;

template <int SHAPE, int R>
struct Sten {
    __host__ __device__ static constexpr bool in(int a, int b) {
        return SHAPE == 0 ? true
             : SHAPE == 1 ? ((a < 0 ? -a : a) + (b < 0 ? -b : b) <= R)
                          : (a == 0 || b == 0);
    }
    __host__ __device__ static constexpr int count() {
        int k = 0;
        for (int a = -R; a <= R; ++a)
            for (int b = -R; b <= R; ++b)
                if (in(a, b)) ++k;
        return k;
    }
    __host__ __device__ static constexpr int dr(int idx) {
        int k = 0;
        for (int a = -R; a <= R; ++a)
            for (int b = -R; b <= R; ++b)
                if (in(a, b)) {
                    if (k == idx) return a;
                    ++k;
                }
        return 0;
    }
    __host__ __device__ static constexpr int dc(int idx) {
        int k = 0;
        for (int a = -R; a <= R; ++a)
            for (int b = -R; b <= R; ++b)
                if (in(a, b)) {
                    if (k == idx) return b;
                    ++k;
                }
        return 0;
    }
    static constexpr int K = count();
};

__device__ __forceinline__ float lds_f(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// Context values k = 0..count-1 at p + k*stride (halo layout: no modulo)
// into slots CAP-count .. CAP-1, by entering a straight-line sequence.
template <int CAP>
__device__ __forceinline__ void ctx_fetch(float (&cv)[CAP], const float *p, int stride, int count) {
    const int s0 = CAP - count;
#define LMT_CF(s)                           \
    case s:                                 \
        if constexpr (CAP > s) {            \
            cv[s] = __ldg(p);               \
            p += stride;                    \
        }                                   \
        [[fallthrough]];
    switch (s0) {
        LMT_CF(0) LMT_CF(1) LMT_CF(2) LMT_CF(3) LMT_CF(4) LMT_CF(5) LMT_CF(6) LMT_CF(7)
        LMT_CF(8) LMT_CF(9) LMT_CF(10) LMT_CF(11) LMT_CF(12) LMT_CF(13) LMT_CF(14) LMT_CF(15)
        default:
            break;
    }
#undef LMT_CF
}

// acc[u] += value k for k = 0..count-1, in order (slot CAP-count+k).
template <int U, int CAP>
__device__ __forceinline__ void ctx_add(float (&acc)[U], const float (&cv)[CAP], int count) {
    const int s0 = CAP - count;
#define LMT_CA(s)                                                                                      \
    case s:                                                                                            \
        if constexpr (CAP > s) {                                                                       \
            _Pragma("unroll") for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], cv[s]);           \
        }                                                                                              \
        [[fallthrough]];
    switch (s0) {
        LMT_CA(0) LMT_CA(1) LMT_CA(2) LMT_CA(3) LMT_CA(4) LMT_CA(5) LMT_CA(6) LMT_CA(7)
        LMT_CA(8) LMT_CA(9) LMT_CA(10) LMT_CA(11) LMT_CA(12) LMT_CA(13) LMT_CA(14) LMT_CA(15)
        default:
            break;
    }
#undef LMT_CA
}

// MADs of phases 0 .. n-1 (n < 10) on every accumulator.
template <int U, int N>
__device__ __forceinline__ void mad_run(float (&acc)[U]) {
#pragma unroll
    for (int p = 0; p < N; ++p)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = __fmaf_rn(acc[u], mad_c1(p), mad_c2(p));
}

template <int U>
__device__ __forceinline__ void mad_ilb_u(float (&acc)[U], int q, int rem) {
    for (int b = 0; b < q; ++b) mad_run<U, 10>(acc);
    switch (rem) {  // one jump instead of nine predicated steps
        case 1: mad_run<U, 1>(acc); break;
        case 2: mad_run<U, 2>(acc); break;
        case 3: mad_run<U, 3>(acc); break;
        case 4: mad_run<U, 4>(acc); break;
        case 5: mad_run<U, 5>(acc); break;
        case 6: mad_run<U, 6>(acc); break;
        case 7: mad_run<U, 7>(acc); break;
        case 8: mad_run<U, 8>(acc); break;
        case 9: mad_run<U, 9>(acc); break;
        default: break;
    }
}

template <int U>
__device__ __forceinline__ void epilogue_u(const SynthArgs &A, float (&acc)[U], const float *in2c,
                                           const float *in2u) {
    int phase = A.comp_ep_phase;
    for (int k = 0; k < A.comp_ep; ++k) {
        const float c1 = (phase & 1) ? 0.5f : 2.0f;
        const float c2 = ((phase & 1) ? -1.0f : 1.0f) * (float)(1 + phase % 5) * (1.0f / 64.0f);
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = __fmaf_rn(acc[u], c1, c2);
        phase = (phase == 9) ? 0 : phase + 1;
    }
    for (int k = 0; k < A.coal_ep; ++k) {
        const float x = __ldg(in2c + (size_t)wrap_add(A.ep_row0, k, A.H2) * A.P2);
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], x);
    }
    for (int k = 0; k < A.uncoal_ep; ++k) {
        const float x = __ldg(in2u + wrap_add(A.ep_col0, k, A.W2));
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], x);
    }
}

// Target-array source: global float pointers (K1) or shared byte addresses (K2).
template <bool SMEM>
struct TAddr;
template <>
struct TAddr<false> {
    using T = const float *;
    __device__ static __forceinline__ float load(T base, int off) { return __ldg(base + off); }
};
template <>
struct TAddr<true> {
    using T = uint32_t;
    __device__ static __forceinline__ float load(T base, int off) { return lds_f(base + 4u * (uint32_t)off); }
};

// U work units of one thread in lockstep. base[u] addresses the home
// coordinate (i=0, j=0) of work unit u; `pitch` is the row pitch of the
// source (in floats).
template <int SHAPE, int R, int U, bool SMEM>
__device__ __forceinline__ void group_compute(const SynthArgs &A, const typename TAddr<SMEM>::T (&base)[U],
                                              int pitch, const float *in2c, const float *in2u, float (&acc)[U]) {
    using S = Sten<SHAPE, R>;
    constexpr int K = S::K;
    const int step_i = A.a[2] * pitch + A.a[6];
    const int step_j = A.a[3] * pitch + A.a[7];
    const bool fast = A.coal_ilb <= kCoalCap && A.uncoal_ilb <= kUncoalCap;
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.0f;
    int trow = 0, tcol = 0;       // (i*M + j) mod IN2_H / IN2_W
    const float *crow = in2c;     // coal row trow (halo rows cover trow + k, k < 16)
    const float *ucol = in2u;     // uncoal column tcol (halo columns cover tcol + k, k < 8)
    for (int i = 0; i < A.N; ++i) {
        int off = i * step_i;
        for (int j = 0; j < A.M; ++j, off += step_j) {
            float v[U][K];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < K; ++k) v[u][k] = TAddr<SMEM>::load(base[u], off + S::dr(k) * pitch + S::dc(k));
            float cv[kCoalCap], uv[kUncoalCap];
            if (fast) {
                ctx_fetch<kCoalCap>(cv, crow, A.P2, A.coal_ilb);
                ctx_fetch<kUncoalCap>(uv, ucol, 1, A.uncoal_ilb);
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], v[u][k]);
            mad_ilb_u<U>(acc, A.comp_q, A.comp_rem);
            if (fast) {
                ctx_add<U, kCoalCap>(acc, cv, A.coal_ilb);
                ctx_add<U, kUncoalCap>(acc, uv, A.uncoal_ilb);
            } else {
                for (int k = 0; k < A.coal_ilb; ++k) {
                    const float x = __ldg(in2c + (size_t)wrap_add(trow, k, A.H2) * A.P2);
#pragma unroll
                    for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], x);
                }
                for (int k = 0; k < A.uncoal_ilb; ++k) {
                    const float x = __ldg(in2u + wrap_add(tcol, k, A.W2));
#pragma unroll
                    for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], x);
                }
            }
            if (++trow == A.H2) {
                trow = 0;
                crow = in2c;
            } else {
                crow += A.P2;
            }
            if (++tcol == A.W2) {
                tcol = 0;
                ucol = in2u;
            } else {
                ucol += 1;
            }
        }
    }
    epilogue_u<U>(A, acc, in2c, in2u);
}

// Threads per CTA each instantiation is compiled for (register budget
// 64K / threads): U = 4 with the 25-point stencil needs ~190 registers.
template <int U, int K>
struct Bounds {
    static constexpr int threads = U == 1 ? 1024 : (U == 2 ? 512 : (K <= 13 ? 512 : 256));
};
__host__ __device__ constexpr int bound_threads(int U, int K) {
    return U == 1 ? 1024 : (U == 2 ? 512 : (K <= 13 ? 512 : 256));
}

// ------------------------------------------------------------------ K1 (ILP)

template <int SHAPE, int R, int U>
__global__ void __launch_bounds__(Bounds<U, Sten<SHAPE, R>::K>::threads, 1) k_synth_base_g(const SynthArgs A) {
    const int wi_x = threadIdx.x, wi_y = threadIdx.y;
    const int wg_w = blockDim.x, wg_h = blockDim.y;
    const int glin = (blockIdx.y * wg_h + wi_y) * A.grid_x + blockIdx.x * wg_w + wi_x;
    const float *in2c = A.in2 + (glin % A.W2);
    const float *in2u = A.in2 + (size_t)(glin % A.H2) * A.P2;
    const int wux0 = blockIdx.x * (wg_w * A.nwx) + wi_x;
    const int wuy0 = blockIdx.y * (wg_h * A.nwy) + wi_y;
    const float *in0 = A.in + (A.pad * A.P + A.pad);
    const int nit = A.nwx * A.nwy;
    int it = 0;
    for (; it + U <= nit; it += U) {
        const float *b[U];
        size_t o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int ix = (it + u) % A.nwx, iy = (it + u) / A.nwx;
            const int wu_x = wux0 + ix * wg_w, wu_y = wuy0 + iy * wg_h;
            b[u] = in0 + ((A.a[0] * wu_x + A.a[1] * wu_y) * A.P + A.a[4] * wu_x + A.a[5] * wu_y);
            o[u] = (size_t)wu_y * A.out_w + wu_x;
        }
        float acc[U];
        group_compute<SHAPE, R, U, false>(A, b, A.P, in2c, in2u, acc);
#pragma unroll
        for (int u = 0; u < U; ++u) A.out[o[u]] = acc[u];
    }
    for (; it < nit; ++it) {
        const int ix = it % A.nwx, iy = it / A.nwx;
        const int wu_x = wux0 + ix * wg_w, wu_y = wuy0 + iy * wg_h;
        const float *b[1] = {in0 + ((A.a[0] * wu_x + A.a[1] * wu_y) * A.P + A.a[4] * wu_x + A.a[5] * wu_y)};
        float acc[1];
        group_compute<SHAPE, R, 1, false>(A, b, A.P, in2c, in2u, acc);
        A.out[(size_t)wu_y * A.out_w + wu_x] = acc[0];
    }
}

// ------------------------------------------------------------------ K2 (ILP)

// Slots: iteration `it` lives in slot it % S; the producer (thread 0)
// re-arms a slot as soon as every warp has released it, for iteration
// it + S. With S >= 2U a group's regions are in flight while the previous
// group computes.
template <int SHAPE, int R, int U>
__global__ void __launch_bounds__(Bounds<U, Sten<SHAPE, R>::K>::threads, 1)
    k_synth_opt_g(const __grid_constant__ CUtensorMap tmap, const SynthArgs A) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full[kMaxStagesG], empty[kMaxStagesG];

    const int wi_x = threadIdx.x, wi_y = threadIdx.y;
    const int wg_w = blockDim.x, wg_h = blockDim.y;
    const int tid = wi_y * wg_w + wi_x;
    const int nwarps = (wg_w * wg_h + 31) >> 5;
    const int lane = tid & 31;
    const int S = A.nstages;
    const int nit = A.nwx * A.nwy;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (int s = 0; s < S && s < nit; ++s) stage_region(A, &tmap, smem, full, s, s);
    }
    const int glin = (blockIdx.y * wg_h + wi_y) * A.grid_x + blockIdx.x * wg_w + wi_x;
    const float *in2c = A.in2 + (glin % A.W2);
    const float *in2u = A.in2 + (size_t)(glin % A.H2) * A.P2;
    const int hr0 = A.a[0] * wi_x + A.a[1] * wi_y - A.off_min_row;
    const int hc0 = A.a[4] * wi_x + A.a[5] * wi_y - A.off_min_col;
    const int wux0 = blockIdx.x * (wg_w * A.nwx) + wi_x;
    const int wuy0 = blockIdx.y * (wg_h * A.nwy) + wi_y;
    const uint32_t sbase = smem_u32(smem) + 4u * (uint32_t)(hr0 * A.bw + hc0);

    int prev0 = 0, prevcnt = 0;
    for (int it0 = 0; it0 < nit;) {
        const int cnt = (it0 + U <= nit) ? U : 1;
        // re-arm the slots the previous group released
        if (tid == 0) {
            for (int q = 0; q < prevcnt; ++q) {
                const int pit = prev0 + q;
                if (pit + S < nit) {
                    mbar_wait(&empty[pit % S], (pit / S) & 1);
                    stage_region(A, &tmap, smem, full, pit % S, pit + S);
                }
            }
        }
        if (cnt == U) {
            uint32_t b[U];
            size_t o[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int it = it0 + u;
                mbar_wait(&full[it % S], (it / S) & 1);
                b[u] = sbase + 4u * (uint32_t)((it % S) * A.stage_floats + region_shift(A, it));
                const int ix = it % A.nwx, iy = it / A.nwx;
                o[u] = (size_t)(wuy0 + iy * wg_h) * A.out_w + (wux0 + ix * wg_w);
            }
            float acc[U];
            group_compute<SHAPE, R, U, true>(A, b, A.bw, in2c, in2u, acc);
#pragma unroll
            for (int u = 0; u < U; ++u) A.out[o[u]] = acc[u];
        } else {
            const int it = it0;
            mbar_wait(&full[it % S], (it / S) & 1);
            const uint32_t b[1] = {sbase + 4u * (uint32_t)((it % S) * A.stage_floats + region_shift(A, it))};
            float acc[1];
            group_compute<SHAPE, R, 1, true>(A, b, A.bw, in2c, in2u, acc);
            const int ix = it % A.nwx, iy = it / A.nwx;
            A.out[(size_t)(wuy0 + iy * wg_h) * A.out_w + (wux0 + ix * wg_w)] = acc[0];
        }
        __syncwarp();
        if (lane == 0)
            for (int q = 0; q < cnt; ++q) mbar_arrive(&empty[(it0 + q) % S]);
        prev0 = it0;
        prevcnt = cnt;
        it0 += cnt;
    }
}

}  // namespace lmt
