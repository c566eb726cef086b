// lmt_jit.cuh -- K1/K2 specialised per compile tuple, compiled at run time
// by NVRTC for sm_100a (see lmt_jit_host.cuh). No system headers: the host
// prepends lmt_args.h and a block of -D style #defines.
//
// Why specialise: the reference emits every kernel instance as OpenCL C with
// its counts and loop bounds as #defines (codegen.py:150-182) and the inner
// body fully unrolled (_inner_body 207-224, _epilogue 227-237). Run-time
// counts force either per-step loops or jump tables around each category of
// operation; on B200 those compile to compare/branch trees that cost more
// than the arithmetic (ncu: branch_resolving + no_inst + short_sb ~35% of
// stall samples in the ahead-of-time kernels). Here the stencil, the six
// counts, the work units per thread U and the prefetch depth D are
// compile-time, so one (i, j) step is straight-line code: its loads, then a
// dependent fp32 chain interleaved across U independent work units.
//
// Latency: the loads of step t + D - 1 are issued before the chain of step t
// consumes its own (a D-slot register ring, the step loop unrolled by D), so
// global/L2 latency hides behind D - 1 steps of arithmetic even when a
// workgroup is a single warp.
//
// Numerics: identical to lmt_kernels.cuh (see its header): per work unit the
// order is stencil taps row-major, comp_ilb MADs (k restarting every step),
// coal_ilb reads, uncoal_ilb reads, then the epilogue; every add is one
// __fadd_rn, every MAD one __fmaf_rn (exact for c1 in {2, 0.5}).
//
// Compile-time parameters (all required):
//   LMT_SHAPE LMT_R                      stencil (0 rect, 1 diamond, 2 star)
//   LMT_CI LMT_CE                        num_comp_ilb, num_comp_ep
//   LMT_NC LMT_NCE LMT_NU LMT_NUE        coal/uncoal ilb/ep counts
//   LMT_U LMT_D                          work units per thread, prefetch depth
//   LMT_OPT                              0 baseline (global loads), 1 optimized (TMA -> smem)
//   LMT_WIDE                             optimized variant with several 256-column TMA chunks
//   LMT_CTXWRAP                          context counts exceed the in2 halo: reduce indices mod IN2_H/W
//   LMT_VEC                              baseline: 128-bit loads for stencil rows of >= 5 taps
//   LMT_MAXT LMT_MINB                    launch bounds (max threads per CTA, min resident CTAs per SM)
//   LMT_PF                               L1 prefetch distance in steps for the in2 context lines (0 off)
//   LMT_SHARE                            the U work units of a group read the same `in` values (their
//                                        home coordinates do not depend on the work unit within the
//                                        group: xy_reuse, or x_reuse_* with the group inside one row of
//                                        work units), so a step loads them once for all U
//   LMT_NM1                              N * M == 1 (one (i, j) step per work unit): the step loops
//                                        and the cursor advance are compile-time
//   LMT_H2 LMT_W2 LMT_P2                 in2 shape (IN2_H, IN2_W: #defines in the reference too) and
//                                        its physical pitch, so every context read of a step is
//                                        one base register plus an immediate offset

namespace lmt {

constexpr int SHAPE = LMT_SHAPE, RAD = LMT_R;
constexpr int CI = LMT_CI, CE = LMT_CE, NC = LMT_NC, NCE = LMT_NCE, NU = LMT_NU, NUE = LMT_NUE;
constexpr int U = LMT_U, D = LMT_D;
constexpr bool SHARE = LMT_SHARE != 0;
// stencil value sets a step loads for NU_ work units
template <int NU_>
constexpr int kSets = SHARE ? 1 : NU_;
constexpr int kMaxStagesJ = 16;
constexpr int H2 = LMT_H2, W2 = LMT_W2, P2 = LMT_P2;
constexpr int PF = LMT_PF;
constexpr long long CS = (long long)(H2 + kIn2PhysHaloRows) * P2;  // floats per in2 copy (lmt_args.h)

// ----------------------------------------------------- stencil (kernel_model.py:115-130)
__host__ __device__ constexpr bool tap_in(int a, int b) {
    return SHAPE == 0 ? true
         : SHAPE == 1 ? ((a < 0 ? -a : a) + (b < 0 ? -b : b) <= RAD)
                      : (a == 0 || b == 0);
}
__host__ __device__ constexpr int tap_count() {
    int k = 0;
    for (int a = -RAD; a <= RAD; ++a)
        for (int b = -RAD; b <= RAD; ++b)
            if (tap_in(a, b)) ++k;
    return k;
}
__host__ __device__ constexpr int tap_dr(int idx) {
    int k = 0;
    for (int a = -RAD; a <= RAD; ++a)
        for (int b = -RAD; b <= RAD; ++b)
            if (tap_in(a, b)) {
                if (k == idx) return a;
                ++k;
            }
    return 0;
}
__host__ __device__ constexpr int tap_dc(int idx) {
    int k = 0;
    for (int a = -RAD; a <= RAD; ++a)
        for (int b = -RAD; b <= RAD; ++b)
            if (tap_in(a, b)) {
                if (k == idx) return b;
                ++k;
            }
    return 0;
}
constexpr int KT = tap_count();

// ----------------------------------------------------- MAD constants (codegen.py:58-66)
__host__ __device__ constexpr float mad_c1(int k) { return (k & 1) ? 0.5f : 2.0f; }
__host__ __device__ constexpr float mad_c2(int k) {
    return ((k & 1) ? -1.0f : 1.0f) * (float)(1 + k % 5) * (1.0f / 64.0f);
}

// ----------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The suspend-time hint (10 ms, the CUTLASS value) lets a waiting warp sleep
// until the phase completes instead of spinning on try_wait: ncu on a
// memory-bound K2 launch showed the spin loop at 38 % of all issued
// instructions (SYNCS + BRA), stealing issue slots from the computing warps.
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(unsigned long long *bar, unsigned parity) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(r)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return r != 0;
}

// L1 prefetch: no destination register, so no scoreboard for the step
// that consumes the line later to wait on.
__device__ __forceinline__ void prefetch_l1(const float *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct alignas(64) TensorMap {
    unsigned long long opaque[16];
};

__device__ __forceinline__ void tma_load_2d(float *dst, const TensorMap *map, unsigned long long *bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// ----------------------------------------------------- target-array sources

// Row structure of the stencil: half-width of row dr and index of its
// first tap (taps are row-major, dc ascending).
__host__ __device__ constexpr int row_w(int dr) {
    return SHAPE == 0 ? RAD : SHAPE == 1 ? RAD - (dr < 0 ? -dr : dr) : (dr == 0 ? RAD : 0);
}
__host__ __device__ constexpr int row_first(int dr) {
    int k = 0;
    for (int a = -RAD; a < dr; ++a) k += 2 * row_w(a) + 1;
    return k;
}

// K1: plain global loads through the read-only path. One pointer per work
// unit; a step adds the (i, j) offset once per work unit and every stencil
// row once more. Rows of >= 5 taps are read with 128-bit loads (LMT_VEC):
// the row's first tap lives at a 16-byte-aligned address of shifted copy
// (addr & 3) of `in` (k_in_shift), so ceil(taps / 4) LDG.128 replace the
// scalar loads -- the "coalesced, vectorised (128-bit) global loads" of the
// baseline, fewer L1 wavefronts when the lanes of a warp walk different rows.
struct GlobalSrc {
    const float *p[U];  // element of the step being loaded next, per work unit
    int pitch;
    long long cs;       // floats between copies of `in`
    template <int NU_>
    __device__ __forceinline__ void load(float (&v)[kSets<NU_>][KT]) const {
#pragma unroll
        for (int u = 0; u < kSets<NU_>; ++u) {
            const float *q = p[u];
            const int qa = (int)(reinterpret_cast<unsigned long long>(q) >> 2);
#pragma unroll
            for (int dr = -RAD; dr <= RAD; ++dr) {
                const int w = row_w(dr), k0 = row_first(dr), nt = 2 * w + 1;
                if (LMT_VEC && nt >= 5) {
                    // the copy is the same for every row of the unit (pitch % 4 == 0):
                    // one shifted base per unit and row width, rows as offsets of it
                    const int sh = (qa - w) & 3;
                    const float4 *vp =
                        reinterpret_cast<const float4 *>(q + ((long long)sh * cs - sh - w) + dr * pitch);
#pragma unroll
                    for (int b = 0; b < (nt + 3) / 4; ++b) {
                        const float4 x = __ldg(vp + b);
                        if (4 * b + 0 < nt) v[u][k0 + 4 * b + 0] = x.x;
                        if (4 * b + 1 < nt) v[u][k0 + 4 * b + 1] = x.y;
                        if (4 * b + 2 < nt) v[u][k0 + 4 * b + 2] = x.z;
                        if (4 * b + 3 < nt) v[u][k0 + 4 * b + 3] = x.w;
                    }
                } else {
                    // the row pointer once, the taps as immediate offsets of it
                    const float *rp = q + dr * pitch;
#pragma unroll
                    for (int t = 0; t < nt; ++t) v[u][k0 + t] = __ldg(rp + (t - w));
                }
            }
        }
    }
    // move every work unit's pointer by (dr, dc) home-coordinate steps: one
    // 64-bit add per work unit (the offset is uniform)
    template <int NU_>
    __device__ __forceinline__ void step(int dr, int dc) {
        const long long d = (long long)dr * pitch + dc;
#pragma unroll
        for (int u = 0; u < NU_; ++u) p[u] += d;
    }
};

// K2: the staged region, row-major with pitch bw (one TMA column chunk).
struct SmemSrc {
    const float *p[U];  // shared-memory element of (i=0, j=0), per work unit
    int pitch;
    int r = 0, c = 0;   // home-coordinate offset of the step being loaded next
    template <int NU_>
    __device__ __forceinline__ void load(float (&v)[kSets<NU_>][KT]) const {
        const int off = r * pitch + c;  // 32-bit shared addresses: recomputing is cheaper than more live pointers
#pragma unroll
        for (int u = 0; u < kSets<NU_>; ++u) {
            const float *q = p[u] + off;
#pragma unroll
            for (int dr = -RAD; dr <= RAD; ++dr) {
                const float *rp = q + dr * pitch;
#pragma unroll
                for (int t = 0; t < 2 * row_w(dr) + 1; ++t) v[u][row_first(dr) + t] = rp[t - row_w(dr)];
            }
        }
    }
    template <int NU_>
    __device__ __forceinline__ void step(int dr, int dc) {
        r += dr;
        c += dc;
    }
};

// K2 with several 256-wide column chunks: smem [ccol][rows_padded][256].
struct SmemWideSrc {
    const float *slot[U];  // stage base per work unit
    int hr[U], hc[U];      // region coordinate of the step being loaded next, per work unit
    int chunk;             // rows_padded * 256
    template <int NU_>
    __device__ __forceinline__ void load(float (&v)[kSets<NU_>][KT]) const {
#pragma unroll
        for (int u = 0; u < kSets<NU_>; ++u) {
#pragma unroll
            for (int k = 0; k < KT; ++k) {
                const int row = hr[u] + tap_dr(k), col = hc[u] + tap_dc(k);
                v[u][k] = slot[u][(col >> 8) * chunk + row * 256 + (col & 255)];
            }
        }
    }
    template <int NU_>
    __device__ __forceinline__ void step(int dr, int dc) {
#pragma unroll
        for (int u = 0; u < NU_; ++u) {
            hr[u] += dr;
            hc[u] += dc;
        }
    }
};

// ----------------------------------------------------- the step pipeline

constexpr int NCs = NC > 0 ? NC : 1;
constexpr int NUs = NU > 0 ? NU : 1;

template <int NU_>
struct Slot {
    float v[kSets<NU_>][KT];
    float c[NCs];
    float w[NUs];
};

// Load cursor: the (i, j) step a slot is filled for.
struct Cursor {
    int j;
    const float *crow; // coal: in2 row trow at column glin % IN2_W
    int trow;
    const float *ucol; // uncoal: in2 row glin % IN2_H, column tcol
    int tcol;
};

__device__ __forceinline__ float ctx_coal(const SynthArgs &A, const float *in2c, const float *crow, int trow,
                                          int k) {
#if LMT_CTXWRAP
    return __ldg(in2c + (size_t)((trow + k) % H2) * P2);
#else
    return __ldg(crow + k * P2);
#endif
}
__device__ __forceinline__ float ctx_uncoal(const SynthArgs &A, const float *in2u, const float *ucol, int tcol,
                                            int k) {
#if LMT_CTXWRAP
    return __ldg(in2u + (tcol + k) % W2);
#else
    return __ldg(ucol + k);
#endif
}

// The uncoalesced context reads in2[row][t .. t + N - 1] (N <= 8) as one or
// two 128-bit loads from the shifted copy (t & 3) (lmt_args.h): `p` points at
// column t of copy 0.
template <int N, int CAP>
__device__ __forceinline__ void uncoal_vec(float (&w)[CAP], const float *p, int t) {
    if constexpr (N > 0) {
        const int sh = t & 3;
        const float4 *v = reinterpret_cast<const float4 *>(p + (sh * CS - sh));
        const float4 a = __ldg(v);
        w[0] = a.x;
        if constexpr (N > 1) w[1] = a.y;
        if constexpr (N > 2) w[2] = a.z;
        if constexpr (N > 3) w[3] = a.w;
        if constexpr (N > 4) {
            const float4 b = __ldg(v + 1);
            w[4] = b.x;
            if constexpr (N > 5) w[5] = b.y;
            if constexpr (N > 6) w[6] = b.z;
            if constexpr (N > 7) w[7] = b.w;
        }
    }
}

template <int NU_, class Src>
__device__ __forceinline__ void fill(Slot<NU_> &s, const Src &src, const Cursor &q, const SynthArgs &A,
                                     const float *in2c, const float *in2u) {
#if LMT_PF > 0 && !LMT_CTXWRAP
    // the one new coal row a step touches (rows trow .. trow+NC-1), PF steps ahead
    if (NC > 0) prefetch_l1(q.crow + (NC - 1 + PF) * P2);
#endif
    src.template load<NU_>(s.v);
#pragma unroll
    for (int k = 0; k < NC; ++k) s.c[k] = ctx_coal(A, in2c, q.crow, q.trow, k);
#if LMT_CTXWRAP
#pragma unroll
    for (int k = 0; k < NU; ++k) s.w[k] = ctx_uncoal(A, in2u, q.ucol, q.tcol, k);
#else
    uncoal_vec<NU>(s.w, q.ucol, q.tcol);
#endif
}

template <int NU_, class Src>
__device__ __forceinline__ void advance(Cursor &q, Src &src, const SynthArgs &A, const float *in2c,
                                        const float *in2u) {
    // j-walk, then the i carriage return (home coordinate affine in i, j)
    int dr = A.a[3], dc = A.a[7];
    if (++q.j == A.M) {
        q.j = 0;
        dr += A.a[2] - A.M * A.a[3];
        dc += A.a[6] - A.M * A.a[7];
    }
    src.template step<NU_>(dr, dc);
    // (i*M + j) mod IN2_H / IN2_W
    if (++q.trow == H2) {
        q.trow = 0;
        q.crow = in2c;
    } else {
        q.crow += P2;
    }
    if (++q.tcol == W2) {
        q.tcol = 0;
        q.ucol = in2u;
    } else {
        q.ucol += 1;
    }
}

template <int NU_>
__device__ __forceinline__ void consume(float (&acc)[NU_], const Slot<NU_> &s) {
#pragma unroll
    for (int k = 0; k < KT; ++k)
#pragma unroll
        for (int u = 0; u < NU_; ++u) acc[u] = __fadd_rn(acc[u], s.v[SHARE ? 0 : u][k]);
#pragma unroll
    for (int k = 0; k < CI; ++k)
#pragma unroll
        for (int u = 0; u < NU_; ++u) acc[u] = __fmaf_rn(acc[u], mad_c1(k), mad_c2(k));
#pragma unroll
    for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int u = 0; u < NU_; ++u) acc[u] = __fadd_rn(acc[u], s.c[k]);
#pragma unroll
    for (int k = 0; k < NU; ++k)
#pragma unroll
        for (int u = 0; u < NU_; ++u) acc[u] = __fadd_rn(acc[u], s.w[k]);
}

// Epilogue context (codegen.py:227-237): the reads depend only on the
// workitem (glin) and N*M, so a thread loads them once; the chain applies
// comp_ep MADs, then the coal and uncoal values, per work unit.
struct EpCtx {
    float ce[NCE > 0 ? NCE : 1], ue[NUE > 0 ? NUE : 1];
    __device__ __forceinline__ void load(const SynthArgs &A, const float *in2c, const float *in2u) {
#pragma unroll
        for (int k = 0; k < NCE; ++k) ce[k] = ctx_coal(A, in2c, in2c + (size_t)A.ep_row0 * P2, A.ep_row0, k);
#if LMT_CTXWRAP
#pragma unroll
        for (int k = 0; k < NUE; ++k) ue[k] = ctx_uncoal(A, in2u, in2u + A.ep_col0, A.ep_col0, k);
#else
        uncoal_vec<NUE>(ue, in2u + A.ep_col0, A.ep_col0);
#endif
    }
    template <int NU_>
    __device__ __forceinline__ void apply(float (&acc)[NU_]) const {
#pragma unroll
        for (int k = 0; k < CE; ++k)
#pragma unroll
            for (int u = 0; u < NU_; ++u) acc[u] = __fmaf_rn(acc[u], mad_c1(CI + k), mad_c2(CI + k));
#pragma unroll
        for (int k = 0; k < NCE; ++k)
#pragma unroll
            for (int u = 0; u < NU_; ++u) acc[u] = __fadd_rn(acc[u], ce[k]);
#pragma unroll
        for (int k = 0; k < NUE; ++k)
#pragma unroll
            for (int u = 0; u < NU_; ++u) acc[u] = __fadd_rn(acc[u], ue[k]);
    }
};

// NU_ work units of one thread: the full i/j nest then the epilogue.
template <int NU_, class Src>
__device__ __forceinline__ void run_units(const SynthArgs &A, Src src, const float *in2c, const float *in2u,
                                          float (&acc)[NU_]) {
#pragma unroll
    for (int u = 0; u < NU_; ++u) acc[u] = 0.0f;
    const int NM = LMT_NM1 ? 1 : A.N * A.M;  // one step per work unit: the loops fold away
    Cursor q{0, in2c, 0, in2u, 0};
    Slot<NU_> s[D];
#pragma unroll
    for (int d = 0; d < D - 1; ++d)
        if (d < NM) {
            fill<NU_>(s[d], src, q, A, in2c, in2u);
            advance<NU_>(q, src, A, in2c, in2u);
        }
    int t0 = 0;
    // steady state: whole blocks of D steps whose prefetches are all in range,
    // straight-line (no per-step guards) so each slot's loads can sit on
    // their own dependency scoreboard
    for (; t0 + 2 * D - 1 <= NM; t0 += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            fill<NU_>(s[(d + D - 1) % D], src, q, A, in2c, in2u);
            advance<NU_>(q, src, A, in2c, in2u);
            consume<NU_>(acc, s[d]);
        }
    }
    for (; t0 < NM; t0 += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int t = t0 + d;
            if (t < NM) {
                if (t + D - 1 < NM) {
                    fill<NU_>(s[(d + D - 1) % D], src, q, A, in2c, in2u);
                    advance<NU_>(q, src, A, in2c, in2u);
                }
                consume<NU_>(acc, s[d]);
            }
        }
    }
    EpCtx e;
    e.load(A, in2c, in2u);
    e.apply<NU_>(acc);
}

// ----------------------------------------------------- K1

#if !LMT_OPT
// blockDim = (WG_W, WG_H), gridDim = (GRID_X/WG_W, GRID_Y/WG_H); work units
// blocked across workgroups, cyclic across workitems (kernel_model.py:158-170).
extern "C" __global__ void __launch_bounds__(LMT_MAXT, LMT_MINB) lmt_kernel(const SynthArgs A) {
    const int wi_x = threadIdx.x, wi_y = threadIdx.y;
    const int wg_w = blockDim.x, wg_h = blockDim.y;
    const int glin = (blockIdx.y * wg_h + wi_y) * A.grid_x + blockIdx.x * wg_w + wi_x;
    const float *in2c = A.in2 + (glin % W2);
    const float *in2u = A.in2 + (size_t)(glin % H2) * P2;
    const int wux0 = blockIdx.x * (wg_w * A.nwx) + wi_x;
    const int wuy0 = blockIdx.y * (wg_h * A.nwy) + wi_y;
    const int nit = A.nwx * A.nwy;
    // Work-unit iterations in order, ix fastest: iteration (ix, iy) reads
    // home pointer prow + ix * sx of the row of work units iy (prow moves by
    // sy per row) and writes orow + ix * wg_w -- no division per work unit.
    const int sx = (A.a[0] * A.P + A.a[4]) * wg_w;
    const long long sy = ((long long)A.a[1] * A.P + A.a[5]) * wg_h;
    const float *prow = A.in + (A.pad * A.P + A.pad) +
                        ((long long)(A.a[0] * wux0 + A.a[1] * wuy0) * A.P + A.a[4] * wux0 + A.a[5] * wuy0);
    float *orow = A.out + ((size_t)wuy0 * A.out_w + wux0);
    const size_t oy = (size_t)wg_h * A.out_w;
    EpCtx ep;
    ep.load(A, in2c, in2u);
    // The thread's full groups of U work units as one stream of (group,
    // step) slots: the D-slot load ring runs across group boundaries, so the
    // loads of the next group are in flight while this one finishes and is
    // stored (with N*M = 1 a group is a single step: without this every
    // group would wait out a full memory latency on its own).
    const int NM = LMT_NM1 ? 1 : A.N * A.M;  // one step per work unit: the loops fold away
    const int ng = nit / U;
    const int total = ng * NM;
    int fix = 0;  // fill cursor: column of work units and row pointer of the next group to load
    const float *fprow = prow;
    int cix = 0;  // consumer cursor: the group being accumulated
    float *corow = orow;
    GlobalSrc src;
    src.pitch = A.P;
    src.cs = A.in_copy;
    Cursor q{0, in2c, 0, in2u, 0};
    int ft = 0, fg = 0, ct = 0;
    auto set_group = [&]() {  // src for the group at the fill cursor; cursor moves on by U units
        if (fix + U <= A.nwx) {
#pragma unroll
            for (int u = 0; u < U; ++u) src.p[u] = fprow + (fix + u) * sx;
            fix += U;
            if (fix == A.nwx) {
                fix = 0;
                fprow += sy;
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                src.p[u] = fprow + fix * sx;
                if (++fix == A.nwx) {
                    fix = 0;
                    fprow += sy;
                }
            }
        }
    };
    auto fill_next = [&](Slot<U> &sl) {
        fill<U>(sl, src, q, A, in2c, in2u);
        if (++ft == NM) {
            ft = 0;
            if (++fg < ng) set_group();
            q = Cursor{0, in2c, 0, in2u, 0};
        } else {
            advance<U>(q, src, A, in2c, in2u);
        }
    };
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.0f;
    auto consume_next = [&](const Slot<U> &sl) {
        consume<U>(acc, sl);
        if (++ct == NM) {  // the group's last step: epilogue, store, next group
            ct = 0;
            ep.apply<U>(acc);
            if (cix + U <= A.nwx) {
#pragma unroll
                for (int u = 0; u < U; ++u) corow[(cix + u) * wg_w] = acc[u];
                cix += U;
                if (cix == A.nwx) {
                    cix = 0;
                    corow += oy;
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    corow[cix * wg_w] = acc[u];
                    if (++cix == A.nwx) {
                        cix = 0;
                        corow += oy;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = 0.0f;
        }
    };
    if (ng > 0) {
        set_group();
        Slot<U> sl[D];
#pragma unroll
        for (int d = 0; d < D - 1; ++d)
            if (d < total) fill_next(sl[d]);
        int k = 0;
        for (; k + 2 * D - 1 <= total; k += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                fill_next(sl[(d + D - 1) % D]);
                consume_next(sl[d]);
            }
        }
        for (; k < total; k += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                if (k + d < total) {
                    if (k + d + D - 1 < total) fill_next(sl[(d + D - 1) % D]);
                    consume_next(sl[d]);
                }
            }
        }
    }
    // the nit % U work units left over, one at a time
    for (int it = ng * U; it < nit; ++it) {
        GlobalSrc s1;
        s1.pitch = A.P;
        s1.cs = A.in_copy;
        s1.p[0] = fprow + fix * sx;
        float *o0 = corow + cix * wg_w;
        if (++fix == A.nwx) {
            fix = 0;
            fprow += sy;
        }
        if (++cix == A.nwx) {
            cix = 0;
            corow += oy;
        }
        float a1[1];
        run_units<1>(A, s1, in2c, in2u, a1);
        *o0 = a1[0];
    }
}
#endif

// ----------------------------------------------------- K2

#if LMT_OPT
// Work-unit iteration -> (ix, iy), ix fastest (kernel_model.py:158-170).
__device__ __forceinline__ void iter_xy(const SynthArgs &A, int it, int &ix, int &iy) {
    if (A.nwx_shift >= 0) {
        ix = it & (A.nwx - 1);
        iy = it >> A.nwx_shift;
    } else {
        ix = it % A.nwx;
        iy = it / A.nwx;
    }
}

// Regions staged per group of U work-unit iterations: one per unit, or one
// for the whole group when its units read the same region (LMT_SHARE).
constexpr int RPS = SHARE ? 1 : U;

// Stage the region of work-unit iteration `it` at `dst` (the cooperative
// copy of codegen.py:296-311, done by the TMA engine). The innermost box
// coordinate must be 16-byte aligned, so the box starts at org_col rounded
// down to 4 floats; region column 0 sits at (org_col & 3).
__device__ __forceinline__ void stage_region(const SynthArgs &A, const TensorMap *map, float *dst,
                                             unsigned long long *bar, int it) {
    int ix, iy;
    iter_xy(A, it, ix, iy);
    const int wu_x0 = blockIdx.x * (blockDim.x * A.nwx) + ix * blockDim.x;
    const int wu_y0 = blockIdx.y * (blockDim.y * A.nwy) + iy * blockDim.y;
    const int org_row = A.a[0] * wu_x0 + A.a[1] * wu_y0 + A.off_min_row + A.pad;
    const int org_col = (A.a[4] * wu_x0 + A.a[5] * wu_y0 + A.off_min_col + A.pad) & ~3;
    for (int cc = 0; cc < A.ncc; ++cc)
        for (int rc = 0; rc < A.nrc; ++rc)
            tma_load_2d(dst + (cc * A.nrc + rc) * A.bh * A.bw, map, bar, org_col + cc * A.bw, org_row + rc * A.bh);
}

// Stage group g (iterations gU .. gU + cnt - 1) into group stage s: one
// full barrier for all of its regions.
__device__ __forceinline__ void stage_group(const SynthArgs &A, const TensorMap *map, float *smem,
                                            unsigned long long *full, int s, int g, int nit) {
    const int it0 = g * U;
    const int nreg = SHARE ? 1 : min(U, nit - it0);
    float *base = smem + (size_t)s * RPS * A.stage_floats;
    mbar_expect_tx(&full[s], (unsigned)nreg * A.stage_bytes);
    for (int r = 0; r < nreg; ++r) stage_region(A, map, base + r * A.stage_floats, &full[s], it0 + r);
}

// A warp is done with group g: arrive on its stage's empty barrier;
// whichever warp then sees the phase complete (the last to arrive, or one
// that checks after it) and wins the claim re-arms the stage with group
// g + G. No warp waits for another to reach a group boundary.
__device__ __forceinline__ void release_group(const SynthArgs &A, const TensorMap *map, float *smem,
                                              unsigned long long *full, unsigned long long *empty, int *claim, int g,
                                              int s, unsigned phase, int G, int ngr, int nit) {
    mbar_arrive(&empty[s]);
    if (g + G < ngr && mbar_test(&empty[s], phase) && atomicCAS(&claim[s], g, g + G) == g)
        stage_group(A, map, smem, full, s, g + G, nit);
}

// The ring holds G group stages (A.nstages); group g (U work-unit
// iterations) lives in stage g % G behind one full and one empty mbarrier,
// so a warp synchronises once per group, not once per work unit, and the
// next G - 1 groups' regions are in flight while it computes. The consumer
// walks the iterations in order with a cursor (ix, row pointers), so no
// division runs per work unit.
extern "C" __global__ void __launch_bounds__(LMT_MAXT, LMT_MINB)
    lmt_kernel(const __grid_constant__ TensorMap tmap, const SynthArgs A) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) unsigned long long full[kMaxStagesJ], empty[kMaxStagesJ];
    __shared__ int claim[kMaxStagesJ];  // group stage s holds / was last armed for

    const int wi_x = threadIdx.x, wi_y = threadIdx.y;
    const int wg_w = blockDim.x, wg_h = blockDim.y;
    const int tid = wi_y * wg_w + wi_x;
    const int nwarps = (wg_w * wg_h + 31) >> 5;
    const int lane = tid & 31;
    const int G = A.nstages;
    const int nit = A.nwx * A.nwy;
    const int ngr = (nit + U - 1) / U;

    if (tid == 0) {
        for (int s = 0; s < G; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwarps);
            claim[s] = s;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmap)) : "memory");
        for (int g = 0; g < G && g < ngr; ++g) stage_group(A, &tmap, smem, full, g, g, nit);
    }
    const int glin = (blockIdx.y * wg_h + wi_y) * A.grid_x + blockIdx.x * wg_w + wi_x;
    const float *in2c = A.in2 + (glin % W2);
    const float *in2u = A.in2 + (size_t)(glin % H2) * P2;
    // home coordinate of (i=0, j=0) relative to the region origin: the same
    // for every iteration (a0*wi_x + a1*wi_y - off_min_row, ...)
    const int hr0 = A.a[0] * wi_x + A.a[1] * wi_y - A.off_min_row;
    const int hc0 = A.a[4] * wi_x + A.a[5] * wi_y - A.off_min_col;
    const int wux0 = blockIdx.x * (wg_w * A.nwx) + wi_x;
    const int wuy0 = blockIdx.y * (wg_h * A.nwy) + wi_y;
    // region column shift of iteration (ix, iy): (cb + cx * ix + cy * iy) & 3
    const int cb = A.a[4] * (blockIdx.x * wg_w * A.nwx) + A.a[5] * (blockIdx.y * wg_h * A.nwy) + A.off_min_col + A.pad;
    const int cx = A.a[4] * wg_w, cy = A.a[5] * wg_h;
    float *orow = A.out + ((size_t)wuy0 * A.out_w + wux0);
    const size_t oy = (size_t)wg_h * A.out_w;
    int ix = 0, iy = 0;  // cursor: the group's first iteration

    int s = 0;
    unsigned phase = 0;  // stage g % G and the parity of its use (g / G) & 1, kept incrementally
    for (int g = 0; g < ngr; ++g) {
        const float *stage = smem + (size_t)s * RPS * A.stage_floats;
        const int cnt = min(U, nit - g * U);
        mbar_wait(&full[s], phase);
        if (cnt == U) {
#if LMT_WIDE
            SmemWideSrc src;
            src.chunk = A.nrc * A.bh * 256;
#else
            SmemSrc src;
            src.pitch = A.bw;
#endif
            float *o[U];
            int sh[U];
            if (ix + U <= A.nwx) {  // the group lies in one row of work units
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    o[u] = orow + (ix + u) * wg_w;
                    sh[u] = (cb + cx * (ix + u) + cy * iy) & 3;
                }
                ix += U;
                if (ix == A.nwx) {
                    ix = 0;
                    ++iy;
                    orow += oy;
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    o[u] = orow + ix * wg_w;
                    sh[u] = (cb + cx * ix + cy * iy) & 3;
                    if (++ix == A.nwx) {
                        ix = 0;
                        ++iy;
                        orow += oy;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float *slot = stage + (SHARE ? 0 : u) * A.stage_floats;
#if LMT_WIDE
                src.slot[u] = slot;
                src.hr[u] = hr0;
                src.hc[u] = hc0 + sh[u];
#else
                src.p[u] = slot + sh[u] + (hr0 * A.bw + hc0);
#endif
            }
            float acc[U];
            run_units<U>(A, src, in2c, in2u, acc);
#pragma unroll
            for (int u = 0; u < U; ++u) *o[u] = acc[u];
        } else {
            for (int u = 0; u < cnt; ++u) {  // the last, short group: one unit at a time
                const int sh0 = (cb + cx * ix + cy * iy) & 3;
                float *o0 = orow + ix * wg_w;
                if (++ix == A.nwx) {
                    ix = 0;
                    ++iy;
                    orow += oy;
                }
                const float *slot = stage + (SHARE ? 0 : u) * A.stage_floats;
#if LMT_WIDE
                SmemWideSrc src;
                src.chunk = A.nrc * A.bh * 256;
                src.slot[0] = slot;
                src.hr[0] = hr0;
                src.hc[0] = hc0 + sh0;
#else
                SmemSrc src;
                src.pitch = A.bw;
                src.p[0] = slot + sh0 + (hr0 * A.bw + hc0);
#endif
                float acc[1];
                run_units<1>(A, src, in2c, in2u, acc);
                *o0 = acc[0];
            }
        }
        __syncwarp();
        if (lane == 0) release_group(A, &tmap, smem, full, empty, claim, g, s, phase, G, ngr, nit);
        if (++s == G) {
            s = 0;
            phase ^= 1;
        }
    }
}
#endif

}  // namespace lmt
