// lmt_args.h -- launch arguments shared by the ahead-of-time kernels
// (lmt_kernels.cuh) and the NVRTC-specialised kernels (lmt_jit.cuh). Plain
// built-in types only: NVRTC compiles this without any system header.
#pragma once

namespace lmt {

constexpr int kMaxGenericOffsets = 128;

struct SynthArgs {
    const float *in;
    const float *in2;
    float *out;
    int P;                   // physical row pitch of `in`, floats (multiple of 4)
    int H2, W2;              // in2 dims (IN2_H, IN2_W)
    int P2;                  // physical row pitch of in2 (W2 + wrapped halo)
    int out_w, grid_x;
    int N, M, nwx, nwy;
    int comp_q, comp_rem;    // comp_ilb = 10*comp_q + comp_rem (AOT kernels)
    int comp_ep, comp_ep_phase;
    int coal_ilb, coal_ep, uncoal_ilb, uncoal_ep;
    int ep_row0, ep_col0;    // (N*M) % IN2_H, (N*M) % IN2_W
    int a[8];                // pattern_affine: row_wu_x,row_wu_y,row_i,row_j,col_wu_x,col_wu_y,col_i,col_j
    int pad;
    // optimized variant: region origin offsets and TMA staging geometry
    int off_min_row, off_min_col;
    int bw, bh, nrc, ncc;    // box width/height, row/col chunk counts
    int stage_floats, nstages;
    unsigned stage_bytes;
    // generic stencil (radius > 2, AOT kernels only)
    int K;
    signed char sdr[kMaxGenericOffsets], sdc[kMaxGenericOffsets];
    // floats between the kInCopies shifted copies of `in` (0: one copy only);
    // copy_s[r][x] = in[r][x + s] (see k_in_shift)
    long long in_copy;
    // log2(nwx) when the number of work-unit columns per workitem is a power
    // of two (iteration -> (ix, iy) by shift and mask), else -1 (division)
    int nwx_shift;
};

// Shifted copies of `in` for the baseline's 128-bit loads of stencil rows
// with >= 5 taps (the row's first tap is read from copy (addr & 3) at a
// 16-byte-aligned address).
constexpr int kInCopies = 4;

// in2 is stored with a wrapped halo: physical [IN2_H + 16][P2 >= IN2_W + 8],
// cell (r, c) = logical in2[r % IN2_H][c % IN2_W]. A context read
// (t + k) mod IN2_H / IN2_W with k < 16 / 8 then needs no modulo.
constexpr int kIn2HaloRows = 16;
constexpr int kIn2HaloCols = 8;
// The physical halo is wider: the specialised kernels prefetch the in2 lines
// of the step kPfMax steps ahead into L1 without wrapping the index, so
// those addresses must stay inside the buffer (they hold wrapped copies too).
constexpr int kPfMax = 32;
constexpr int kIn2PhysHaloRows = kIn2HaloRows + kPfMax;
constexpr int kIn2PhysHaloCols = kIn2HaloCols + kPfMax;
// kIn2Copies copies of the (haloed) in2 buffer, copy s shifted left by s
// columns: copy_s[r][x] = in2[r % IN2_H][(x + s) % IN2_W]. The uncoalesced
// context reads of a step, in2[glin % IN2_H][t .. t + 3], are then one
// 16-byte-aligned 128-bit load from copy (t & 3) at column t - (t & 3).
constexpr int kIn2Copies = 4;

}  // namespace lmt
