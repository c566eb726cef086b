// Single-warp FFMA chain fed from shared memory, the inner loop of the MVT
// ring kernel 1 without TMA or barriers: cycles per element with y staged
// as is (a_j and y_j land in registers of equal parity: an even/odd register
// bank conflict on every FFMA) vs y rotated within each 16-byte quad (a_j and
// y_j of opposite parity).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chainp tools/probes/chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 lds4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

template <bool ROT>
__global__ void __launch_bounds__(32) chain(float *out, long long *cyc, int steps) {
    constexpr int T = 32, BW = 132, KB = 4;
    __shared__ __align__(16) float st[32 * BW];
    __shared__ __align__(16) float ys[4096];
    const int tid = threadIdx.x;
    for (int i = tid; i < 32 * BW; i += 32) st[i] = 1.0f + (i & 7) * 1e-3f;
    for (int i = tid; i < 4096; i += 32) ys[i] = 0.5f + (i & 15) * 1e-3f;
    __syncwarp();
    const unsigned rowb = (unsigned)__cvta_generic_to_shared(st) + tid * BW * 4;
    const unsigned yb = (unsigned)__cvta_generic_to_shared(ys);
    float acc = tid;
    float4 a[2][T / 4], y[2][T / 4];
    auto load = [&](int b, unsigned pa, unsigned py) {
#pragma unroll
        for (int c = 0; c < T / 4; ++c) {
            a[b][c] = lds4(pa + (c << 4));
            y[b][c] = lds4(py + (c << 4));
        }
    };
    long long t0 = clock64();
    load(0, rowb, yb);
    for (int step = 0; step < steps; ++step) {
        const unsigned ysb = yb + (step & 31) * 128 * 4;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            if (kb + 1 < KB) load((kb + 1) & 1, rowb + (kb + 1) * T * 4, ysb + (kb + 1) * T * 4);
            else load(0, rowb, yb + ((step + 1) & 31) * 128 * 4);
#pragma unroll
            for (int c = 0; c < T / 4; ++c) {
                const float4 &A = a[kb & 1][c], &Y = y[kb & 1][c];
                if (ROT) {  // the quad holds (y1, y2, y3, y0)
                    acc = __fmaf_rn(A.x, Y.w, acc);
                    acc = __fmaf_rn(A.y, Y.x, acc);
                    acc = __fmaf_rn(A.z, Y.y, acc);
                    acc = __fmaf_rn(A.w, Y.z, acc);
                } else {
                    acc = __fmaf_rn(A.x, Y.x, acc);
                    acc = __fmaf_rn(A.y, Y.y, acc);
                    acc = __fmaf_rn(A.z, Y.z, acc);
                    acc = __fmaf_rn(A.w, Y.w, acc);
                }
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + tid] = acc;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float *out; long long *cyc;
    cudaMalloc(&out, 148 * 32 * 4); cudaMalloc(&cyc, 148 * 8);
    const int steps = 32;  // 4096 elements
    for (int rep = 0; rep < 2; rep++) {
        long long c;
        chain<false><<<148, 32>>>(out, cyc, steps); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("plain  : %.2f cycles/element\n", (double)c / (steps * 128));
        chain<true><<<148, 32>>>(out, cyc, steps); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("rotated: %.2f cycles/element\n", (double)c / (steps * 128));
    }
    return 0;
}
