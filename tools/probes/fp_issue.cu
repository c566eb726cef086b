// Single-SMSP fp32 issue-rate probe: cycles per warp-instruction for the
// instruction forms the specialised kernels use, with U independent chains
// per thread and W warps per CTA (W <= 4: one warp per SM sub-partition).
#include <cstdio>
#include <cuda_runtime.h>

template <int U, int FORM>
__global__ void probe(float *out, long long *cycles, int iters, float c2r) {
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = threadIdx.x * 1e-3f + u;
    float x = out[threadIdx.x];  // runtime addend
    __syncwarp();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (FORM == 0) acc[u] = __fadd_rn(acc[u], x);                       // FADD R, R, R
                if (FORM == 1) acc[u] = __fmaf_rn(acc[u], (k & 1) ? 0.5f : 2.0f, x); // FFMA R, imm, R
                if (FORM == 2) {                                                      // FFMA R, R, imm(c2)
                    float c1 = (k & 1) ? 0.5f : 2.0f;
                    asm volatile("" : "+f"(c1));
                    acc[u] = __fmaf_rn(acc[u], c1, (k & 1) ? -0.03125f : 0.015625f);
                }
                if (FORM == 3) acc[u] = __fmaf_rn(acc[u], (k & 1) ? 0.5f : 2.0f, (k & 1) ? -0.03125f : 0.015625f);
                if (FORM == 4) acc[u] = __fmaf_rn(acc[u], (k & 1) ? 0.5f : 2.0f, c2r);  // imm c1, reg c2
                if (FORM == 5) acc[u] = __fmaf_rn(x, c2r, acc[u]);                     // FFMA R,R,R (matmul form)
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) s += acc[u];
    out[threadIdx.x + 1024] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int U, int FORM>
void run(const char *name, int warps) {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 4096 * 4);
    cudaMemset(out, 0, 4096 * 4);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    probe<U, FORM><<<1, 32 * warps>>>(out, cyc, iters, 0.015625f);
    probe<U, FORM><<<1, 32 * warps>>>(out, cyc, iters, 0.015625f);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double instr = (double)iters * 16 * U;  // per warp
    printf("%-28s U=%d warps=%d  cycles/instr/warp %.3f  (SMSP issue %.3f instr/cycle)\n", name, U, warps,
           c / instr, warps <= 4 ? instr / c : instr * warps / 4 / c);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 4, 8}) {
        run<4, 0>("FADD R,R,R", w);
        run<8, 0>("FADD R,R,R", w);
        run<8, 1>("FFMA R,R,imm(c1),R", w);
        run<8, 2>("FFMA R,R,R(c1),imm(c2)", w);
        run<8, 3>("FFMA const c1,c2", w);
        run<8, 4>("FFMA imm c1, reg c2", w);
        run<16, 0>("FADD R,R,R", w);
        run<8, 5>("FFMA R,R,R", w);
        run<16, 5>("FFMA R,R,R", w);
    }
    return 0;
}
