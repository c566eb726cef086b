// Full-chip fp32 FMA throughput (the roofline denominator for the
// issue-bound synthetic kernels; MEASURED_PEAKS.json holds only HBM copy and
// bf16 tensor peaks). 8 independent FFMA chains per thread, every SM full,
// best of 10 launches timed with CUDA events. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) ffma(float *out, int iters) {
    float a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = threadIdx.x * 1e-7f + u * 1e-3f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 32; ++k)
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __fmaf_rn(a[u], 0.999f, 1e-4f);
    }
    float s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u];
    if (s == 12345.0f) out[0] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out;
    cudaMalloc(&out, 64);
    const int iters = 2000, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ffma<<<blocks, threads>>>(out, 10);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        ffma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * blocks * threads * (double)iters * 32 * 8;
    printf("{\"fp32_fma_tflops\": %.2f, \"fp32_lane_ops_per_s\": %.4e, \"sms\": %d, \"clock_khz_attr\": %d, "
           "\"ms\": %.3f, \"how\": \"FFMA chains, %d CTAs x %d threads x 8 chains, best of 10, CUDA events\"}\n",
           flops / (best * 1e-3) / 1e12, flops / 2 / (best * 1e-3), sms, clk, best, blocks, threads);
    return 0;
}
