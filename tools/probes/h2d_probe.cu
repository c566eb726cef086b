// Host -> device copy rates from pinned memory: one 1D copy vs a 2D copy into
// a pitched (halo-padded) device layout, for the e2e leg's `in` shapes.
//   nvcc -O3 -o /tmp/h2dp tools/probes/h2d_probe.cu && /tmp/h2dp
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const int shapes[][2] = {{2048, 2048}, {4096, 4096}, {1024, 1024}, {8192, 2048}, {2048, 512}};
    for (auto &sh : shapes) {
        const int rows = sh[0], cols = sh[1];
        const size_t bytes = (size_t)rows * cols * 4;
        float *h, *d, *d2;
        cudaMallocHost(&h, bytes);
        const int pitch = cols + 8;  // halo-padded device rows
        cudaMalloc(&d, (size_t)(rows + 8) * pitch * 4);
        cudaMalloc(&d2, bytes);
        cudaStream_t s;
        cudaStreamCreate(&s);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float t1 = 1e9, t2 = 1e9, t3 = 1e9;
        for (int r = 0; r < 5; r++) {
            float ms;
            cudaEventRecord(a, s);
            cudaMemcpyAsync(d2, h, bytes, cudaMemcpyHostToDevice, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            t1 = ms < t1 ? ms : t1;
            cudaEventRecord(a, s);
            cudaMemcpy2DAsync(d + 4 * pitch + 4, (size_t)pitch * 4, h, (size_t)cols * 4, (size_t)cols * 4, rows,
                              cudaMemcpyHostToDevice, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            t2 = ms < t2 ? ms : t2;
            cudaEventRecord(a, s);  // 1D H2D + on-device 2D placement
            cudaMemcpyAsync(d2, h, bytes, cudaMemcpyHostToDevice, s);
            cudaMemcpy2DAsync(d + 4 * pitch + 4, (size_t)pitch * 4, d2, (size_t)cols * 4, (size_t)cols * 4, rows,
                              cudaMemcpyDeviceToDevice, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            t3 = ms < t3 ? ms : t3;
        }
        printf("%5d x %5d (%6.1f MB): 1D %6.2f GB/s   2D pitched %6.2f GB/s   1D + D2D placement %6.2f GB/s\n", rows,
               cols, bytes / 1e6, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6);
        cudaFreeHost(h);
        cudaFree(d);
        cudaFree(d2);
    }
    return 0;
}
