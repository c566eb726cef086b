// Transpose variants at n = 8192 (256 MB per array, beyond L2): GB/s of
// 2 * n^2 * 4 bytes per launch, L2 flushed before each. Picks the design of
// K5's optimized transpose (lmt_real.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o transpose_probe transpose_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_copy(const float4 *a, float4 *b, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_scrub(float4 *b, long n4, float t) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
        b[i] = make_float4(t, t, t, t);
}
// V0/V1: SDK transposeCoalesced, T x (T+1) tile, block (T, wy)
__global__ void k_sdk(const float *A, float *B, int n, int T) {
    extern __shared__ float tile[];
    const int P = T + 1, tx = threadIdx.x;
    for (int j = threadIdx.y; j < T; j += blockDim.y) tile[j * P + tx] = A[(size_t)(blockIdx.y * T + j) * n + blockIdx.x * T + tx];
    __syncthreads();
    for (int j = threadIdx.y; j < T; j += blockDim.y) B[(size_t)(blockIdx.x * T + j) * n + blockIdx.y * T + tx] = tile[tx * P + j];
}
// V2: same, diagonal block order (partition camping)
__global__ void k_sdk_diag(const float *A, float *B, int n, int T) {
    extern __shared__ float tile[];
    const int nb = gridDim.x;
    const int by = blockIdx.x, bx = (blockIdx.x + blockIdx.y) % nb;
    const int P = T + 1, tx = threadIdx.x;
    for (int j = threadIdx.y; j < T; j += blockDim.y) tile[j * P + tx] = A[(size_t)(by * T + j) * n + bx * T + tx];
    __syncthreads();
    for (int j = threadIdx.y; j < T; j += blockDim.y) B[(size_t)(bx * T + j) * n + by * T + tx] = tile[tx * P + j];
}
// V3: TMA tile load (box T x T, dense) + TMA tile store of the transposed tile
struct alignas(64) Tm { unsigned long long o[16]; };
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k_tma(const __grid_constant__ Tm tin, const __grid_constant__ Tm tout, int T) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) unsigned long long bar;
    float *a = sm, *b = sm + T * T;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(T * T * 4) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(sa(a)), "l"(&tin), "r"(sa(&bar)), "r"((int)blockIdx.x * T), "r"((int)blockIdx.y * T) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sa(&bar)) : "memory");
    // b[x][y] = a[y][x]; a read down a column: (T+1)-free dense tile -> skew the column index
    for (int e = tid; e < T * T; e += blockDim.x * blockDim.y) {
        const int x = e / T, y = e % T;  // b row x, col y  (lanes: consecutive y)
        b[x * T + y] = a[y * T + x];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                     ::"l"(&tout), "r"(sa(b)), "r"((int)blockIdx.y * T), "r"((int)blockIdx.x * T) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}
// V4: 64-wide tiles, float2 loads, each thread 2 columns; pitch 65
__global__ void k_t64(const float *A, float *B, int n) {
    __shared__ float tile[64][65];
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    const int bx = blockIdx.x * 64, by = blockIdx.y * 64;
    for (int j = ty; j < 64; j += 8) {
        const float2 v = *reinterpret_cast<const float2 *>(A + (size_t)(by + j) * n + bx + 2 * tx);
        tile[j][2 * tx] = v.x;
        tile[j][2 * tx + 1] = v.y;
    }
    __syncthreads();
    for (int j = ty; j < 64; j += 8) {
        float2 v = make_float2(tile[2 * tx][j], tile[2 * tx + 1][j]);
        *reinterpret_cast<float2 *>(B + (size_t)(bx + j) * n + by + 2 * tx) = v;
    }
}

int main() {
    const int n = 8192;
    const size_t bytes = (size_t)n * n * 4;
    float *A, *B, *S;
    CK(cudaMalloc(&A, bytes));
    CK(cudaMalloc(&B, bytes));
    CK(cudaMalloc(&S, 256 << 20));
    CK(cudaMemset(A, 0, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    auto time = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 6; r++) {
            k_scrub<<<592, 256>>>((float4 *)S, (256 << 20) / 16, (float)r);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r && ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("%-28s %8.1f us  %7.0f GB/s %s\n", name, best * 1e3, 2.0 * bytes / (best * 1e-3) / 1e9,
               err ? cudaGetErrorString(err) : "");
    };
    time("copy float4", [&] { k_copy<<<148 * 16, 256>>>((float4 *)A, (float4 *)B, (long)n * n / 4); });
    for (int T : {16, 32})
        for (int wy : {2, 4, 8, 16}) {
            if (wy > T) continue;
            char nm[64];
            snprintf(nm, 64, "sdk T%d wy%d", T, wy);
            time(nm, [&] { k_sdk<<<dim3(n / T, n / T), dim3(T, wy), T * (T + 1) * 4>>>(A, B, n, T); });
            snprintf(nm, 64, "sdk diag T%d wy%d", T, wy);
            time(nm, [&] { k_sdk_diag<<<dim3(n / T, n / T), dim3(T, wy), T * (T + 1) * 4>>>(A, B, n, T); });
        }
    time("t64 32x8 float2", [&] { k_t64<<<dim3(n / 64, n / 64), dim3(32, 8)>>>(A, B, n); });
    for (int T : {32, 64}) {
        CUtensorMap ti, to;
        cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n}, str[1] = {(cuuint64_t)n * 4};
        cuuint32_t box[2] = {(cuuint32_t)T, (cuuint32_t)T}, es[2] = {1, 1};
        enc(&ti, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        enc(&to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        Tm a = *(Tm *)&ti, b = *(Tm *)&to;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * T * T * 4);
        char nm[64];
        snprintf(nm, 64, "tma T%d", T);
        time(nm, [&] { k_tma<<<dim3(n / T, n / T), dim3(32, 8), 2 * T * T * 4>>>(a, b, T); });
    }
    return 0;
}
