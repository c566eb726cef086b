// green_probe.cu -- can the B200 be split into disjoint SM partitions (green
// contexts) that run independent small launches concurrently, and does a
// few-CTA kernel take the same time in a partition as alone on the chip?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o green_probe green_probe.cu -lcuda
//
// Prints: split granularity per flag/minCount, per-group SM ids of a probe
// launch, overlap of concurrent launches, and the time of a fixed-work
// 4-CTA kernel (a) alone on the full device, (b) alone in a partition,
// (c) in a partition while every other partition runs the same kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        CUresult r_ = (x);                                                                 \
        if (r_ != CUDA_SUCCESS) {                                                          \
            const char *s_ = nullptr;                                                      \
            cuGetErrorString(r_, &s_);                                                     \
            printf("FAIL %s -> %d %s (line %d)\n", #x, (int)r_, s_ ? s_ : "?", __LINE__);  \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)
#define CR(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            printf("FAIL %s -> %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__);      \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %smid;" : "=r"(s));
    return s;
}

// fixed dependent fp32 chain per thread (issue-bound like the sweep's long launches)
__global__ void k_work(float *out, int iters, unsigned *sm, unsigned long long *t) {
    float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.999f, d = 0.5f;
    const unsigned long long t0 = gtime();
    for (int i = 0; i < iters; i++) {
        a = fmaf(a, b, c);
        d = fmaf(d, c, b);
        b = fmaf(b, 0.9999f, 1e-6f);
        c = fmaf(c, 1.0001f, -1e-6f);
    }
    if (threadIdx.x == 0) {
        sm[blockIdx.x] = smid();
        t[2 * blockIdx.x] = t0;
        t[2 * blockIdx.x + 1] = gtime();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + d;
}

static const char *kPtx = R"(
.version 8.0
.target sm_100a
.address_size 64
.visible .entry k_ptx(.param .u64 p) {
  .reg .u64 %rd<3>;
  .reg .u32 %r<3>;
  ld.param.u64 %rd1, [p];
  cvta.to.global.u64 %rd2, %rd1;
  mov.u32 %r1, %smid;
  st.global.u32 [%rd2], %r1;
  ret;
}
)";

int main() {
    CR(cudaSetDevice(0));
    CR(cudaFree(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    for (unsigned flags : {0u, (unsigned)CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING}) {
        for (unsigned mc : {1u, 2u, 4u, 8u, 16u, 32u, 36u, 64u, 72u, 74u}) {
            unsigned nb = 0;
            CUresult r = cuDevSmResourceSplitByCount(nullptr, &nb, &all, nullptr, flags, mc);
            std::vector<CUdevResource> g(std::max(1u, nb));
            CUdevResource rem;
            unsigned nb2 = nb;
            unsigned sz = 0, remsz = 0;
            if (r == CUDA_SUCCESS && nb) {
                r = cuDevSmResourceSplitByCount(g.data(), &nb2, &all, &rem, flags, mc);
                if (r == CUDA_SUCCESS) { sz = g[0].sm.smCount; remsz = rem.sm.smCount; }
            }
            printf("split flags=%u minCount=%u -> rc=%d groups=%u size=%u remainder=%u\n", flags, mc, (int)r, nb2, sz,
                   remsz);
        }
    }
    // ---- 8-SM groups (default flags)
    unsigned nb = 0;
    CK(cuDevSmResourceSplitByCount(nullptr, &nb, &all, nullptr, 0, 8));
    std::vector<CUdevResource> groups(nb);
    CUdevResource rem;
    CK(cuDevSmResourceSplitByCount(groups.data(), &nb, &all, &rem, 0, 8));
    std::vector<CUgreenCtx> gctx(nb);
    std::vector<CUstream> gs(nb);
    for (unsigned i = 0; i < nb; i++) {
        CUdevResourceDesc desc;
        CK(cuDevResourceGenerateDesc(&desc, &groups[i], 1));
        CK(cuGreenCtxCreate(&gctx[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
        CK(cuGreenCtxStreamCreate(&gs[i], gctx[i], CU_STREAM_NON_BLOCKING, 0));
    }
    printf("created %u green contexts of %u SMs\n", nb, groups[0].sm.smCount);

    const int ctas = 4, threads = 128;
    float *out;
    unsigned *sm;
    unsigned long long *tt;
    CR(cudaMalloc(&out, sizeof(float) * 64 * 1024 * 64));
    CR(cudaMalloc(&sm, sizeof(unsigned) * 64 * 64));
    CR(cudaMalloc(&tt, sizeof(unsigned long long) * 2 * 64 * 64));
    const int iters = 2000000;
    cudaStream_t full;
    CR(cudaStreamCreateWithFlags(&full, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CR(cudaEventCreate(&e0));
    CR(cudaEventCreate(&e1));
    // (a) alone on the full device
    k_work<<<ctas, threads, 0, full>>>(out, iters / 10, sm, tt);
    CR(cudaStreamSynchronize(full));
    float ms_full = 0;
    CR(cudaEventRecord(e0, full));
    k_work<<<ctas, threads, 0, full>>>(out, iters, sm, tt);
    CR(cudaEventRecord(e1, full));
    CR(cudaStreamSynchronize(full));
    CR(cudaEventElapsedTime(&ms_full, e0, e1));
    printf("(a) full device: %.3f ms\n", ms_full);
    // (b) alone in partition 0, runtime launch onto a green stream
    k_work<<<ctas, threads, 0, (cudaStream_t)gs[0]>>>(out, iters / 10, sm, tt);
    CR(cudaGetLastError());
    CR(cudaStreamSynchronize((cudaStream_t)gs[0]));
    CR(cudaEventRecord(e0, (cudaStream_t)gs[0]));
    k_work<<<ctas, threads, 0, (cudaStream_t)gs[0]>>>(out, iters, sm, tt);
    CR(cudaEventRecord(e1, (cudaStream_t)gs[0]));
    CR(cudaStreamSynchronize((cudaStream_t)gs[0]));
    float ms_part = 0;
    CR(cudaEventElapsedTime(&ms_part, e0, e1));
    unsigned hsm[64];
    CR(cudaMemcpy(hsm, sm, sizeof(unsigned) * ctas, cudaMemcpyDeviceToHost));
    printf("(b) partition 0 alone: %.3f ms, SMs:", ms_part);
    for (int i = 0; i < ctas; i++) printf(" %u", hsm[i]);
    printf("\n");
    // (c) every partition at once, each with its own events
    std::vector<cudaEvent_t> a(nb), b(nb);
    for (unsigned i = 0; i < nb; i++) {
        CR(cudaEventCreate(&a[i]));
        CR(cudaEventCreate(&b[i]));
    }
    for (unsigned i = 0; i < nb; i++) {
        CR(cudaEventRecord(a[i], (cudaStream_t)gs[i]));
        k_work<<<ctas, threads, 0, (cudaStream_t)gs[i]>>>(out + i * 1024 * 64, iters, sm + i * 64, tt + i * 128);
        CR(cudaEventRecord(b[i], (cudaStream_t)gs[i]));
    }
    CR(cudaDeviceSynchronize());
    std::vector<unsigned> hs(nb * 64);
    std::vector<unsigned long long> ht(nb * 128);
    CR(cudaMemcpy(hs.data(), sm, sizeof(unsigned) * nb * 64, cudaMemcpyDeviceToHost));
    CR(cudaMemcpy(ht.data(), tt, sizeof(unsigned long long) * nb * 128, cudaMemcpyDeviceToHost));
    unsigned long long tmin = ~0ull, tmax = 0;
    std::set<unsigned> used;
    int dup = 0;
    for (unsigned i = 0; i < nb; i++) {
        float ms = 0;
        CR(cudaEventElapsedTime(&ms, a[i], b[i]));
        printf("(c) partition %2u: %.3f ms  SMs:", i, ms);
        for (int k = 0; k < ctas; k++) {
            printf(" %u", hs[i * 64 + k]);
            if (!used.insert(hs[i * 64 + k]).second) dup++;
            tmin = std::min(tmin, ht[i * 128 + 2 * k]);
            tmax = std::max(tmax, ht[i * 128 + 2 * k + 1]);
        }
        printf("\n");
    }
    printf("(c) all partitions: span %.3f ms (one kernel %.3f ms), SMs shared by two launches: %d\n",
           (tmax - tmin) / 1e6, ms_part, dup);
    // (d) a module loaded in the primary context, launched on a green stream
    CUmodule mod;
    CUfunction fn;
    CK(cuModuleLoadData(&mod, kPtx));
    CK(cuModuleGetFunction(&fn, mod, "k_ptx"));
    unsigned *p = sm;
    void *args[] = {&p};
    CK(cuLaunchKernel(fn, 1, 1, 1, 1, 1, 1, 0, gs[3], args, nullptr));
    CK(cuStreamSynchronize(gs[3]));
    CR(cudaMemcpy(hsm, sm, sizeof(unsigned), cudaMemcpyDeviceToHost));
    printf("(d) primary-context module on green stream 3: ok, ran on SM %u\n", hsm[0]);
    // (e) 16 SM and 32 SM partitions via IGNORE_SM_COSCHEDULING 2-SM split
    for (unsigned mc : {2u, 4u}) {
        unsigned n2 = 0;
        if (cuDevSmResourceSplitByCount(nullptr, &n2, &all, nullptr, CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING,
                                        mc) != CUDA_SUCCESS)
            continue;
        std::vector<CUdevResource> g2(n2);
        CK(cuDevSmResourceSplitByCount(g2.data(), &n2, &all, &rem, CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING, mc));
        CUdevResourceDesc desc;
        CK(cuDevResourceGenerateDesc(&desc, &g2[0], 1));
        CUgreenCtx gc;
        CK(cuGreenCtxCreate(&gc, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
        CUstream st;
        CK(cuGreenCtxStreamCreate(&st, gc, CU_STREAM_NON_BLOCKING, 0));
        const int c2 = (int)g2[0].sm.smCount;
        k_work<<<c2, threads, 0, (cudaStream_t)st>>>(out, iters, sm, tt);
        CR(cudaGetLastError());
        CR(cudaStreamSynchronize((cudaStream_t)st));
        CR(cudaMemcpy(hsm, sm, sizeof(unsigned) * c2, cudaMemcpyDeviceToHost));
        printf("(e) ignore-cosched minCount %u: %u groups of %d SMs; launch of %d CTAs on SMs:", mc, n2, c2, c2);
        for (int i = 0; i < c2; i++) printf(" %u", hsm[i]);
        printf("\n");
    }
    printf("probe done\n");
    return 0;
}
