// Standalone probe of the K2 staging pipeline: stage every work-unit
// iteration's region with TMA into an S-slot ring (exactly k_synth_opt's
// protocol), copy each staged slot out, compare with the host's view.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>
#include "../paper_1412_6986_b200/csrc/lmt_kernels.cuh"
using namespace lmt;

__global__ void probe(const __grid_constant__ CUtensorMap tmap, const SynthArgs A, float *out, int mode) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nthreads = blockDim.x * blockDim.y;
    const int nwarps = (nthreads + 31) >> 5, lane = tid & 31, S = A.nstages, nit = A.nwx * A.nwy;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nwarps); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) for (int s = 0; s < S && s < nit; ++s) stage_region(A, &tmap, smem, full, s, s);
    for (int it = 0; it < nit; ++it) {
        const int slot = it % S;
        if (mode == 0) {
            if (tid == 0 && it > 0 && it - 1 + S < nit) {
                const int ps = (it - 1) % S;
                mbar_wait(&empty[ps], ((it - 1) / S) & 1);
                stage_region(A, &tmap, smem, full, ps, it - 1 + S);
            }
        } else {
            if ((tid >> 5) == 0 && it > 0 && it - 1 + S < nit) {
                const int ps = (it - 1) % S;
                mbar_wait(&empty[ps], ((it - 1) / S) & 1);
                if (lane == 0) stage_region(A, &tmap, smem, full, ps, it - 1 + S);
                __syncwarp();
            }
        }
        mbar_wait(&full[slot], (it / S) & 1);
        const float *region = smem + slot * A.stage_floats;
        for (int e = tid; e < A.stage_floats; e += nthreads) out[(size_t)it * A.stage_floats + e] = region[e];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }
}

int main(int argc, char **argv) {
    // args: rows cols bw bh nrc ncc S nwx nwy wgx wgy a0 a1 a4 a5 offr offc
    int rows = atoi(argv[1]), cols = atoi(argv[2]);
    SynthArgs A{};
    A.bw = atoi(argv[3]); A.bh = atoi(argv[4]); A.nrc = atoi(argv[5]); A.ncc = atoi(argv[6]);
    A.nstages = atoi(argv[7]); A.nwx = atoi(argv[8]); A.nwy = atoi(argv[9]);
    int wgx = atoi(argv[10]), wgy = atoi(argv[11]);
    A.a[0] = atoi(argv[12]); A.a[1] = atoi(argv[13]); A.a[4] = atoi(argv[14]); A.a[5] = atoi(argv[15]);
    A.off_min_row = atoi(argv[16]); A.off_min_col = atoi(argv[17]); A.pad = 0;
    A.stage_floats = A.ncc * A.nrc * A.bh * A.bw; A.stage_bytes = A.stage_floats * 4;
    int pitch = (cols + 3) / 4 * 4, nit = A.nwx * A.nwy;
    std::vector<float> h((size_t)rows * pitch);
    for (size_t i = 0; i < h.size(); i++) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&o, (size_t)nit * A.stage_floats * 4); cudaMemset(o, 0xff, (size_t)nit * A.stage_floats * 4);
    void *fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box[2] = {(cuuint32_t)A.bw, (cuuint32_t)A.bh}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); return 1; }
    size_t sm = (size_t)A.nstages * A.stage_bytes;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    probe<<<1, dim3(wgx, wgy), sm>>>(map, A, o, argc > 18 ? atoi(argv[18]) : 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("kernel error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> got((size_t)nit * A.stage_floats);
    cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0; int first_it = -1, first_e = -1;
    for (int it = 0; it < nit; it++) {
        int ix = it % A.nwx, iy = it / A.nwx;
        int wx0 = ix * wgx, wy0 = iy * wgy;
        int orow = A.a[0] * wx0 + A.a[1] * wy0 + A.off_min_row, ocol = A.a[4] * wx0 + A.a[5] * wy0 + A.off_min_col;
        for (int cc = 0; cc < A.ncc; cc++) for (int rr = 0; rr < A.nrc * A.bh; rr++) for (int c = 0; c < A.bw; c++) {
            int R = orow + rr, C = ocol + cc * A.bw + c;
            float want = (R >= 0 && R < rows && C >= 0 && C < cols) ? h[(size_t)R * pitch + C] : 0.0f;
            float g = got[(size_t)it * A.stage_floats + ((size_t)cc * A.nrc * A.bh + rr) * A.bw + c];
            if (g != want) { if (!bad) { first_it = it; first_e = rr * 1000 + c; printf("first bad it=%d rr=%d c=%d got=%f want=%f\n", it, rr, c, g, want); } bad++; }
        }
    }
    printf("rows=%d cols=%d box=%dx%d S=%d nit=%d bad=%ld\n", rows, cols, A.bh, A.bw, A.nstages, nit, bad);
    return 0;
}
