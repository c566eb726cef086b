// lmt_capi.cu -- host side of liblmt_b200.so: the C ABI declared in
// include/lmt_b200.h. Validation, geometry, device-memory cache, TMA
// descriptor encoding, kernel dispatch, the measurement engine (CUDA-event
// timing on the whole device or in SM partitions) and the ABI wrappers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lmt_b200.h"
#include "lmt_kernels.cuh"
#include "lmt_jit_host.cuh"
#include "lmt_features.cuh"
#include "lmt_real.cuh"
#include "lmt_train.h"
#include "lmt_train_gpu.cuh"

#ifndef LMT_VERSION
#define LMT_VERSION "lmt_b200 0.1.0 sm_100a"
#endif

using namespace lmt;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return fail(LMT_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                        __LINE__);                                                           \
    } while (0)

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

const lmt_device kDefaultDevice = {128, 32, 4, 48 * 1024, 32768, 63, 48, 8, 400, 4};

// ------------------------------------------------------------ validation

// kernel_model.py:173-219 (validate_params + validate_instance); same
// messages in the same order, joined by "; " like InvalidInstance.
std::vector<std::string> violations(const lmt_instance &p) {
    std::vector<std::string> v;
    char b[160];
    const struct {
        const char *n;
        int32_t x;
    } pos[] = {{"in_h", p.in_h}, {"in_w", p.in_w}, {"out_h", p.out_h},
               {"out_w", p.out_w}, {"n", p.n},       {"m", p.m}};
    for (auto &f : pos)
        if (f.x < 1) { snprintf(b, sizeof b, "%s %d < 1", f.n, f.x); v.push_back(b); }
    const struct {
        const char *n;
        int32_t x;
    } cnt[] = {{"num_comp_ilb", p.num_comp_ilb},     {"num_comp_ep", p.num_comp_ep},
               {"num_coal_ilb", p.num_coal_ilb},     {"num_coal_ep", p.num_coal_ep},
               {"num_uncoal_ilb", p.num_uncoal_ilb}, {"num_uncoal_ep", p.num_uncoal_ep}};
    for (auto &f : cnt)
        if (f.x < 0) { snprintf(b, sizeof b, "%s %d < 0", f.n, f.x); v.push_back(b); }
    if (p.stencil_radius < 0) {
        snprintf(b, sizeof b, "stencil radius %d < 0", p.stencil_radius);
        v.push_back(b);
    }
    const struct {
        const char *n;
        int32_t x;
    } l[] = {{"grid_x", p.grid_x}, {"grid_y", p.grid_y}, {"wg_x", p.wg_x}, {"wg_y", p.wg_y}};
    for (auto &f : l)
        if (!is_pow2(f.x)) { snprintf(b, sizeof b, "%s %d is not a power of two", f.n, f.x); v.push_back(b); }
    if (p.wg_x > p.grid_x) { snprintf(b, sizeof b, "wg_x %d > grid_x %d", p.wg_x, p.grid_x); v.push_back(b); }
    if (p.wg_y > p.grid_y) { snprintf(b, sizeof b, "wg_y %d > grid_y %d", p.wg_y, p.grid_y); v.push_back(b); }
    const int64_t wgs = (int64_t)p.wg_x * p.wg_y, gs = (int64_t)p.grid_x * p.grid_y;
    if (wgs > 1024) { snprintf(b, sizeof b, "workgroup size %lld > 1024", (long long)wgs); v.push_back(b); }
    if (gs < 512) { snprintf(b, sizeof b, "grid size %lld < 512", (long long)gs); v.push_back(b); }
    if (p.grid_x > 0 && p.out_w % p.grid_x != 0) {
        snprintf(b, sizeof b, "grid_x %d does not divide out_w %d", p.grid_x, p.out_w);
        v.push_back(b);
    }
    if (p.grid_y > 0 && p.out_h % p.grid_y != 0) {
        snprintf(b, sizeof b, "grid_y %d does not divide out_h %d", p.grid_y, p.out_h);
        v.push_back(b);
    }
    return v;
}

// ------------------------------------------------------------- geometry

// access_analysis.py:51-62
bool pattern_affine(int pattern, int n, int m, int32_t c[8]) {
    static const int32_t tab[5][8] = {{0, 0, 1, 0, 0, 0, 0, 1}, {0, 1, 0, 0, 0, 0, 0, 1},
                                      {0, 0, 0, 1, 0, 1, 0, 0}, {1, 0, 0, 0, 0, 0, 0, 1},
                                      {0, 0, 0, 1, 1, 0, 0, 0}};
    if (pattern >= 0 && pattern < 5) { memcpy(c, tab[pattern], sizeof tab[0]); return true; }
    if (pattern == 5) { const int32_t t[8] = {0, n, 1, 0, m, 0, 0, 1}; memcpy(c, t, sizeof t); return true; }
    if (pattern == 6) { const int32_t t[8] = {0, m, 0, 1, n, 0, 1, 0}; memcpy(c, t, sizeof t); return true; }
    return false;
}

// kernel_model.py:115-130
int stencil_offsets(int shape, int r, std::vector<int> *dr, std::vector<int> *dc) {
    int k = 0;
    for (int a = -r; a <= r; a++)
        for (int b = -r; b <= r; b++) {
            if (shape == 1 && std::abs(a) + std::abs(b) > r) continue;
            if (shape == 2 && a != 0 && b != 0) continue;
            if (dr) { dr->push_back(a); dc->push_back(b); }
            k++;
        }
    return k;
}

// access_analysis.py:169-181
int64_t pad_col_span(int64_t span, int64_t tx) {
    if (span % tx == 0) return span;
    if (span > tx) return (span / tx + 1) * tx;
    int64_t b = 1;
    while (b < span) b <<= 1;
    return b;
}

// access_analysis.py:184-213 + codegen.py:94-132
int compute_geometry(const lmt_instance &p, const lmt_device &d, lmt_geometry *g) {
    int32_t c[8];
    if (!pattern_affine(p.pattern, p.n, p.m, c)) return fail(LMT_ERR_ARG, "unknown pattern %d", p.pattern);
    if (p.stencil_shape < 0 || p.stencil_shape > 2) return fail(LMT_ERR_ARG, "unknown stencil shape %d", p.stencil_shape);
    if (p.stencil_radius < 0 || p.stencil_radius > 64) return fail(LMT_ERR_ARG, "stencil radius %d out of range", p.stencil_radius);
    if (d.transaction_bytes <= 0 || d.element_bytes <= 0 || d.warp_size <= 0) return fail(LMT_ERR_ARG, "bad device descriptor");
    std::vector<int> dr, dc;
    const int K = stencil_offsets(p.stencil_shape, p.stencil_radius, &dr, &dc);
    const int omin_r = *std::min_element(dr.begin(), dr.end()), omax_r = *std::max_element(dr.begin(), dr.end());
    const int omin_c = *std::min_element(dc.begin(), dc.end()), omax_c = *std::max_element(dc.begin(), dc.end());
    const int64_t hrm = (int64_t)c[0] * (p.wg_x - 1) + (int64_t)c[1] * (p.wg_y - 1) + (int64_t)c[2] * (p.n - 1) +
                        (int64_t)c[3] * (p.m - 1);
    const int64_t hcm = (int64_t)c[4] * (p.wg_x - 1) + (int64_t)c[5] * (p.wg_y - 1) + (int64_t)c[6] * (p.n - 1) +
                        (int64_t)c[7] * (p.m - 1);
    const int64_t row_span = hrm + 1 + (omax_r - omin_r);
    const int64_t col_span = hcm + 1 + (omax_c - omin_c);
    const int64_t tx = d.transaction_bytes / d.element_bytes;
    const int64_t padded = pad_col_span(col_span, tx);
    const int64_t seg = std::min<int64_t>(tx, padded);
    const int64_t wgs = (int64_t)p.wg_x * p.wg_y;
    const int64_t mx0 = (int64_t)p.out_w - p.wg_x, my0 = (int64_t)p.out_h - p.wg_y;
    const int64_t max_org_row = c[0] * mx0 + c[1] * my0 + omin_r;
    const int64_t max_org_col = c[4] * mx0 + c[5] * my0 + omin_c;
    g->pad = p.stencil_radius;
    g->off_min_row = omin_r;
    g->off_min_col = omin_c;
    g->r_rows = (int32_t)row_span;
    g->r_cols = (int32_t)col_span;
    g->r_cols_pad = (int32_t)padded;
    g->seg_elems = (int32_t)seg;
    g->segs_per_row = (int32_t)(padded / seg);
    g->num_segs = (int32_t)(row_span * (padded / seg));
    g->num_warps = (int32_t)((wgs + d.warp_size - 1) / d.warp_size);
    g->lanes_per_warp = (int32_t)std::min<int64_t>(d.warp_size, wgs);
    g->alloc_h = p.stencil_radius + max_org_row + row_span;
    g->alloc_w = p.stencil_radius + max_org_col + padded;
    g->org_row_wu_x = c[0];
    g->org_row_wu_y = c[1];
    g->row_i = c[2];
    g->row_j = c[3];
    g->org_col_wu_x = c[4];
    g->org_col_wu_y = c[5];
    g->col_i = c[6];
    g->col_j = c[7];
    g->footprint_bytes = row_span * padded * d.element_bytes;
    g->num_offsets = K;
    return LMT_OK;
}

// ------------------------------------------------------- device context

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

// Driver entry points of the green-context (SM partition) API, resolved at
// run time like the TMA encoder (no libcuda at link time).
struct GreenApi {
    PFN_cuDeviceGet_v2000 device_get = nullptr;
    PFN_cuDeviceGetDevResource_v12040 get_resource = nullptr;
    PFN_cuDevSmResourceSplitByCount_v12040 split = nullptr;
    PFN_cuDevResourceGenerateDesc_v12040 gen_desc = nullptr;
    PFN_cuGreenCtxCreate_v12040 create = nullptr;
    PFN_cuGreenCtxStreamCreate_v12050 stream_create = nullptr;
    PFN_cuCtxFromGreenCtx_v12040 to_ctx = nullptr;
    bool tried = false, ok = false;
} g_green;

PFN_cuCtxGetCurrent_v4000 g_ctx_current = nullptr;

bool green_init() {
    if (g_green.tried) return g_green.ok;
    g_green.tried = true;
    struct {
        const char *name;
        void **slot;
    } fns[] = {{"cuDeviceGet", (void **)&g_green.device_get},
               {"cuDeviceGetDevResource", (void **)&g_green.get_resource},
               {"cuDevSmResourceSplitByCount", (void **)&g_green.split},
               {"cuDevResourceGenerateDesc", (void **)&g_green.gen_desc},
               {"cuGreenCtxCreate", (void **)&g_green.create},
               {"cuGreenCtxStreamCreate", (void **)&g_green.stream_create},
               {"cuCtxFromGreenCtx", (void **)&g_green.to_ctx}};
    for (auto &f : fns) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(f.name, f.slot, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !*f.slot)
            return false;
    }
    g_green.ok = true;
    return true;
}

// Where instances run: the whole device (isolated: one instance at a time,
// L2 flushed before each variant), or one SM partition (a green context).
// A lane owns its input/output buffers; its stream orders its instances.
struct Lane {
    int sms = 0;  // SMs of the partition; 0 = the whole device
    cudaStream_t s = nullptr;
    CUcontext ctx = nullptr;  // the (green) context its stream belongs to
    // host mode: the copied `in` (+ the baseline's shifted copies); device
    // mode: the baseline's shifted copies of the shared `in` only
    float *in[2] = {nullptr, nullptr};
    size_t in_cap[2] = {0, 0};
    float *ob[2] = {nullptr, nullptr}, *oo[2] = {nullptr, nullptr};
    size_t out_cap[2] = {0, 0};
    float *in2[2] = {nullptr, nullptr};  // host mode: this lane's in2 in the kernels' layout
    size_t in2_cap[2] = {0, 0};
    // host mode on the whole device: copies on their own streams, two buffer
    // sets, so the copies of instances i +- 1 overlap the kernels of i
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t copied[2] = {}, consumed[2] = {}, drained[2] = {};
    CUgreenCtx gctx = nullptr;  // the partition's green context (copy streams are created in it)
    unsigned seq = 0;           // instances enqueued on this lane (buffer set = seq & 1)
    std::vector<int64_t> inflight;  // instances enqueued, in order
};

struct DevCtx {
    int device = -1;
    int sms = 0;
    size_t smem_optin = 0;
    cudaStream_t stream = nullptr;  // the library stream: the whole-device lane
    Lane full;
    std::vector<Lane> parts;        // SM partitions, largest first
    bool parts_tried = false;
    // device-generated inputs, shared read-only by every lane: `in` per
    // logical width (its content is hash(r * alloc_w + c) whatever the
    // instance), in2 per shape in the kernels' wrapped-halo layout
    struct SharedIn {
        float *p = nullptr;
        int64_t rows = 0, pitch = 0;
        uint64_t used = 0;
    };
    std::map<int64_t, SharedIn> ins;
    size_t ins_bytes = 0;
    uint64_t batch_no = 0;
    std::map<std::pair<int64_t, int64_t>, float *> in2s;
    cudaEvent_t inputs_ready = nullptr;  // shared inputs and per-batch scratch are ready
    float4 *scrub = nullptr;        // L2 flush buffer
    int64_t scrub_n4 = 0;
    float scrub_tag = 0.0f;
    unsigned long long *dres = nullptr;
    size_t dres_cap = 0;
    int64_t *didx = nullptr;
    size_t didx_cap = 0;
    float *dsamp = nullptr;
    size_t dsamp_cap = 0;
    std::vector<cudaEvent_t> events;
};

std::mutex g_mu;
DevCtx g_ctx[64];

constexpr int kEvPerInst = 8;  // base start/end, opt start/end, done, fill start/end, spare
constexpr int64_t kScrubBytes = 192ll << 20;  // > 126 MB L2

template <class T>
int ensure(T **p, size_t *cap, size_t need) {
    if (*cap >= need && *p) return LMT_OK;
    if (*p) CUDA_TRY(cudaFree(*p));
    *p = nullptr;
    *cap = 0;
    CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(p), std::max<size_t>(need, 64) * sizeof(T)));
    *cap = std::max<size_t>(need, 64);
    return LMT_OK;
}

int lane_streams(Lane &L) {
    if (L.h2d) return LMT_OK;
    if (L.gctx) {  // a partition: its copy streams live in its green context too
        CUstream a, b;
        if (g_green.stream_create(&a, L.gctx, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
            g_green.stream_create(&b, L.gctx, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
            return fail(LMT_ERR_CUDA, "green-context copy streams");
        L.h2d = (cudaStream_t)a;
        L.d2h = (cudaStream_t)b;
    } else {
        CUDA_TRY(cudaStreamCreateWithFlags(&L.h2d, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&L.d2h, cudaStreamNonBlocking));
    }
    for (int b = 0; b < 2; b++) {
        CUDA_TRY(cudaEventCreateWithFlags(&L.copied[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&L.consumed[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&L.drained[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(L.consumed[b], L.s));  // complete: nothing in flight yet
        CUDA_TRY(cudaEventRecord(L.drained[b], L.s));
    }
    return LMT_OK;
}

int get_ctx(DevCtx **out) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(LMT_ERR_ARG, "device %d out of range", dev);
    DevCtx &c = g_ctx[dev];
    if (c.device < 0) {
        CUDA_TRY(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
        int optin = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        c.smem_optin = (size_t)optin;
        CUDA_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        c.full.s = c.stream;
        CUDA_TRY(cudaFree(0));  // the primary context exists and is current
        if (!g_ctx_current) {
            cudaDriverEntryPointQueryResult q;
            CUDA_TRY(cudaGetDriverEntryPoint("cuCtxGetCurrent", (void **)&g_ctx_current, cudaEnableDefault, &q));
            if (!g_ctx_current || q != cudaDriverEntryPointSuccess) return fail(LMT_ERR_CUDA, "cuCtxGetCurrent unavailable");
        }
        if (g_ctx_current(&c.full.ctx) != CUDA_SUCCESS) return fail(LMT_ERR_CUDA, "no current CUDA context");
        CUDA_TRY(cudaEventCreateWithFlags(&c.inputs_ready, cudaEventDisableTiming));
        CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(k_rf_mean),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(k_mvt1_tma<16>),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(k_mvt1_tma<32>),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(k_mvt2_tma<16>),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(k_mvt2_tma<32>),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        for (const void *kf : {reinterpret_cast<const void *>(k_matmul_opt_t<64, 4, 4>),
                               reinterpret_cast<const void *>(k_matmul_opt_t<64, 8, 4>),
                               reinterpret_cast<const void *>(k_matmul_opt88)})
            CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        for (const void *kf : {reinterpret_cast<const void *>(k_mvt1_ring<16>), reinterpret_cast<const void *>(k_mvt1_ring<32>),
                               reinterpret_cast<const void *>(k_mvt2_ring<16, 32>), reinterpret_cast<const void *>(k_mvt2_ring<16, 64>),
                               reinterpret_cast<const void *>(k_mvt2_ring<16, 128>), reinterpret_cast<const void *>(k_mvt2_ring<32, 32>),
                               reinterpret_cast<const void *>(k_mvt2_ring<32, 64>), reinterpret_cast<const void *>(k_mvt2_ring<32, 128>)})
            CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        for (const void *kf : {reinterpret_cast<const void *>(k_conv_rows_opt<0>), reinterpret_cast<const void *>(k_conv_rows_opt<1>),
                               reinterpret_cast<const void *>(k_conv_rows_opt<2>), reinterpret_cast<const void *>(k_conv_rows_opt<4>),
                               reinterpret_cast<const void *>(k_conv_rows_opt<8>), reinterpret_cast<const void *>(k_conv_cols_opt<0>),
                               reinterpret_cast<const void *>(k_conv_cols_opt<1>), reinterpret_cast<const void *>(k_conv_cols_opt<2>),
                               reinterpret_cast<const void *>(k_conv_cols_opt<4>), reinterpret_cast<const void *>(k_conv_cols_opt<8>)})
            CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        c.device = dev;
    }
    if (!g_encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(LMT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    *out = &c;
    return LMT_OK;
}

// The SM partitions of the concurrent measurement: one split of the device
// into 2-SM groups (the finest the driver offers), regrouped into
// partitions of 74, 36, 16, 8, 8, 4 and 2 SMs. The sizes come from a
// scheduling simulation over the round-1 40k-instance sweep:
// any layout of this kind packs the sweep within a few percent of the
// others; what bounds the gain is the launches too wide for a partition.
const int kLayout[] = {74, 36, 16, 8, 8, 4, 2};

// Module loading is lazy and per context: launch every ahead-of-time kernel
// a lane uses once, so none of them loads inside a timed window later.
int warm_lane(Lane &L) {
    float *buf = nullptr;
    CUDA_TRY(cudaMalloc(&buf, 4096 * sizeof(float)));
    int64_t *idx = reinterpret_cast<int64_t *>(buf + 2048);
    CUDA_TRY(cudaMemsetAsync(buf, 0, 4096 * sizeof(float), L.s));
    k_fill<<<1, 32, 0, L.s>>>(buf, 1, 4, 4, 0);
    k_in2_halo<<<1, 32, 0, L.s>>>(buf, 1, 1, 4);
    k_in2_shift<<<1, 32, 0, L.s>>>(buf, 1, 1, 4, 0);
    k_in_shift<<<1, 32, 0, L.s>>>(buf, 0, 4);
    k_in_copy4<<<1, 32, 0, L.s>>>(buf, buf + 512, 0, 4);
    k_digest<<<1, 32, 0, L.s>>>(buf, buf, 0, reinterpret_cast<unsigned long long *>(buf + 1024));
    k_gather<<<1, 32, 0, L.s>>>(buf, buf, idx, 0, buf + 1536);
    k_scrub<<<1, 32, 0, L.s>>>(reinterpret_cast<float4 *>(buf), 0, 0.0f);
    k_lead<<<1, 32, 0, L.s>>>(0ll);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(L.s));
    CUDA_TRY(cudaFree(buf));
    return LMT_OK;
}

int ensure_parts(DevCtx *c) {
    if (c->parts_tried) return LMT_OK;
    c->parts_tried = true;
    if (!green_init()) return LMT_OK;
    CUdevice dev;
    if (g_green.device_get(&dev, c->device) != CUDA_SUCCESS) return LMT_OK;
    CUdevResource all;
    if (g_green.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return LMT_OK;
    unsigned ng = 0;
    const unsigned fl = CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING;
    if (g_green.split(nullptr, &ng, &all, nullptr, fl, 2) != CUDA_SUCCESS || ng == 0) return LMT_OK;
    std::vector<CUdevResource> g(ng);
    CUdevResource rem;
    if (g_green.split(g.data(), &ng, &all, &rem, fl, 2) != CUDA_SUCCESS) return LMT_OK;
    const unsigned per = g[0].sm.smCount;
    unsigned next = 0;
    for (int size : kLayout) {
        const unsigned k = (unsigned)size / std::max(1u, per);
        if (k == 0 || next + k > ng) break;
        CUdevResourceDesc desc;
        if (g_green.gen_desc(&desc, &g[next], k) != CUDA_SUCCESS) break;
        CUgreenCtx gc;
        if (g_green.create(&gc, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) break;
        CUstream st;
        if (g_green.stream_create(&st, gc, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) break;
        Lane L;
        L.sms = (int)(k * per);
        L.s = (cudaStream_t)st;
        L.gctx = gc;
        if (g_green.to_ctx(&L.ctx, gc) != CUDA_SUCCESS) break;
        int rc = warm_lane(L);
        if (rc) return rc;
        c->parts.push_back(L);
        next += k;
    }
    return LMT_OK;
}

// ------------------------------------------------------ launch planning

struct Plan {
    lmt_geometry g;
    SynthArgs A;
    bool feasible;      // footprint <= lmem cap (codegen.py:351)
    bool wide;
    JitKey kb, ko;      // specialised kernels (baseline, optimized)
    int in_copies;      // shifted copies of `in` the baseline reads (1 or kInCopies)
    size_t dyn_smem;
    dim3 grid, block;
    int64_t ctas;
    double alg_bytes, alg_flops;
    double est_s;       // launch floor of one variant (scheduling only)
};

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
int64_t in2_pitch(int64_t w) { return round_up(w + kIn2PhysHaloCols, 32); }  // rows start on 128-byte lines
size_t in2_copy_elems(int64_t h, int64_t w) { return (size_t)(h + kIn2PhysHaloRows) * (size_t)in2_pitch(w); }
size_t in2_phys_elems(int64_t h, int64_t w) { return kIn2Copies * in2_copy_elems(h, w); }

// |U_in2|: union of the in2 cells the context reads touch.
double in2_union(const lmt_instance &p) {
    const int64_t H = p.in_h, W = p.in_w, nm = (int64_t)p.n * p.m;
    const int64_t gs = (int64_t)p.grid_x * p.grid_y;
    // glin takes every value in [0, grid_size), so glin % W covers
    // [0, min(gs, W)) and glin % H covers [0, min(gs, H)).
    const int64_t gcols = std::min(gs, W), grows = std::min(gs, H);
    int64_t coal_rows = 0, coal_rows_lo = 0, uncoal_cols = 0, uncoal_cols_lo = 0;
    auto count_set = [&](int64_t lo_count, int64_t extra_start, int64_t extra_count, int64_t mod, int64_t below,
                         int64_t *in_range) {
        std::vector<char> seen((size_t)mod, 0);
        int64_t c = 0, c_lo = 0;
        auto add = [&](int64_t r) {
            if (!seen[(size_t)r]) { seen[(size_t)r] = 1; c++; if (r < below) c_lo++; }
        };
        for (int64_t t = 0; t < std::min(lo_count, mod); t++) add(t);
        for (int64_t k = 0; k < std::min(extra_count, mod); k++) add((extra_start + k) % mod);
        *in_range = c_lo;
        return c;
    };
    if (p.num_coal_ilb > 0 || p.num_coal_ep > 0)
        coal_rows = count_set(p.num_coal_ilb > 0 ? nm + p.num_coal_ilb - 1 : 0, nm, p.num_coal_ep, H, grows, &coal_rows_lo);
    if (p.num_uncoal_ilb > 0 || p.num_uncoal_ep > 0)
        uncoal_cols = count_set(p.num_uncoal_ilb > 0 ? nm + p.num_uncoal_ilb - 1 : 0, nm, p.num_uncoal_ep, W, gcols,
                                &uncoal_cols_lo);
    // coal cells: coal_rows x gcols; uncoal cells: grows x uncoal_cols;
    // their intersection: (coal rows < grows) x (uncoal cols < gcols)
    const double cells = (double)coal_rows * gcols + (double)grows * uncoal_cols - (double)coal_rows_lo * uncoal_cols_lo;
    return cells;
}

// |U_in| in closed form: home rectangle dilated by the stencil.
double in_union(const lmt_instance &p) {
    const int64_t n = p.n, m = p.m, oh = p.out_h, ow = p.out_w, r = p.stencil_radius;
    int64_t H = 0, W = 0;
    switch (p.pattern) {
        case 0: H = n; W = m; break;
        case 1: H = oh; W = m; break;
        case 2: H = m; W = oh; break;
        case 3: H = ow; W = m; break;
        case 4: H = m; W = ow; break;
        case 5: H = oh * n; W = ow * m; break;
        default: H = oh * m; W = ow * n; break;
    }
    if (r == 0) return (double)H * W;
    if (p.stencil_shape == 0) return (double)(H + 2 * r) * (W + 2 * r);
    if (p.stencil_shape == 2) return (double)H * W + 2.0 * r * (H + W);
    return (double)H * W + 2.0 * r * (H + W) + 4.0 * (r * (r - 1) / 2);
}

constexpr int kMaxStagesJ = 16;
constexpr int kPfDist = 8;  // L1 prefetch distance of the in2 context lines, steps
JitCache g_jit;

// kernel_id of a specialised pair: 1 B D O E with B/O = log2 U + 1 of the
// baseline/optimized kernel and D/E their prefetch depths (e.g. 14342:
// baseline U=8 D=3, optimized U=8 D=2)
int jit_kid(const JitKey &b, const JitKey &o) {
    auto lg = [](int u) { int l = 0; while ((1 << l) < u) l++; return l + 1; };
    return 10000 + lg(b.U) * 1000 + b.D * 100 + lg(o.U) * 10 + o.D;
}

// Work units per thread U, prefetch depth D (and, for the optimized
// variant, staging slots S) for the specialised kernels.
//
// A thread's work units are independent fp32 chains, so U of them in
// lockstep give U-way ILP, and the in2 context loads of a step are shared by
// its U work units; D prefetched steps hide load latency. Each work unit
// still issues its own stencil loads (the emitted kernel's semantics)
// unless `regblock` lets units with identical home coordinates share them.
// Measured on B200 (round 1, tools/gpu_ud.sh): the largest U and D the
// register file holds win on every representative launch shape, so the
// baseline asks for U = 16, D = 3 and JitCache::resolve steps D, then U,
// down until ptxas does not spill.
//
// The optimized variant also needs S >= U staged regions per CTA (S >= 2U to
// overlap the next group's TMA with the current group), and shared memory
// bounds residency: score = independent chains per SM sub-partition, then
// TMA overlap, then U, then D.
constexpr double kLoopInstrBudget = 2100.0;

int64_t jit_regs_guess(int K, int64_t slot, int U, int D) {
    return std::min<int64_t>(255, D * slot + 100 + 6 * U + K);
}

// Whether the U work units of an aligned group (iterations it0 .. it0+U-1,
// it0 % U == 0) read identical `in` values: their home coordinates do not
// depend on wu_x (a0 = a4 = 0) and either not on wu_y either (xy_reuse) or
// the group lies in one row of work units (nwx % U == 0, or one row).
// Only used by the register-blocked variants (LMT_MEASURE_REGBLOCK).
bool jit_share(const SynthArgs &A, int U, bool regblock) {
    if (!regblock || U <= 1 || A.a[0] != 0 || A.a[4] != 0) return false;
    return (A.a[1] == 0 && A.a[5] == 0) || A.nwy == 1 || A.nwx % U == 0;
}

void choose_jit(int K, const lmt_instance &p, const SynthArgs &A, int64_t maxt, int64_t ctas, int64_t warps,
                int64_t nit, int64_t sms, bool opt, int64_t stage_bytes, int64_t smem_cap, bool regblock, bool membound,
                int *U_out, int *D_out, int *S_out, int *minb_out) {
    auto sets = [&](int U) -> int64_t { return jit_share(A, U, regblock) ? 1 : U; };
    const int64_t nm = (int64_t)p.n * p.m;  // (i, j) steps per work unit: a deeper prefetch ring is dead weight
    const int dmax = (int)std::min<int64_t>(3, std::max<int64_t>(1, nm));
    int bu = 1, bd = dmax, bs = 1;
    if (minb_out) *minb_out = 1;
    for (int U : {16, 8, 4, 2, 1})
        if (U <= nit) { bu = U; break; }
    // optimized variant: U work units per thread and a ring of G group
    // stages, each holding the regions of one group of U iterations (one
    // region when the group's units share it) behind one mbarrier pair.
    auto rps = [&](int U) -> int64_t { return jit_share(A, U, regblock) ? 1 : U; };
    const auto ngroups = [&](int U) { return std::max<int64_t>(1, (nit + U - 1) / U); };
    if (opt && membound) {
        // HBM-bound launch with CTAs to spare: as many resident CTAs as the
        // warps and shared memory allow (launch bounds hold the registers to
        // it), U = 4 work units per group and 4 group stages in flight per
        // CTA. Measured on B200 over (U, stages, CTAs/SM) on the HBM legs
        // (tools/tune_hbm.py, profiles/r02_tune_hbm.json): within 2% of the
        // best shape on each. Stencils of several taps: launch bounds of 2
        // CTAs/SM instead (registers for the group body; residency then
        // follows shared memory), 4-10 % faster on the star legs
        // (tools/tune_hbm_deep.py, profiles/r02_tune_hbm_deep.json).
        bd = 1;
        bu = (int)std::min<int64_t>(4, std::max<int64_t>(1, nit));
        while (bu & (bu - 1)) bu &= bu - 1;
        while (bu > 1 && rps(bu) * stage_bytes > smem_cap) bu >>= 1;  // one group's regions must fit
        int64_t G = std::min<int64_t>(4, ngroups(bu));
        while (G > 1 && G * rps(bu) * stage_bytes > smem_cap) G--;
        // ... leaving at least 48 registers per thread (32 spill the U = 4 group body)
        const int64_t res = std::min<int64_t>({64 / std::max<int64_t>(1, warps), 32,
                                               (228 * 1024) / (G * rps(bu) * stage_bytes + 1024),
                                               std::max<int64_t>(1, ctas / std::max<int64_t>(1, sms)),
                                               65536 / (48 * 32 * std::max<int64_t>(1, warps))});
        if (minb_out) *minb_out = (int)std::max<int64_t>(1, K > 1 ? std::min<int64_t>(res, 2) : res);
        *U_out = bu;
        *D_out = bd;
        *S_out = (int)G;
        return;
    }
    if (!opt && membound) {
        // The baseline walks a thread's groups of U units as one stream of
        // (group, step) slots with a D-slot load ring across group
        // boundaries (lmt_jit.cuh). Stencils of several taps: 48 resident
        // warps per SM (launch bounds), U = 4, D = 3 -- within 1 % of the best
        // measured shape on the star legs (tools/tune_hbm_deep.py,
        // profiles/r02_tune_hbm_deep.json; 32 warps and U = 8: 3-6 % slower).
        // One tap: 32 warps, U = 8, D = 3 (within 4 % of the best,
        // tools/tune_hbm.py; the tuned 64-warp shape does not survive the
        // automatic spill step-down).
        bu = (int)std::min<int64_t>(K > 1 ? 4 : 8, std::max<int64_t>(1, nit));
        while (bu & (bu - 1)) bu &= bu - 1;
        *U_out = bu;
        *D_out = 3;
        *S_out = 1;
        return;
    }
    if (!opt) {
        // start where the register estimate fits (ptxas has the last word in
        // JitCache::resolve; a good start saves the compiles of the step-down)
        const int64_t regcap = std::min<int64_t>(255, 65536 / maxt);
        const int64_t ctx = p.num_coal_ilb + p.num_uncoal_ilb;
        auto est = [&](int U, int D) { return D * (sets(U) * K + ctx) + U + 16; };
        while (bu > 1 || bd > 1) {
            if (est(bu, bd) <= regcap) break;
            if (bd > 1) bd--;
            else { bu >>= 1; bd = 3; }
        }
        // Launches of many 1-2-warp CTAs: resident warps hide latency better
        // than a deep prefetch ring once fewer than 16 warps per SM would fit
        // (measured on B200, tools/tune_records.py, profiles/r02_tune_top.json:
        // a 131,072-CTA launch of 2-thread workgroups, D = 3 -> 1: 143 -> 119 ms).
        auto resident = [&](int U, int D) {
            // ptxas allocates ~1.45x the live-value estimate (address registers, temporaries)
            const int64_t regs = std::min<int64_t>(255, ((int64_t)(1.45 * est(U, D)) + 7) / 8 * 8);
            const int64_t ctas_sm = std::min<int64_t>({32, 64 / std::max<int64_t>(1, warps),
                                                       65536 / std::max<int64_t>(1, regs * 32 * warps)});
            return ctas_sm * warps;
        };
        if (warps <= 2 && ctas >= 2 * sms * (16 / warps))
            while (bd > 1 && resident(bu, bd) < 16) bd--;
        // single-warp CTAs with at least two waves of 4 per SM: no prefetch
        // ring at all (the 12 longest isolated launches of a bench batch,
        // tools/tune_records.py, profiles/r02_tune_iso.json: D = 1 at the
        // chosen U was never slower, and 6-20 % faster where D = 2-3 had been
        // chosen; whole bench: neutral to +0.4 %)
        if (warps == 1 && ctas >= 2 * sms * 4) bd = 1;
    } else {
        bd = std::min(2, dmax);  // shared-memory loads: one step of lookahead covers them
        bu = 1;  // when no shape fits (the region alone exceeds shared memory) the variant is infeasible
        bs = 1;
        double best = -1.0;
        for (int U : {8, 4, 2, 1}) {
            if (U > nit) continue;
            const int64_t slot = sets(U) * K + p.num_coal_ilb + p.num_uncoal_ilb;
            const int64_t regs = std::min<int64_t>(jit_regs_guess(K, slot, U, 2), 65536 / maxt);
            const int64_t rregs = (regs + 7) / 8 * 8;
            for (int Gx : {2, 1}) {
                const int64_t G = std::min<int64_t>(Gx, ngroups(U));
                const int64_t sbytes = G * rps(U) * stage_bytes;
                if (sbytes > smem_cap) continue;
                int64_t res = std::min<int64_t>(32, 64 / std::max<int64_t>(1, warps));
                res = std::min<int64_t>(res, 65536 / std::max<int64_t>(1, rregs * warps * 32));
                res = std::min<int64_t>(res, (228 * 1024) / (sbytes + 1024));
                res = std::max<int64_t>(res, 1);
                const int64_t act = std::min<int64_t>(res, (ctas + sms - 1) / sms);
                const double chains = std::min(64.0, (double)act * (double)warps * U / 4.0);
                // two stages: the next group's regions land while this one computes
                const bool overlap = G >= 2 || ngroups(U) == 1;
                // stagings in flight per SM (resident CTAs x stages): with one CTA and one
                // stage every group waits out its own TMA (measured, profiles/r02_tune_top.json:
                // an xy_reuse launch of 8-thread workgroups, U = 8 -> 2: 170 -> 88 ms)
                const double staging = (double)std::min<int64_t>(4, act * G);
                const double score = chains * 64.0 + staging * 8.0 + (overlap ? 16.0 : 0.0) + U * 2.0;
                if (score > best) { best = score; bu = U; bs = (int)G; }
            }
        }
    }
    // The steady-state loop is D unrolled steps of ~U * (K + comp + ctx)
    // instructions. Past the 32 KB instruction cache (~2,000 SASS
    // instructions) the loop runs up to 2x slower (measured on B200,
    // tools/gpu_icache.sh: a 2,600-instruction body vs 1,300), so D is capped.
    {
        const int64_t ctx = p.num_coal_ilb + p.num_uncoal_ilb;
        auto step_instr = [&](int U) {
            return 1.1 * U * (K + p.num_comp_ilb + ctx) + (jit_share(A, U, regblock) ? 0.0 : 0.8 * U * K) + ctx;
        };
        while (bd > 1 && bd * step_instr(bu) > kLoopInstrBudget) bd--;
    }
    if (opt) {
        bs = std::max(bs, 1);
        while (bs > 1 && (int64_t)bs * rps(bu) * stage_bytes > smem_cap) bs--;
    }
    *U_out = bu;
    *D_out = bd;
    *S_out = bs;
}

// Launch floor of one variant (sweep.floor_seconds): the per-thread chain,
// the per-SM issue of the CTAs' warps, and the algorithmic bytes at HBM
// speed -- used to order and place instances, never as a result.
double launch_floor_s(const lmt_instance &p, int K, int64_t ctas, int64_t warps, double bytes, int sms) {
    const double chain = (double)p.n * p.m * (K + p.num_comp_ilb + p.num_coal_ilb + p.num_uncoal_ilb) +
                         p.num_comp_ep + p.num_coal_ep + p.num_uncoal_ep;
    const double wus = (double)p.out_h * p.out_w / std::max<double>(1.0, (double)p.grid_x * p.grid_y);
    const double clk = 1.965e9;
    const double chain_s = wus * chain / clk;
    const double issue_s = std::ceil((double)ctas / sms) * warps * wus * chain / 4.0 / clk;
    return std::max({chain_s, issue_s, bytes / 6.5e12}) + 3e-6;
}

int make_plan(const lmt_instance &p, const lmt_device &d, int64_t in_pitch, int32_t flags, const DevCtx *ctx,
              Plan *pl, const int32_t *tune = nullptr) {
    std::vector<std::string> v = violations(p);
    if (!v.empty()) {
        std::string m;
        for (size_t i = 0; i < v.size(); i++) m += (i ? "; " : "") + v[i];
        return fail(LMT_ERR_INVALID_INSTANCE, "%s", m.c_str());
    }
    int rc = compute_geometry(p, d, &pl->g);
    if (rc) return rc;
    const lmt_geometry &g = pl->g;
    if (g.alloc_h * in_pitch >= (int64_t)1 << 31 || (int64_t)p.in_h * p.in_w >= (int64_t)1 << 31 ||
        (int64_t)p.out_h * p.out_w >= (int64_t)1 << 31)
        return fail(LMT_ERR_TOO_LARGE, "arrays exceed 2^31 elements");
    const bool regblock = (flags & LMT_MEASURE_REGBLOCK) != 0;
    const int K = stencil_offsets(p.stencil_shape, p.stencil_radius, nullptr, nullptr);
    SynthArgs &A = pl->A;
    memset(&A, 0, sizeof A);
    A.P = (int32_t)in_pitch;
    A.H2 = p.in_h;
    A.W2 = p.in_w;
    A.out_w = p.out_w;
    A.grid_x = p.grid_x;
    A.N = p.n;
    A.M = p.m;
    A.nwx = p.out_w / p.grid_x;
    A.nwy = p.out_h / p.grid_y;
    A.nwx_shift = -1;
    if (is_pow2(A.nwx))
        for (A.nwx_shift = 0; (1 << A.nwx_shift) < A.nwx; A.nwx_shift++) {}
    const int64_t nm = (int64_t)p.n * p.m;
    A.ep_row0 = (int32_t)(nm % p.in_h);
    A.ep_col0 = (int32_t)(nm % p.in_w);
    A.a[0] = g.org_row_wu_x; A.a[1] = g.org_row_wu_y; A.a[2] = g.row_i; A.a[3] = g.row_j;
    A.a[4] = g.org_col_wu_x; A.a[5] = g.org_col_wu_y; A.a[6] = g.col_i; A.a[7] = g.col_j;
    A.pad = g.pad;
    A.off_min_row = g.off_min_row;
    A.off_min_col = g.off_min_col;
    pl->block = dim3(p.wg_x, p.wg_y);
    pl->grid = dim3(p.grid_x / p.wg_x, p.grid_y / p.wg_y);
    pl->feasible = g.footprint_bytes <= d.lmem_capacity_bytes;

    // TMA staging geometry: only the `col_span` columns are read
    // (interp.py:94-97 bounds the reads by r_rows x r_cols_pad, and the
    // footprint bounding box guarantees < col_span).
    // +3 columns: the box x is aligned down to 16 bytes (see stage_region)
    const int64_t rows = g.r_rows, cols = g.r_cols + 3;
    int64_t bw, ncc;
    if (round_up(cols, 4) <= 256) {
        bw = round_up(cols, 4);
        if ((bw & 7) == 0 && bw + 4 <= 256) bw += 4;  // pitch = 4 * odd: column walks hit 8 banks, not 1
        ncc = 1;
        pl->wide = false;
    } else {
        bw = 256;
        ncc = (cols + 255) / 256;
        pl->wide = true;
    }
    const int64_t nrc = (rows + 255) / 256;
    // one row chunk: the box is exactly the region's rows (no rows fetched
    // that nobody reads); several: equal chunks whose stride stays 128-byte aligned
    const int64_t bh = nrc == 1 ? rows : round_up((rows + nrc - 1) / nrc, 8);
    A.bw = (int32_t)bw;
    A.bh = (int32_t)bh;
    A.nrc = (int32_t)nrc;
    A.ncc = (int32_t)ncc;
    const int64_t stage_tx = ncc * nrc * bh * bw;  // floats the TMA writes per region
    A.stage_floats = (int32_t)round_up(stage_tx, 32);  // slot stride: slots start on 128-byte boundaries
    A.stage_bytes = (uint32_t)(stage_tx * 4);
    const int64_t nit = (int64_t)A.nwx * A.nwy;
    const int64_t warps = ((int64_t)p.wg_x * p.wg_y + 31) / 32;
    const int64_t ctas = (int64_t)pl->grid.x * pl->grid.y;
    pl->ctas = ctas;
    const int64_t sms = ctx ? ctx->sms : 148;
    const int64_t smem_cap = ctx ? (int64_t)ctx->smem_optin - 1024 : 227 * 1024;
    const int64_t wgs = (int64_t)p.wg_x * p.wg_y;
    const int64_t maxt = wgs <= 256 ? 256 : (wgs <= 512 ? 512 : 1024);
    const bool ctxwrap = p.num_coal_ilb > kIn2HaloRows || p.num_coal_ep > kIn2HaloRows ||
                         p.num_uncoal_ilb > kIn2HaloCols || p.num_uncoal_ep > kIn2HaloCols;
    JitKey k0{p.stencil_shape, p.stencil_radius, p.num_comp_ilb, p.num_comp_ep, p.num_coal_ilb,
              p.num_coal_ep, p.num_uncoal_ilb, p.num_uncoal_ep, 1, 1, 0, 0, ctxwrap ? 1 : 0, (int)maxt,
              p.in_h, p.in_w, (int)in2_pitch(p.in_w), kPfDist, 0, 1, 0, (int64_t)p.n * p.m == 1 ? 1 : 0};

    pl->alg_bytes = 4.0 * (in_union(p) + in2_union(p) + (double)p.out_h * p.out_w);
    const double per_wu = (double)nm * (K + 2.0 * p.num_comp_ilb + p.num_coal_ilb + p.num_uncoal_ilb) +
                          2.0 * p.num_comp_ep + p.num_coal_ep + p.num_uncoal_ep;
    pl->alg_flops = per_wu * p.out_h * p.out_w;
    pl->est_s = launch_floor_s(p, K, ctas, warps, pl->alg_bytes, (int)sms);

    // 128-bit stencil-row loads (rows of >= 5 taps, radius >= 2) read three
    // shifted copies of `in` that the baseline builds inside its own timed
    // window (k_in_shift); used only where that copy is cheap next to the
    // launch (<= 2% of its floor, at the bandwidth share of its SMs).
    if (p.stencil_radius >= 2) {
        const double shift_bytes = 6.0 * 4.0 * (double)g.alloc_h * (double)in_pitch;  // 3 copies, read + write
        const double bw_share = 6.0e12 * std::min<double>(1.0, std::max<double>(8.0, (double)ctas) / (double)sms);
        k0.vec = shift_bytes / bw_share <= 0.02 * pl->est_s ? 1 : 0;
    }
    // Baseline launches with few work units per thread (U <= 2) and CTAs to
    // spare get their ILP from resident warps instead: launch bounds that
    // keep 32 warps per SM resident (8 per scheduler) cap the registers.
    // HBM-bound launches (the algorithmic bytes at HBM speed outlast the
    // per-SM issue floor) with at least two full waves of CTAs are latency
    // hidden by resident warps, not by work units in lockstep: a CTA loads,
    // computes and stores its units once, so several CTAs per SM are what
    // overlap one CTA's loads with another's stores.
    const double chain_ops = (double)nm * (K + p.num_comp_ilb + p.num_coal_ilb + p.num_uncoal_ilb) +
                             p.num_comp_ep + p.num_coal_ep + p.num_uncoal_ep;
    const double issue_s = std::ceil((double)ctas / sms) * warps * (double)nit * chain_ops / 4.0 / 1.965e9;
    const bool membound = pl->alg_bytes / 6.5e12 >= issue_s && ctas >= 2 * sms;
    int64_t maxt_b = maxt, minb = 1;
    if ((nit <= 2 || membound) && ctas >= 2 * sms) {
        // memory-bound: 48 resident warps per SM (32 for a one-tap stencil);
        // a compute chain with few
        // units per thread: 16 (forcing 32 spilled the U = 2 body to U = 1 on a
        // launch of 4-thread workgroups: 85 -> 69 ms at 16, profiles/r02_tune_tiny.json)
        const int64_t want = membound ? (K > 1 ? 48 : 32) : 16;
        minb = std::min<int64_t>({(want + warps - 1) / warps, 64 / std::max<int64_t>(1, warps), 32,
                                  ctas / std::max<int64_t>(1, sms)});
        if (minb > 1) maxt_b = warps * 32;
        else minb = 1;
    }
    int Ub, Db, Uo, Do, Sb, So, minb_o = 1;
    choose_jit(K, p, A, maxt_b * minb, ctas, warps, nit, sms, false, 0, smem_cap, regblock, membound, &Ub, &Db, &Sb,
               nullptr);
    choose_jit(K, p, A, maxt, ctas, warps, nit, sms, true, (int64_t)A.stage_floats * 4, smem_cap, regblock, membound, &Uo,
               &Do, &So, &minb_o);
    pl->kb = k0;
    pl->kb.maxt = (int)maxt_b;
    pl->kb.minb = (int)minb;
    pl->kb.U = Ub;
    pl->kb.D = Db;
    pl->kb.share = jit_share(A, Ub, regblock) ? 1 : 0;  // stays valid when the spill step-down halves U
    pl->ko = k0;
    pl->ko.vec = 0;
    pl->ko.U = Uo;
    pl->ko.D = Do;
    pl->ko.opt = 1;
    pl->ko.share = jit_share(A, Uo, regblock) ? 1 : 0;
    pl->ko.wide = pl->wide ? 1 : 0;
    if (tune) {  // explicit overrides (lmt_measure_opts.tune), for tuning studies
        if (tune[0] > 0) pl->kb.U = std::min<int>(tune[0], 16);
        if (tune[1] > 0) pl->kb.D = std::min(tune[1], 3);
        if (tune[2] > 0) { pl->kb.minb = tune[2]; pl->kb.maxt = (int)(warps * 32); }
        if (tune[3] > 0) pl->ko.U = std::min<int>(tune[3], 8);
        if (tune[4] > 0) So = std::min<int>(tune[4], kMaxStagesJ);
        if (tune[5] > 0) minb_o = tune[5];
        if (pl->kb.share && !jit_share(A, pl->kb.U, regblock)) pl->kb.share = 0;
        if (pl->ko.share && !jit_share(A, pl->ko.U, regblock)) pl->ko.share = 0;
        while (So > 1 && (int64_t)So * (pl->ko.share ? 1 : pl->ko.U) * A.stage_floats * 4 > smem_cap) So--;
    }
    if (minb_o > 1) {  // launch bounds that keep minb_o CTAs of this size resident
        pl->ko.minb = minb_o;
        pl->ko.maxt = (int)(warps * 32);
    }
    pl->in_copies = pl->kb.vec ? kInCopies : 1;
    A.nstages = (int32_t)So;  // group stages of the optimized variant's ring
    pl->dyn_smem = (size_t)So * (pl->ko.share ? 1 : pl->ko.U) * A.stage_floats * 4;
    if ((int64_t)A.stage_floats * 4 > smem_cap) pl->feasible = false;  // cannot stage even once on this device
    return LMT_OK;
}

int encode_tmap(CUtensorMap *map, const float *d_in, int64_t rows, int64_t cols, int64_t pitch, const Plan &pl) {
    if (((uintptr_t)d_in & 15) || (pitch & 3)) return fail(LMT_ERR_ARG, "in must be 16-byte aligned with pitch %% 4 == 0");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box[2] = {(cuuint32_t)pl.A.bw, (cuuint32_t)pl.A.bh};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(d_in), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LMT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) box %dx%d", (int)r, pl.A.bw, pl.A.bh);
    return LMT_OK;
}

// A variant ready to launch: the kernel resolved and loaded, its arguments
// (and, optimized, the TMA descriptor) built -- everything the host does
// before a launch, kept outside the timed window.
struct Ready {
    CUfunction f = nullptr;
    SynthArgs A;
    CUtensorMap map;
    size_t smem = 0;
    bool opt = false;
    JitKey got;
};

// d_in holds pl.in_copies shifted copies (copy stride in_rows * pitch)
// when the baseline reads 128-bit rows; d_in2x is in2 in the wrapped-halo
// layout (k_in2_halo), pitch in2_pitch(in_w).
int ready_variant(const Plan &pl, int variant, int device, CUcontext ctx, const float *d_in, int64_t in_rows,
                  int64_t in_cols, int64_t pitch, const float *d_in2x, float *d_out, Ready *r) {
    r->A = pl.A;
    r->A.in = d_in;
    r->A.in_copy = (variant == 0 && pl.in_copies > 1) ? in_rows * pitch : 0;
    r->A.in2 = d_in2x;
    r->A.P2 = (int32_t)in2_pitch(pl.A.W2);
    r->A.out = d_out;
    r->opt = variant == 1;
    std::string err;
    int rc = g_jit.get(device, variant == 0 ? pl.kb : pl.ko, &r->f, &r->got, &err);
    if (!rc) rc = g_jit.load_in(ctx, r->f, &err);  // no lazy load inside a timed window
    if (rc) return fail(LMT_ERR_CUDA, "%s", err.c_str());
    if (r->opt) {
        rc = encode_tmap(&r->map, d_in, in_rows, in_cols, pitch, pl);
        if (rc) return rc;
        r->smem = pl.dyn_smem;
    }
    return LMT_OK;
}

int launch_ready(Ready &r, const Plan &pl, cudaStream_t s) {
    std::string err;
    int rc;
    if (!r.opt) {
        void *args[] = {&r.A};
        rc = g_jit.launch(r.f, pl.grid, pl.block, 0, s, args, &err);
    } else {
        void *args[] = {&r.map, &r.A};
        rc = g_jit.launch(r.f, pl.grid, pl.block, r.smem, s, args, &err);
    }
    if (rc) return fail(LMT_ERR_CUDA, "%s", err.c_str());
    return LMT_OK;
}

int launch_in2_halo(float *buf, int64_t h, int64_t w, cudaStream_t s, int blocks_cap) {
    const int64_t total = (h + kIn2PhysHaloRows) * in2_pitch(w);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, blocks_cap));
    k_in2_halo<<<(unsigned)blocks, 256, 0, s>>>(buf, (int)h, (int)w, (int)in2_pitch(w));
    CUDA_TRY(cudaGetLastError());
    k_in2_shift<<<(unsigned)blocks, 256, 0, s>>>(buf, (int)h, (int)w, (int)in2_pitch(w),
                                                 (long long)in2_copy_elems(h, w));
    CUDA_TRY(cudaGetLastError());
    return LMT_OK;
}

int launch_fill(float *d, int64_t rows, int64_t cols, int64_t pitch, uint32_t salt, cudaStream_t s, int blocks_cap) {
    const int64_t vecs = rows * (pitch / 4);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((vecs + 255) / 256, blocks_cap));
    k_fill<<<(unsigned)blocks, 256, 0, s>>>(d, rows, cols, pitch, salt);
    CUDA_TRY(cudaGetLastError());
    return LMT_OK;
}

int launch_digest(const float *a, const float *b, int64_t count, unsigned long long *res, cudaStream_t s,
                  int blocks_cap) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, blocks_cap));
    k_digest<<<(unsigned)blocks, 256, 0, s>>>(a, b, count, res);
    CUDA_TRY(cudaGetLastError());
    return LMT_OK;
}

lmt_device dev_or_default(const lmt_device *d) { return d ? *d : kDefaultDevice; }

// ------------------------------------------------------ measurement engine

struct Batch {
    const lmt_instance *insts;
    int64_t n;
    lmt_device d;
    int32_t flags;
    int samples;
    const int64_t *sample_idx;
    float *sample_vals;
    const float *const *h_in;
    const int64_t *h_rows, *h_cols;
    const float *const *h_in2;
    float *const *h_ob, *const *h_oo;
    lmt_measurement *out;
    int32_t tune[6] = {0, 0, 0, 0, 0, 0};
    std::vector<Plan> plans;
    std::vector<char> ok, ran_base, ran_opt, filled;
    bool host() const { return h_in != nullptr; }
};

bool run_opt_of(const Batch &B, const Plan &pl, const DevCtx *c) {
    return !(B.flags & LMT_MEASURE_SKIP_OPT) &&
           (pl.feasible || ((B.flags & LMT_MEASURE_ALLOW_LARGE_LMEM) &&
                            (int64_t)pl.A.stage_bytes <= (int64_t)c->smem_optin - 1024));
}

// The lane's own `in` buffer: host mode holds the copied `in` (and its
// shifted copies); device mode only the baseline's shifted copies of the
// shared `in` (0 when the baseline reads the shared one directly).
size_t need_in_elems(const Batch &B, int64_t i, const Plan &pl) {
    const int64_t rows = B.host() ? B.h_rows[i] : pl.g.alloc_h;
    const int64_t cols = B.host() ? B.h_cols[i] : pl.g.alloc_w;
    if (!B.host() && pl.in_copies == 1) return 0;
    return (size_t)(rows * round_up(cols, 4)) * pl.in_copies + 64;
}

// Enqueue instance i on lane L: its inputs, both variants each bracketed by
// its own events (in alternating order), digest + comparison, sampled cells,
// and (host mode) the copies. Stream-ordered on L.s; never blocks unless a
// buffer has to grow.
int enqueue(DevCtx *c, Batch &B, Lane &L, int64_t i) {
    const lmt_instance &p = B.insts[i];
    const Plan &pl = B.plans[(size_t)i];
    lmt_measurement &m = B.out[i];
    cudaStream_t s = L.s;
    const bool whole = L.sms == 0;
    const int cap_blocks = (whole ? c->sms : L.sms) * 8;
    cudaEvent_t *ev = &c->events[(size_t)i * kEvPerInst];
    const int64_t rows = B.host() ? B.h_rows[i] : pl.g.alloc_h;
    const int64_t cols = B.host() ? B.h_cols[i] : pl.g.alloc_w;
    const int64_t pitch = round_up(cols, 4);
    const size_t need_in = need_in_elems(B, i, pl), need_out = (size_t)p.out_h * p.out_w;
    const bool ropt = run_opt_of(B, pl, c);
    // host buffers: copies on the lane's own copy streams, two buffer sets, so
    // the copies of the lane's neighbouring instances overlap its kernels
    const bool pipelined = B.host();
    const int b = pipelined ? (int)(L.seq++ & 1) : 0;
    int rc;
    if (pipelined && (rc = lane_streams(L))) return rc;
    // ---- buffers (growing one waits for everything in flight on the lane)
    if (need_in > L.in_cap[b] || need_out > L.out_cap[b] ||
        (B.host() && in2_phys_elems(p.in_h, p.in_w) > L.in2_cap[b])) {
        CUDA_TRY(cudaStreamSynchronize(s));
        if (L.h2d) {
            CUDA_TRY(cudaStreamSynchronize(L.h2d));
            CUDA_TRY(cudaStreamSynchronize(L.d2h));
        }
        if (need_in > L.in_cap[b]) {
            size_t fr = 0, tot = 0;
            CUDA_TRY(cudaMemGetInfo(&fr, &tot));
            if (need_in * 4 + ((size_t)256 << 20) > fr + L.in_cap[b] * 4)
                return fail(LMT_ERR_TOO_LARGE, "instance %lld: in needs %zu bytes", (long long)i, need_in * 4);
            if ((rc = ensure(&L.in[b], &L.in_cap[b], need_in))) return rc;
        }
        if (need_out > L.out_cap[b]) {
            size_t oc = L.out_cap[b];
            if ((rc = ensure(&L.ob[b], &oc, need_out))) return rc;
            oc = L.out_cap[b];
            if ((rc = ensure(&L.oo[b], &oc, need_out))) return rc;
            L.out_cap[b] = oc;
        }
        if (B.host() && (rc = ensure(&L.in2[b], &L.in2_cap[b], in2_phys_elems(p.in_h, p.in_w)))) return rc;
    }
    float *dob = L.ob[b], *doo = L.oo[b];
    // din: the `in` the optimized variant (and a scalar baseline) reads;
    // dcp: the baseline's 128-bit layout (4 shifted copies) when it uses one
    const float *din = nullptr, *din2 = nullptr;
    float *dcp = pl.in_copies > 1 ? L.in[b] : nullptr;
    // ---- inputs (make_inputs, interp.py:30-38)
    if (B.host()) {
        float *dst = L.in[b];
        cudaStream_t cs = pipelined ? L.h2d : s;
        if (pipelined) CUDA_TRY(cudaStreamWaitEvent(cs, L.consumed[b], 0));  // instance i - 2 done with slot b
        CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)pitch * 4, B.h_in[i], (size_t)cols * 4, (size_t)cols * 4,
                                   (size_t)rows, cudaMemcpyHostToDevice, cs));
        CUDA_TRY(cudaMemcpy2DAsync(L.in2[b], (size_t)in2_pitch(p.in_w) * 4, B.h_in2[i], (size_t)p.in_w * 4,
                                   (size_t)p.in_w * 4, (size_t)p.in_h, cudaMemcpyHostToDevice, cs));
        if (pipelined) {
            CUDA_TRY(cudaEventRecord(L.copied[b], cs));
            CUDA_TRY(cudaStreamWaitEvent(s, L.copied[b], 0));
        }
        CUDA_TRY(cudaEventRecord(ev[5], s));
        if ((rc = launch_in2_halo(L.in2[b], p.in_h, p.in_w, s, cap_blocks))) return rc;
        CUDA_TRY(cudaEventRecord(ev[6], s));
        m.launches += 2;
        B.filled[(size_t)i] = 1;
        if (pipelined) CUDA_TRY(cudaStreamWaitEvent(s, L.drained[b], 0));  // outs of i - 2 reached the host
        din = dst;
        din2 = L.in2[b];
    } else {  // the shared inputs, generated for the whole batch before it started
        din = c->ins.at(cols).p;
        din2 = c->in2s.at({p.in_h, p.in_w});
    }
    m.in_copies = pl.in_copies;
    // ---- both variants, resolved before any event is recorded
    Ready rb, ro;
    if ((rc = ready_variant(pl, 0, c->device, L.ctx, dcp ? dcp : din, rows, cols, pitch, din2, dob, &rb))) return rc;
    if (ropt && (rc = ready_variant(pl, 1, c->device, L.ctx, din, rows, cols, pitch, din2, doo, &ro))) return rc;
    m.kernel_id = jit_kid(rb.got, ropt ? ro.got : pl.ko);
    m.lane_sms = L.sms;
    m.order = (ropt && (i & 1)) ? 1 : 0;
    const bool flush = whole && !(B.flags & LMT_MEASURE_WARM_L2);
    // an idle lane would start timing before the host has enqueued the
    // kernel: give the GPU a short head start first
    if (!flush && L.inflight.empty() && !B.filled[(size_t)i]) {
        k_lead<<<1, 32, 0, s>>>(20000ll);
        CUDA_TRY(cudaGetLastError());
    }
    for (int k = 0; k < 2; k++) {
        const int variant = (k == 0) == (m.order == 0) ? 0 : 1;
        if (variant == 1 && !ropt) continue;
        if (flush) {
            c->scrub_tag += 1.0f;
            k_scrub<<<c->sms * 4, 256, 0, s>>>(c->scrub, c->scrub_n4, c->scrub_tag);
            CUDA_TRY(cudaGetLastError());
            m.launches += 1;
        }
        CUDA_TRY(cudaEventRecord(ev[variant * 2], s));
        if (variant == 0 && dcp) {  // the baseline's own layout, inside its window
            const int blocks = (int)std::max<int64_t>(
                1, std::min<int64_t>((rows * pitch * kInCopies + 255) / 256, (whole ? c->sms : L.sms) * 16));
            if (B.host()) {
                k_in_shift<<<blocks, 256, 0, s>>>(dcp, rows, pitch);
            } else {
                k_in_copy4<<<blocks, 256, 0, s>>>(din, dcp, rows, pitch);
            }
            CUDA_TRY(cudaGetLastError());
            m.launches += 1;
        }
        if ((rc = launch_ready(variant == 0 ? rb : ro, pl, s))) return rc;
        CUDA_TRY(cudaEventRecord(ev[variant * 2 + 1], s));
        m.launches += 1;
        (variant == 0 ? B.ran_base : B.ran_opt)[(size_t)i] = 1;
    }
    if (!ropt && !pl.feasible) m.status = LMT_ERR_INFEASIBLE;
    m.nstages = pl.A.nstages;
    if ((rc = launch_digest(dob, ropt ? doo : nullptr, (int64_t)need_out, c->dres + i * 3, s, cap_blocks))) return rc;
    m.launches += 1;
    if (B.samples > 0) {
        k_gather<<<1, 256, 0, s>>>(dob, ropt ? doo : nullptr, c->didx + i * B.samples, B.samples,
                                   c->dsamp + i * B.samples * 2);
        CUDA_TRY(cudaGetLastError());
        m.launches += 1;
    }
    if (B.host()) {
        cudaStream_t cs = s;
        if (pipelined) {
            CUDA_TRY(cudaEventRecord(L.consumed[b], s));
            CUDA_TRY(cudaStreamWaitEvent(L.d2h, L.consumed[b], 0));
            cs = L.d2h;
        }
        if (B.h_ob && B.h_ob[i]) CUDA_TRY(cudaMemcpyAsync(B.h_ob[i], dob, need_out * 4, cudaMemcpyDeviceToHost, cs));
        if (ropt && B.h_oo && B.h_oo[i])
            CUDA_TRY(cudaMemcpyAsync(B.h_oo[i], doo, need_out * 4, cudaMemcpyDeviceToHost, cs));
        if (pipelined) CUDA_TRY(cudaEventRecord(L.drained[b], cs));
    }
    CUDA_TRY(cudaEventRecord(ev[4], s));
    L.inflight.push_back(i);
    return LMT_OK;
}

// Device-generated inputs shared read-only by every lane (make_inputs,
// interp.py:30-38): in2 (salt 1) per shape in the kernels' wrapped-halo
// layout, and `in` (salt 0) per logical width with the most rows any
// instance needs -- hash(r * alloc_w + c) does not depend on the instance
// otherwise. Generated on the library stream before a batch's kernels;
// widths unused for the longest are evicted past kSharedInBudget.
constexpr size_t kSharedInBudget = (size_t)48 << 30;

int ensure_shared_in2(DevCtx *c, int64_t h, int64_t w) {
    if (c->in2s.count({h, w})) return LMT_OK;
    float *p = nullptr;
    size_t cap = 0;
    int rc;
    if ((rc = ensure(&p, &cap, in2_phys_elems(h, w)))) return rc;
    if ((rc = launch_fill(p, h, w, in2_pitch(w), 1, c->stream, c->sms * 8))) return rc;
    if ((rc = launch_in2_halo(p, h, w, c->stream, c->sms * 8))) return rc;
    c->in2s[{h, w}] = p;
    return LMT_OK;
}

int ensure_shared_ins(DevCtx *c, const std::map<int64_t, int64_t> &need) {
    c->batch_no++;
    for (auto &kv : need) {
        auto it = c->ins.find(kv.first);
        if (it != c->ins.end() && it->second.rows >= kv.second) { it->second.used = c->batch_no; continue; }
        const int64_t pitch = round_up(kv.first, 4);
        const size_t bytes = (size_t)kv.second * pitch * 4;
        CUDA_TRY(cudaDeviceSynchronize());  // no lane still reads what gets replaced or evicted
        if (it != c->ins.end()) {
            CUDA_TRY(cudaFree(it->second.p));
            c->ins_bytes -= (size_t)it->second.rows * it->second.pitch * 4;
            c->ins.erase(it);
        }
        while (c->ins_bytes + bytes > kSharedInBudget) {  // least recently used width not in this batch
            auto victim = c->ins.end();
            for (auto e = c->ins.begin(); e != c->ins.end(); ++e)
                if (!need.count(e->first) && (victim == c->ins.end() || e->second.used < victim->second.used))
                    victim = e;
            if (victim == c->ins.end()) break;
            CUDA_TRY(cudaFree(victim->second.p));
            c->ins_bytes -= (size_t)victim->second.rows * victim->second.pitch * 4;
            c->ins.erase(victim);
        }
        DevCtx::SharedIn e;
        e.rows = kv.second;
        e.pitch = pitch;
        e.used = c->batch_no;
        CUDA_TRY(cudaMalloc(&e.p, bytes + 256));
        int rc = launch_fill(e.p, e.rows, kv.first, pitch, 0, c->stream, c->sms * 16);
        if (rc) return rc;
        c->ins[kv.first] = e;
        c->ins_bytes += bytes;
    }
    return LMT_OK;
}

// Lane picks for the concurrent phase: the costliest pending instance that
// needs this lane's size (too wide for the next smaller lane), else the
// costliest that fits at all (list scheduling, longest first).
int64_t pick(std::vector<int64_t> &pending, const Batch &B, int lane_sms, int smaller_sms) {
    size_t best = pending.size();
    for (size_t k = 0; k < pending.size(); k++) {
        const int64_t ct = B.plans[(size_t)pending[k]].ctas;
        if (ct > lane_sms) continue;
        if (ct > smaller_sms) { best = k; break; }
        if (best == pending.size()) best = k;
    }
    if (best == pending.size()) return -1;
    const int64_t i = pending[best];
    pending.erase(pending.begin() + (long)best);
    return i;
}

int retire(DevCtx *c, Lane &L, bool wait) {
    while (!L.inflight.empty()) {
        cudaEvent_t done = c->events[(size_t)L.inflight.front() * kEvPerInst + 4];
        if (wait) {
            CUDA_TRY(cudaEventSynchronize(done));
        } else {
            cudaError_t q = cudaEventQuery(done);
            if (q == cudaErrorNotReady) break;
            if (q != cudaSuccess) return fail(LMT_ERR_CUDA, "instance failed: %s", cudaGetErrorString(q));
        }
        L.inflight.erase(L.inflight.begin());
    }
    return LMT_OK;
}

int measure_run(Batch &B);

// An aborted batch still leaves every record defined: the instances that
// did not run carry the error.
int measure_impl(Batch &B) {
    const int rc = measure_run(B);
    if (rc != LMT_OK && B.out)
        for (int64_t i = 0; i < B.n; i++)
            if (i >= (int64_t)B.ran_base.size() || !B.ran_base[(size_t)i])
                if (B.out[i].status == LMT_OK) B.out[i].status = rc;
    return rc;
}

int measure_run(Batch &B) {
    if (!B.insts || !B.out || B.n < 0) return fail(LMT_ERR_ARG, "bad measure arguments");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    const int64_t n = B.n;
    for (int64_t i = 0; i < n; i++) {  // every record defined, whatever happens later
        memset(&B.out[i], 0, sizeof(lmt_measurement));
        B.out[i].t_opt_ms = -1.0;
        B.out[i].mismatches = -1;
        B.out[i].status = LMT_ERR_CUDA;
    }
    B.plans.assign((size_t)n, Plan{});
    B.ok.assign((size_t)n, 0);
    B.ran_base.assign((size_t)n, 0);
    B.ran_opt.assign((size_t)n, 0);
    B.filled.assign((size_t)n, 0);
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    if ((rc = ensure(&c->dres, &c->dres_cap, nn * 3))) return rc;
    CUDA_TRY(cudaMemsetAsync(c->dres, 0, nn * 3 * sizeof(unsigned long long), c->stream));
    if (B.samples > 0) {
        if ((rc = ensure(&c->didx, &c->didx_cap, nn * B.samples))) return rc;
        if ((rc = ensure(&c->dsamp, &c->dsamp_cap, nn * B.samples * 2))) return rc;
    }
    while (c->events.size() < (size_t)n * kEvPerInst) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        c->events.push_back(e);
    }
    if (!(B.flags & LMT_MEASURE_WARM_L2) && !c->scrub) {
        size_t cap = 0;
        if ((rc = ensure(&c->scrub, &cap, (size_t)(kScrubBytes / 16)))) return rc;
        c->scrub_n4 = kScrubBytes / 16;
    }
    // ---- plans; the shared in2
    for (int64_t i = 0; i < n; i++) {
        const lmt_instance &p = B.insts[i];
        lmt_geometry g0;
        std::vector<std::string> v = violations(p);
        if (!v.empty()) {
            std::string msg;
            for (size_t k = 0; k < v.size(); k++) msg += (k ? "; " : "") + v[k];
            B.out[i].status = fail(LMT_ERR_INVALID_INSTANCE, "%s", msg.c_str());
            continue;
        }
        if ((rc = compute_geometry(p, B.d, &g0))) { B.out[i].status = rc; continue; }
        const int64_t cols = B.host() ? B.h_cols[i] : g0.alloc_w;
        Plan &pl = B.plans[(size_t)i];
        if ((rc = make_plan(p, B.d, round_up(cols, 4), B.flags, c, &pl, B.tune))) { B.out[i].status = rc; continue; }
        if (B.host() && (B.h_rows[i] < pl.g.alloc_h || B.h_cols[i] < pl.g.alloc_w)) {
            B.out[i].status = fail(LMT_ERR_ARG, "instance %lld: in too small", (long long)i);
            continue;
        }
        B.out[i].status = LMT_OK;
        B.out[i].alg_bytes = pl.alg_bytes;
        B.out[i].alg_flops = pl.alg_flops;
        B.out[i].ctas = (int32_t)pl.ctas;
        B.ok[(size_t)i] = 1;
        if (!B.host() && (rc = ensure_shared_in2(c, p.in_h, p.in_w))) return rc;
    }
    if (!B.host()) {  // the shared `in` of every width the batch reads
        std::map<int64_t, int64_t> need;
        for (int64_t i = 0; i < n; i++)
            if (B.ok[(size_t)i]) {
                const Plan &pl = B.plans[(size_t)i];
                int64_t &r = need[pl.g.alloc_w];
                r = std::max<int64_t>(r, pl.g.alloc_h);
            }
        if ((rc = ensure_shared_ins(c, need))) return rc;
    }
    CUDA_TRY(cudaEventRecord(c->inputs_ready, c->stream));
    if (B.samples > 0)
        CUDA_TRY(cudaMemcpyAsync(c->didx, B.sample_idx, (size_t)n * B.samples * 8, cudaMemcpyHostToDevice,
                                 c->stream));
    // ---- placement: partitions for launches that fit one, the whole device otherwise
    const bool conc = (B.flags & LMT_MEASURE_CONCURRENT) != 0;
    if (conc && (rc = ensure_parts(c))) return rc;
    const int max_part = (conc && !c->parts.empty()) ? c->parts.front().sms : 0;
    std::vector<int64_t> iso, pending;
    for (int64_t i = 0; i < n; i++) {
        if (!B.ok[(size_t)i]) continue;
        const Plan &pl = B.plans[(size_t)i];
        // a partition lane keeps its own `in`; bound that memory
        const bool fits = pl.ctas <= max_part && need_in_elems(B, i, pl) * 4 <= ((size_t)6 << 30);
        (fits ? pending : iso).push_back(i);
    }
    // every lane's buffers sized up front for the largest instance it can be
    // given: growing one inside the batch drains the lane and cudaFree /
    // cudaMalloc synchronise the whole device (a first host-buffer batch paid
    // that on every new largest instance). Skipped past 40 % of free memory
    // (the lanes then grow on demand as before).
    {
        struct Need {
            size_t in = 0, out = 0, in2 = 0;
        };
        auto need_of = [&](const std::vector<int64_t> &idx, int lane_sms) {
            Need nd;
            for (int64_t i : idx) {
                const Plan &pl = B.plans[(size_t)i];
                if (lane_sms > 0 && pl.ctas > lane_sms) continue;
                nd.in = std::max(nd.in, need_in_elems(B, i, pl));
                nd.out = std::max(nd.out, (size_t)B.insts[i].out_h * B.insts[i].out_w);
                if (B.host()) nd.in2 = std::max(nd.in2, in2_phys_elems(B.insts[i].in_h, B.insts[i].in_w));
            }
            return nd;
        };
        const int sets = B.host() ? 2 : 1;
        std::vector<std::pair<Lane *, Need>> plan_bufs;
        plan_bufs.push_back({&c->full, need_of(iso, 0)});
        for (Lane &P : c->parts) plan_bufs.push_back({&P, need_of(pending, P.sms)});
        size_t extra = 0;  // bytes beyond what the lanes hold now
        for (auto &pb : plan_bufs)
            for (int b = 0; b < sets; b++) {
                const Lane &L = *pb.first;
                const Need &nd = pb.second;
                if (nd.in > L.in_cap[b]) extra += nd.in * 4;
                if (nd.out > L.out_cap[b]) extra += nd.out * 8;
                if (nd.in2 > L.in2_cap[b]) extra += nd.in2 * 4;
            }
        size_t fr = 0, tot = 0;
        CUDA_TRY(cudaMemGetInfo(&fr, &tot));
        if (extra > 0 && extra < fr / 10 * 4) {
            CUDA_TRY(cudaDeviceSynchronize());
            for (auto &pb : plan_bufs)
                for (int b = 0; b < sets; b++) {
                    Lane &L = *pb.first;
                    const Need &nd = pb.second;
                    if (nd.in > L.in_cap[b] && (rc = ensure(&L.in[b], &L.in_cap[b], nd.in))) return rc;
                    if (nd.out > L.out_cap[b]) {
                        size_t oc = L.out_cap[b];
                        if ((rc = ensure(&L.ob[b], &oc, nd.out))) return rc;
                        oc = L.out_cap[b];
                        if ((rc = ensure(&L.oo[b], &oc, nd.out))) return rc;
                        L.out_cap[b] = oc;
                    }
                    if (nd.in2 > L.in2_cap[b] && (rc = ensure(&L.in2[b], &L.in2_cap[b], nd.in2))) return rc;
                }
        }
    }
    auto by_cost = [&](int64_t a, int64_t b) { return B.plans[(size_t)a].est_s > B.plans[(size_t)b].est_s; };
    std::stable_sort(pending.begin(), pending.end(), by_cost);
    auto mark_fail = [&](int64_t i, int code) { B.out[i].status = code; B.ok[(size_t)i] = 0; };
    // phase 1: whole-device instances, one at a time, L2 flushed per variant
    for (int64_t i : iso) {
        rc = enqueue(c, B, c->full, i);
        if (rc == LMT_ERR_CUDA) return rc;
        if (rc) mark_fail(i, rc);
        if ((rc = retire(c, c->full, false))) return rc;
    }
    if (!pending.empty()) {
        if ((rc = retire(c, c->full, true))) return rc;
        if (B.host() && c->full.d2h) CUDA_TRY(cudaStreamSynchronize(c->full.d2h));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    // phase 2: partitions, list-scheduled. A lane commits to its next
    // instance only when the previous one has finished: a lane that queues
    // two commits to work other lanes could have started sooner (simulated
    // on the bench sample with its measured times: 2 in flight 40.0 vs 1 in
    // flight 43.8 instances/s; measured 36.5 -> 40.1). With host buffers an
    // instance's copies then run just before its kernels (a few ms against
    // launches of ~100 ms).
    const size_t depth = 1;
    for (Lane &L : c->parts) CUDA_TRY(cudaStreamWaitEvent(L.s, c->inputs_ready, 0));
    while (!pending.empty()) {
        bool progressed = false;
        for (size_t l = c->parts.size(); l-- > 0;) {  // smallest lanes choose first
            Lane &L = c->parts[l];
            if ((rc = retire(c, L, false))) return rc;
            const int smaller = l + 1 < c->parts.size() ? c->parts[l + 1].sms : 0;
            while (L.inflight.size() < depth) {
                const int64_t i = pick(pending, B, L.sms, smaller);
                if (i < 0) break;
                rc = enqueue(c, B, L, i);
                if (rc == LMT_ERR_CUDA) return rc;
                if (rc) mark_fail(i, rc);
                progressed = true;
            }
        }
        if (!progressed) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    for (Lane &L : c->parts) {
        if ((rc = retire(c, L, true))) return rc;
        if (L.d2h) CUDA_TRY(cudaStreamSynchronize(L.d2h));
    }
    if ((rc = retire(c, c->full, true))) return rc;
    if (c->full.d2h) CUDA_TRY(cudaStreamSynchronize(c->full.d2h));
    // ---- results
    std::vector<unsigned long long> res(nn * 3);
    CUDA_TRY(cudaMemcpyAsync(res.data(), c->dres, res.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             c->stream));
    if (B.samples > 0)
        CUDA_TRY(cudaMemcpyAsync(B.sample_vals, c->dsamp, (size_t)n * B.samples * 2 * sizeof(float),
                                 cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < n; i++) {
        lmt_measurement &m = B.out[i];
        cudaEvent_t *ev = &c->events[(size_t)i * kEvPerInst];
        float ms = 0.0f;
        if (B.ran_base[(size_t)i]) {
            CUDA_TRY(cudaEventElapsedTime(&ms, ev[0], ev[1]));
            m.t_base_ms = ms;
            m.digest_base = res[(size_t)i * 3];
        }
        if (B.filled[(size_t)i]) {
            CUDA_TRY(cudaEventElapsedTime(&ms, ev[5], ev[6]));
            m.t_fill_ms = ms;
        }
        if (B.ran_opt[(size_t)i]) {
            CUDA_TRY(cudaEventElapsedTime(&ms, ev[2], ev[3]));
            m.t_opt_ms = ms;
            m.digest_opt = res[(size_t)i * 3 + 1];
            m.mismatches = (int64_t)res[(size_t)i * 3 + 2];
        }
    }
    return LMT_OK;
}

}  // namespace

// =================================================================== C ABI

extern "C" {

const char *lmt_version(void) { return LMT_VERSION; }
const char *lmt_last_error(void) { return g_err.c_str(); }

int lmt_validate(const lmt_instance *inst, char *msg, int64_t cap) {
    if (!inst) return -1;
    std::vector<std::string> v = violations(*inst);
    if (msg && cap > 0) {
        std::string m;
        for (size_t i = 0; i < v.size(); i++) m += (i ? "; " : "") + v[i];
        snprintf(msg, (size_t)cap, "%s", m.c_str());
    }
    return (int)v.size();
}

int lmt_emit_geometry(const lmt_instance *inst, const lmt_device *dev, lmt_geometry *out) {
    if (!inst || !out) return fail(LMT_ERR_ARG, "null argument");
    return compute_geometry(*inst, dev_or_default(dev), out);
}

int lmt_fill(float *d_dst, int64_t rows, int64_t cols, int64_t pitch, uint32_t salt, void *stream) {
    if (!d_dst || rows < 0 || cols < 0 || pitch < cols || (pitch & 3)) return fail(LMT_ERR_ARG, "bad fill arguments");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    return launch_fill(d_dst, rows, cols, pitch, salt, (cudaStream_t)stream, c->sms * 16);
}

int lmt_execute(const lmt_instance *inst, const lmt_device *dev, int variant, const float *d_in, int64_t in_rows,
                int64_t in_cols, int64_t in_pitch, const float *d_in2, float *d_out, void *stream) {
    if (!inst || !d_in || !d_in2 || !d_out) return fail(LMT_ERR_ARG, "null argument");
    if (variant != 0 && variant != 1) return fail(LMT_ERR_ARG, "variant must be 0 or 1");
    // the TMA descriptor needs 16-byte rows; rows must not overlap
    if (in_pitch < in_cols || in_pitch % 4 || reinterpret_cast<uintptr_t>(d_in) % 16)
        return fail(LMT_ERR_ARG, "in pitch must be >= in_cols and a multiple of 4 floats, the base 16-byte aligned");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    const lmt_device d = dev_or_default(dev);
    Plan pl;
    rc = make_plan(*inst, d, in_pitch, 0, c, &pl);
    if (rc) return rc;
    if (in_rows < pl.g.alloc_h || in_cols < pl.g.alloc_w)
        return fail(LMT_ERR_ARG, "in is %lldx%lld, instance needs %lldx%lld", (long long)in_rows, (long long)in_cols,
                    (long long)pl.g.alloc_h, (long long)pl.g.alloc_w);
    // interp.execute runs the optimized variant whatever its footprint; the
    // only hard limit here is that one staged region fits the SM's shared memory.
    if (variant == 1 && (int64_t)pl.A.stage_bytes > (int64_t)c->smem_optin - 1024)
        return fail(LMT_ERR_INFEASIBLE, "local-memory footprint %lld bytes exceeds capacity %d",
                    (long long)pl.g.footprint_bytes, (int)c->smem_optin - 1024);
    // the caller's `in` is read as is: the baseline uses scalar stencil loads here
    pl.kb.vec = 0;
    pl.in_copies = 1;
    // stage the caller's in2 into the wrapped-halo layout (stream-ordered scratch)
    cudaStream_t s = (cudaStream_t)stream;
    float *x = nullptr;
    CUDA_TRY(cudaMallocAsync(&x, in2_phys_elems(inst->in_h, inst->in_w) * sizeof(float), s));
    rc = LMT_OK;
    cudaError_t ce = cudaMemcpy2DAsync(x, (size_t)in2_pitch(inst->in_w) * 4, d_in2, (size_t)inst->in_w * 4,
                                       (size_t)inst->in_w * 4, (size_t)inst->in_h, cudaMemcpyDeviceToDevice, s);
    if (ce != cudaSuccess) rc = fail(LMT_ERR_CUDA, "in2 staging: %s", cudaGetErrorString(ce));
    if (rc == LMT_OK) rc = launch_in2_halo(x, inst->in_h, inst->in_w, s, c->sms * 8);
    Ready r;
    if (rc == LMT_OK) rc = ready_variant(pl, variant, c->device, nullptr, d_in, in_rows, in_cols, in_pitch, x, d_out, &r);
    if (rc == LMT_OK) rc = launch_ready(r, pl, s);
    ce = cudaFreeAsync(x, s);
    if (rc == LMT_OK && ce != cudaSuccess) rc = fail(LMT_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(ce));
    return rc;
}

int lmt_digest(const float *d, int64_t count, uint64_t *h_out, void *stream) {
    if (!d || !h_out || count < 0) return fail(LMT_ERR_ARG, "bad digest arguments");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *res = nullptr;
    CUDA_TRY(cudaMallocAsync(&res, 3 * sizeof(unsigned long long), s));
    unsigned long long h[3] = {0, 0, 0};
    cudaError_t e = cudaMemsetAsync(res, 0, 3 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) rc = launch_digest(d, nullptr, count, res, s, c->sms * 8);
    if (e == cudaSuccess && rc == LMT_OK) e = cudaMemcpyAsync(h, res, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(res, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(LMT_ERR_CUDA, "digest: %s", cudaGetErrorString(e));
    if (rc) return rc;
    *h_out = h[0];
    return LMT_OK;
}

int lmt_measure_batch_ex(const lmt_instance *insts, int64_t n, const lmt_device *dev, const lmt_measure_opts *opts,
                         const float *const *h_in, const int64_t *in_rows, const int64_t *in_cols,
                         const float *const *h_in2, float *const *h_out_base, float *const *h_out_opt,
                         lmt_measurement *out) {
    if (h_in && (!in_rows || !in_cols || !h_in2)) return fail(LMT_ERR_ARG, "host inputs need rows, cols and in2");
    if (opts && opts->samples > 0 && (!opts->sample_idx || !opts->h_sample_vals))
        return fail(LMT_ERR_ARG, "samples need sample_idx and h_sample_vals");
    if (opts && opts->samples > 0 && opts->sample_idx)
        for (int64_t i = 0; i < n; i++)
            for (int k = 0; k < opts->samples; k++) {
                const int64_t v = opts->sample_idx[i * opts->samples + k];
                if (v < 0 || v >= (int64_t)insts[i].out_h * insts[i].out_w)
                    return fail(LMT_ERR_ARG, "sample index %lld out of range for instance %lld", (long long)v,
                                (long long)i);
            }
    Batch B;
    B.insts = insts;
    B.n = n;
    B.d = dev_or_default(dev);
    B.flags = opts ? opts->flags : 0;
    B.samples = opts ? std::max(0, opts->samples) : 0;
    B.sample_idx = opts ? opts->sample_idx : nullptr;
    B.sample_vals = opts ? opts->h_sample_vals : nullptr;
    B.h_in = h_in;
    B.h_rows = in_rows;
    B.h_cols = in_cols;
    B.h_in2 = h_in2;
    B.h_ob = h_out_base;
    B.h_oo = h_out_opt;
    B.out = out;
    if (opts) memcpy(B.tune, opts->tune, sizeof B.tune);
    return measure_impl(B);
}

int lmt_measure_batch(const lmt_instance *insts, int64_t n, const lmt_device *dev, int32_t flags,
                      lmt_measurement *out) {
    lmt_measure_opts o{flags, 0, nullptr, nullptr, {0, 0, 0, 0, 0, 0}};
    return lmt_measure_batch_ex(insts, n, dev, &o, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, out);
}

int lmt_measure_batch_host(const lmt_instance *insts, int64_t n, const lmt_device *dev, int32_t flags,
                           const float *const *h_in, const int64_t *in_rows, const int64_t *in_cols,
                           const float *const *h_in2, float *const *h_out_base, float *const *h_out_opt,
                           lmt_measurement *out) {
    if (!h_in || !in_rows || !in_cols || !h_in2) return fail(LMT_ERR_ARG, "host inputs required");
    lmt_measure_opts o{flags, 0, nullptr, nullptr, {0, 0, 0, 0, 0, 0}};
    return lmt_measure_batch_ex(insts, n, dev, &o, h_in, in_rows, in_cols, h_in2, h_out_base, h_out_opt, out);
}

int lmt_partitions(int32_t *sizes, int32_t cap, int32_t *count) {
    if (!count) return fail(LMT_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    if ((rc = ensure_parts(c))) return rc;
    *count = (int32_t)c->parts.size();
    for (int32_t k = 0; sizes && k < cap && k < (int32_t)c->parts.size(); k++) sizes[k] = c->parts[(size_t)k].sms;
    return LMT_OK;
}

int lmt_prepare(const lmt_instance *insts, int64_t n, const lmt_device *dev, int32_t flags, int32_t nthreads,
                int64_t *kernels_out) {
    if ((!insts && n > 0) || n < 0) return fail(LMT_ERR_ARG, "bad prepare arguments");
    std::vector<JitKey> keys;
    int device = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        DevCtx *c;
        int rc = get_ctx(&c);
        if (rc) return rc;
        device = c->device;
        if ((flags & LMT_MEASURE_CONCURRENT) && (rc = ensure_parts(c))) return rc;
        const lmt_device d = dev_or_default(dev);
        size_t fr = 0, tot = 0;
        CUDA_TRY(cudaMemGetInfo(&fr, &tot));
        size_t max_in = 0, max_out = 0;
        for (int64_t i = 0; i < n; i++) {
            const lmt_instance &p = insts[i];
            if (!violations(p).empty()) continue;
            lmt_geometry g0;
            if (compute_geometry(p, d, &g0)) continue;
            Plan pl;
            if (make_plan(p, d, round_up(g0.alloc_w, 4), flags, c, &pl)) continue;
            // the whole-device lane's buffers (measure_impl's sizes): the
            // baseline's shifted copies, when it reads them
            const size_t need_in =
                pl.in_copies > 1 ? (size_t)(g0.alloc_h * round_up(g0.alloc_w, 4)) * pl.in_copies + 64 : 0;
            if (need_in * 4 + ((size_t)1 << 30) <= fr + c->full.in_cap[0] * 4) max_in = std::max(max_in, need_in);
            max_out = std::max(max_out, (size_t)p.out_h * p.out_w);
            if (!violations(p).empty() || !p.in_h) continue;
            if ((rc = ensure_shared_in2(c, p.in_h, p.in_w))) return rc;
            keys.push_back(pl.kb);
            const bool run_opt = !(flags & LMT_MEASURE_SKIP_OPT) &&
                                 (pl.feasible || ((flags & LMT_MEASURE_ALLOW_LARGE_LMEM) &&
                                                  (int64_t)pl.A.stage_bytes <= (int64_t)c->smem_optin - 1024));
            if (run_opt) keys.push_back(pl.ko);
        }
        // reserve them now: growing a buffer inside a timed batch means a
        // stream sync and a multi-GB cudaFree/cudaMalloc with the GPU idle
        Lane &L = c->full;
        if (max_in > L.in_cap[0]) {
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            if ((rc = ensure(&L.in[0], &L.in_cap[0], max_in))) return rc;
        }
        if (max_out > L.out_cap[0]) {
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            size_t oc = L.out_cap[0];
            if ((rc = ensure(&L.ob[0], &oc, max_out))) return rc;
            oc = L.out_cap[0];
            if ((rc = ensure(&L.oo[0], &oc, max_out))) return rc;
            L.out_cap[0] = oc;
        }
        for (Lane &P : c->parts) {  // partition lanes: outputs up front, inputs grow on demand
            if (max_out > P.out_cap[0]) {
                size_t oc = P.out_cap[0];
                if ((rc = ensure(&P.ob[0], &oc, max_out))) return rc;
                oc = P.out_cap[0];
                if ((rc = ensure(&P.oo[0], &oc, max_out))) return rc;
                P.out_cap[0] = oc;
            }
        }
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    std::string err;
    int nt = nthreads;
    if (nt <= 0) {  // all cores, shared among the processes of this node (one per GPU)
        const char *lw = getenv("LOCAL_WORLD_SIZE");
        const int procs = lw ? std::max(1, atoi(lw)) : 1;
        nt = std::max(1, (int)std::thread::hardware_concurrency() / procs);
    }
    int rc = g_jit.prepare(keys, nt, &err);
    if (rc) return fail(LMT_ERR_CUDA, "%s", err.c_str());
    std::vector<CUcontext> ctxs;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        ctxs.push_back(g_ctx[device].full.ctx);
        for (const Lane &P : g_ctx[device].parts) ctxs.push_back(P.ctx);
    }
    for (const JitKey &k : keys) {  // load the kernels into every context now, not inside a timed batch
        CUfunction f;
        rc = g_jit.get(device, k, &f, nullptr, &err);
        for (size_t q = 0; !rc && q < ctxs.size(); q++) rc = g_jit.load_in(ctxs[q], f, &err);
        if (rc) return fail(LMT_ERR_CUDA, "%s", err.c_str());
    }
    if (kernels_out) *kernels_out = (int64_t)keys.size();
    return LMT_OK;
}

int lmt_features(const lmt_instance *insts, int64_t n, const lmt_device *devs, int64_t ndev,
                 const double *coal_override, const int64_t *lmem_override, double *h_X, double *h_label,
                 double *h_times, int32_t *h_status) {
    if (n < 0 || (n > 0 && (!insts || !h_X || !h_label || !h_status)) || (ndev != 1 && ndev != n && devs))
        return fail(LMT_ERR_ARG, "bad features arguments");
    if (n == 0) return LMT_OK;
    static_assert(sizeof(lmt_instance) == sizeof(FeatInst), "lmt_instance layout");
    static_assert(sizeof(lmt_device) == sizeof(FeatDev), "lmt_device layout");
    DevCtx *c;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int rc = get_ctx(&c);
        if (rc) return rc;
    }
    const lmt_device dflt = kDefaultDevice;
    if (!devs) { devs = &dflt; ndev = 1; }
    int max_tx = 0, max_w = 0;
    for (int64_t k = 0; k < ndev; k++) {
        max_tx = std::max(max_tx, std::min(devs[k].transaction_bytes, kFeatMaxTx));
        max_w = std::max(max_w, devs[k].warp_size);
    }
    const int smem_longs = 3 * std::max(max_tx, 1) + (max_w > 32 ? std::min(max_w, 1024) : 0);
    const size_t smem = (size_t)smem_longs * 8 * 4;  // 4 warps per CTA
    if (smem > c->smem_optin - 1024) return fail(LMT_ERR_ARG, "device descriptor too large for K4");
    cudaStream_t s = c->stream;
    CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(k_features),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char *buf = nullptr;
    const size_t bi = (size_t)n * sizeof(lmt_instance), bd = (size_t)ndev * sizeof(lmt_device);
    const size_t bco = coal_override ? (size_t)n * 8 : 0, blo = lmem_override ? (size_t)n * 8 : 0;
    const size_t bx = (size_t)n * 18 * 8, bl = (size_t)n * 8, bt = h_times ? (size_t)n * 64 : 0, bs = (size_t)n * 4;
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t total = al(bi) + al(bd) + al(bco) + al(blo) + al(bx) + al(bl) + al(bt) + al(bs);
    CUDA_TRY(cudaMallocAsync(&buf, total, s));
    char *q = buf;
    auto take = [&](size_t b) { char *r = q; q += al(b); return r; };
    FeatInst *d_i = (FeatInst *)take(bi);
    FeatDev *d_d = (FeatDev *)take(bd);
    double *d_co = bco ? (double *)take(bco) : nullptr;
    long long *d_lo = blo ? (long long *)take(blo) : nullptr;
    double *d_x = (double *)take(bx), *d_l = (double *)take(bl);
    double *d_t = bt ? (double *)take(bt) : nullptr;
    int *d_s = (int *)take(bs);
    CUDA_TRY(cudaMemcpyAsync(d_i, insts, bi, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(d_d, devs, bd, cudaMemcpyHostToDevice, s));
    if (d_co) CUDA_TRY(cudaMemcpyAsync(d_co, coal_override, bco, cudaMemcpyHostToDevice, s));
    if (d_lo) CUDA_TRY(cudaMemcpyAsync(d_lo, lmem_override, blo, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(d_s, 0xff, bs, s));
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 3) / 4, (int64_t)c->sms * 16));
    k_features<<<(unsigned)blocks, 128, smem, s>>>(d_i, n, d_d, (int)ndev, d_co, d_lo, d_x, d_l, d_t, d_s,
                                                   smem_longs);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h_X, d_x, bx, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(h_label, d_l, bl, cudaMemcpyDeviceToHost, s));
    if (d_t) CUDA_TRY(cudaMemcpyAsync(h_times, d_t, bt, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(h_status, d_s, bs, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaFreeAsync(buf, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return LMT_OK;
}

// ------------------------------------------------------------ K5 real kernels

namespace {

const uint32_t kRealSalt[8] = {21, 22, 23, 24, 25, 26, 27, 28};  // A, B, conv in, y1, y2, x1_0, x2_0, w

std::string real_violations(const lmt_real_instance &r) {
    char b[256];
    const int64_t n = r.n, wx = r.wg_x, wy = r.wg_y, T = r.tile;
    if (n < 1) return "n < 1";
    if (wx < 1 || wy < 1 || wx * wy > 1024) { snprintf(b, sizeof b, "workgroup %lldx%lld", (long long)wx, (long long)wy); return b; }
    switch (r.kernel) {
        case 0:
            if (T > 64 || T % wx || (T / wx != 1 && T / wx != 2 && T / wx != 4) || T % wy || n % T)
                return "transpose needs tile <= 64, tile / wg_x in {1, 2, 4} (columns per thread), wg_y | tile, "
                       "tile | n";
            return "";
        case 1:
            if (T > 64 || T % wx || T % wy || n % T || T % 4 || n % 4)
                return "matrixMul needs tile <= 64, a multiple of 4 dividing n, wg_x | tile, wg_y | tile";
            if (T / wy != 1 && T / wy != 2 && T / wy != 4 && T / wy != 8) return "matrixMul rows per thread tile/wg_y must be 1, 2, 4 or 8";
            if (T / wx == 8 && T == 64 && wy == 8) return "";  // the 8 x 8 register tile
            if (T / wx != 1 && T / wx != 2 && T / wx != 4)
                return "matrixMul columns per thread tile/wg_x must be 1, 2 or 4 (8 with tile 64, wg 8 x 8)";
            return "";
        case 2:
            if (T < 1) return "convolution outputs per thread (tile) must be >= 1";
            if (n % (wx * T) || n % (wy * T)) return "convolution needs wg_x * tile | n and wg_y * tile | n";
            if (r.radius < 1 || r.radius > kConvMaxRadius) return "convolution radius must be in [1, 16]";
            return "";
        case 3:
            if (wy != 1 || n % wx || T < 1 || n % T) return "MVT needs wg_y == 1, wg_x | n, tile | n";
            if (wx % 32 || wx > 512 || (T != 16 && T != 32) || n % 256)
                return "MVT needs wg_x a multiple of 32 (<= 512), tile 16 or 32, n % 256 == 0";
            return "";
        default:
            return "unknown real kernel";
    }
}

double real_hash(uint64_t idx) {  // interp._hash_fill's value, on the host (exact double math)
    const uint32_t v = (uint32_t)(idx * 2654435761ull);
    return (double)(float)((double)v / 4294967296.0 - 0.5);
}

RealConv real_weights(int R) {
    RealConv c{};
    for (int k = 0; k <= 2 * R; k++) c.w[k] = (float)real_hash((uint64_t)k + kRealSalt[7]);
    return c;
}

// MVT: the side stream kernel 2 runs on (per device, created on first use;
// callers hold g_mu)
struct RealSide {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    int sms = 0;
};
RealSide g_real_side[64];

RealSide &real_side() {
    int dev = 0;
    cudaGetDevice(&dev);
    RealSide &sd = g_real_side[dev];
    if (!sd.s) {
        cudaStream_t st = nullptr;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming) != cudaSuccess ||
            cudaDeviceGetAttribute(&sd.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            return sd;
        sd.s = st;
    }
    return sd;
}

// tensor map of the n x n matrix A (fp32, row-major) with a box of bx columns x by rows
int mvt_tmap(RealTmap *t, const float *A, int n, int bx, int by) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult e = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(A), dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) return fail(LMT_ERR_CUDA, "MVT tensor map (%d)", (int)e);
    *t = *reinterpret_cast<const RealTmap *>(&m);
    return LMT_OK;
}

// MVT optimized variant: kernel 1 on s, kernel 2 on the side stream. When
// the two grids together exceed the SM count (32-row workgroups: 2 x 128
// CTAs), each kernel's ring is sized to half an SM's shared memory so one CTA
// of each can share an SM; otherwise each CTA has an SM to itself.
int mvt_opt_launch(const lmt_real_instance &r, const float *const *in, float *out, cudaStream_t s, const RealSide &sd,
                   int smem_optin) {
    const int n = r.n, wx = r.wg_x, T = r.tile;
    const dim3 grd(n / wx);
    const int64_t ybytes = (int64_t)n * 4;
    const bool share = 2 * (n / wx) > sd.sms;
    const int64_t budget = share ? 110 * 1024 : smem_optin - 2048;
    // kernel 1: ring kernel for workgroups of <= 128 rows (stages of 128 + 4 columns)
    const int64_t st1 = (int64_t)wx * (kMvtRingCols + 4) * 4;
    const int S1 = (int)std::min<int64_t>({(int64_t)kMvtMaxStages, (budget - 128 - ybytes) / st1, (int64_t)n / kMvtRingCols});
    const int64_t st2 = (int64_t)wx * kMvtRingRows * 4;
    const int S2 = (int)std::min<int64_t>({(int64_t)kMvtMaxStages, (budget - 128 - ybytes) / st2, (int64_t)n / kMvtRingRows});
    const bool ring1 = wx <= 128 && n % kMvtRingCols == 0 && S1 >= 2;
    const bool ring2 = (wx == 32 || wx == 64 || wx == 128) && n % kMvtRingRows == 0 && S2 >= 2;
    if (ring1) {
        RealTmap t1;
        if (int rc = mvt_tmap(&t1, in[0], n, kMvtRingCols + 4, wx)) return rc;
        const size_t sm = (size_t)S1 * st1 + 128 + ybytes;
        if (T == 32) k_mvt1_ring<32><<<grd, wx, sm, s>>>(t1, in[1], in[3], out, n, S1);
        else k_mvt1_ring<16><<<grd, wx, sm, s>>>(t1, in[1], in[3], out, n, S1);
    }
    if (ring2) {
        RealTmap t2;
        if (int rc = mvt_tmap(&t2, in[0], n, wx, kMvtRingRows)) return rc;
        const size_t sm = (size_t)S2 * st2 + 128 + ybytes;
#define LMT_MVT2(TT, W_) \
    if (T == TT && wx == W_) k_mvt2_ring<TT, W_><<<grd, wx, sm, sd.s>>>(t2, in[2], in[4], out + n, n, S2);
        LMT_MVT2(16, 32) LMT_MVT2(16, 64) LMT_MVT2(16, 128) LMT_MVT2(32, 32) LMT_MVT2(32, 64) LMT_MVT2(32, 128)
#undef LMT_MVT2
    }
    CUDA_TRY(cudaGetLastError());
    if (ring1 && ring2) return LMT_OK;
    // wide workgroups (few CTAs: each has an SM to itself): the general ring kernels
    // A streamed through a ring of S stages of [wg][T] (kernel 1) and [T][wg] (kernel 2)
    // tiles by TMA; y is staged whole in shared memory after each kernel's ring
    const int64_t stage = (int64_t)wx * T * 4, cap = smem_optin - 2048 - (int64_t)n * 4;
    const int S = (int)std::min<int64_t>({(int64_t)kMvtMaxStages, cap / stage, (int64_t)n / T});
    // kernel 1: stages of NB boxes of bwu + 4 columns (2 x 128 when two stages fit,
    // else one box, then narrower ones for wide workgroups)
    int bwu = kMvtBoxCols, NB = kMvtStageCols / kMvtBoxCols;
    auto st1f = [&]() { return (int64_t)wx * (bwu + 4) * 4 * NB; };
    while (st1f() * 2 > cap && (NB > 1 || bwu > 16)) {
        if (NB > 1) NB--;
        else bwu >>= 1;
    }
    const int64_t stage1 = st1f();
    const int S1w = (int)std::min<int64_t>({(int64_t)kMvtMaxStages, cap / stage1, (int64_t)n / (NB * bwu)});
    if (S < 1 || S1w < 1 || n % (NB * bwu))
        return fail(LMT_ERR_TOO_LARGE, "MVT needs n %% %d == 0 and %lld bytes of shared memory per stage", NB * bwu,
                    (long long)stage1);
    if (!ring1) {
        RealTmap t1;
        if (int rc = mvt_tmap(&t1, in[0], n, bwu + 4, std::min(wx, 256))) return rc;
        int bwl = 0;
        while ((1 << bwl) < bwu) bwl++;
        const size_t sm = (size_t)S1w * stage1 + 128 + ybytes;
        if (T == 32 && wx <= 256 && bwu >= 32)
            k_mvt1_tma<32><<<grd, wx, sm, s>>>(t1, in[1], in[3], out, n, S1w, bwl, NB);
        else
            k_mvt1_tma<16><<<grd, wx, sm, s>>>(t1, in[1], in[3], out, n, S1w, bwl, NB);
        CUDA_TRY(cudaGetLastError());
    }
    if (!ring2) {
        if (T == 32 && wx <= 256) {
            RealTmap t2;
            if (int rc = mvt_tmap(&t2, in[0], n, std::min(wx, 256), T)) return rc;
            k_mvt2_tma<32><<<grd, wx, (size_t)S * stage + 128 + ybytes, sd.s>>>(t2, in[2], in[4], out + n, n, S);
        } else {  // T = 16 stages (same results: T only sets the staging granularity)
            const int64_t stage16 = (int64_t)wx * 16 * 4;
            const int S16 = (int)std::min<int64_t>({(int64_t)kMvtMaxStages, cap / stage16, (int64_t)n / 16});
            RealTmap t2;
            if (int rc = mvt_tmap(&t2, in[0], n, std::min(wx, 256), 16)) return rc;
            k_mvt2_tma<16><<<grd, wx, (size_t)S16 * stage16 + 128 + ybytes, sd.s>>>(t2, in[2], in[4], out + n, n, S16);
        }
        CUDA_TRY(cudaGetLastError());
    }
    return LMT_OK;
}

// inputs: transpose {A}; matrixMul {A, B}; convolution {in} (+ scratch `tmp`
// of n*n floats); MVT {A, y1, y2, x1_0, x2_0}; out: n*n floats, MVT 2n (x1 then x2)
int real_launch(const lmt_real_instance &r, int variant, const float *const *in, float *out, float *tmp,
                cudaStream_t s, int smem_optin) {
    const int n = r.n, wx = r.wg_x, wy = r.wg_y, T = r.tile;
    const dim3 blk(wx, wy);
    switch (r.kernel) {
        case 0: {
            const dim3 grd(n / T, n / T);
            const int C = T / wx;
            const size_t sm = (size_t)T * (T + 1) * 4;
            if (variant == 0) {
                if (C == 1) k_transpose_base<1><<<grd, blk, 0, s>>>(in[0], out, n, T);
                else if (C == 2) k_transpose_base<2><<<grd, blk, 0, s>>>(in[0], out, n, T);
                else k_transpose_base<4><<<grd, blk, 0, s>>>(in[0], out, n, T);
            } else {
                if (C == 1) k_transpose_opt<1><<<grd, blk, sm, s>>>(in[0], out, n, T);
                else if (C == 2) k_transpose_opt<2><<<grd, blk, sm, s>>>(in[0], out, n, T);
                else k_transpose_opt<4><<<grd, blk, sm, s>>>(in[0], out, n, T);
            }
            break;
        }
        case 1: {
            const dim3 grd(n / T, n / T);
            const int W = T / wy, CC = T / wx;
            if (variant == 0) {
                if (CC == 1) k_matmul_base<1><<<grd, blk, 0, s>>>(in[0], in[1], out, n, T, W);
                else if (CC == 2) k_matmul_base<2><<<grd, blk, 0, s>>>(in[0], in[1], out, n, T, W);
                else if (CC == 4) k_matmul_base<4><<<grd, blk, 0, s>>>(in[0], in[1], out, n, T, W);
                else k_matmul_base<8><<<grd, blk, 0, s>>>(in[0], in[1], out, n, T, W);
                break;
            }
            if (T == 64 && W == 8 && CC == 8) {
                k_matmul_opt88<<<grd, blk, (size_t)4 * 64 * 68 * 4, s>>>(in[0], in[1], out, n);
                break;
            }
            // compile-time tile shapes (the instance set's T = 16, 32, 64): double-buffered
#define LMT_MMT(TT, WW, C_)                                                                                 \
    if (T == TT && W == WW && CC == C_) {                                                                   \
        k_matmul_opt_t<TT, WW, C_><<<grd, blk, (size_t)4 * TT * (TT + 4) * 4, s>>>(in[0], in[1], out, n); \
        break;                                                                                              \
    }
            LMT_MMT(16, 1, 1) LMT_MMT(16, 2, 1) LMT_MMT(16, 4, 1) LMT_MMT(16, 8, 1)
            LMT_MMT(32, 1, 1) LMT_MMT(32, 2, 1) LMT_MMT(32, 4, 1) LMT_MMT(32, 8, 1)
            LMT_MMT(32, 8, 2) LMT_MMT(32, 4, 4) LMT_MMT(32, 8, 4)
            LMT_MMT(64, 4, 4) LMT_MMT(64, 8, 4)
#undef LMT_MMT
            const size_t sm = (size_t)2 * T * (T + 4) * 4;
#define LMT_MM(WW, C_)                                                                    \
    if (W == WW && CC == C_) {                                                            \
        k_matmul_opt<WW, C_><<<grd, blk, sm, s>>>(in[0], in[1], out, n, T);              \
        break;                                                                            \
    }
            LMT_MM(1, 1) LMT_MM(2, 1) LMT_MM(4, 1) LMT_MM(8, 1)
            LMT_MM(1, 2) LMT_MM(2, 2) LMT_MM(4, 2) LMT_MM(8, 2)
            LMT_MM(1, 4) LMT_MM(2, 4) LMT_MM(4, 4) LMT_MM(8, 4)
#undef LMT_MM
            return fail(LMT_ERR_INVALID_INSTANCE, "matrixMul shape");
        }
        case 2: {
            const RealConv c = real_weights(r.radius);
            const int R = r.radius, W = T;
            const dim3 grr(n / (wx * W), n / wy), grc(n / wx, n / (wy * W));
            const size_t smr = (size_t)wy * (W * wx + 2 * ((R + 3) & ~3)) * 4, smc = (size_t)(W * wy + 2 * R) * wx * 4;
#define LMT_CONV(RR)                                                                     \
    if (variant == 0) {                                                                  \
        k_conv_rows_base<RR><<<grr, blk, 0, s>>>(in[0], tmp, n, R, W, c);                \
        k_conv_cols_base<RR><<<grc, blk, 0, s>>>(tmp, out, n, R, W, c);                  \
    } else {                                                                             \
        k_conv_rows_opt<RR><<<grr, blk, smr, s>>>(in[0], tmp, n, R, W, c);               \
        k_conv_cols_opt<RR><<<grc, blk, smc, s>>>(tmp, out, n, R, W, c);                 \
    }
            switch (R) {
                case 1: LMT_CONV(1) break;
                case 2: LMT_CONV(2) break;
                case 4: LMT_CONV(4) break;
                case 8: LMT_CONV(8) break;
                default: LMT_CONV(0) break;
            }
#undef LMT_CONV
            break;
        }
        case 3: {
            // kernel 1 (x1, row dots) and kernel 2 (x2, column dots) are independent
            // (Polybench launches them back to back): both variants run them
            // concurrently, kernel 2 on a side stream forked from and joined back
            // into `s`, so the events around a variant bracket both
            RealSide &sd = real_side();
            if (!sd.s) return fail(LMT_ERR_CUDA, "MVT side stream");
            CUDA_TRY(cudaEventRecord(sd.fork, s));
            CUDA_TRY(cudaStreamWaitEvent(sd.s, sd.fork, 0));
            const dim3 grd(n / wx);
            if (variant == 0) {
                k_mvt1_base<<<grd, wx, 0, s>>>(in[0], in[1], in[3], out, n);
                k_mvt2_base<<<grd, wx, 0, sd.s>>>(in[0], in[2], in[4], out + n, n);
            } else {
                const int rc = mvt_opt_launch(r, in, out, s, sd, smem_optin);
                if (rc) return rc;
            }
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaEventRecord(sd.join, sd.s));
            CUDA_TRY(cudaStreamWaitEvent(s, sd.join, 0));
            break;
        }
    }
    CUDA_TRY(cudaGetLastError());
    return LMT_OK;
}

void real_work(const lmt_real_instance &r, double *bytes, double *flops) {
    const double n = r.n;
    switch (r.kernel) {
        case 0: *bytes = 8.0 * n * n; *flops = 0.0; break;
        case 1: *bytes = 12.0 * n * n; *flops = 2.0 * n * n * n; break;
        case 2: *bytes = 16.0 * n * n; *flops = 4.0 * (2 * r.radius + 1) * n * n; break;
        default: *bytes = 8.0 * n * n + 24.0 * n; *flops = 4.0 * n * n; break;
    }
}

struct RealBufs {
    int64_t n = -1;
    float *in[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    float *tmp = nullptr, *ob = nullptr, *oo = nullptr;
    unsigned long long *dres = nullptr;
} g_real[64];

// L2 flush before a timed K5 variant (k_scrub writes a buffer larger than L2)
int real_scrub(DevCtx *c, cudaStream_t s) {
    if (!c->scrub) {
        size_t cap = 0;
        int rc = ensure(&c->scrub, &cap, (size_t)(kScrubBytes / 16));
        if (rc) return rc;
        c->scrub_n4 = kScrubBytes / 16;
    }
    c->scrub_tag += 1.0f;
    k_scrub<<<c->sms * 4, 256, 0, s>>>(c->scrub, c->scrub_n4, c->scrub_tag);
    CUDA_TRY(cudaGetLastError());
    return LMT_OK;
}

}  // namespace

int lmt_real_validate(const lmt_real_instance *inst, char *msg, int64_t cap) {
    if (!inst) return -1;
    const std::string v = real_violations(*inst);
    if (msg && cap > 0) snprintf(msg, (size_t)cap, "%s", v.c_str());
    return v.empty() ? 0 : 1;
}

int lmt_real_execute(const lmt_real_instance *inst, int variant, const float *const *d_inputs, float *d_out,
                     void *stream) {
    if (!inst || !d_inputs || !d_out || (variant != 0 && variant != 1)) return fail(LMT_ERR_ARG, "bad real arguments");
    const std::string v = real_violations(*inst);
    if (!v.empty()) return fail(LMT_ERR_INVALID_INSTANCE, "%s", v.c_str());
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    float *tmp = nullptr;
    if (inst->kernel == 2) CUDA_TRY(cudaMallocAsync(&tmp, (size_t)inst->n * inst->n * 4, s));
    rc = real_launch(*inst, variant, d_inputs, d_out, tmp, s, (int)c->smem_optin);
    if (tmp) CUDA_TRY(cudaFreeAsync(tmp, s));
    return rc;
}

int lmt_real_measure(const lmt_real_instance *insts, int64_t n, int32_t flags, lmt_measurement *out) {
    if ((!insts && n > 0) || !out || n < 0) return fail(LMT_ERR_ARG, "bad real measure arguments");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    RealBufs &B = g_real[c->device];
    cudaStream_t s = c->stream;
    std::vector<cudaEvent_t> ev((size_t)n * 4);
    for (auto &e : ev) CUDA_TRY(cudaEventCreate(&e));
    if (!B.dres) CUDA_TRY(cudaMalloc(&B.dres, 3 * sizeof(unsigned long long) * 4096));
    std::vector<char> ran((size_t)n, 0);
    std::vector<unsigned long long> res((size_t)n * 3, 0);
    for (int64_t i = 0; i < n; i++) {  // every record defined, whatever happens later
        memset(&out[i], 0, sizeof(lmt_measurement));
        out[i].t_opt_ms = -1.0;
        out[i].mismatches = -1;
        out[i].status = LMT_ERR_CUDA;
    }
    for (int64_t i = 0; i < n; i++) {
        lmt_measurement &m = out[i];
        m.status = LMT_OK;
        const lmt_real_instance &r = insts[i];
        const std::string v = real_violations(r);
        if (!v.empty()) { m.status = fail(LMT_ERR_INVALID_INSTANCE, "%s", v.c_str()); continue; }
        const int64_t N = r.n;
        if (B.n != N) {  // (re)generate the hashed inputs of this size
            CUDA_TRY(cudaStreamSynchronize(s));
            for (auto *p : {&B.in[0], &B.in[1], &B.in[2], &B.in[3], &B.in[4], &B.tmp, &B.ob, &B.oo})
                if (*p) { CUDA_TRY(cudaFree(*p)); *p = nullptr; }
            const size_t nn = (size_t)N * N;
            CUDA_TRY(cudaMalloc(&B.in[0], nn * 4));
            CUDA_TRY(cudaMalloc(&B.in[1], nn * 4));
            CUDA_TRY(cudaMalloc(&B.tmp, nn * 4));
            CUDA_TRY(cudaMalloc(&B.ob, nn * 4 + 8 * N));
            CUDA_TRY(cudaMalloc(&B.oo, nn * 4 + 8 * N));
            for (int k = 2; k < 5; k++) CUDA_TRY(cudaMalloc(&B.in[k], (size_t)N * 4 + 16));
            B.n = N;
        }
        // the inputs of this kernel (salts per array; the conv input shares the A buffer slot 0)
        const size_t nn = (size_t)N * N;
        if (r.kernel == 2) {
            rc = launch_fill(B.in[0], N, N, N, kRealSalt[2], s, c->sms * 16);
        } else {
            rc = launch_fill(B.in[0], N, N, N, kRealSalt[0], s, c->sms * 16);
            if (!rc && r.kernel == 1) rc = launch_fill(B.in[1], N, N, N, kRealSalt[1], s, c->sms * 16);
            if (!rc && r.kernel == 3) {
                for (int k = 0; k < 4 && !rc; k++)
                    rc = launch_fill(B.in[1 + k], 1, N, (N + 3) / 4 * 4, kRealSalt[3 + k], s, c->sms * 16);
            }
        }
        if (rc) return rc;
        const float *ins[5] = {B.in[0], B.in[1], B.in[2], B.in[3], B.in[4]};
        if (r.kernel == 3) { ins[1] = B.in[1]; ins[2] = B.in[2]; ins[3] = B.in[3]; ins[4] = B.in[4]; }
        real_work(r, &m.alg_bytes, &m.alg_flops);
        cudaEvent_t *e = &ev[(size_t)i * 4];
        // each variant starts from a cold L2 (the 192 MB scrub, outside its events)
        if ((rc = real_scrub(c, s))) return rc;
        CUDA_TRY(cudaEventRecord(e[0], s));
        rc = real_launch(r, 0, ins, B.ob, B.tmp, s, (int)c->smem_optin);
        if (rc) { m.status = rc; continue; }
        CUDA_TRY(cudaEventRecord(e[1], s));
        m.launches = r.kernel >= 2 ? 2 : 1;
        const bool run_opt = !(flags & LMT_MEASURE_SKIP_OPT);
        if (run_opt) {
            if ((rc = real_scrub(c, s))) return rc;
            CUDA_TRY(cudaEventRecord(e[2], s));
            rc = real_launch(r, 1, ins, B.oo, B.tmp, s, (int)c->smem_optin);
            if (rc) { m.status = rc; continue; }
            CUDA_TRY(cudaEventRecord(e[3], s));
            m.launches *= 2;
        }
        const int64_t count = r.kernel == 3 ? 2 * N : (int64_t)nn;
        const size_t slot = (size_t)(i % 4096) * 3;
        CUDA_TRY(cudaMemsetAsync(B.dres + slot, 0, 3 * sizeof(unsigned long long), s));
        rc = launch_digest(B.ob, run_opt ? B.oo : nullptr, count, B.dres + slot, s, c->sms * 8);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(&res[(size_t)i * 3], B.dres + slot, 3 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
        m.launches += 1;
        m.kernel_id = 50000 + r.kernel;
        ran[(size_t)i] = run_opt ? 2 : 1;
        if ((i + 1) % 4096 == 0) CUDA_TRY(cudaStreamSynchronize(s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; i++) {
        if (!ran[(size_t)i]) continue;
        lmt_measurement &m = out[i];
        cudaEvent_t *e = &ev[(size_t)i * 4];
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e[0], e[1]));
        m.t_base_ms = ms;
        m.digest_base = res[(size_t)i * 3];
        if (ran[(size_t)i] == 2) {
            CUDA_TRY(cudaEventElapsedTime(&ms, e[2], e[3]));
            m.t_opt_ms = ms;
            m.digest_opt = res[(size_t)i * 3 + 1];
            m.mismatches = (int64_t)res[(size_t)i * 3 + 2];
        }
    }
    for (auto &e : ev) cudaEventDestroy(e);
    return LMT_OK;
}

int lmt_rf_train_tree(const double *X, const double *y, int64_t nrows, int32_t nfeat, const int64_t *sample,
                      int64_t nsample, const int32_t *draws, int64_t ndraws, int32_t k, int32_t max_depth,
                      int32_t min_samples_leaf, int32_t *feature, double *threshold, int32_t *left, int32_t *right,
                      double *value, int64_t cap, int64_t *nodes_out, int64_t *draws_used) {
    if (!X || !y || !sample || nsample < 1 || nfeat < 1 || k < 1 || (!draws && ndraws > 0) || !nodes_out ||
        !draws_used)
        return fail(LMT_ERR_ARG, "bad train arguments");
    for (int64_t i = 0; i < nsample; i++)
        if (sample[i] < 0 || sample[i] >= nrows) return fail(LMT_ERR_ARG, "sample row out of range");
    TreeOut t;
    if (build_tree(X, y, nfeat, sample, nsample, draws, ndraws, k, max_depth, min_samples_leaf, &t)) {
        *draws_used = -1;
        return fail(LMT_ERR_TOO_LARGE, "tree needs more than %lld feature draws", (long long)ndraws);
    }
    const int64_t nn = (int64_t)t.feature.size();
    *nodes_out = nn;
    *draws_used = t.draws_used;
    if (nn > cap) return fail(LMT_ERR_TOO_LARGE, "tree has %lld nodes > capacity %lld", (long long)nn, (long long)cap);
    std::copy(t.feature.begin(), t.feature.end(), feature);
    std::copy(t.threshold.begin(), t.threshold.end(), threshold);
    std::copy(t.left.begin(), t.left.end(), left);
    std::copy(t.right.begin(), t.right.end(), right);
    std::copy(t.value.begin(), t.value.end(), value);
    return LMT_OK;
}

int lmt_rf_feature_draws(const uint64_t *state4, int32_t has_uint32, uint32_t uinteger, int32_t nfeat, int32_t k,
                         int64_t ndraws, int32_t *out) {
    if (!state4 || !out || nfeat < 1 || nfeat > 10000 || k < 1 || k > nfeat || k > 64 || ndraws < 0)
        return fail(LMT_ERR_ARG, "bad draw arguments");
    NpPcg64 g;
    g.state = ((unsigned __int128)state4[0] << 64) | state4[1];
    g.inc = ((unsigned __int128)state4[2] << 64) | state4[3];
    g.has32 = has_uint32 != 0;
    g.u32 = uinteger;
    for (int64_t i = 0; i < ndraws; i++) g.choice_sorted(nfeat, k, out + i * k);
    return LMT_OK;
}

int lmt_rf_train_gpu(const double *X, const double *y, int64_t nrows, int32_t nfeat, int32_t ntrees,
                     const int64_t *samples, const int32_t *draws, int64_t ndraws, int32_t k, int32_t max_depth,
                     int32_t min_samples_leaf, int32_t *feature, double *threshold, int32_t *left, int32_t *right,
                     double *value, int64_t cap, int64_t *nodes_out, int64_t *draws_used) {
    if (!X || !y || !samples || !draws || !nodes_out || !draws_used || nrows < 1 || nfeat < 1 || ntrees < 1 ||
        k < 1 || k > kRfMaxK || k > nfeat || ndraws < 1 || cap < 1 || min_samples_leaf < 1)
        return fail(LMT_ERR_ARG, "bad train arguments");
    if (nrows >= (1ll << 30) / (nfeat + 1)) return fail(LMT_ERR_TOO_LARGE, "training set too large");
    const int64_t n = nrows, T = ntrees;
    std::vector<int32_t> s32((size_t)(T * n));
    for (int64_t i = 0; i < T * n; i++) {
        if (samples[i] < 0 || samples[i] >= nrows) return fail(LMT_ERR_ARG, "sample row out of range");
        s32[(size_t)i] = (int32_t)samples[i];
    }
    for (int64_t i = 0; i < T * ndraws * k; i++)
        if (draws[i] < 0 || draws[i] >= nfeat) return fail(LMT_ERR_ARG, "feature draw out of range");
    DevCtx *c;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int rc = get_ctx(&c);
        if (rc) return rc;
    }
    cudaStream_t s = c->stream;
    int64_t N2 = 1;
    while (N2 < n) N2 <<= 1;
    // device buffers, released on every path
    std::vector<void *> bufs;
    struct Guard {
        std::vector<void *> *b;
        ~Guard() {
            for (void *p : *b) cudaFree(p);
        }
    } guard{&bufs};
    auto alloc = [&](void **p, size_t bytes) -> int {
        CUDA_TRY(cudaMalloc(p, std::max<size_t>(bytes, 16)));
        bufs.push_back(*p);
        return LMT_OK;
    };
    RfTrainArgs A{};
    double *dX, *dy, *keys;
    int32_t *dsamp, *ddraws, *pos;
    int rc = 0;
    if ((rc = alloc((void **)&dX, sizeof(double) * n * nfeat)) || (rc = alloc((void **)&dy, sizeof(double) * n)) ||
        (rc = alloc((void **)&dsamp, sizeof(int32_t) * T * n)) ||
        (rc = alloc((void **)&ddraws, sizeof(int32_t) * T * ndraws * k)) ||
        (rc = alloc((void **)&keys, sizeof(double) * T * nfeat * N2)) ||
        (rc = alloc((void **)&pos, sizeof(int32_t) * T * nfeat * N2)) ||
        (rc = alloc((void **)&A.sorted, sizeof(int32_t) * T * (nfeat + 1) * n)) ||
        (rc = alloc((void **)&A.tmp, sizeof(int32_t) * T * n)) || (rc = alloc((void **)&A.flag, T * n)) ||
        (rc = alloc((void **)&A.xs, sizeof(double) * T * k * n)) ||
        (rc = alloc((void **)&A.ys, sizeof(double) * T * k * n)) ||
        (rc = alloc((void **)&A.s1, sizeof(double) * T * k * n)) ||
        (rc = alloc((void **)&A.s2, sizeof(double) * T * k * n)) ||
        (rc = alloc((void **)&A.stack, sizeof(int32_t) * T * (n + 1) * 4)) ||
        (rc = alloc((void **)&A.feature, sizeof(int32_t) * T * cap)) ||
        (rc = alloc((void **)&A.left, sizeof(int32_t) * T * cap)) ||
        (rc = alloc((void **)&A.right, sizeof(int32_t) * T * cap)) ||
        (rc = alloc((void **)&A.threshold, sizeof(double) * T * cap)) ||
        (rc = alloc((void **)&A.value, sizeof(double) * T * cap)) ||
        (rc = alloc((void **)&A.nodes_out, sizeof(int64_t) * T)) ||
        (rc = alloc((void **)&A.draws_used, sizeof(int64_t) * T)))
        return rc;
    CUDA_TRY(cudaMemcpyAsync(dX, X, sizeof(double) * n * nfeat, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dsamp, s32.data(), sizeof(int32_t) * T * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ddraws, draws, sizeof(int32_t) * T * ndraws * k, cudaMemcpyHostToDevice, s));
    k_rf_presort<<<dim3((unsigned)nfeat + 1, (unsigned)T), kRfTrainThreads, 0, s>>>(dX, dsamp, (int)n, nfeat, (int)N2,
                                                                                  keys, pos, A.sorted);
    CUDA_TRY(cudaGetLastError());
    A.X = dX;
    A.y = dy;
    A.samples = dsamp;
    A.draws = ddraws;
    A.n = (int)n;
    A.nfeat = nfeat;
    A.k = k;
    A.ndraws = (int)ndraws;
    A.max_depth = max_depth;
    A.msl = min_samples_leaf;
    A.cap = cap;
    k_rf_build<<<(unsigned)T, kRfTrainThreads, 0, s>>>(A);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(nodes_out, A.nodes_out, sizeof(int64_t) * T, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(draws_used, A.draws_used, sizeof(int64_t) * T, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(feature, A.feature, sizeof(int32_t) * T * cap, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(threshold, A.threshold, sizeof(double) * T * cap, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(left, A.left, sizeof(int32_t) * T * cap, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(right, A.right, sizeof(int32_t) * T * cap, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(value, A.value, sizeof(double) * T * cap, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t t = 0; t < T; t++) {
        if (draws_used[t] == -1) return fail(LMT_ERR_TOO_LARGE, "tree %lld needs more than %lld feature draws",
                                             (long long)t, (long long)ndraws);
        if (draws_used[t] == -2) return fail(LMT_ERR_TOO_LARGE, "tree %lld exceeds %lld nodes", (long long)t,
                                             (long long)cap);
    }
    return LMT_OK;
}

int lmt_plan_info(const lmt_instance *inst, const lmt_device *dev, int32_t flags, int64_t *out16) {
    if (!inst || !out16) return fail(LMT_ERR_ARG, "bad plan_info arguments");
    if (!violations(*inst).empty()) return fail(LMT_ERR_INVALID_INSTANCE, "invalid instance");
    const lmt_device d = dev_or_default(dev);
    lmt_geometry g0;
    int rc = compute_geometry(*inst, d, &g0);
    if (rc) return rc;
    Plan pl;
    rc = make_plan(*inst, d, round_up(g0.alloc_w, 4), flags, nullptr, &pl);
    if (rc) return rc;
    const int64_t v[16] = {pl.kb.U, pl.kb.D, pl.kb.minb, pl.kb.maxt, pl.kb.vec, pl.ko.U, pl.ko.D, pl.ko.minb,
                           pl.ko.maxt, pl.A.nstages, (int64_t)pl.dyn_smem, (int64_t)pl.A.stage_bytes,
                           (int64_t)pl.A.stage_floats, pl.feasible ? 1 : 0, pl.ctas, pl.ko.share};
    memcpy(out16, v, sizeof v);
    return LMT_OK;
}

int lmt_kernel_source(const lmt_instance *inst, const lmt_device *dev, int variant, int32_t flags, char *buf,
                      int64_t cap, int64_t *len_out) {
    if (!inst || (variant != 0 && variant != 1)) return fail(LMT_ERR_ARG, "bad kernel_source arguments");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c = nullptr;
    lmt_geometry g0;
    const lmt_device d = dev_or_default(dev);
    int rc = compute_geometry(*inst, d, &g0);
    if (rc) return rc;
    Plan pl;
    if (!violations(*inst).empty()) {
        std::string m;
        for (auto &v : violations(*inst)) m += (m.empty() ? "" : "; ") + v;
        return fail(LMT_ERR_INVALID_INSTANCE, "%s", m.c_str());
    }
    rc = make_plan(*inst, d, round_up(g0.alloc_w, 4), flags, c, &pl);
    if (rc) return rc;
    const std::string src = (variant == 0 ? pl.kb : pl.ko).defines() + kLmtJitSource;
    if (len_out) *len_out = (int64_t)src.size();
    if (buf && cap > 0) snprintf(buf, (size_t)cap, "%s", src.c_str());
    return LMT_OK;
}

int lmt_jit_stats(int64_t *kernels_compiled, double *compile_seconds) {
    if (kernels_compiled) *kernels_compiled = g_jit.compiled();
    if (compile_seconds) *compile_seconds = g_jit.compile_seconds();
    return LMT_OK;
}

int lmt_get_stream(void **stream_out) {
    if (!stream_out) return fail(LMT_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    *stream_out = (void *)c->stream;
    return LMT_OK;
}

int lmt_current_device(int32_t *dev_out) {
    if (!dev_out) return fail(LMT_ERR_ARG, "null argument");
    int d = 0;
    CUDA_TRY(cudaGetDevice(&d));
    *dev_out = d;
    return LMT_OK;
}

int lmt_sync(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx *c;
    int rc = get_ctx(&c);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LMT_OK;
}

// ------------------------------------------------------------ forest

struct lmt_forest {
    int device = -1;
    int32_t ntrees = 0, nfeat = 0;
    RfNode *nodes = nullptr;
    int64_t *tree_off = nullptr;
    int32_t *cached_off = nullptr;
    int32_t ncached = 0;
};

int lmt_rf_create(const int32_t *feature, const double *threshold, const int32_t *left, const int32_t *right,
                  const double *value, const int64_t *tree_off, int32_t ntrees, int32_t nfeat, lmt_forest **out) {
    if (!feature || !threshold || !left || !right || !value || !tree_off || !out || ntrees < 1 || nfeat < 1)
        return fail(LMT_ERR_ARG, "bad forest arguments");
    // breadth-first renumbering per tree: the two children of a node become
    // adjacent (right = left + 1) and the top levels form a prefix
    std::vector<RfNode> flat;
    std::vector<int64_t> off((size_t)ntrees + 1, 0);
    std::vector<int32_t> coff((size_t)ntrees + 1, 0);
    for (int32_t t = 0; t < ntrees; t++) {
        const int64_t b = tree_off[t], e = tree_off[t + 1];
        const int64_t nn = e - b;
        if (nn < 1) return fail(LMT_ERR_ARG, "tree %d is empty", t);
        std::vector<int64_t> newid((size_t)nn, -1), order;
        order.reserve((size_t)nn);
        newid[0] = 0;
        order.push_back(0);
        int64_t next = 1;
        for (size_t q = 0; q < order.size(); q++) {
            const int64_t u = order[q];
            if (feature[b + u] < 0) continue;
            if (feature[b + u] >= nfeat) return fail(LMT_ERR_ARG, "tree %d node %lld: feature out of range", t, (long long)u);
            const int64_t l = left[b + u], r = right[b + u];
            if (l < 0 || l >= nn || r < 0 || r >= nn || newid[l] >= 0 || newid[r] >= 0 || l == r)
                return fail(LMT_ERR_ARG, "tree %d node %lld: bad children", t, (long long)u);
            newid[l] = next++;
            newid[r] = next++;
            order.push_back(l);
            order.push_back(r);
        }
        off[(size_t)t] = (int64_t)flat.size();
        std::vector<RfNode> tn(order.size());
        for (size_t q = 0; q < order.size(); q++) {
            const int64_t u = order[q];
            RfNode nd;
            if (feature[b + u] < 0) {
                nd.v = value[b + u];
                nd.feature = -1;
                nd.left = -1;
            } else {
                nd.v = threshold[b + u];
                nd.feature = feature[b + u];
                nd.left = (int32_t)newid[left[b + u]];
            }
            tn[(size_t)newid[u]] = nd;
        }
        flat.insert(flat.end(), tn.begin(), tn.end());
    }
    off[(size_t)ntrees] = (int64_t)flat.size();
    // shared-memory prefix per tree (top levels), kRfSmemNodes in total
    const int32_t per = kRfSmemNodes / ntrees;
    for (int32_t t = 0; t < ntrees; t++)
        coff[(size_t)t + 1] = coff[(size_t)t] + (int32_t)std::min<int64_t>(per, off[(size_t)t + 1] - off[(size_t)t]);
    lmt_forest *f = new lmt_forest();
    CUDA_TRY(cudaGetDevice(&f->device));
    f->ntrees = ntrees;
    f->nfeat = nfeat;
    f->ncached = coff[(size_t)ntrees];
    cudaError_t e1 = cudaMalloc(&f->nodes, flat.size() * sizeof(RfNode));
    cudaError_t e2 = cudaMalloc(&f->tree_off, off.size() * sizeof(int64_t));
    cudaError_t e3 = cudaMalloc(&f->cached_off, coff.size() * sizeof(int32_t));
    if (e1 || e2 || e3) { lmt_rf_destroy(f); return fail(LMT_ERR_CUDA, "forest allocation failed"); }
    CUDA_TRY(cudaMemcpy(f->nodes, flat.data(), flat.size() * sizeof(RfNode), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(f->tree_off, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(f->cached_off, coff.data(), coff.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    *out = f;
    return LMT_OK;
}

int lmt_rf_mean(const lmt_forest *f, const double *d_X, int64_t nrows, double *d_mean, int32_t *d_votes, void *stream) {
    if (!f || (!d_X && nrows > 0) || (!d_mean && nrows > 0) || nrows < 0) return fail(LMT_ERR_ARG, "bad rf arguments");
    if (nrows == 0) return LMT_OK;
    DevCtx *c;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int rc = get_ctx(&c);
        if (rc) return rc;
    }
    if (c->device != f->device)
        return fail(LMT_ERR_ARG, "forest was uploaded to device %d, current device is %d", f->device, c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t warps = (nrows + 0);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)c->sms * 8));
    const size_t smem = (size_t)f->ncached * sizeof(RfNode);
    k_rf_mean<<<(unsigned)blocks, 256, smem, s>>>(f->nodes, f->tree_off, f->cached_off, f->ntrees, d_X, nrows, f->nfeat,
                                                  d_mean, d_votes);
    CUDA_TRY(cudaGetLastError());
    return LMT_OK;
}

int lmt_rf_mean_host(const lmt_forest *f, const double *h_X, int64_t nrows, double *h_mean, int32_t *h_votes) {
    if (!f || nrows < 0 || (nrows > 0 && (!h_X || !h_mean))) return fail(LMT_ERR_ARG, "bad rf arguments");
    if (nrows == 0) return LMT_OK;
    DevCtx *c;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int rc = get_ctx(&c);
        if (rc) return rc;
    }
    cudaStream_t s = c->stream;
    double *dX = nullptr, *dm = nullptr;
    int32_t *dv = nullptr;
    // scratch is released on every path (stream-ordered)
    struct Scratch {
        cudaStream_t s;
        void *p[3];
        ~Scratch() {
            for (void *q : p)
                if (q) cudaFreeAsync(q, s);
        }
    } guard{s, {nullptr, nullptr, nullptr}};
    CUDA_TRY(cudaMallocAsync(&dX, (size_t)nrows * f->nfeat * sizeof(double), s));
    guard.p[0] = dX;
    CUDA_TRY(cudaMallocAsync(&dm, (size_t)nrows * sizeof(double), s));
    guard.p[1] = dm;
    if (h_votes) {
        CUDA_TRY(cudaMallocAsync(&dv, (size_t)nrows * sizeof(int32_t), s));
        guard.p[2] = dv;
    }
    CUDA_TRY(cudaMemcpyAsync(dX, h_X, (size_t)nrows * f->nfeat * sizeof(double), cudaMemcpyHostToDevice, s));
    int rc = lmt_rf_mean(f, dX, nrows, dm, dv, s);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(h_mean, dm, (size_t)nrows * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (h_votes) CUDA_TRY(cudaMemcpyAsync(h_votes, dv, (size_t)nrows * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return LMT_OK;
}

void lmt_rf_destroy(lmt_forest *f) {
    if (!f) return;
    if (f->nodes) cudaFree(f->nodes);
    if (f->tree_off) cudaFree(f->tree_off);
    if (f->cached_off) cudaFree(f->cached_off);
    delete f;
}

}  // extern "C"
