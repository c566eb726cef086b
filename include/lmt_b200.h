/*
 * lmt_b200.h -- C ABI of the B200-native lmtune hot path (liblmt_b200.so).
 *
 * The reference (lmtune, pure Python + numpy) has no FFI; its boundary is the
 * public Python API (/root/reference/pkg/src/lmtune/__init__.py:9-84). Each
 * entry point below replaces one reference function; the Python shim in
 * paper_1412_6986_b200/ binds them with ctypes behind the reference's own
 * signatures (INTEGRATION.md shows the binding a maintainer would add).
 *
 * Conventions
 *  - plain pointers and sizes; no torch types. "d_" pointers are device
 *    memory, "h_" pointers host memory. `stream` is a cudaStream_t taken as
 *    is (NULL = the legacy default stream, as in the CUDA runtime); the
 *    batch entry points (lmt_measure_batch*) run on the library's own
 *    stream, see lmt_get_stream().
 *  - every function returns LMT_OK (0) or an LMT_ERR_* code; the message of
 *    the last failure on the calling thread is in lmt_last_error().
 *    LMT_ERR_INVALID_INSTANCE maps to lmtune.errors.InvalidInstance
 *    (errors.py:10-15), LMT_ERR_INFEASIBLE to OptimizationInfeasible
 *    (errors.py:18-24), everything else to LmtuneError.
 *  - device memory for inputs/outputs inside lmt_measure_batch* is owned by
 *    the library (a per-device cache guarded by a mutex).
 */
#ifndef LMT_B200_H
#define LMT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMT_OK 0
#define LMT_ERR_INVALID_INSTANCE 1
#define LMT_ERR_INFEASIBLE 2
#define LMT_ERR_CUDA 3
#define LMT_ERR_ARG 4
#define LMT_ERR_TOO_LARGE 5

/* TemplateParams + LaunchConfig (kernel_model.py:54-90), flattened.
 * pattern: HomeAccessPattern declaration order (kernel_model.py:15-24):
 *   0 xy_reuse 1 x_reuse_row 2 x_reuse_col 3 y_reuse_row 4 y_reuse_col
 *   5 no_reuse_row_major 6 no_reuse_col_major
 * stencil_shape: StencilShape order (kernel_model.py:27-30): 0 rect 1 diamond 2 star */
typedef struct lmt_instance {
    int32_t in_h, in_w, out_h, out_w;
    int32_t pattern, n, m;
    int32_t stencil_shape, stencil_radius;
    int32_t num_comp_ilb, num_comp_ep;
    int32_t num_coal_ilb, num_coal_ep;
    int32_t num_uncoal_ilb, num_uncoal_ep;
    int32_t grid_x, grid_y, wg_x, wg_y;
} lmt_instance;

/* DeviceDescriptor (device.py:11-37); the defaults are DEFAULT_DEVICE. */
typedef struct lmt_device {
    int32_t transaction_bytes, warp_size, element_bytes, lmem_capacity_bytes;
    int32_t register_file_per_sm, max_regs_per_thread, max_warps_per_sm;
    int32_t max_workgroups_per_sm, dram_latency_cycles, issue_cycles_per_op;
} lmt_device;

/* EmitGeometry (codegen.py:69-91) + Footprint (access_analysis.py:158-166)
 * + the rest of AffineAccess (access_analysis.py:32-48). */
typedef struct lmt_geometry {
    int32_t pad, off_min_row, off_min_col;
    int32_t r_rows, r_cols, r_cols_pad;
    int32_t seg_elems, segs_per_row, num_segs, num_warps, lanes_per_warp;
    int64_t alloc_h, alloc_w;
    int32_t org_row_wu_x, org_row_wu_y, org_col_wu_x, org_col_wu_y;
    int32_t row_i, row_j, col_i, col_j;
    int64_t footprint_bytes;
    int32_t num_offsets;
} lmt_geometry;

/* One measured instance (the GPU counterpart of cost_model.label_speedup,
 * cost_model.py:144-158, which only *models* these times). */
typedef struct lmt_measurement {
    double t_base_ms;        /* CUDA-event time of the baseline kernel */
    double t_opt_ms;         /* optimized kernel; < 0 when not run (infeasible) */
    uint64_t digest_base;    /* order-independent digest of the baseline out */
    uint64_t digest_opt;     /* same for the optimized out (0 if not run) */
    int64_t mismatches;      /* elements whose bits differ base vs opt; -1 if not run */
    double alg_bytes;        /* algorithmic bytes per variant */
    double alg_flops;        /* algorithmic fp32 ops per variant (MAD = 2) */
    double t_fill_ms;        /* input generation (K0) time; 0 when inputs were reused */
    int32_t status;          /* LMT_OK, LMT_ERR_INFEASIBLE (opt skipped), or an error */
    int32_t kernel_id;       /* which specialised kernel ran (diagnostics) */
    int32_t launches;        /* kernels this instance launched (fill, K1, K2, digest) */
    int32_t nstages;         /* shared-memory stages the optimized variant used */
    int32_t lane_sms;        /* SMs of the partition it ran in; 0 = the whole device (isolated) */
    int32_t order;           /* 0: baseline timed first, 1: optimized timed first */
    int32_t in_copies;       /* 4: the baseline read 128-bit shifted copies of `in`; building them is
                                inside t_base_ms. 1: plain `in` */
    int32_t ctas;            /* CTAs (workgroups) per launch */
} lmt_measurement;

typedef struct lmt_forest lmt_forest;

/* flags for lmt_measure_batch*
 *
 * Measurement contract: each variant is timed alone on
 * its SMs with CUDA events on its launching stream; the variant order
 * alternates between instances (odd instances time the optimized variant
 * first). On the whole device the L2 is flushed before each variant (a
 * 192 MB scrub outside the events), so both variants start L2-cold. With
 * LMT_MEASURE_CONCURRENT, instances whose launch has at most as many CTAs as
 * the largest SM partition run inside disjoint SM partitions (green
 * contexts), several at once; a CTA still gets an SM of its own, as on the
 * whole device, and these long launches are not flushed (a flush would evict
 * the neighbouring partitions' working sets too). */
#define LMT_MEASURE_SKIP_OPT         0x1  /* run the baseline only */
#define LMT_MEASURE_ALLOW_LARGE_LMEM 0x4  /* run the optimized variant past the device lmem cap (B200 has 227 KB) */
#define LMT_MEASURE_CONCURRENT       0x8  /* few-CTA launches run concurrently in disjoint SM partitions */
#define LMT_MEASURE_REGBLOCK         0x10 /* register-blocked variants: the work units of a thread whose home
                                             coordinates coincide share their stencil loads (and, optimized,
                                             their staged region); default: every work unit issues its own
                                             loads, like the emitted kernel (codegen.py:268-283) */
#define LMT_MEASURE_WARM_L2          0x20 /* no L2 flush before the isolated variants */

/* Options of lmt_measure_batch_ex. */
typedef struct lmt_measure_opts {
    int32_t flags;
    int32_t samples;            /* output cells gathered per instance (0: none) */
    const int64_t *sample_idx;  /* [n][samples] linear indices into out (row * out_w + col) */
    float *h_sample_vals;       /* [n][samples][2]: baseline, optimized value (0 when not run) */
    /* Kernel-shape overrides for tuning studies, 0 = the library's choice:
     * baseline work units per thread, prefetch depth, min resident CTAs per
     * SM; optimized work units per thread, staging slots, min resident CTAs.
     * Outputs do not depend on them (every shape is bit-identical). */
    int32_t tune[6];
} lmt_measure_opts;

const char *lmt_version(void);
const char *lmt_last_error(void);

/* kernel_model.validate_instance (kernel_model.py:196-219). Returns the number
 * of violations; their messages, joined by "; " as InvalidInstance does
 * (errors.py:13-15), are written to msg (cap bytes, NUL-terminated). */
int lmt_validate(const lmt_instance *inst, char *msg, int64_t cap);

/* codegen.emit_geometry + access_analysis.footprint (codegen.py:94-132,
 * access_analysis.py:184-213). */
int lmt_emit_geometry(const lmt_instance *inst, const lmt_device *dev, lmt_geometry *out);

/* interp._hash_fill / make_inputs (interp.py:22-38) into device memory:
 * d_dst[r * pitch + c] = hash(r * cols + c + salt) for r < rows, c < cols. */
int lmt_fill(float *d_dst, int64_t rows, int64_t cols, int64_t pitch, uint32_t salt, void *stream);

/* interp.execute (interp.py:41-114) on the GPU. variant 0 = BASELINE
 * (plain global loads), 1 = OPTIMIZED (region staged in shared memory by
 * TMA). d_in is [in_rows, in_cols] with row pitch in_pitch floats (in_pitch
 * >= in_cols, a multiple of 4, 16-byte aligned base); d_in2 is [in_h, in_w];
 * d_out [out_h, out_w]. Asynchronous on `stream`; d_in is read as is (no
 * copy), in2 is staged into the kernels' wrapped-halo layout in stream-
 * ordered scratch. */
int lmt_execute(const lmt_instance *inst, const lmt_device *dev, int variant,
                const float *d_in, int64_t in_rows, int64_t in_cols, int64_t in_pitch,
                const float *d_in2, float *d_out, void *stream);

/* The measurement path: for each instance generate its inputs on the device,
 * run and time both variants with CUDA events, digest and compare the two
 * outputs. Blocks until the batch is done. out[i] is always written; a failing
 * instance gets a non-zero status (the batch continues, like build_dataset's
 * skip log, dataset.py:264-281). Returns LMT_OK unless the arguments or the
 * device are unusable. */
int lmt_measure_batch(const lmt_instance *insts, int64_t n, const lmt_device *dev,
                      int32_t flags, lmt_measurement *out);

/* Same, end to end from host buffers: instance i's `in` is h_in[i]
 * ([in_rows[i], in_cols[i]] contiguous, ideally pinned) and `in2` is h_in2[i];
 * both are copied to the device inside the timed batch, and both outputs are
 * copied back into h_out_base[i] / h_out_opt[i] (may be NULL to skip). */
int lmt_measure_batch_host(const lmt_instance *insts, int64_t n, const lmt_device *dev,
                           int32_t flags, const float *const *h_in, const int64_t *in_rows,
                           const int64_t *in_cols, const float *const *h_in2,
                           float *const *h_out_base, float *const *h_out_opt,
                           lmt_measurement *out);

/* Both of the above, plus sampled output cells for an independent check
 * (the CPU oracle) of every measured instance. h_in == NULL: device-generated
 * inputs (lmt_measure_batch); otherwise host buffers (lmt_measure_batch_host). */
int lmt_measure_batch_ex(const lmt_instance *insts, int64_t n, const lmt_device *dev,
                         const lmt_measure_opts *opts, const float *const *h_in, const int64_t *in_rows,
                         const int64_t *in_cols, const float *const *h_in2, float *const *h_out_base,
                         float *const *h_out_opt, lmt_measurement *out);

/* The SM partitions LMT_MEASURE_CONCURRENT runs in on the current device:
 * their sizes in SMs (largest first) into sizes[cap]; *count = partitions
 * (0 when the driver offers no green contexts: every instance then runs on
 * the whole device). */
int lmt_partitions(int32_t *sizes, int32_t cap, int32_t *count);

/* Order-independent 64-bit digest of an fp32 device array (the digest in
 * lmt_measurement). */
int lmt_digest(const float *d, int64_t count, uint64_t *h_out, void *stream);

/* Random-forest inference (forest.py:49-58, 208-219). Trees use the
 * reference's node arrays (tree-local child indices, feature -1 = leaf);
 * tree t owns nodes [tree_off[t], tree_off[t+1]). */
int lmt_rf_create(const int32_t *feature, const double *threshold, const int32_t *left,
                  const int32_t *right, const double *value, const int64_t *tree_off,
                  int32_t ntrees, int32_t nfeat, lmt_forest **out);
/* mean[r] = (sum over trees in tree order of leaf value) / T, bit-identical to
 * forest.predict's acc / len(trees); votes[r] = number of trees whose leaf is
 * > 0 (log2-speedup > 0), via warp ballot. d_votes may be NULL. */
int lmt_rf_mean(const lmt_forest *f, const double *d_X, int64_t nrows, double *d_mean,
                int32_t *d_votes, void *stream);
/* Host-buffer convenience: copies X in, means (and votes) out. */
int lmt_rf_mean_host(const lmt_forest *f, const double *h_X, int64_t nrows, double *h_mean,
                     int32_t *h_votes);
void lmt_rf_destroy(lmt_forest *f);

/* Compile (NVRTC, sm_100a) and load every specialised kernel a batch of
 * instances will launch, using up to nthreads host threads (<= 0: all
 * cores). The reference compiles each kernel instance from its emitted
 * source with the instance's #defines (codegen.py:150-182); this is that
 * step, done once per compile tuple and variant. Optional: the measure and
 * execute entry points compile on first use. *kernels_out = keys needed. */
int lmt_prepare(const lmt_instance *insts, int64_t n, const lmt_device *dev, int32_t flags,
                int32_t nthreads, int64_t *kernels_out);

/* K4: the feature vector and modelled label of n instances on the GPU
 * (access_analysis.extract_features, access_analysis.py:272-308, and
 * cost_model.label_speedup with the coalescing override build_dataset passes,
 * cost_model.py:94-158, dataset.py:264-271), bit-identical to the reference.
 * devs: ndev == 1 descriptor for all instances or ndev == n (NULL: defaults).
 * coal_override[i] (NaN = none) / lmem_override[i] (< 0 = none) may be NULL.
 * Outputs (host): X [n][18] in FEATURE_NAMES order, label [n] (0.0 when the
 * optimized variant is infeasible), times [n][8] = kernel_time of the
 * baseline then the optimized variant (compute_cycles, mem_transactions,
 * active_warps, total_cycles; NaN when infeasible; may be NULL), status [n]:
 * 0 ok, 1 invalid instance (X, label NaN), 2 infeasible, 5 unsupported device. */
int lmt_features(const lmt_instance *insts, int64_t n, const lmt_device *devs, int64_t ndev,
                 const double *coal_override, const int64_t *lmem_override, double *h_X,
                 double *h_label, double *h_times, int32_t *h_status);

/* K5: the real-world kernel set of the paper (BASELINE.json
 * configs[1]) in both variants. The reference has no implementation of it
 * (SPEC.md:15); semantics are defined in csrc/lmt_real.cuh and pinned by the
 * C oracle. kernel: 0 transpose, 1 matrixMul, 2 convolution-separable,
 * 3 MVT. tile: transpose / matrixMul tile (== wg_x; wg_y = tile / work per
 * thread), MVT j-tile, convolution outputs per thread; radius: convolution
 * radius (1..16). */
typedef struct lmt_real_instance {
    int32_t kernel, n, wg_x, wg_y, tile, radius;
} lmt_real_instance;

/* 0 when valid, else 1 with the reason in msg. */
int lmt_real_validate(const lmt_real_instance *inst, char *msg, int64_t cap);
/* One variant on caller buffers: inputs transpose {A}, matrixMul {A, B},
 * convolution {in}, MVT {A, y1, y2, x1_0, x2_0}; d_out n*n floats (MVT: 2n,
 * x1 then x2). Asynchronous on `stream` (MVT runs its kernel 2 on an
 * internal stream forked from and joined back into `stream`, so stream order
 * holds). Inputs 16-byte aligned (MVT's y1/y2 are copied to shared memory in
 * one bulk copy). */
int lmt_real_execute(const lmt_real_instance *inst, int variant, const float *const *d_inputs, float *d_out,
                     void *stream);
/* Hash-filled inputs, both variants timed with CUDA events, outputs digested
 * and compared bitwise on the device (same record as lmt_measure_batch). */
int lmt_real_measure(const lmt_real_instance *insts, int64_t n, int32_t flags, lmt_measurement *out);

/* Random-forest training, one tree (forest.py:72-163 _best_split /
 * _build_tree), on the host, bit-identical to the reference. The random
 * draws are numpy's, generated by the caller from the tree's PCG64 stream in
 * the reference's order: `sample` = the bootstrap rows (or 0..n-1), `draws`
 * = ndraws x k sorted feature subsets, one per split attempt in DFS order.
 * Outputs the node arrays (capacity `cap`, >= 2*nsample - 1 suffices).
 * LMT_ERR_TOO_LARGE with *draws_used = -1: call again with more draws. */
int lmt_rf_train_tree(const double *X, const double *y, int64_t nrows, int32_t nfeat, const int64_t *sample,
                      int64_t nsample, const int32_t *draws, int64_t ndraws, int32_t k, int32_t max_depth,
                      int32_t min_samples_leaf, int32_t *feature, double *threshold, int32_t *left,
                      int32_t *right, double *value, int64_t cap, int64_t *nodes_out, int64_t *draws_used);

/* The per-split feature subsets of forest._best_split (forest.py:77:
 * np.sort(rng.choice(nfeat, k, replace=False)), ndraws times) continued
 * from a numpy Generator(PCG64) state: state4 = {state >> 64, state & mask,
 * inc >> 64, inc & mask}, plus its buffered 32-bit half. Bit-identical to
 * numpy's draws (nfeat <= 10000: Floyd's algorithm path). out: [ndraws][k]. */
int lmt_rf_feature_draws(const uint64_t *state4, int32_t has_uint32, uint32_t uinteger, int32_t nfeat, int32_t k,
                         int64_t ndraws, int32_t *out);

/* forest.train's trees on the GPU (forest.py:117-163), all `ntrees` trees in
 * one call, bit-identical to lmt_rf_train_tree / the reference: samples =
 * [ntrees][nrows] bootstrap rows, draws = [ntrees][ndraws][k] sorted feature
 * subsets (numpy's draws, as for lmt_rf_train_tree). Outputs [ntrees][cap]
 * node arrays and the node count per tree. LMT_ERR_TOO_LARGE when a tree
 * needs more draws (draws_used[t] = -1) or more than `cap` nodes (-2). */
int lmt_rf_train_gpu(const double *X, const double *y, int64_t nrows, int32_t nfeat, int32_t ntrees,
                     const int64_t *samples, const int32_t *draws, int64_t ndraws, int32_t k, int32_t max_depth,
                     int32_t min_samples_leaf, int32_t *feature, double *threshold, int32_t *left,
                     int32_t *right, double *value, int64_t cap, int64_t *nodes_out, int64_t *draws_used);

/* The CUDA source the specialised kernel of (instance, variant) is compiled
 * from -- its #defines then the kernel text -- the counterpart of
 * codegen.emit_baseline / emit_optimized (codegen.py:336-354). flags: the
 * lmt_measure_batch flags that shape the kernel (LMT_MEASURE_REGBLOCK).
 * *len_out = bytes needed (without the NUL); buf may be NULL to query. */
int lmt_kernel_source(const lmt_instance *inst, const lmt_device *dev, int variant, int32_t flags, char *buf,
                      int64_t cap, int64_t *len_out);

/* The launch plan of an instance as the measurement engine would build it on
 * a 148-SM B200 (no GPU needed): out16 = baseline U, D, min CTAs/SM, max
 * threads, 128-bit shifted copies; optimized U, D, min CTAs/SM, max threads,
 * group stages, dynamic shared memory bytes, bytes per staged region, floats
 * per region slot, feasible, CTAs, shared-region groups. */
int lmt_plan_info(const lmt_instance *inst, const lmt_device *dev, int32_t flags, int64_t *out16);

/* Kernels compiled by NVRTC so far in this process (disk-cache hits are not
 * compiles) and the host seconds spent compiling. */
int lmt_jit_stats(int64_t *kernels_compiled, double *compile_seconds);

/* The current CUDA device of the calling thread (the device every other
 * entry point works on; a forest handle is bound to the device it was
 * created on and lmt_rf_mean rejects it on another). */
int lmt_current_device(int32_t *dev_out);

/* Synchronise the library stream of the current device. */
int lmt_sync(void);

/* The library's stream on the current device (where lmt_measure_batch*
 * launch), so callers can bracket a batch with their own CUDA events. */
int lmt_get_stream(void **stream_out);

#ifdef __cplusplus
}
#endif
#endif
