/*
 * lmt_oracle.h -- CPU ORACLE for the lmtune hot path. TEST INFRASTRUCTURE ONLY.
 *
 * This is a plain-C restatement of the reference's CPU semantics, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg as the *checker*. Nothing in paper_1412_6986_b200/ links,
 * loads or calls it; the product path is the CUDA library only.
 *
 * Parity pinning: the restatement is checked against golden vectors that
 * tests/golden/make_golden.py generates by importing the reference package
 * (/root/reference/pkg/src/lmtune) in the build container, and against the
 * reference's own KATs (test_interp.py:32-58, test_codegen.py:112-127,
 * test_access_analysis.py:151-190, test_forest.py:81-104).
 *
 * Every function cites the reference file:line it follows.
 */
#ifndef LMT_ORACLE_H
#define LMT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors TemplateParams + LaunchConfig (kernel_model.py:54-90).
 * pattern: HomeAccessPattern declaration order (kernel_model.py:15-24)
 *   0 xy_reuse, 1 x_reuse_row, 2 x_reuse_col, 3 y_reuse_row, 4 y_reuse_col,
 *   5 no_reuse_row_major, 6 no_reuse_col_major
 * stencil_shape: StencilShape declaration order (kernel_model.py:27-30)
 *   0 rect, 1 diamond, 2 star */
typedef struct ora_instance {
    int32_t in_h, in_w, out_h, out_w;
    int32_t pattern, n, m;
    int32_t stencil_shape, stencil_radius;
    int32_t num_comp_ilb, num_comp_ep;
    int32_t num_coal_ilb, num_coal_ep;
    int32_t num_uncoal_ilb, num_uncoal_ep;
    int32_t grid_x, grid_y, wg_x, wg_y;
} ora_instance;

/* DeviceDescriptor (device.py:11-37). */
typedef struct ora_device {
    int32_t transaction_bytes, warp_size, element_bytes, lmem_capacity_bytes;
    int32_t register_file_per_sm, max_regs_per_thread, max_warps_per_sm;
    int32_t max_workgroups_per_sm, dram_latency_cycles, issue_cycles_per_op;
} ora_device;

/* EmitGeometry (codegen.py:69-91) + Footprint (access_analysis.py:158-166). */
typedef struct ora_geometry {
    int32_t pad, off_min_row, off_min_col;
    int32_t r_rows, r_cols, r_cols_pad;
    int32_t seg_elems, segs_per_row, num_segs, num_warps, lanes_per_warp;
    int64_t alloc_h, alloc_w;
    int32_t org_row_wu_x, org_row_wu_y, org_col_wu_x, org_col_wu_y;
    int32_t row_i, row_j, col_i, col_j;   /* rest of pattern_affine */
    int64_t footprint_bytes;
    int32_t num_offsets;
} ora_geometry;

#define ORA_OK 0
#define ORA_ERR_INVALID 1
#define ORA_ERR_INFEASIBLE 2
#define ORA_ERR_BOUNDS 3
#define ORA_ERR_ARG 4

int ora_validate(const ora_instance *inst);
int ora_geometry_of(const ora_instance *inst, const ora_device *dev, ora_geometry *g);
int ora_stencil_offsets(int shape, int radius, int32_t *dr, int32_t *dc, int cap);
void ora_hash_fill(float *dst, int64_t count, uint32_t salt);
int ora_execute(const ora_instance *inst, const ora_device *dev, int variant,
                const float *in, int64_t in_rows, int64_t in_cols,
                const float *in2, float *out, int nthreads,
                int64_t wg_begin, int64_t wg_end);
int ora_execute_prefix(const ora_instance *p, const ora_device *dev, int variant, const float *in, int64_t in_rows,
                       int64_t in_cols, const float *in2, float *out, int nthreads, int64_t wg_begin, int64_t wg_end,
                       int64_t units_per_wg);
uint64_t ora_out_hash(const float *out, int64_t count);
int64_t ora_execute_sample(const ora_instance *p, const ora_device *dev, int variant, const float *in,
                           int64_t in_rows, int64_t in_cols, const float *in2, float *out, int64_t max_units);
/* interp.execute's value at out[idx[k] / out_w][idx[k] % out_w] for each k,
 * with make_inputs' hash evaluated on the fly (see lmt_oracle.c). */
int ora_eval_units(const ora_instance *p, const ora_device *dev, int variant, const int64_t *idx, int64_t count,
                   float *vals, int nthreads);
int ora_forest_mean(const int32_t *feature, const double *threshold,
                    const int32_t *left, const int32_t *right, const double *value,
                    const int64_t *tree_off, int32_t ntrees,
                    const double *X, int64_t nrows, int32_t nfeat, double *mean_out,
                    int nthreads);

/* K5 real-kernel set (paper Table 3; semantics of csrc/lmt_real.cuh, which the
 * reference does not implement: parity is pinned by this restatement, not by
 * reference outputs). Accumulation order k / j / tap ascending with fmaf. */
void ora_real_transpose(const float *A, float *B, int64_t n);
void ora_real_matmul(const float *A, const float *B, float *C, int64_t n, int nthreads);
void ora_real_conv(const float *in, float *tmp, float *out, int64_t n, int radius, const float *w);
void ora_real_mvt(const float *A, const float *y1, const float *y2, const float *x1_0, const float *x2_0,
                  float *x1, float *x2, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
