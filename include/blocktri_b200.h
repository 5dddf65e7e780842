/*
 * blocktri_b200.h -- C ABI of the B200-native block-tridiagonal SPD factor/solve engine.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2509.03015, package
 * `blocktri`).  The reference boundary is Python-level; each entry point below replaces one
 * reference interface:
 *
 *   btd_plan_separators  <- plan_partition            /root/reference/pkg/src/blocktri/schur.py:75-95
 *   btd_create           <- RecursionConfig + the level loop / _should_recurse
 *                                                      schur.py:43-64, 289-326
 *   btd_factorize        <- recursive_factorize        schur.py:289-318  (with _factorize_level 329-343,
 *                           permute_split 98-138, factorize_btd_batch block_cholesky.py:60-68,
 *                           _coupling_panels 141-153, compute_schur 156-193, serial_factorize
 *                           block_cholesky.py:87-92)
 *   btd_solve            <- recursive_solve            schur.py:346-374  (split_rhs 196-211,
 *                           compute_separator_rhs 230-260, update_boundary 263-286,
 *                           solve_btd_batch block_cholesky.py:71-84, assemble_solution 214-227,
 *                           serial_solve block_cholesky.py:95-98)
 *   btd_status           <- NotPositiveDefinite / LevelOverflow / DimensionMismatch
 *                                                      errors.py:10-90
 *
 * Conventions (identical to the reference containers, core.py:23-71):
 *   diag : N blocks of n x n, float64, row-major, contiguous           (N, n, n)
 *   sub  : N-1 blocks, sub[i] = A_{i+1,i}                               (N-1, n, n)
 *   rhs/x: N panels of n x d, row-major                                 (N, n, d)
 * All data pointers are DEVICE pointers.  Every launch goes on the caller's CUDA stream
 * (`stream` is a cudaStream_t; NULL = legacy default stream).  The input matrix and rhs are never
 * written.  Device memory is caller-provided: query the sizes, allocate, pass the pointers.
 */
#ifndef BLOCKTRI_B200_H
#define BLOCKTRI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define BTD_OK 0
#define BTD_ERR_NOT_POSITIVE_DEFINITE 1 /* reference NotPositiveDefinite(pivot, level, member, block) */
#define BTD_ERR_LEVEL_OVERFLOW 2        /* reference LevelOverflow */
#define BTD_ERR_DIMENSION_MISMATCH 3    /* reference DimensionMismatch */
#define BTD_ERR_INVALID_ARGUMENT 4      /* reference ValueError (config / plan preconditions) */
#define BTD_ERR_UNSUPPORTED 5           /* block size outside the compiled kernel set */
#define BTD_ERR_CUDA 6                  /* CUDA runtime error (message carries cudaGetErrorString) */
#define BTD_ERR_NOT_FACTORED 7          /* reference ValueError("batch must be factorized ...") */
#define BTD_ERR_SINGULAR_DIAGONAL 8     /* reference SingularDiagonal(row, member) (errors.py:71-78) */

/* RecursionConfig (schur.py:43-64). All knobs must be >= 1. */
typedef struct btd_config {
  int64_t crossover;      /* default 64 */
  int64_t segment_length; /* rho, default 8 */
  int64_t max_levels;     /* default 32 */
  int32_t auto_crossover; /* default 0 */
  int32_t reserved;
} btd_config;

/* Failure coordinates (errors.py:31-68). Coordinates that do not apply are -1. */
typedef struct btd_status {
  int32_t code;
  int32_t pivot; /* 1-based pivot row inside the failing block */
  int64_t level; /* recursion level (level-local coordinates, like the reference) */
  int64_t member;
  int64_t block;
  char message[256];
} btd_status;

typedef struct btd_hierarchy btd_hierarchy; /* opaque: plan + device pointers of the factor */

const char* btd_version(void);
void btd_default_config(btd_config* cfg);

/* One level of the partition plan, bit-exact with plan_partition (schur.py:75-95).
 * separators_out may be NULL (count query). Requires num_blocks >= 3. */
int btd_plan_separators(int64_t num_blocks, const btd_config* cfg, int64_t* separators_out,
                        int64_t* count_out, btd_status* st);

/* Plan the whole recursion for (N, n, cfg).  Fails with BTD_ERR_UNSUPPORTED when no kernel
 * covers block size n. Host-only; no device work. */
int btd_create(int64_t num_blocks, int64_t block_size, const btd_config* cfg, btd_hierarchy** out,
               btd_status* st);
void btd_destroy(btd_hierarchy* h);

/* Recursion shape: levels that recurse, and the base (serial) block count.
 * `overflow` = 1 when the plan would exceed max_levels (factorize then reports LevelOverflow). */
int btd_num_levels(const btd_hierarchy* h, int64_t* num_levels, int64_t* base_blocks, int32_t* overflow);
/* Level introspection: block count and separators of level `level` (separators_out may be NULL). */
int btd_level_info(const btd_hierarchy* h, int64_t level, int64_t* num_blocks, int64_t* num_separators,
                   int64_t* separators_out);

/* Device memory: `persistent` holds the factor (kept for solves); `scratch` only lives during
 * btd_factorize. Both 256-byte aligned. */
int btd_factor_workspace(const btd_hierarchy* h, size_t* persistent_bytes, size_t* scratch_bytes);

/* Factor. diag/sub: device pointers (read-only). With check != 0 the call synchronizes the stream
 * once at the end and reports NotPositiveDefinite / LevelOverflow in `st`; with check == 0 it is
 * fully asynchronous and btd_check() reports later. */
int btd_factorize(btd_hierarchy* h, const double* diag, const double* sub, void* persistent, void* scratch,
                  void* stream, int32_t check, btd_status* st);
int btd_check(btd_hierarchy* h, void* stream, btd_status* st);

/* Solve A X = B against a factored hierarchy. rhs (read-only) and x: device (N, n, d). The
 * hierarchy is not modified, so concurrent solves on distinct buffers/streams are safe. */
int btd_solve_workspace(const btd_hierarchy* h, int64_t num_columns, size_t* scratch_bytes);
int btd_solve(const btd_hierarchy* h, const double* rhs, double* x, int64_t num_columns, void* scratch,
              void* stream, btd_status* st);

/* Debug/introspection: copy level `level`'s factor blocks (Linv of every row and L_sub / coupling
 * copies) into caller device buffers of N_l*n*n and (N_l-1)*n*n doubles.  level == num_levels
 * addresses the base. */
int btd_level_factor(const btd_hierarchy* h, int64_t level, double* linv_out, double* lsub_out,
                     void* stream, btd_status* st);

/* Debug/introspection: the next-level (Schur complement) system produced by level `level`
 * (compute_schur + new_btd, schur.py:156-193, core.py:205-211): P_l diagonal blocks (symmetric,
 * mirrored from the lower triangle the kernels form) and P_l - 1 sub blocks, copied into caller
 * device buffers.  `scratch` must be the factor scratch of the last btd_factorize on `h`, still
 * unmodified (the Schur systems live there only until it is reused). */
int btd_level_schur(const btd_hierarchy* h, int64_t level, const void* scratch, double* diag_out, double* sub_out,
                    void* stream, btd_status* st);

/* ---- Sharded (multi-GPU) building blocks, SURVEY.md §8e ----
 * The global chain is cut at level-L separators into contiguous chunks [a_g, b_g] (shared boundary
 * separators b_g = a_{g+1}); chunk g factors exactly `local_levels` levels of its own plan (which
 * equals the global plan restricted to the chunk), never its two boundary separators.  The
 * reduced system over the chunk's remaining separators (partial Schur diagonal at the two
 * boundaries) is exported; the caller sums the boundary partials of neighbouring chunks (NCCL),
 * factors the reduced global system with btd_factorize, and solves it between btd_solve_down
 * (exports the chunk's reduced rhs partial) and btd_solve_up (imports the reduced solution).
 * The boundary diagonal block / rhs panel must be given by exactly one side (the other passes 0). */
int btd_create_partial(int64_t num_blocks, int64_t block_size, const btd_config* cfg, int64_t local_levels,
                       btd_hierarchy** out, btd_status* st);
int btd_reduced_size(const btd_hierarchy* h, int64_t* num_blocks);
int btd_factorize_partial(btd_hierarchy* h, const double* diag, const double* sub, void* persistent, void* scratch,
                          double* reduced_diag, double* reduced_sub, void* stream, int32_t check, btd_status* st);
/* scratch (btd_solve_workspace) must be the same buffer for the down and up halves */
int btd_solve_down(const btd_hierarchy* h, const double* rhs, double* x, int64_t num_columns, void* scratch,
                   double* reduced_rhs_out, void* stream, btd_status* st);
int btd_solve_up(const btd_hierarchy* h, const double* rhs, const double* reduced_x, double* x, int64_t num_columns,
                 void* scratch, void* stream, btd_status* st);

/* btd_factorize with HOST-resident inputs (pinned for full overlap): the blocks are copied into the
 * caller's device arrays dev_diag / dev_sub in chunks of whole level-0 segments on a private copy
 * stream, and every chunk is eliminated as soon as it has landed (H2D overlaps the level-0 factor).
 * Same result and errors as btd_factorize(h, dev_diag, dev_sub, ...); the host arrays are read
 * asynchronously until the work on `stream` completes. */
int btd_factorize_from_host(btd_hierarchy* h, const double* host_diag, const double* host_sub, double* dev_diag,
                            double* dev_sub, void* persistent, void* scratch, void* stream, int32_t check,
                            btd_status* st);

/* Optional per-launch timing: when enabled, btd_factorize records CUDA events on the caller's
 * stream around every factor kernel (one per level, then the base).  btd_kernel_times returns the
 * elapsed milliseconds of the last factorization's launches in that order. */
int btd_profile_kernels(btd_hierarchy* h, int32_t enable);
int btd_kernel_times(const btd_hierarchy* h, float* ms_out, int64_t cap, int64_t* count);
/* Block SpMV y = A x (btd_matmul, core.py:280-288) and the fused residual of residual_report
 * (report.py:20-38): norms2[c] = ||b_c - (A x)_c||_2^2, norms2[d + c] = ||b_c||_2^2, reduced in a
 * fixed order (deterministic).  `workspace` holds btd_residual_workspace() bytes; norms2 is a
 * device array of 2d doubles. */
int btd_matmul(const double* diag, const double* sub, int64_t num_blocks, int64_t block_size, const double* x,
               int64_t num_columns, double* y, void* stream, btd_status* st);
int btd_residual_workspace(int64_t num_blocks, int64_t block_size, int64_t num_columns, size_t* bytes);
int btd_residual_norms(const double* diag, const double* sub, int64_t num_blocks, int64_t block_size,
                       const double* x, const double* b, int64_t num_columns, void* workspace, double* norms2,
                       void* stream, btd_status* st);

/* Kalman MAP-smoothing normal equations (build_normal_equations, kalman.py:130-162): one device
 * pass assembling diag (N,n,n), sub (N-1,n,n), rhs (N,n) from the model arrays (device pointers,
 * reference layouts).  flags: BTD_KALMAN_DIAG_R (meas_cov is (N,m) variances, else (N,m,m)),
 * BTD_KALMAN_SHARED_{H,Q,R} (the array is one block shared by every step).  n <= 64; dense R:
 * m <= 64.  A failing covariance returns BTD_ERR_NOT_POSITIVE_DEFINITE with pivot, block = step,
 * member = 0 (process) / 1 (measurement).  workspace: btd_kalman_workspace() bytes. */
#define BTD_KALMAN_DIAG_R 1
#define BTD_KALMAN_SHARED_H 2
#define BTD_KALMAN_SHARED_Q 4
#define BTD_KALMAN_SHARED_R 8
int btd_kalman_workspace(int64_t horizon, int64_t state_dim, size_t* bytes);
int btd_kalman_normal_equations(int64_t horizon, int64_t state_dim, int64_t obs_dim, const double* transition,
                                const double* observation, const double* process_cov, const double* meas_cov,
                                const double* observations, const double* prior_offsets, int32_t flags,
                                double* diag, double* sub, double* rhs, void* workspace, void* stream,
                                btd_status* st);

/* Process-wide count of kernels this library has launched (evidence for bench.py gpu_launches);
 * a replayed CUDA graph adds the kernel launches it contains. */
long long btd_launch_count(void);

/* CUDA graphs (no reference counterpart: replaces the per-kernel launches of the paper's batched
 * BLAS calls, §5).  With device-resident inputs, btd_factorize / btd_solve (and the
 * partial variants) capture their whole launch sequence -- every level, assembly and the base --
 * into one graph per (shape, config, buffer addresses) and replay it on later calls with the same
 * buffers.  Enabled by default (environment BTD_GRAPHS=0 disables); returns the previous setting.
 * Disabling drops the cached graphs. */
int btd_set_graphs(int32_t enable);
/* Process-wide count of factor / solve calls served by replaying a cached graph. */
long long btd_graph_replays(void);

/* ---- The reference's accelerator seam (bt/kernels.py:164-338) ----
 * Batched dense kernels over `count` same-shaped members of ANY element strides (member, row,
 * column) -- the reference solves through transposed views (block_cholesky.py:32).  All pointers are
 * device pointers; launches are asynchronous on `stream`.  Failures accumulate in a device error
 * word (btd_seam_error_bytes() bytes, reset by btd_seam_error_init) exactly as the reference's
 * chunked batch reports them: NotPositiveDefinite = earliest `block_coord`, then lowest member,
 * 1-based pivot; SingularDiagonal = lowest (member, row).  btd_seam_error_read synchronizes `stream`
 * and returns BTD_OK / BTD_ERR_NOT_POSITIVE_DEFINITE (pivot, member, block) /
 * BTD_ERR_SINGULAR_DIAGONAL (pivot = 1-based row, member). */
size_t btd_seam_error_bytes(void);
int btd_seam_error_init(void* err, void* stream);
int btd_seam_error_read(const void* err, void* stream, btd_status* st);
/* chol_factor_batch (kernels.py:164-181): member = L L^T in place, strict upper triangle zeroed.
 * block_coord = the block step reported with a failure (_chol_step, block_cholesky.py:40-42). */
int btd_chol_batch(double* blocks, const int64_t strides[3], int64_t count, int64_t n, int64_t block_coord, void* err,
                   void* stream, btd_status* st);
/* trsm_lower_batch (kernels.py:215-259): panels (count, n, cols) <- L^{-1} P (trans = 0) or
 * L^{-T} P (trans = 1), L = lower triangle of factors (count, n, n).  A zero diagonal anywhere is
 * reported and no panel is modified. */
int btd_trsm_batch(const double* factors, const int64_t fstrides[3], double* panels, const int64_t pstrides[3],
                   int64_t count, int64_t n, int64_t cols, int32_t trans, void* err, void* stream, btd_status* st);
/* gemm_acc_batch (kernels.py:270-310): out (count, m, p) <- alpha op(a) op(b) + beta out, op(a) m x q,
 * op(b) q x p; alpha == 0 skips the product, beta == 0 ignores out's contents.  out must not alias
 * a or b.  At most 65535 members per call. */
int btd_gemm_batch(double* out, const int64_t ostrides[3], const double* a, const int64_t astrides[3], const double* b,
                   const int64_t bstrides[3], int64_t count, int64_t m, int64_t q, int64_t p, int32_t trans_a,
                   int32_t trans_b, double alpha, double beta, void* stream, btd_status* st);

#ifdef __cplusplus
}
#endif

#endif /* BLOCKTRI_B200_H */
