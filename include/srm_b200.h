/*
 * srm_b200.h -- C ABI of the B200-native SRM EM engine (libsrm_b200.so).
 *
 * This is the drop-in boundary for the reference's SRM fit path
 * (/root/reference/pkg/src/factorfit/srm.py).  The reference has no FFI of
 * its own (it is numpy/scipy); each entry point below names the reference
 * function or call site whose work it replaces.  Signatures use plain
 * pointers and sizes only: device pointers, host arrays of dimensions, and an
 * opaque cudaStream_t passed as void*.  No torch types cross this boundary.
 *
 * Error convention (mirrors factorfit/errors.py):
 *   every function returns an srm_status code; SRM_OK == 0.  Device-side
 *   failures (non-finite input, rank deficiency, Cholesky breakdown) are
 *   recorded asynchronously in a device status word -- {code, arg, iteration,
 *   warnings} -- and surface through srm_read_status().  `arg` is the failing
 *   Cholesky pivot (0-based, DefinitenessError.pivot) or the global subject
 *   index (RankError / InvalidInputError).  srm_last_error() returns a
 *   thread-local message for the last host-side failure.
 *
 * Threading: one plan per GPU process; plans are not shared between threads
 * (reference SPEC.md:177-178: communicators and workers are not shareable).
 */
#ifndef SRM_B200_H_
#define SRM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRM_B200_ABI_VERSION 1

/* storage dtype of the demeaned data X-hat (all arithmetic is fp64) */
enum srm_dtype { SRM_F64 = 0, SRM_F32 = 1 };

/* status codes <-> factorfit.errors exception classes */
enum srm_status {
  SRM_OK = 0,
  SRM_ERR_CONFIG = 1,        /* ConfigError            */
  SRM_ERR_SHAPE = 2,         /* ShapeError             */
  SRM_ERR_INVALID_INPUT = 3, /* InvalidInputError      */
  SRM_ERR_DEFINITENESS = 4,  /* DefinitenessError(pivot) */
  SRM_ERR_RANK = 5,          /* RankError              */
  SRM_ERR_CUDA = 6,          /* CUDA runtime failure   */
  SRM_ERR_UNSUPPORTED = 7,   /* outside this build's limits (k > 128) */
  SRM_ERR_FORMAT = 8,        /* malformed SFAB container (srm_sfab_last_error) */
  SRM_ERR_IO = 9             /* file system error (srm_sfab_last_error) */
};

/* warning bits of the device status word (element 3), sticky until
 * srm_clear_status / srm_reset */
enum srm_warning {
  SRM_WARN_POLAR_CONDITION = 1 /* a subject's A^T A was too ill-conditioned for the
                                  Gram-route polar transform (sigma_min / sigma_max
                                  below ~3e-3): redo the fit with SRM_FLAG_EXACT_POLAR,
                                  which resolves it -- or raises RankError -- like the
                                  reference's SVD (kernels.py:190-212) */
};

/* plan flags */
enum srm_flags {
  SRM_FLAG_ORDERED = 1,   /* E-step terms summed in ascending global subject order
                             from a gathered per-subject table (srm.py:193-213);
                             otherwise per-rank sums are all-reduced */
  SRM_FLAG_TOLERANCE = 2, /* compute |S - S_prev| / |S_prev| every iteration (srm.py:275-287) */
  SRM_FLAG_GRAM = 4,      /* per-iteration contractions through the T x T data Gram
                             (one-time X^T X); exact algebra, fewer flops when
                             4*K*iterations > T */
  SRM_FLAG_TC = 8,        /* fp32 X-hat: streaming passes on the tcgen05 tensor cores
                             as 3xTF32 split-precision MMAs (ignored for fp64
                             storage, K > 128, or with SRM_FLAG_GRAM) */
  SRM_FLAG_GRAM_I8 = 16,  /* with SRM_FLAG_GRAM and fp64 storage: X^T X from seven
                             exact int8 slices per value (power-of-two column
                             scales) on the tcgen05 int8 tensor cores, ~2^-48
                             relative to the column maxima; otherwise fp64 DMMA */
  SRM_FLAG_EXACT_POLAR = 32, /* every polar transform (init and M-step) from A itself:
                             Householder TSQR + one-sided Jacobi SVD of R, never
                             A^T A; implies the fp64 streaming path (A_i = X_i S^T / 2
                             formed each iteration; clears GRAM, GRAM_I8, TC) */
  SRM_FLAG_COLBLOCK = 64  /* world_size > 1: the ordered accumulation of srm.py:193-213
                             by TR column blocks -- each rank's terms cut into
                             world_size column blocks and exchanged all-to-all
                             (SRM_R_XSEND -> SRM_R_XRECV), every rank sums its block
                             over all subjects in ascending global order
                             (srm_xchg_reduce), the K x T / world_size results are
                             all-gathered (SRM_R_XRED) and unpacked into SRM_R_RED.
                             Bit-identical to one rank, with 1 / world_size of the
                             all-gather's traffic; overrides SRM_FLAG_ORDERED */
};

/* workspace regions (srm_plan_region) */
enum srm_region {
  SRM_R_XHAT = 0,     /* [rows_total x ldx] X-hat, dtype                              */
  SRM_R_AMAT = 1,     /* [rows_total x kp] f64: A_i = X_i S^T / 2 (init: N(0,1) draw)  */
  SRM_R_WOUT = 2,     /* [rows_total x k] f64: final W_i (srm.py:315-327 model.W)     */
  SRM_R_MU = 3,       /* [rows_total] f64: voxel means (model.mu)                      */
  SRM_R_TERMS = 4,    /* [n_slots x term_stride] f64: per-subject E-step records       */
  SRM_R_RED = 5,      /* [red_stride] f64: reduced K x ldx sum + scalars               */
  SRM_R_REDLOCAL = 6, /* [red_stride] f64: this rank's partial (unordered mode)        */
  SRM_R_S = 7,        /* [kp x ldx] f64: shared response S (model.S)                   */
  SRM_R_SIGMA = 8,    /* [kp x kp] f64: Sigma_s (model.sigma_s)                        */
  SRM_R_HIST = 9,     /* [iterations x hist_stride] f64: per-iteration scalars         */
  SRM_R_STATUS = 10,  /* int32[4] device status word                                   */
  SRM_R_MMAT = 11,    /* [n_local x kp x kp] f64: polar transforms M_i                 */
  SRM_R_SCAL = 12,    /* [n_local x 8] f64: per-subject scalars                        */
  SRM_R_GRAM = 13,    /* [n_local x ldx x ldx] f64/f32: X_i^T X_i (SRM_FLAG_GRAM only) */
  SRM_R_VAR = 14,     /* [kp x kp] f64: posterior covariance var_s                     */
  SRM_R_XSEND = 15,   /* SRM_FLAG_COLBLOCK: [world x max_local x xrec] f64 column blocks  */
  SRM_R_XRECV = 16,   /*   ... received: [world (source rank) x max_local x xrec]          */
  SRM_R_XRED = 17,    /*   [world x xred] f64: the reduced blocks (this rank's at `rank`) */
  SRM_R_COUNT = 18
};

/* plan dimensions (srm_plan_dim) */
enum srm_dim {
  SRM_D_LDX = 0,          /* padded T (row stride of X-hat, S, terms)   */
  SRM_D_KP = 1,           /* padded K                                   */
  SRM_D_ROWS = 2,         /* sum of local voxel counts                  */
  SRM_D_TERM_STRIDE = 3,  /* doubles per subject record in SRM_R_TERMS  */
  SRM_D_RED_STRIDE = 4,   /* doubles in SRM_R_RED                       */
  SRM_D_HIST_STRIDE = 5,  /* doubles per iteration in SRM_R_HIST        */
  SRM_D_N_SLOTS = 6,      /* subject records in SRM_R_TERMS             */
  SRM_D_SLOT_OFFSET = 7,  /* first record slot owned by this rank       */
  SRM_D_ITEMS_E = 8,      /* work items of the V-contraction kernel     */
  SRM_D_ITEMS_A = 9,      /* work items of the T-contraction kernel     */
  SRM_D_CHUNK_ROWS = 10,  /* rows per V chunk                           */
  SRM_D_LAUNCHES = 11,    /* kernel launches per EM iteration (e+m step) */
  SRM_D_FLAGS = 12,       /* effective plan flags                        */
  SRM_D_XREC = 13,        /* SRM_FLAG_COLBLOCK: doubles per block record */
  SRM_D_XRED = 14         /*   doubles per reduced block                  */
};

/* per-iteration history columns (SRM_R_HIST, hist_stride doubles per row) */
enum srm_hist {
  SRM_H_LL = 0,       /* log-likelihood of the parameters entering the iteration */
  SRM_H_TRACE = 1,    /* tr(Sigma_s_new)                                         */
  SRM_H_RHO0 = 2,     /* sum_i 1/rho_i^2 used by the E-step                      */
  SRM_H_SDIFF = 3,    /* |S - S_prev|_F                                          */
  SRM_H_SPREV = 4,    /* |S_prev|_F                                              */
  SRM_H_RHO2 = 8      /* first of n_local post-M-step rho_i^2                    */
};

typedef struct srm_plan srm_plan;

/* ---- version / errors ---------------------------------------------------- */
int srm_abi_version(void);
const char* srm_last_error(void);

/* ---- plan ------------------------------------------------------------------
 * srm_plan_create replaces the bookkeeping of factorfit.srm.fit
 * (srm.py:216-246: validation, rank_offsets, per-subject state).
 *   n_local subjects with voxel counts n_voxels[n_local] (host array), T TRs,
 *   k factors; world_size ranks with counts_per_rank[world_size] subjects
 *   each (contiguous shards, cli.py:82-85); this rank is `rank`.
 */
int srm_plan_create(srm_plan** out, int dtype, int n_local, const int64_t* n_voxels,
                    int64_t n_trs, int64_t k, int iterations, int world_size, int rank,
                    const int32_t* counts_per_rank, int flags);
int srm_plan_destroy(srm_plan* plan);
int64_t srm_plan_workspace_bytes(const srm_plan* plan);
int64_t srm_plan_dim(const srm_plan* plan, int which);
/* bind a device workspace of srm_plan_workspace_bytes() bytes (256-B aligned).
 * Every region is zeroed except SRM_R_XHAT and SRM_R_GRAM (and the internal
 * int8 slices), which srm_load_subject / srm_prepare_gram write in full. */
int srm_plan_bind(srm_plan* plan, void* workspace, int64_t bytes);
int srm_plan_region(const srm_plan* plan, int region, int64_t* offset, int64_t* bytes);

/* ---- one-time work ----------------------------------------------------------
 * srm_load_subject: srm.py:94-98 `demean` + kernels.py:45 finite check +
 *   the loop-invariant kernels.py:152-155 `trace_ata` (hoisted out of the EM
 *   loop, srm.py:152).  x is a device array [V_i x ld] of x_dtype; it is not
 *   modified (srm.py:98 returns a copy).
 * srm_init_mapping: srm.py:101-113 `init_subject` after the host RNG draw
 *   (the N(0,1) matrix, PCG64-seeded as the reference, is written to
 *   SRM_R_AMAT first): polar transform of the draw, and the first E-step term
 *   W_i^T X_i = M_0^T (G^T X_i) (srm.py:116-118) with rho_i^2 = 1.  On int8
 *   Gram plans G^T X_i runs on the int8 tensor cores from seven-slice records
 *   of G and the slices of X-hat (srm_prepare_gram_range is enqueued first for
 *   any subject it has not covered yet).
 */
int srm_load_subject(srm_plan* plan, int local_index, const void* x, int x_dtype,
                     int64_t ld, void* stream);
int srm_finish_load(srm_plan* plan, void* stream);
int srm_init_mapping(srm_plan* plan, void* stream);
/* the same for local subjects [first, first + count) only (their draws and
 * X-hat must be in place), so the loader can overlap it with later uploads;
 * srm_init_mapping = this over all subjects + iteration counter reset */
int srm_init_mapping_range(srm_plan* plan, int first, int count, void* stream);
/* SRM_FLAG_GRAM plans: G_i = Xhat_i^T Xhat_i (T x T, fp64) for every local
 * subject, after srm_load_subject.  The per-iteration M-step then needs
 * B_i = A_i^T Xhat_i = S G_i / 2 and A_i^T A_i = B_i S^T / 2 only; A_i itself is
 * formed once in srm_finalize.  No-op for streaming plans. */
int srm_prepare_gram(srm_plan* plan, void* stream);
/* the same for local subjects [first, first + count) -- lets the loader
 * overlap each subject's Gram with the next subject's host-to-device copy */
int srm_prepare_gram_range(srm_plan* plan, int first, int count, void* stream);
/* restart the EM state (Sigma_s = I, status cleared, iteration 0); the next
 * srm_init_mapping draws a fresh start (used to time repeated fits) */
int srm_reset(srm_plan* plan, void* stream);

/* ---- per-iteration work (srm.py:254-287) -----------------------------------
 * The iteration index lives in a device counter (set to 0 by
 * srm_init_mapping, advanced by srm_m_step) so one captured CUDA graph of
 * {e_step, m_step} serves every iteration.  History rows wrap modulo
 * `iterations`.
 * srm_set_iteration: overwrite the device counter (asynchronous).
 * srm_reduce_local: unordered mode only -- this rank's sum of its E-step
 *   terms into SRM_R_REDLOCAL, to be all-reduced into SRM_R_RED.
 * srm_e_step: srm.py:193-213 ordered accumulation (ordered mode), then
 *   srm.py:121-129 `e_step_global` and srm.py:132-142 `update_sigma_s`:
 *   K x K Cholesky inverses, S, Sigma_s, tr(Sigma_s), the Woodbury
 *   log-likelihood and the tolerance statistic.
 * srm_m_step: srm.py:145-155 `m_step_subject` for every local subject:
 *   A_i = X_i S^T / 2, the polar factor W_i = A_i (A_i^T A_i)^{-1/2}, the
 *   cross term and rho_i^2, and the next E-step term W_i^T X_i / rho_i^2
 *   (srm.py:151 and :118 share one product).
 * srm_finalize: materialise W_i = A_i M_i (model.W).
 * srm_finalize_range: the same for local subjects [first, first + count);
 *   calls must cover 0 .. n_local - 1 in ascending order, starting with
 *   first = 0 (which runs the shared prelude).  Lets a caller read W_i of
 *   earlier subjects back while later ones are formed (srm.py:315-327).
 */
int srm_set_iteration(srm_plan* plan, int iteration, void* stream);
int srm_reduce_local(srm_plan* plan, void* stream);
/* SRM_FLAG_COLBLOCK exchange, around an all-to-all of SRM_R_XSEND into
 * SRM_R_XRECV (equal splits of max_local * xrec doubles) and an all-gather of
 * this rank's block of SRM_R_XRED:
 *   srm_xchg_pack: this rank's E-step terms (and record scalars) cut into
 *     world column blocks of ceil(ldx / world) TRs -> SRM_R_XSEND;
 *   srm_xchg_reduce: its own block summed over every subject of every rank in
 *     ascending global order (srm.py:193-213, the same left fold as one rank),
 *     plus the scalar sums -> SRM_R_XRED[rank];
 *   srm_xchg_unpack: the gathered blocks -> SRM_R_RED. */
int srm_xchg_pack(srm_plan* plan, void* stream);
int srm_xchg_reduce(srm_plan* plan, void* stream);
int srm_xchg_unpack(srm_plan* plan, void* stream);
int srm_e_step(srm_plan* plan, void* stream);
int srm_m_step(srm_plan* plan, void* stream);
int srm_finalize(srm_plan* plan, void* stream);
int srm_finalize_range(srm_plan* plan, int first, int count, void* stream);

/* one EM iteration as a CUDA graph: srm_graph_capture records
 * {srm_e_step, srm_m_step} once (single-rank plans; call after one eager
 * iteration so every kernel is configured); srm_graph_launch replays it on
 * `stream` (the device iteration counter advances inside the graph). */
int srm_graph_capture(srm_plan* plan);
int srm_graph_launch(srm_plan* plan, void* stream);

/* measurement: run one e_step + m_step eagerly with a CUDA event between every
 * kernel, synchronise, and write each kernel's duration (ms) to ms_out; *n_out
 * receives the number of kernels.  srm_profile_name(i) names kernel i of the
 * last profiled iteration. */
int srm_profile_iteration(srm_plan* plan, float* ms_out, int capacity, int* n_out, void* stream);
/* the same for srm_prepare_gram over all local subjects (SRM_FLAG_GRAM plans;
 * *n_out = 0 otherwise) */
int srm_profile_gram(srm_plan* plan, float* ms_out, int capacity, int* n_out, void* stream);
/* the same for srm_finalize */
int srm_profile_finalize(srm_plan* plan, float* ms_out, int capacity, int* n_out, void* stream);
const char* srm_profile_name(int index);

/* synchronous copy of the device status word {code, arg, iteration, warnings}
 * (warnings: SRM_WARN_* bits) */
int srm_read_status(srm_plan* plan, int32_t* out4);
/* clear the device status word (asynchronous) */
int srm_clear_status(srm_plan* plan, void* stream);

/* ---- stateless kernels (step-function API, srm.py:116-155, kernels.py) ---- */
/* out[k x t] = alpha * W^T X over all V rows; W [V x ldw] f64, X [V x ldx]
 * dtype; replaces srm.py:118 (e_step_local) and srm.py:151 (W_new^T Xhat). */
int srm_gemm_tn(const double* w, int64_t ldw, const void* x, int x_dtype, int64_t ldx,
                int64_t v, int64_t k, int64_t t, double alpha, double* out, int64_t ldo,
                void* workspace, int64_t ws_bytes, void* stream);
/* out[v x k] = alpha * X S^T; replaces srm.py:147 (A = Xhat S^T / 2). */
int srm_gemm_nt(const void* x, int x_dtype, int64_t ldx, const double* s, int64_t lds,
                int64_t v, int64_t t, int64_t k, double alpha, double* out, int64_t ldo,
                void* workspace, int64_t ws_bytes, void* stream);
/* srm.py:330-333 `project`, batched over the t columns of a block of volumes:
 * out[k x t] = W^T (X - mu 1^T) with W [v x k] f64, X [v x t] dtype, mu [v] f64
 * (null: no centering); the subtraction is fused into the fp64 staging of X,
 * so projecting mu itself gives exactly 0 (reference test_srm.py:343-345). */
int srm_project(const double* w, int64_t ldw, const void* x, int x_dtype, int64_t ldx,
                const double* mu, int64_t v, int64_t k, int64_t t, double* out, int64_t ldo,
                void* workspace, int64_t ws_bytes, void* stream);
/* srm.py:336-338 `map_between` after the projection: out[v x t] = W z + mu 1^T
 * with W [v x k], z [k x t], mu [v] (null: none); k <= 128 */
int srm_unproject(const double* w, int64_t ldw, const double* z, int64_t ldz, const double* mu,
                  int64_t v, int64_t k, int64_t t, double* out, int64_t ldo, void* stream);
/* trace(A^T A) = sum of squares of a [rows x cols] f64 block (kernels.py:152-155)
 * into *out (device), summed in a fixed order; non-finite entries raise
 * InvalidInputError through status4 (kernels.py:45-46).  workspace >= 8 KB. */
int srm_trace_ata(const double* a, int64_t lda, int64_t rows, int64_t cols, double* out,
                  int32_t* status4, void* workspace, int64_t ws_bytes, void* stream);
/* *out = sum_{r,c} a[r][c] b[r][c] over [rows x cols] f64 blocks, fixed order
 * (srm.py:151 cross term einsum("kt,kt->", W^T Xhat, S)); workspace >= 8 KB */
int srm_dot(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t rows, int64_t cols,
            double* out, void* workspace, int64_t ws_bytes, void* stream);
/* srm.py:140-142 `update_sigma_s` after var_s: out = sym(var_s + ss / t) with
 * ss = S S^T [k x k], and *trace_out = tr(out) (device pointers) */
int srm_sigma_update(const double* var, int64_t ldv, const double* ss, int64_t ldss, int64_t k, int64_t t,
                     double* out, int64_t ldo, double* trace_out, void* stream);
/* out = A + c I for a [n x n] f64 matrix (kernels.py:158-165); off-diagonal
 * entries are copied bit for bit. */
int srm_add_diag(const double* a, int64_t lda, int64_t n, double c, double* out, int64_t ldo,
                 void* stream);
/* in-place SPD inverse of a [n x n] f64 matrix (kernels.py:168-187).  Status
 * (DefinitenessError pivot) goes to status4 (device int32[4]). */
int srm_spd_inverse(double* a, int64_t n, int32_t* status4, void* stream);
/* srm.py:121-142 e_step_global + update_sigma_s for one reduced K x T sum:
 * S (k x t), var_s (k x k), Sigma_new (k x k) and tr(Sigma_new) (one double),
 * all device pointers; DefinitenessError pivots go to status4.  Synchronous. */
int srm_tail_step(const double* reduced, int64_t ldr, const double* sigma, int64_t ldsig,
                  int64_t k, int64_t t, double rho0, double* s_out, int64_t lds_out,
                  double* var_out, double* sigma_out, double* trace_out, int32_t* status4,
                  void* workspace, int64_t ws_bytes, void* stream);
/* orthogonal polar factor W = U V^T of a [v x k] f64 matrix (kernels.py:190-212):
 * Householder TSQR A = Q R, one-sided Jacobi SVD of R (never forms A^T A, so
 * singular values resolve to ~eps sigma_max like gesdd), W = A V diag(1/sigma) V^T,
 * then one exact polar step of W.  RankError (sigma_min < 1e-12 sigma_max, or
 * sigma_max = 0) goes to status4.  Synchronous. */
int srm_polar(const double* a, int64_t lda, int64_t v, int64_t k, double* w, int64_t ldw,
              int32_t* status4, void* workspace, int64_t ws_bytes, void* stream);
/* workspace bytes needed by srm_gemm_tn / srm_gemm_nt / srm_project / srm_polar / srm_tail_step */
int64_t srm_stateless_workspace_bytes(int64_t v, int64_t k, int64_t t);

/* ---- SFAB subject containers (data_io.py:1-30 layout, :130-196 checks) ------
 * Host functions (no GPU needed).  Failures return SRM_ERR_FORMAT (the
 * reference's FormatError: srm_sfab_last_error gives the message, the byte
 * offset and the field name of the first failed check), SRM_ERR_IO (open /
 * read / write), SRM_ERR_SHAPE (destination too small) or
 * SRM_ERR_INVALID_INPUT (non-finite values on write).
 */
/* read_header (data_io.py:144-157): validated (rows, cols) without the payload */
int srm_sfab_header(const char* path, int64_t* rows, int64_t* cols);
/* load_matrix (data_io.py:160-179): validate and read the row-major f64
 * payload into dst (>= rows*cols*8 bytes; normally a pinned host slot that an
 * asynchronous H2D copy drains into srm_load_subject) with `threads` parallel
 * preads (<= 0: 8) */
int srm_sfab_read(const char* path, void* dst, int64_t capacity_bytes, int threads);
/* save_matrix (data_io.py:130-141): header + payload; rejects non-finite entries */
int srm_sfab_write(const char* path, const double* src, int64_t rows, int64_t cols);
/* message of the last SFAB failure on this thread; *offset / *field locate the
 * failed check of a SRM_ERR_FORMAT (-1 / "" otherwise) */
const char* srm_sfab_last_error(int64_t* offset, const char** field);

#ifdef __cplusplus
}
#endif

#endif /* SRM_B200_H_ */
