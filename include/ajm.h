/*
 * ajm.h -- C ABI of the B200-native accelerated Jacobi-type method (AJM) solver, arXiv 2407.03272.
 *
 * The library solves a consistent symmetric positive semidefinite system Q x = b
 * (eq-linear-sys), equivalently min f(x) = 1/2<x,Qx> - <b,x> (PAPER.md:25-28,
 * eq-qp), with the parallel Nesterov-accelerated Jacobi-type method with adaptive restart,
 * Algorithm 3 on one GPU (s = 1 block: the GPU's row-parallel pass is the
 * "for i parallel" loop of Alg. 3 line 3).  Everything is FP64.  Every step of every iteration runs
 * in this library's own sm_100a kernels; there is no CPU fallback.
 *
 * Conventions shared by every entry point
 *   - extern "C", plain pointers and sizes.  An array pointer may be HOST memory (pageable or
 *     pinned) or DEVICE memory of the current CUDA device; the library detects which with
 *     cudaPointerGetAttributes and copies accordingly (host<->device copies are stream-ordered on
 *     `cuda_stream`).
 *   - `cuda_stream` is a cudaStream_t (NULL = the legacy default stream); all device work of a call
 *     is ordered on it.  ajm_create and ajm_solve return only after the stream reaches the end of
 *     their work (their results are host-visible).
 *   - A handle is not thread-safe; distinct handles are independent and may be used from different
 *     host threads at the same time: the solver kernels' attributes (shared by every handle of the
 *     same layout class) are only set, queried and launched with under one library-wide lock.
 *   - On error a call returns a non-zero ajm_status_t and ajm_last_error() explains it; no output
 *     argument is written except where stated.
 */
#ifndef AJM_H_
#define AJM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AJM_ABI_VERSION 5  /* 2: AJM_D_JBLOCK, ajm_get_jblock, ajm_info_t.l2_mode / launches_per_solve;
                              3: layout create flags (AJM_INT32_COLUMNS, AJM_GLOBAL_TABLES, AJM_SEGMENTS_*,
                                 AJM_DEBUG_POISON), ajm_estimate_spectrum;
                              4: the row-block sharded API (ajm_partition_rows, ajm_shard_*,
                                 ajm_group_solve), ajm_info_t.nranks / halo;
                              5: pair-coded SELL entries (AJM_VALUE_STREAM, ajm_info_t.val_bytes) */

typedef struct ajm_ctx* ajm_handle_t;

typedef enum {
    AJM_OK = 0,
    AJM_ERR_INVALID_ARG = 1,   /* NULL / size mismatch, tol < 0 or NaN, maxit < 1, k0 < 2,
                                  restart without momentum, n or nnz out of range */
    AJM_ERR_CSR_INVALID = 2,   /* row_ptr[0] != 0, row_ptr decreasing, row_ptr[n] != nnz, column out of
                                  range or not strictly increasing within a row            */
    AJM_ERR_NOT_SYMMETRIC = 3, /* Q_ij != Q_ji (only checked with AJM_VALIDATE_SYMMETRY)   */
    AJM_ERR_NONFINITE = 4,     /* NaN/Inf in Q, b, d or x0                                     */
    AJM_ERR_NEGATIVE_DIAG = 5, /* some Q_kk < 0: Q cannot be SPSD                                     */
    AJM_ERR_ZERO_DIAG = 6,     /* some D_kk = 0 (zero row / isolated node) or user d_k <= 0 */
    AJM_ERR_ZERO_RHS = 7,      /* ||b|| = 0: the relative-residual stopping rule is undefined */
    AJM_ERR_CUDA = 8,          /* a CUDA runtime call failed (message in ajm_last_error)              */
    AJM_ERR_OOM = 9,           /* device allocation failed                                            */
    AJM_ERR_UNSUPPORTED = 10   /* e.g. n >= 2^31, or nnz >= 2^31 with rows of > 64 nonzeros          */
} ajm_status_t;

/* The diagonal metric D of the Jacobi-type step x = y + D^{-1}(b - Q y). */
typedef enum {
    AJM_D_JDIAG = 0, /* eq-J-diag: D_kk = J_kk = Q_kk + sum_{j != k}|Q_kj|, built on
                        the device, summed in ascending column order.  S = J - Q is PSD,
                        which is what Thm 2.3 / 2.5 need.  The default and the paper's experiments. */
    AJM_D_USER = 1,  /* the caller's positive diagonal d[n], e.g. diag(Q)/omega for weighted Jacobi */
    AJM_D_QDIAG = 2, /* D = diag(Q): classical Jacobi metric; no S >= 0 guarantee */
    AJM_D_JBLOCK = 3 /* block-diagonal J of eq-J-blkdiag: contiguous row blocks of bs rows
                        (bs = AJM_JBLOCK_SIZE in the create flags; the last block ragged),
                        J^{ii} = Q^{ii} + (sum_{j != i} ||Q^{ij}||_2) I, the spectral norms summed in
                        ascending j; the step applies J^{-1} block by block (Alg. 3 line 4).  S = J - Q
                        is PSD.  Requires every row to have <= 64 nonzeros (the blocks are
                        solved inside a warp); otherwise AJM_ERR_UNSUPPORTED.  A block that is not SPD
                        gives AJM_ERR_ZERO_DIAG.  DESIGN.md R23. */
} ajm_dmode_t;

/* ajm_create flags */
#define AJM_VALIDATE_SYMMETRY 0x1u /* also check Q_ij == Q_ji bitwise (O(nnz log rowlen) kernel)    */
#define AJM_LOOP_HOST 0x10u        /* debug: one solver-kernel launch per pass, driven by the host,
                                      instead of the single persistent launch (same kernel, same
                                      results bit for bit)                                          */
/* layout switches (defaults are chosen from the row-length histogram; these force one choice):   */
#define AJM_INT32_COLUMNS 0x10000u    /* keep int32 SELL columns even when the column offsets col - row
                                         take <= 256 values (no byte-coded columns; same iterates)     */
#define AJM_GLOBAL_TABLES 0x20000u    /* per-CTA unit/chunk tables in global memory instead of shared
                                         memory (what huge layouts use; same iterates)                 */
#define AJM_SEGMENTS_STATIC 0x40000u  /* rows of > 64 nonzeros: static LPT plan of warp segments        */
#define AJM_SEGMENTS_DYNAMIC 0x80000u /* ... or a per-pass claim queue (default: dynamic only when long
                                         rows carry >= 90% of the nonzeros); same iterates either way   */
#define AJM_DEBUG_POISON 0x100000u    /* debug: fill every device allocation of this create with 0xff   */
#define AJM_VALUE_STREAM 0x400000u    /* keep streaming the SELL values even when the (column offset,
                                         value) pairs take <= 256 values (no pair codes; same iterates) */
#define AJM_NO_BAND_STAGING 0x800000u /* pair-coded stencils: gather x~ from global memory instead of
                                         staging its bands and the row operands through the TMA ring
                                         (same iterates)                                              */
/* block size of AJM_D_JBLOCK, bits 8..15 of the flags: bs in {1, 2, 4, 8, 16, 32} */
#define AJM_JBLOCK_SIZE(bs) (((uint32_t)(bs) & 0xffu) << 8)
#define AJM_JBLOCK_SIZE_OF(flags) (((uint32_t)(flags) >> 8) & 0xffu)

/* Iteration policy. */
typedef struct {
    int32_t momentum; /* 1: Nesterov alpha schedule alpha_{t+1} = (1 + sqrt(1 + 4 alpha_t^2))/2,
                         beta_t = (alpha_t - 1)/alpha_{t+1} (Alg. 1/3);
                         0: beta = 0, the variable-metric gradient / Jacobi step (eq-gd)   */
    int32_t restart;  /* 1: adaptive restart = Alg. 3 IsRestart; 0: Alg. 1.
                         restart = 1 with momentum = 0 -> AJM_ERR_INVALID_ARG                       */
    int64_t k0;       /* K_0 >= 2, the first prohibition period ("K_l >= 2"); default 2      */
} ajm_policy_t;

typedef enum { AJM_CONVERGED = 0, AJM_MAXITER = 1, AJM_DIVERGED = 2 } ajm_term_t;

typedef struct {
    int32_t status;          /* ajm_term_t                                                          */
    int32_t n_restarts;      /* restarts executed (Alg. 3 line 6 taken), ell at exit                */
    int64_t iterations;      /* t at exit; 0 if x0 already satisfies the tolerance                  */
    double rel_residual;     /* ||b - Q x~^t|| / ||b|| of the last evaluated iterate        */
    double f;                /* f(x~^t) = 1/2<x,Qx> - <b,x> of the same iterate           */
    int32_t x_is_prerestart; /* 1 if converged at an iteration whose restart test fired: x_out is the
                                pre-restart x~^t (R5)                                     */
    int32_t restarts_logged; /* entries written to restart_iters                                    */
} ajm_result_t;

/* Layout / launch facts of a handle (for benchmarks and tests). */
typedef struct {
    int64_t n, nnz;
    int64_t units;            /* work items: SELL chunks + warp segments                         */
    int64_t long_rows;        /* rows split into several warp segments (> 2048 nonzeros)        */
    int32_t grid;             /* CTAs of the persistent solver kernel (#SMs x resident/SM)      */
    int32_t block;            /* threads per CTA                                                */
    int32_t sm_count;
    int32_t ctas_per_sm;
    double model_bytes_per_iter; /* nnz*12 + 7*n*8 + 4*(n+1)  */
    double last_loop_ms;      /* device time of the last solve's iteration loop (CUDA events)  */
    int64_t last_passes;      /* fused passes run by the last solve (= iterations + 1)        */
    int64_t last_launches;    /* solver-kernel launches of the last solve (1: persistent loop) */
    int64_t sell_rows;        /* rows in the SELL-32-sigma copy (<= 64 nonzeros)               */
    int64_t seg_rows;         /* rows handled by warp segments                                 */
    int64_t split_rows;       /* rows spanning several segments (finished by an owner CTA)     */
    int64_t sell_elems;       /* SELL entries including padding                                */
    int32_t sigma;            /* SELL sorting window (1 = natural order)                       */
    int32_t variant;          /* 0 (one kernel family; kept for layout compatibility)           */
    int64_t l2_window_bytes;  /* iterate vectors covered by the persisting-L2 access window     */
    double l2_hit_ratio;      /* persisting fraction of that window                            */
    int32_t mode;             /* 0 cooperative grid with a TMA ring, 5 single thread-block cluster,
                                 6 single cluster with the whole solve resident on chip            */
    int32_t l2_mode;          /* L2 policy: 2 all vectors persist, 3 only the x~ buffers persist */
    int32_t launches_per_solve; /* kernel launches of one ajm_solve (L2 priming + init + solver)   */
    int32_t col_bytes;        /* bytes streamed per SELL column index: 4 (int32), or 1 when the
                                 column offsets col - row take <= 256 values and the layout stores
                                 byte codes into an offset table (stencils)        */
    int64_t seg_nnz;          /* nonzeros streamed by warp segments (rows of > 64 nonzeros)       */
    int32_t rank, nranks;     /* sharded handles: this rank / group size (1 for ajm_create)        */
    int64_t halo;             /* sharded handles: halo entries H_lo + H_hi received per pass       */
    int64_t send;             /* sharded handles: entries pushed to other ranks per pass           */
    int64_t group_rows;       /* rows of 65..256 nonzeros run four to a warp (8-lane sub-warp groups) */
    int32_t val_bytes;        /* bytes streamed per SELL value: 8, or 0 when the byte code indexes a
                                 table of <= 256 (value, column offset) pairs (pair-coded entries:
                                 constant-coefficient stencils)                       */
    int32_t band_staged;      /* 1: x~ bands and the row operands are staged by the TMA ring
                                 (ajm_band_kernel; natural-order pair-coded stencils)              */
} ajm_info_t;

/*
 * ajm_create -- validate Q, b (and d), build the device layout and the diagonal metric D.
 *   out       : receives the handle (written only on AJM_OK)
 *   n, nnz    : 1 <= n < 2^31, nnz >= 0 (nnz >= 2^31 only when every row has <= 64 nonzeros,
 *               else AJM_ERR_UNSUPPORTED)
 *   row_ptr   : int64[n+1], canonical CSR offsets (row_ptr[0] = 0, nondecreasing, row_ptr[n] = nnz)
 *   col_idx   : int32[nnz], strictly increasing within each row, 0 <= col < n
 *   vals      : double[nnz]; BOTH triangles of the symmetric Q are stored
 *   b         : double[n], consistent right-hand side (b in range(Q) is assumed, not checked)
 *   dmode     : ajm_dmode_t
 *   d         : double[n] (> 0) for AJM_D_USER, otherwise ignored (may be NULL)
 *   flags     : AJM_VALIDATE_SYMMETRY | AJM_LOOP_HOST | AJM_JBLOCK_SIZE(bs) (AJM_D_JBLOCK only) |
 *               the layout switches above
 * Ownership: the handle deep-copies (and re-lays-out) Q, b and D into device memory it owns; the
 * caller's buffers may be freed when the call returns.
 * Side effects: device memory comes from a library-owned stream-ordered pool that keeps up to
 * 16 GiB of freed memory for later creates; when the six iterate vectors fit the L2 the call
 * raises the device's cudaLimitPersistingL2CacheSize to min(their size, the device maximum) so a
 * persisting access-policy window can keep them resident (a device-wide setting); when
 * the last handle that raised it is destroyed the previous limit is restored and the persisting
 * lines are reset (cudaCtxResetPersistingL2Cache).
 */
ajm_status_t ajm_create(ajm_handle_t* out, int64_t n, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const double* vals, const double* b,
                        int32_t dmode, const double* d, uint32_t flags, void* cuda_stream);

/*
 * ajm_solve -- run Algorithm 3 from x0 until ||b - Q x~^t||/||b|| <= tol (converged; x_out = x~^t,
 * R5), t = maxit (x_out = post-iteration x^t, R10) or divergence (res > 1e8 or non-finite, R19).
 *   x0            : double[n] initial point (NULL = zeros, the paper's/configs' x0 = 0)
 *   tol           : >= 0 (0 = run to maxit unless the residual is exactly 0)
 *   maxit         : >= 1
 *   policy        : see ajm_policy_t
 *   x_out         : double[n] (host or device), receives the answer
 *   res           : host, receives the ajm_result_t (may be NULL)
 *   res_hist,f_hist : host double[maxit+1] or NULL; entry t (0 <= t <= iterations) is the relative
 *                   residual / f of the pre-restart iterate x~^t; t = 0 is x0
 *   restart_iters : host int64[restart_cap] or NULL; iterations t at which a restart executed, in
 *                   order (ell <= log2(t+2) - 1 < 64)
 * The whole iteration loop runs on the device: ONE cooperative launch of a persistent kernel with a
 * grid barrier per iteration; the restart rule, the alpha/beta schedule and the stopping test are
 * evaluated on the device; there is no host round trip and no relaunch per iteration.  The
 * handle's previous solve state is overwritten.
 */
ajm_status_t ajm_solve(ajm_handle_t h, const double* x0, double tol, int64_t maxit,
                       ajm_policy_t policy, double* x_out, ajm_result_t* res, double* res_hist,
                       double* f_hist, int64_t* restart_iters, int64_t restart_cap,
                       void* cuda_stream);

/*
 * ajm_get_trace -- copy a per-iteration trace of the last solve to host out[count]:
 *   which = 0 res (as res_hist), 1 f (as f_hist), 2 the restart inner product
 *   d_t = <Q y^t - b, x~^t - x^{t-1}> (entry 0 = 0), 3 sum_i |(Qy^t - b)_i (x~^t - x^{t-1})_i|
 *   (the tie-ratio denominator of DESIGN.md R17).  count <= iterations + 1.
 */
ajm_status_t ajm_get_trace(ajm_handle_t h, int32_t which, double* out, int64_t count);

/* ajm_get_diag -- copy the diagonal metric D actually used (J for AJM_D_JDIAG; the diagonal of the
 * block J for AJM_D_JBLOCK) to out[n] (host/device). */
ajm_status_t ajm_get_diag(ajm_handle_t h, double* out);

/* ajm_get_jblock -- AJM_D_JBLOCK handles only: copy the blocks J^{ii} of eq-J-blkdiag to
 * out[s * bs * bs] (host/device), s = ceil(n / bs), block i row-major at out + i*bs*bs; the ragged
 * last block is padded with the identity.  Other handles: AJM_ERR_INVALID_ARG. */
ajm_status_t ajm_get_jblock(ajm_handle_t h, double* out);

/* Extreme eigenvalues of D^{-1} Q for the handle's metric D (AJM_D_QDIAG: the Jacobi metric diag(Q)
 * of P:54-69, whose omega_opt = 2 / (lambda_min + lambda_max)(D^{-1} Q) is the optimal weight of
 * weighted Jacobi, eq-weighted-jacobi P:61-69; AJM_D_JDIAG: J^{-1} Q, whose lambda_max <= 1 since
 * S = J - Q is PSD). */
typedef struct {
    double lambda_min, lambda_max; /* extreme Ritz values of the Lanczos tridiagonal T_k            */
    double err_min, err_max;       /* residual bounds beta_k |s_k|: |lambda - theta| <= err (each
                                      extreme Ritz value is within err of an eigenvalue)            */
    double omega_opt;              /* 2 / (lambda_min + lambda_max)                                 */
    int64_t steps;                 /* k, the Lanczos steps in T_k (one SpMV pass each, plus one)    */
    int32_t converged;             /* err_min, err_max <= tol * max(|lambda_min|, |lambda_max|)     */
    int32_t breakdown;             /* beta_k = 0: an invariant subspace, the values are exact       */
} ajm_spectrum_t;

/*
 * ajm_estimate_spectrum -- Lanczos on M = D^{-1} Q in the D-inner product (M is similar to the
 * symmetric D^{-1/2} Q D^{-1/2}) without reorthogonalisation (the extreme Ritz values
 * converge regardless), running on the handle's own SpMV: one fused persistent pass per step with
 * the Lanczos recurrence in the epilogue, launched in chunks of passes; between
 * chunks the host computes the extreme eigenvalues of T_k (Sturm bisection) and their residual
 * bounds (inverse iteration), and stops once both bounds are <= tol * max|lambda| or at max_steps.
 *   v0        : double[n] start vector (host/device, caller's row order), or NULL = a fixed
 *               counter-based pseudo-random vector of `seed` (independent of the layout)
 *   max_steps : 1 .. 2^20;  tol >= 0 (0: run max_steps)
 *   out       : host, the estimate;  alpha, beta: host double[max_steps] or NULL, receive the
 *               coefficients alpha_1..alpha_k (diagonal of T_k) and beta_1..beta_k
 * Errors: AJM_ERR_UNSUPPORTED for AJM_D_JBLOCK handles; AJM_ERR_NONFINITE for a non-finite v0 or
 * coefficient.  The handle's solver state is not touched (a workspace of 8 n-vectors is allocated
 * on first use and kept).
 */
ajm_status_t ajm_estimate_spectrum(ajm_handle_t h, const double* v0, uint64_t seed, int64_t max_steps,
                                   double tol, ajm_spectrum_t* out, double* alpha, double* beta,
                                   void* cuda_stream);

/*
 * ---- Row-block sharded solve (NEXT-2): the paper's own parallel design ----
 * Alg. 3 lines 3-5 ("for i = 1, ..., s parallel") with the row partition of
 * §3 and §4.4 (Q, x, y partitioned by rows, J built locally): rank r of an
 * s = nranks group owns the contiguous global rows [row_starts[r], row_starts[r+1]) of Q, b, D and
 * of every iterate.  Each pass, every rank multiplies its rows by x~^t -- its own entries plus a
 * halo of the entries its rows reference on other ranks -- and the ranks exchange (a) the halo
 * entries of x~^{t+1}, pushed straight into the readers' buffers by the producing CTA (peer stores
 * over NVLink / NVSwitch; IPC-mapped between processes), and (b) the five partial sums of the
 * residual / f / restart reductions, summed in rank order so every rank takes the same (bitwise)
 * control decisions.  One persistent kernel per rank runs the whole solve; there is no host round
 * trip per pass.  D = eq-J-diag needs only the rank's own rows (J built locally), so the
 * iterates are those of the single-GPU solve up to the summation order of the reductions.
 * Local numbering of a rank with n_loc own rows: own row i (global row_starts[r] + i) is i; the
 * halo entries, sorted by global index, are -H_lo .. -1 (owned by lower ranks) and
 * n_loc .. n_loc + H_hi - 1 (higher ranks), so a contiguous slab of a stencil keeps its offsets.
 * Q must be structurally symmetric across the partition (it is, being symmetric): rank r's send
 * list to rank s (the rows of r that s's rows reference) is derived from r's own rows.
 * Supported metrics: AJM_D_JDIAG, AJM_D_USER, AJM_D_QDIAG (not AJM_D_JBLOCK).  Not thread-safe
 * across the ranks of one group except as described per call.
 */
#define AJM_MAX_RANKS 8
#define AJM_SHARD_BLOB_BYTES 1024      /* size of the opaque connection record of one rank            */
#define AJM_SHARD_COLOCATED 0x200000u  /* create flag: every rank of the group lives on this device
                                          (an emulated group, run by ajm_group_solve as ONE launch over
                                          all ranks); the rank's grid is 1/nranks of the device       */

/* ajm_partition_rows -- host only (no GPU): contiguous row blocks balanced by the per-pass bytes
 * 12 B per nonzero + 56 B per row, every block non-empty.
 *   row_ptr    : host int64[n+1] of the whole matrix
 *   row_starts : host int64[nranks+1] out: block r is [row_starts[r], row_starts[r+1])
 * The paper's load imbalance p * max_i nnz(Q^{i,:}) / nnz(Q) follows from it.
 * Errors: INVALID_ARG for nranks < 1, nranks > AJM_MAX_RANKS or nranks > n; CSR_INVALID for a bad
 * row_ptr. */
ajm_status_t ajm_partition_rows(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* row_starts);

/* ajm_shard_plan -- host only (no GPU): rank `rank`'s local numbering and exchange lists.
 *   row_starts : host int64[nranks+1] (row_starts[0] = 0, increasing; row_starts[nranks] = n)
 *   row_ptr    : host int64[n_loc+1] of the rank's rows (local offsets, row_ptr[0] = 0)
 *   col_glob   : host int32[nnz_loc] global columns of those rows
 *   col_loc    : host int32[nnz_loc] out (or NULL): local columns in [-H_lo, n_loc + H_hi)
 *   halo_glob  : host int64[H_lo + H_hi] out (or NULL): global index of local -H_lo + k, in order
 *   send_rows  : host int64[sum send] out (or NULL): local rows to send, grouped by destination rank
 *                (ascending), ascending within a group -- the order of the destination's halo
 *   counts     : host int64[2 + 2*nranks] out: H_lo, H_hi, then halo entries per source rank, then
 *                send entries per destination rank (by symmetry: the rows of this rank that have a
 *                column in the destination's block)
 * Errors: INVALID_ARG, CSR_INVALID (column out of [0, n) or row_ptr inconsistent). */
ajm_status_t ajm_shard_plan(int32_t rank, int32_t nranks, const int64_t* row_starts, const int64_t* row_ptr,
                            const int32_t* col_glob, int32_t* col_loc, int64_t* halo_glob, int64_t* send_rows,
                            int64_t* counts);

/* ajm_shard_create -- rank `rank`'s handle of a sharded group, on the current device.
 *   row_starts        : host int64[nranks+1], the same on every rank (e.g. ajm_partition_rows)
 *   nnz, row_ptr, col_idx, vals : the rank's rows row_starts[rank] .. row_starts[rank+1] as CSR with
 *                       GLOBAL int32 column indices (host or device memory)
 *   b, d              : the rank's slices (d: AJM_D_USER only)
 *   flags             : AJM_SHARD_COLOCATED | the layout switches of ajm_create
 * The handle can be solved only after ajm_shard_connect.  Ownership and errors as ajm_create
 * (a zero local b is allowed; ||b|| = 0 of the whole b is reported by ajm_shard_connect). */
ajm_status_t ajm_shard_create(ajm_handle_t* out, int32_t rank, int32_t nranks, const int64_t* row_starts,
                              int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                              const double* b, int32_t dmode, const double* d, uint32_t flags,
                              void* cuda_stream);

/* ajm_shard_export -- write this rank's connection record (AJM_SHARD_BLOB_BYTES, host) to blob:
 * CUDA IPC handles and offsets of its iterate buffers and exchange block, its halo layout per
 * source rank and its local ||b||^2.  The caller all-gathers the records (e.g. torch.distributed). */
ajm_status_t ajm_shard_export(ajm_handle_t h, void* blob);

/* ajm_shard_connect -- map every rank's buffers (same process: the pointers themselves, with peer
 * access enabled across devices; another process: cudaIpcOpenMemHandle) from the nranks records
 * `blobs` (host, rank order, AJM_SHARD_BLOB_BYTES each), check that each rank's halo from this rank
 * matches this rank's send list (else AJM_ERR_NOT_SYMMETRIC), and set ||b||_2 = sqrt of the ranks'
 * ||b_r||^2 summed in rank order (AJM_ERR_ZERO_RHS if 0).  Once per handle. */
ajm_status_t ajm_shard_connect(ajm_handle_t h, const void* blobs);

/* ajm_solve on a connected shard handle: the same call on every rank of the group, concurrently
 * (one process per GPU), with the same tol / maxit / policy; x0 and x_out are the rank's own rows
 * (n_loc); res, res_hist, f_hist and restart_iters are the whole solve's (identical on every rank).
 * A rank that cannot reach the others fails with AJM_ERR_CUDA after a bounded wait (seconds). */

/* ajm_group_solve -- an AJM_SHARD_COLOCATED group (all ranks on this device, connected): run the
 * sharded solve as ONE cooperative launch over every rank's CTAs (the same kernel and exchange as a
 * multi-GPU group; peers are plain device pointers).
 *   hs     : host array of the nranks handles in rank order
 *   x0     : double[n] of the WHOLE system (host/device) or NULL = zeros;  x_out : double[n] out
 *   other arguments as ajm_solve. */
ajm_status_t ajm_group_solve(const ajm_handle_t* hs, int32_t nranks, const double* x0, double tol,
                             int64_t maxit, ajm_policy_t policy, double* x_out, ajm_result_t* res,
                             double* res_hist, double* f_hist, int64_t* restart_iters, int64_t restart_cap,
                             void* cuda_stream);

/* ajm_get_info -- layout and last-solve timing facts. */
ajm_status_t ajm_get_info(ajm_handle_t h, ajm_info_t* info);

/* ajm_destroy -- free all device memory of the handle (h may be NULL). */
ajm_status_t ajm_destroy(ajm_handle_t h);

/* ajm_last_error -- message of the last failing call on h; h = NULL gives the calling thread's last
 * ajm_create failure.  The string is owned by the library and valid until the next call. */
const char* ajm_last_error(ajm_handle_t h);

/* ajm_abi_version -- AJM_ABI_VERSION of the loaded library. */
int32_t ajm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AJM_H_ */
