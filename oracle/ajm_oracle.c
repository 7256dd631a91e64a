/*
 * ajm_oracle.c -- plain, slow, obviously-correct CPU oracle for the accelerated Jacobi-type
 * method (AJM) of arXiv 2407.03272.  TEST INFRASTRUCTURE ONLY: it may be linked/called only from
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.  It shares
 * no code, header, table or helper with the CUDA path (paper_2407_03272_b200/csrc).
 *
 * FP64, IEEE round-to-nearest, compiled with -O2 -ffp-contract=off -fno-fast-math (no FMA
 * contraction anywhere, reading R14).
 *
 * What it computes (PAPER.md = P, SPEC.md = S; DESIGN.md §2 lists the readings R1..R21):
 *   - eq-J-diag (§3):  J_kk = Q_kk + sum_{j != k} |Q_kj|   (ascending j)
 *   - eq-J-blkdiag (§3): block-diagonal J with J^{ii} = Q^{ii} + sum_{j != i}||Q^{ij}||_2 I
 *     over contiguous row blocks of bs rows (the last block ragged).  The blocks themselves are
 *     built in oracle/__init__.py (numpy: dense blocks, LAPACK SVD for ||.||_2, LAPACK Cholesky);
 *     this file applies J^{-1} per block by forward and back substitution with the Cholesky factor
 *     (Alg. 3 line 4: (x^t)^i = (y^t)^i + (J^{ii})^{-1}(b^i - sum_j Q^{ij}(y^t)^j)).
 *   - eq-qp:            f(x) = 1/2 <x, Qx> - <b, x>
 *   - stopping rule (§4):  ||b - Qx^t||_2 / ||b||_2 <= tol   (R3)
 *   - Alg. 3 with s = 1, LITERALLY: every iteration does the SpMV Q y^t for the step
 *     (line 4) and a second SpMV Q x^t for the stopping test / trace, i.e. two
 *     SpMVs per iteration.  The step is x^t = y^t + D^{-1}(b - Q y^t) with an IEEE division by
 *     D_k.  Restart test (line 5): t > K_re + K_l and
 *     <Q y^t - b, x^t - x^{t-1}> >= 0 and IsRestart; restart branch lines 6-10; else
 *     lines 12-13: alpha_{t+1} = (1 + sqrt(1 + 4 alpha_t^2))/2 and
 *     y^{t+1} = x^t + ((alpha_t - 1)/alpha_{t+1}) (x^t - x^{t-1}).
 *     alpha_1 = 1.  Momentum off (momentum = 0) gives the variable-metric gradient step
 *     eq-gd: beta = 0, so D = diag(Q) is classical Jacobi eq-jacobi.
 *   - Ordering readings: stop test on x~^t before the restart decision (R5), a restart iteration
 *     counts in t (R6), tie <.> = 0 restarts (R7), divergence guard res > 1e8 or non-finite (R19),
 *     output at maxit is the post-iteration x^t (R10).
 *
 * Optional "mirror" mode is a diagnostic only: it replaces the second SpMV by the GPU path's
 * algebraic identity Q y^{t+1} = Q x^t + beta_t (Q x^t - Q x^{t-1}); tests use it
 * to separate reformulation drift from kernel bugs.  The default (mirror = 0) is the literal
 * definition above.
 *
 * Reductions: fixed 4096-row chunks, each summed sequentially, chunk partials summed
 * sequentially in chunk order -> bitwise identical at any OpenMP thread count.
 * Per-row SpMV sums run in ascending column order starting from 0.0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CHUNK 4096

static int g_threads = 1;

void oracle_set_threads(int nt) { g_threads = nt < 1 ? 1 : nt; }
int oracle_get_threads(void) { return g_threads; }

/* y = Q x : y_i = sum_j Q_ij x_j, ascending j, from 0.0 (S:45 deterministic order). */
void oracle_spmv(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                 const double* x, double* y) {
    int64_t i;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

/* fixed-chunk dot product <a, b> */
static double dot_chunked(int64_t n, const double* a, const double* b, double* part) {
    int64_t nch = (n + CHUNK - 1) / CHUNK, c;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (c = 0; c < nch; ++c) {
        int64_t lo = c * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
        double s = 0.0;
        for (int64_t i = lo; i < hi; ++i) s += a[i] * b[i];
        part[c] = s;
    }
    double s = 0.0;
    for (c = 0; c < nch; ++c) s += part[c];
    return s;
}

/* ||b - Qx||^2 given Qx, fixed chunks */
static double resid_sq_chunked(int64_t n, const double* b, const double* qx, double* part) {
    int64_t nch = (n + CHUNK - 1) / CHUNK, c;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (c = 0; c < nch; ++c) {
        int64_t lo = c * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
        double s = 0.0;
        for (int64_t i = lo; i < hi; ++i) {
            double r = b[i] - qx[i];
            s += r * r;
        }
        part[c] = s;
    }
    double s = 0.0;
    for (c = 0; c < nch; ++c) s += part[c];
    return s;
}

/* f(x) = 1/2 <x, Qx> - <b, x>  (eq-qp), given Qx */
static double objective_from_qx(int64_t n, const double* x, const double* qx, const double* b,
                                double* part) {
    double xqx = dot_chunked(n, x, qx, part);
    double bx = dot_chunked(n, b, x, part);
    return 0.5 * xqx - bx;
}

static double* part_alloc(int64_t n) { return (double*)malloc(sizeof(double) * ((n + CHUNK - 1) / CHUNK + 1)); }

double oracle_dot(int64_t n, const double* a, const double* b) {
    double* part = part_alloc(n);
    double s = dot_chunked(n, a, b, part);
    free(part);
    return s;
}

/* f(x) (eq-qp) with its own SpMV */
double oracle_objective(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                        const double* b, const double* x) {
    double* qx = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* part = part_alloc(n);
    oracle_spmv(n, rp, ci, v, x, qx);
    double f = objective_from_qx(n, x, qx, b, part);
    free(qx);
    free(part);
    return f;
}

/* ||b - Qx||_2 / ||b||_2 (R3).  Returns NAN when ||b|| = 0. */
double oracle_rel_residual(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                           const double* b, const double* x) {
    double* qx = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* part = part_alloc(n);
    oracle_spmv(n, rp, ci, v, x, qx);
    double rr = resid_sq_chunked(n, b, qx, part);
    double bb = dot_chunked(n, b, b, part);
    free(qx);
    free(part);
    if (bb == 0.0) return NAN;
    return sqrt(rr) / sqrt(bb);
}

/* eq-J-diag: J_kk = Q_kk + sum_{j != k}|Q_kj|, the off-diagonal sum in ascending j.
 * Returns 0 ok; 1 if some Q_kk < 0 (Q cannot be SPSD); 2 if some J_kk == 0 (zero row);
 * 3 if a value is not finite. */
int oracle_build_jdiag(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                       double* J) {
    int err = 0;
    for (int64_t k = 0; k < n; ++k) {
        double qkk = 0.0, off = 0.0;
        for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
            if (!isfinite(v[p])) err = err ? err : 3;
            if (ci[p] == k) qkk = v[p];
            else off += fabs(v[p]);
        }
        if (qkk < 0.0) err = err ? err : 1;
        J[k] = qkk + off;
        if (J[k] == 0.0) err = err ? err : 2;
    }
    return err;
}

/* diag(Q): D_kk = Q_kk, 0 if absent */
void oracle_diag(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, double* d) {
    for (int64_t k = 0; k < n; ++k) {
        d[k] = 0.0;
        for (int64_t p = rp[k]; p < rp[k + 1]; ++p)
            if (ci[p] == k) d[k] = v[p];
    }
}

/* Alg. 1 line 4 / Alg. 3 line 13: alpha_{t+1} = (1 + sqrt(1 + 4 alpha_t^2)) / 2 */
double oracle_alpha_next(double a) { return (1.0 + sqrt(1.0 + 4.0 * a * a)) / 2.0; }

/* z = J^{-1} r for block-diagonal J given its per-block lower Cholesky factors L (J^{ii} = L L^T,
 * row-major bs x bs per block; the ragged last block uses its leading m x m corner).
 * Forward substitution L w = r, then back substitution L^T z = w, textbook order. */
static void block_chol_solve(int64_t n, int64_t bs, const double* L, const double* r, double* z) {
    int64_t nblk = (n + bs - 1) / bs, blk;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (blk = 0; blk < nblk; ++blk) {
        const int64_t base = blk * bs;
        const int64_t m = (base + bs <= n) ? bs : n - base;
        const double* Lb = L + (size_t)blk * (size_t)(bs * bs);
        double* w = z + base;
        for (int64_t k = 0; k < m; ++k) { /* L w = r */
            double s = r[base + k];
            for (int64_t j = 0; j < k; ++j) s -= Lb[k * bs + j] * w[j];
            w[k] = s / Lb[k * bs + k];
        }
        for (int64_t k = m - 1; k >= 0; --k) { /* L^T z = w (in place) */
            double s = w[k];
            for (int64_t j = k + 1; j < m; ++j) s -= Lb[j * bs + k] * w[j];
            w[k] = s / Lb[k * bs + k];
        }
    }
}

enum { OR_CONVERGED = 0, OR_MAXITER = 1, OR_DIVERGED = 2 };

/*
 * Alg. 3, s = 1, diagonal D (= J from eq-J-diag by default; the caller passes D).
 *
 * inputs : CSR Q (n, rp, ci, v), b[n], D[n] (> 0), x0[n] (NULL = zeros), tol (>= 0), maxit (>= 1),
 *          momentum (0/1), restart (0/1 = IsRestart), k0 (K_0 >= 2), mirror (0 literal / 1 identity),
 *          forced[maxit+1] (NULL, or per-t forced restart decision: -1 none, 0 no, 1 yes; R17 tie
 *          protocol -- the t > K_re + K_l window is still required);
 *          bs, Lfac: block-diagonal J (eq-J-blkdiag) -- if Lfac != NULL the step applies J^{-1} by
 *          per-block Cholesky solves (block_chol_solve) and D is ignored.
 * outputs: x_out[n]; res_hist/f_hist[maxit+1] (entry t is for x~^t, the pre-restart iterate);
 *          d_hist/dabs_hist[maxit+1] (restart inner product <Qy^t - b, x~^t - x^{t-1}> and the sum of
 *          |terms| for the tie ratio, entry 0 unused = 0); xt_hist[(maxit+1)*n] post-iteration x^t
 *          (the returned x~^t at a converged/diverged exit)
 *          and alpha_hist[maxit+1] alpha_t (tiny n only, for the Lyapunov/bound pins); any may be NULL.
 *          restart_iters[restart_cap]; info[6] = {status, iterations, n_restarts, x_is_prerestart,
 *          restarts_logged, 0}.
 * returns 0, or -1 on bad arguments, -2 on ||b|| = 0, -3 on allocation failure.
 */
int oracle_ajm_solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                     const double* b, const double* D, const double* x0, double tol, int64_t maxit,
                     int momentum, int restart, int64_t k0, int mirror, const int8_t* forced,
                     int64_t bs, const double* Lfac, double* x_out, double* res_hist, double* f_hist, double* d_hist,
                     double* dabs_hist, double* xt_hist, double* alpha_hist,
                     int64_t* restart_iters, int64_t restart_cap, int64_t* info) {
    if (n < 1 || maxit < 1 || !(tol >= 0.0) || k0 < 2 || (restart && !momentum)) return -1;
    if (Lfac && bs < 1) return -1;
    size_t bytes = sizeof(double) * (size_t)n;
    double *x = malloc(bytes), *x_prev = malloc(bytes), *y = malloc(bytes), *xt = malloc(bytes);
    double *qy = malloc(bytes), *qx = malloc(bytes), *qx_prev = malloc(bytes);
    double* part = part_alloc(n);
    int rc = 0;
    if (!x || !x_prev || !y || !xt || !qy || !qx || !qx_prev || !part) {
        rc = -3; /* allocation failure: free what was allocated (free(NULL) is a no-op) */
        goto cleanup;
    }

    for (int64_t i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
    double nb2 = dot_chunked(n, b, b, part);
    if (nb2 == 0.0) {
        rc = -2;
        goto cleanup;
    }
    double nb = sqrt(nb2);

    /* t = 0: residual and f of x^0 */
    oracle_spmv(n, rp, ci, v, x, qx);
    double res = sqrt(resid_sq_chunked(n, b, qx, part)) / nb;
    if (res_hist) res_hist[0] = res;
    if (f_hist) f_hist[0] = objective_from_qx(n, x, qx, b, part);
    if (d_hist) d_hist[0] = 0.0;
    if (dabs_hist) dabs_hist[0] = 0.0;
    if (xt_hist) memcpy(xt_hist, x, bytes);
    if (alpha_hist) alpha_hist[0] = 0.0; /* alpha_0 = 0 */
    int64_t status = OR_MAXITER, iters = maxit, nres = 0, prerestart = 0, logged = 0;
    if (res <= tol) {
        status = OR_CONVERGED;
        iters = 0;
        memcpy(x_out, x, bytes);
        goto done;
    }

    /* x^0 = y^1, alpha_1 = 1, l = 0, K_l = K_0, K_re = 0 */
    memcpy(x_prev, x, bytes);
    memcpy(y, x, bytes);
    memcpy(qy, qx, bytes); /* Q y^1 = Q x^0 (used only by the mirror mode) */
    memcpy(qx_prev, qx, bytes);
    double alpha = 1.0;
    int64_t K = k0, Kre = 0;

    for (int64_t t = 1; t <= maxit; ++t) {
        if (alpha_hist) alpha_hist[t] = alpha;
        /* Alg. 3 line 4: x~^t = y^t + D^{-1}(b - Q y^t) */
        if (!mirror) oracle_spmv(n, rp, ci, v, y, qy);
        if (!Lfac) {
            for (int64_t i = 0; i < n; ++i) xt[i] = y[i] + (b[i] - qy[i]) / D[i];
        } else { /* eq-J-blkdiag: x~ = y + J^{-1}(b - Q y), block by block */
            for (int64_t i = 0; i < n; ++i) xt[i] = b[i] - qy[i];
            block_chol_solve(n, bs, Lfac, xt, xt);
            for (int64_t i = 0; i < n; ++i) xt[i] = y[i] + xt[i];
        }

        /* stopping rule on x~^t (R5) and trace */
        oracle_spmv(n, rp, ci, v, xt, qx);
        res = sqrt(resid_sq_chunked(n, b, qx, part)) / nb;
        if (res_hist) res_hist[t] = res;
        if (f_hist) f_hist[t] = objective_from_qx(n, xt, qx, b, part);

        /* restart inner product <Q y^t - b, x~^t - x^{t-1}>, fixed chunks */
        double d = 0.0, dabs = 0.0;
        {
            int64_t nch = (n + CHUNK - 1) / CHUNK, c;
            double* part2 = part_alloc(n);
#pragma omp parallel for schedule(static) num_threads(g_threads)
            for (c = 0; c < nch; ++c) {
                int64_t lo = c * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
                double s = 0.0, sa = 0.0;
                for (int64_t i = lo; i < hi; ++i) {
                    double term = (qy[i] - b[i]) * (xt[i] - x_prev[i]);
                    s += term;
                    sa += fabs(term);
                }
                part[c] = s;
                part2[c] = sa;
            }
            for (c = 0; c < nch; ++c) {
                d += part[c];
                dabs += part2[c];
            }
            free(part2);
        }
        if (d_hist) d_hist[t] = d;
        if (dabs_hist) dabs_hist[t] = dabs;

        int do_restart = 0;
        if (restart && t > Kre + K) {
            do_restart = (d >= 0.0); /* tie => restart (R7) */
            if (forced && forced[t] >= 0) do_restart = forced[t];
        }

        if (res <= tol) { /* converged: answer is x~^t even if a restart would discard it (R5) */
            status = OR_CONVERGED;
            iters = t;
            prerestart = do_restart;
            memcpy(x_out, xt, bytes);
            if (xt_hist) memcpy(xt_hist + (size_t)t * (size_t)n, xt, bytes);
            goto done;
        }
        if (!(res <= 1e8)) { /* divergence guard (R19), also catches NaN */
            status = OR_DIVERGED;
            iters = t;
            memcpy(x_out, xt, bytes);
            if (xt_hist) memcpy(xt_hist + (size_t)t * (size_t)n, xt, bytes);
            goto done;
        }

        if (do_restart) { /* Alg. 3 lines 6-10 */
            Kre = t;
            K = 2 * K;
            nres += 1;
            if (restart_iters && logged < restart_cap) restart_iters[logged++] = t;
            alpha = 1.0; /* alpha_{t+1} = 1 (alpha_t = 0 only names the fresh epoch, R9) */
            memcpy(y, x_prev, bytes); /* y^{t+1} = x^{t-1} */
            memcpy(x, x_prev, bytes); /* x^t = x^{t-1}; x_prev (= x^{t-1}) unchanged */
            if (mirror) memcpy(qy, qx_prev, bytes);
        } else { /* lines 12-13 */
            double a_next = (1.0 + sqrt(1.0 + 4.0 * alpha * alpha)) / 2.0;
            double beta = momentum ? (alpha - 1.0) / a_next : 0.0;
            for (int64_t i = 0; i < n; ++i) y[i] = xt[i] + beta * (xt[i] - x_prev[i]);
            if (mirror)
                for (int64_t i = 0; i < n; ++i) qy[i] = qx[i] + beta * (qx[i] - qx_prev[i]);
            memcpy(x_prev, xt, bytes);
            memcpy(x, xt, bytes);
            if (mirror) memcpy(qx_prev, qx, bytes);
            alpha = a_next;
        }
        if (xt_hist) memcpy(xt_hist + (size_t)t * (size_t)n, x, bytes);
    }
    /* MaxIterReached: output the post-iteration x^t (R10) */
    memcpy(x_out, x, bytes);

done:
    info[0] = status;
    info[1] = iters;
    info[2] = nres;
    info[3] = prerestart;
    info[4] = logged;
    info[5] = 0;
cleanup:
    free(x); free(x_prev); free(y); free(xt); free(qy); free(qx); free(qx_prev); free(part);
    return rc;
}
