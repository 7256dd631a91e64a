/*
 * poisson3d.c -- the C ABI (include/ajm.h) used directly from plain C, no Python: build the 3D
 * 7-point Dirichlet Laplacian on an m^3 grid (BASELINE config 2 at m = 128), b = Q x* with
 * x*_i = sin(i), solve with Alg. 3 (eq-J-diag, adaptive restart) to a relative residual tol, and
 * report iterations, restarts, the final residual, max|x - x*| and the time per iteration.  Runs
 * up to the hardware: m = 680 is n = 314M rows and 2.2e9 nonzeros (> 2^31) on one B200.
 *
 * build: gcc -O2 -std=c11 -I include examples/poisson3d.c -L paper_2407_03272_b200 -lajm \
 *            -Wl,-rpath,$PWD/paper_2407_03272_b200 -lm -o poisson3d
 * run  : ./poisson3d [m] [tol]
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "ajm.h"

int main(int argc, char** argv) {
    const int64_t m = argc > 1 ? atoll(argv[1]) : 64;
    const double tol = argc > 2 ? atof(argv[2]) : 1e-6;
    const int64_t n = m * m * m;
    int64_t* rp = malloc(sizeof(int64_t) * (size_t)(n + 1));
    int32_t* ci = malloc(sizeof(int32_t) * (size_t)(7 * n));
    double* v = malloc(sizeof(double) * (size_t)(7 * n));
    double *xs = malloc(sizeof(double) * (size_t)n), *b = malloc(sizeof(double) * (size_t)n);
    double* x = malloc(sizeof(double) * (size_t)n);
    if (!rp || !ci || !v || !xs || !b || !x) return 2;
    int64_t nnz = 0;
    rp[0] = 0;
    for (int64_t z = 0; z < m; ++z)
        for (int64_t y = 0; y < m; ++y)
            for (int64_t xx = 0; xx < m; ++xx) {
                const int64_t i = (z * m + y) * m + xx;
                /* ascending columns: z-1, y-1, x-1, diagonal, x+1, y+1, z+1 */
                if (z > 0) { ci[nnz] = (int32_t)(i - m * m); v[nnz++] = -1.0; }
                if (y > 0) { ci[nnz] = (int32_t)(i - m); v[nnz++] = -1.0; }
                if (xx > 0) { ci[nnz] = (int32_t)(i - 1); v[nnz++] = -1.0; }
                ci[nnz] = (int32_t)i; v[nnz++] = 6.0;
                if (xx < m - 1) { ci[nnz] = (int32_t)(i + 1); v[nnz++] = -1.0; }
                if (y < m - 1) { ci[nnz] = (int32_t)(i + m); v[nnz++] = -1.0; }
                if (z < m - 1) { ci[nnz] = (int32_t)(i + m * m); v[nnz++] = -1.0; }
                rp[i + 1] = nnz;
            }
    for (int64_t i = 0; i < n; ++i) xs[i] = sin((double)i);
    for (int64_t i = 0; i < n; ++i) { /* b = Q x* */
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * xs[ci[k]];
        b[i] = s;
    }
    ajm_handle_t h = NULL;
    ajm_status_t st = ajm_create(&h, n, nnz, rp, ci, v, b, AJM_D_JDIAG, NULL, 0, NULL);
    if (st != AJM_OK) { fprintf(stderr, "ajm_create: %d %s\n", (int)st, ajm_last_error(NULL)); return 1; }
    ajm_policy_t pol = {1, 1, 2};
    ajm_result_t res;
    int64_t restarts[64];
    st = ajm_solve(h, NULL, tol, 5000, pol, x, &res, NULL, NULL, restarts, 64, NULL);
    if (st != AJM_OK) { fprintf(stderr, "ajm_solve: %d %s\n", (int)st, ajm_last_error(h)); return 1; }
    double err = 0.0;
    for (int64_t i = 0; i < n; ++i) err = fmax(err, fabs(x[i] - xs[i]));
    ajm_info_t info;
    ajm_get_info(h, &info);
    const double us_it = 1e3 * info.last_loop_ms / (double)info.last_passes;
    printf("{\"m\": %lld, \"n\": %lld, \"nnz\": %lld, \"status\": %d, \"iterations\": %lld, \"restarts\": %d, "
           "\"rel_residual\": %.3e, \"max_abs_err\": %.3e, \"us_per_iteration\": %.2f, "
           "\"model_GBps\": %.1f, \"abi\": %d}\n",
           (long long)m, (long long)n, (long long)nnz, (int)res.status, (long long)res.iterations,
           (int)res.n_restarts, res.rel_residual, err, us_it, info.model_bytes_per_iter / (us_it * 1e3),
           (int)ajm_abi_version());
    ajm_destroy(h);
    free(rp); free(ci); free(v); free(xs); free(b); free(x);
    return res.status == AJM_CONVERGED ? 0 : 3;
}
