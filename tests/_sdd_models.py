"""Exact models of the PAPER.md §4.1 experiment on Q = (n+1)I - 11^T, b = 1, x0 = 0.

Every iterate of Jacobi, weighted Jacobi and Alg. 3 on this system is a scalar multiple c*1 of the
all-ones vector (Q(c 1) = c 1 and every diagonal metric used is a multiple of I), so the iterations
reduce to scalar recurrences.  These models are PINNED against the oracle's full iteration in
tests/test_oracle_pins.py (test_sdd_jacobi_closed_form, test_sdd_ajm_scalar_recurrence), and the GPU
test of the experiment (tests/test_gpu_parity.py::test_sdd_paper_experiment) and tools/exp_sdd.py
use these same pinned functions -- there is no second, unpinned copy."""
import math


def closed_form_rate_iters(rate, tol, maxit):
    """Iterations for (Jacobi / weighted-Jacobi) residual rate^t to reach tol."""
    t = math.ceil(math.log(tol) / math.log(rate))
    return (t, "converged") if t <= maxit else (maxit, "maxiter")


def sdd_scalar_ajm(n, tol, maxit, restart=True, k0=2):
    """Alg. 3 restricted to span{1}: J = (2n - 1) I (eq-J-diag), Q(c 1) = c 1 and
    <u 1, v 1> = n u v.  Returns (iterations, residual history, restart iterations)."""
    cx_prev = cy = 0.0
    alpha, K, Kre = 1.0, k0, 0
    res_hist = [1.0]
    rest = []
    for t in range(1, maxit + 1):
        cxt = cy + (1.0 - cy) / (2 * n - 1)
        res = abs(1.0 - cxt)
        res_hist.append(res)
        d = n * (cy - 1.0) * (cxt - cx_prev)
        if res <= tol:
            return t, res_hist, rest
        if restart and t > Kre + K and d >= 0:
            Kre, K = t, 2 * K
            rest.append(t)
            alpha = 1.0
            cy = cx_prev
        else:
            an = (1 + math.sqrt(1 + 4 * alpha * alpha)) / 2
            beta = (alpha - 1) / an
            cy = cxt + beta * (cxt - cx_prev)
            cx_prev = cxt
            alpha = an
    return maxit, res_hist, rest
