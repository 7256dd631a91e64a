"""NEXT-3: the extreme eigenvalues of D^{-1} Q and omega_opt = 2/(lmin + lmax) of
weighted Jacobi, estimated on the GPU by Lanczos on the handle's own SpMV
(ajm_estimate_spectrum), against the oracle (dense LAPACK / ARPACK, pinned in test_oracle_pins.py to
the closed forms and to the definition of omega_opt as the minimiser of rho(I - omega D^{-1}Q)).
Bar: each extreme Ritz value within its own residual bound (plus 1e-12 lambda_max for the oracle's
own accuracy) of the oracle's eigenvalue, and the bound itself <= tol * lambda_max."""
import numpy as np
import pytest

import oracle
import synth
from _gpu_helpers import gpu_solve, requires_cuda

pytestmark = [pytest.mark.gpu, requires_cuda]

TOL = 1e-10


def _estimate(Q, dmode, **kw):
    import paper_2407_03272_b200 as ajm
    with ajm.Solver(Q.n, Q.row_ptr, Q.col, Q.val, np.ones(Q.n), dmode=dmode, **kw) as s:
        sp = s.estimate_spectrum(tol=TOL, max_steps=4000)
        info = s.info()
    return sp, info


def _check(sp, lo, hi):
    assert sp.converged or sp.breakdown
    slack = 1e-12 * abs(hi)
    assert abs(sp.lambda_max - hi) <= sp.err_max + slack, (sp.lambda_max, hi, sp.err_max)
    assert abs(sp.lambda_min - lo) <= sp.err_min + slack, (sp.lambda_min, lo, sp.err_min)
    assert sp.err_max <= TOL * abs(hi) * 1.0001 + slack and sp.err_min <= TOL * abs(hi) * 1.0001 + slack


@pytest.mark.parametrize("n", [50, 1000, 3000])
def test_sdd_omega_opt(n):
    """§4.1 matrix, D = diag(Q): eigenvalues 1/n and (n+1)/n, omega_opt = 2n/(n+2); rows of
    n nonzeros: SELL (50), one warp segment (1000), split rows (3000)."""
    sp, info = _estimate(synth.sdd(n), "qdiag")
    _check(sp, 1.0 / n, (n + 1.0) / n)
    assert sp.omega_opt == pytest.approx(2 * n / (n + 2), rel=1e-9)
    assert (info["seg_rows"] > 0) == (n > 64)


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 0.25)])
def test_poisson_closed_form(cfg, scale):
    """Dirichlet Laplacians with D = diag(Q) = 2 dim I: closed-form extreme eigenvalues
    (single-cluster layout for config 1, byte-coded columns for config 2)."""
    p = synth.config_problem(cfg, scale)
    m, dim = p.meta["m"], (2 if cfg == 1 else 3)
    s = 4 * np.sin(np.arange(1, m + 1) * np.pi / (2 * (m + 1))) ** 2
    sp, info = _estimate(p.Q, "qdiag")
    _check(sp, dim * s[0] / (2 * dim), dim * s[-1] / (2 * dim))
    assert info["mode"] == (6 if cfg == 1 else 0)  # (the Lanczos twin of the resident kernel: kCluster)


@pytest.mark.parametrize("cfg,scale", [(2, 0.25), (3, 0.0025), (4, 0.00075), (5, 0.039)])
def test_jdiag_spectrum_vs_oracle(cfg, scale):
    """D = J of eq-J-diag (the AJM metric): lambda_max(J^{-1}Q) <= 1 (S = J - Q PSD) and both
    ends match the oracle; sorted-window / relabelled (3, singular: lambda_min = 0), warp-segment
    (4: 148 rows of 65-147 nonzeros), wide-row byte-coded (5) layouts.  The graph cases are sized
    for the oracle's dense LAPACK path (n <= 3000): ARPACK on them takes minutes."""
    p = synth.config_problem(cfg, scale)
    sp, _ = _estimate(p.Q, "jdiag")
    o = oracle.spectrum(p.Q, dmode="jdiag")
    _check(sp, o.lambda_min, o.lambda_max)
    assert sp.lambda_max <= 1.0 + 1e-12


def test_layout_independence():
    """The default start vector hashes the caller's row index: the Lanczos coefficients of the
    shared-memory-table and global-table kernels (same SpMV summation order) are bitwise equal."""
    import paper_2407_03272_b200 as ajm
    p = synth.config_problem(4, 0.0125)
    out = []
    for gt in (False, True):
        with ajm.Solver.from_csr(p.Q, p.b, global_tables=gt) as s:
            out.append(s.estimate_spectrum(tol=0.0, max_steps=60))
    np.testing.assert_array_equal(out[0].alpha, out[1].alpha)
    np.testing.assert_array_equal(out[0].beta, out[1].beta)
    assert out[0].steps == 60


def test_weighted_jacobi_with_estimated_omega():
    """Weighted Jacobi (momentum off, D = diag(Q)/omega) with the GPU's own omega_opt on the
    §4.1 matrix converges at the optimal rate 1 - 2/(n+2) (tests/_sdd_models.py)."""
    from _sdd_models import closed_form_rate_iters
    n = 1000
    Q = synth.sdd(n)
    sp, _ = _estimate(Q, "qdiag")
    g = gpu_solve(Q, np.ones(n), tol=1e-4, maxit=5000, momentum=False, restart=False, dmode="user",
                  d=oracle.diag(Q) / sp.omega_opt)
    it, st = closed_form_rate_iters(1 - 2 / (n + 2), 1e-4, 5000)
    assert g.status == st and abs(g.iterations - it) <= 1


def test_estimate_errors():
    import paper_2407_03272_b200 as ajm
    p = synth.config_problem(1)
    with ajm.Solver.from_csr(p.Q, p.b, jblock=4) as s:
        with pytest.raises(ajm.AjmError) as e:
            s.estimate_spectrum()
        assert e.value.status_name == "AJM_ERR_UNSUPPORTED"
    with ajm.Solver.from_csr(p.Q, p.b) as s:
        with pytest.raises(ajm.AjmError) as e:
            s.estimate_spectrum(max_steps=0)
        assert e.value.status_name == "AJM_ERR_INVALID_ARG"
        v0 = np.ones(p.Q.n)
        v0[7] = np.nan
        with pytest.raises(ajm.AjmError) as e:
            s.estimate_spectrum(v0=v0)
        assert e.value.status_name == "AJM_ERR_NONFINITE"
        # the solver still solves after an estimate (its state is separate)
        r = s.solve(tol=0.0, maxit=50)
        o = oracle.solve(p.Q, p.b, tol=0.0, maxit=50)
        assert float(np.abs(r.x.cpu().numpy() - o.x).max() / np.abs(o.x).max()) <= 1e-12
