"""Pins for the CPU oracle (oracle/): each test ties an oracle function to something OTHER than the
oracle itself -- SPEC worked values (tests/golden), dense Cholesky / pseudo-inverse solves, the
paper's theorems (Thm 2.3, Lemma 2.2, Lemma 2.4, Thm 2.5 and its restart-count bound), the alpha
identities, textbook Jacobi / weighted Jacobi, and the §4.1 closed forms.  CPU only.

Citations: PAPER.md = P:<line>, SPEC.md = S:<line>; readings R# are listed in DESIGN.md §2.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth

GOLDEN_MATRICES = {
    "sdd3": lambda: synth.sdd(3),
    "sdd4": lambda: synth.sdd(4),
    "identity3": lambda: synth.diag_matrix(np.ones(3)),
    "path3": lambda: synth.from_dense(np.array([[1., -1, 0], [-1, 2, -1], [0, -1, 1]])),
}


def _instances(kind):
    """Seeded tiny instances (S:570-572 acceptance #2-#4 sizes)."""
    out = []
    if kind in ("spd", "all"):
        for k, n in enumerate([8, 16, 32, 64] * 5):
            out.append(("spd", synth.random_spd(n, seed=100 + k)))
        out.append(("spd", synth.sdd(50)))
    if kind in ("lap", "all"):
        for k, n in enumerate([8, 12, 16, 32, 48]):
            out.append(("lap", synth.random_laplacian(n, seed=200 + k)))
    return out


def _xstar(kind, A, b):
    if kind == "spd":
        return sla.cho_solve(sla.cho_factor(A), b)
    return np.linalg.pinv(A) @ b


def _rhs(A, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    xs = g.uniform(-1, 1, A.shape[0])
    return A @ xs


# ------------------------------------------------------------------------------------------------
# golden worked values (tests/golden/spec_worked_values.json, each entry carries its citation)
# ------------------------------------------------------------------------------------------------

def test_golden_alpha(golden):
    for e in golden["alpha_next"]:
        assert oracle.alpha_next(e["alpha"]) == pytest.approx(e["expected"], rel=1e-15), e["cite"]


def test_golden_jdiag(golden):
    for e in golden["jdiag"]:
        J = oracle.build_jdiag(GOLDEN_MATRICES[e["matrix"]]())
        np.testing.assert_array_equal(J, e["expected"], err_msg=e["cite"])


def test_golden_residual_objective(golden):
    for e in golden["rel_residual"]:
        Q = GOLDEN_MATRICES[e["matrix"]]()
        assert oracle.rel_residual(Q, e["b"], e["x"]) == pytest.approx(e["expected"], abs=1e-15), e["cite"]
    for e in golden["objective"]:
        Q = GOLDEN_MATRICES[e["matrix"]]()
        assert oracle.objective(Q, e["b"], e["x"]) == pytest.approx(e["expected"], abs=1e-15), e["cite"]


def test_golden_one_step(golden):
    for e in golden["one_step"]:
        Q = GOLDEN_MATRICES[e["matrix"]]()
        jb = int(e["dmode"][6:]) if e["dmode"].startswith("jblock") else None
        r = oracle.solve(Q, np.array(e["b"], float), tol=0.0, maxit=1, restart=False,
                         momentum=(e["dmode"] != "qdiag"), dmode=e["dmode"] if jb is None else "jdiag",
                         jblock=jb)
        np.testing.assert_allclose(r.x, e["expected_x1"], rtol=1e-15, err_msg=e["cite"])


def test_golden_omega_opt(golden):
    """omega_opt = 2/(lmin + lmax)(D^-1 Q) on the §4.1 matrix, by dense eigenvalues."""
    for e in golden["omega_opt"]:
        A = synth.to_dense(synth.sdd(e["n"]))
        D = np.diag(oracle.diag(synth.sdd(e["n"])))
        lam = np.linalg.eigvals(np.linalg.solve(D, A)).real
        assert 2.0 / (lam.min() + lam.max()) == pytest.approx(e["expected"], rel=1e-12), e["cite"]


# ------------------------------------------------------------------------------------------------
# spectrum / omega_opt
# ------------------------------------------------------------------------------------------------

def test_spectrum_golden_and_sdd_closed_form(golden):
    """§4.1 matrix with D = diag(Q) = nI: D^{-1}Q has eigenvalues 1/n and (n+1)/n, so omega_opt =
    2n/(n+2) (golden 4/3 at n = 4)."""
    for e in golden["omega_opt"]:
        r = oracle.spectrum(synth.sdd(e["n"]))
        assert r.omega_opt == pytest.approx(e["expected"], rel=1e-12), e["cite"]
    for n in (4, 50, 700):
        r = oracle.spectrum(synth.sdd(n))
        assert r.lambda_min == pytest.approx(1 / n, rel=1e-11)
        assert r.lambda_max == pytest.approx((n + 1) / n, rel=1e-12)
        assert r.omega_opt == pytest.approx(2 * n / (n + 2), rel=1e-12)


def _poisson_closed_form(m, dim):
    """Dirichlet Laplacian on an m^dim grid, D = diag(Q) = 2 dim I: the eigenvalues of D^{-1}Q are
    (1/(2 dim)) sum_a 4 sin^2(k_a pi / (2(m+1))), k_a = 1..m."""
    s = 4 * np.sin(np.arange(1, m + 1) * np.pi / (2 * (m + 1))) ** 2
    return dim * s[0] / (2 * dim), dim * s[-1] / (2 * dim)


@pytest.mark.parametrize("dim,m", [(2, 12), (2, 64), (3, 9), (3, 40)])
def test_spectrum_poisson_closed_form(dim, m):
    """Dense (n <= 3000) and ARPACK (larger n) paths against the closed form."""
    Q = synth.poisson2d(m) if dim == 2 else synth.poisson3d(m)
    lo, hi = _poisson_closed_form(m, dim)
    r = oracle.spectrum(Q)
    assert r.lambda_min == pytest.approx(lo, rel=1e-9)
    assert r.lambda_max == pytest.approx(hi, rel=1e-12)
    assert r.method == ("dense eigvalsh" if Q.n <= 3000 else "ARPACK eigsh")


def test_spectrum_diagonal_and_jdiag_bound():
    """Q diagonal: D^{-1}Q = I, omega_opt = 1; with D = J of eq-J-diag, S = J - Q is PSD
    (P:482), so lambda_max(J^{-1}Q) <= 1 -- and = 1 exactly for a bipartite Laplacian (a path)."""
    r = oracle.spectrum(synth.diag_matrix(np.array([1.0, 3.0, 0.25, 8.0])))
    assert r.lambda_min == pytest.approx(1.0) and r.lambda_max == pytest.approx(1.0) and r.omega_opt == pytest.approx(1.0)
    for seed in range(3):
        Q = synth.random_spd(40, seed=seed)
        assert oracle.spectrum(Q, dmode="jdiag").lambda_max <= 1.0 + 1e-12
    P = synth.from_dense(np.diag([1.0, 2.0, 2.0, 1.0]) - np.diag([1.0] * 3, 1) - np.diag([1.0] * 3, -1))
    r = oracle.spectrum(P, dmode="jdiag")
    assert r.lambda_min == pytest.approx(0.0, abs=1e-14) and r.lambda_max == pytest.approx(1.0, rel=1e-13)


@pytest.mark.parametrize("seed", range(3))
def test_omega_opt_minimises_spectral_radius(seed):
    """omega_opt is the minimiser of rho(I - omega D^{-1} Q): a brute-force scan of the
    spectral radius (nonsymmetric dense eigenvalues of I - omega D^{-1}Q) over omega never beats it,
    and rho at omega_opt equals (kappa - 1)/(kappa + 1)."""
    Q = synth.random_spd(12, seed=seed)
    A = synth.to_dense(Q)
    M = A / np.diag(A)[:, None]
    r = oracle.spectrum(Q)
    rho = lambda w: float(np.abs(np.linalg.eigvals(np.eye(12) - w * M)).max())
    best = min(rho(w) for w in np.linspace(1e-3, 2.0 / r.lambda_max, 4001))
    kappa = r.lambda_max / r.lambda_min
    assert rho(r.omega_opt) <= best + 1e-12
    assert rho(r.omega_opt) == pytest.approx((kappa - 1) / (kappa + 1), rel=1e-10)


# ------------------------------------------------------------------------------------------------
# building blocks against dense brute force
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(5))
def test_spmv_objective_residual_vs_dense(seed):
    Q = synth.random_spd(16, seed=seed)
    A = synth.to_dense(Q)
    x = np.random.Generator(np.random.PCG64(seed)).uniform(-1, 1, 16)
    b = np.arange(16.0) - 3
    np.testing.assert_allclose(oracle.spmv(Q, x), A @ x, rtol=1e-13, atol=1e-13)
    assert oracle.objective(Q, b, x) == pytest.approx(0.5 * x @ A @ x - b @ x, rel=1e-13, abs=1e-13)
    assert oracle.rel_residual(Q, b, x) == pytest.approx(np.linalg.norm(b - A @ x) / np.linalg.norm(b), rel=1e-13)


def test_jdiag_makes_S_psd():
    """eq-J-diag is chosen so that S = J - Q is PSD; S:567 acceptance #5."""
    for kind, Q in _instances("all"):
        A = synth.to_dense(Q)
        J = oracle.build_jdiag(Q)
        # J_kk = Q_kk + sum_{j != k}|Q_kj| restated from the dense matrix
        np.testing.assert_allclose(J, np.diag(A) + (np.abs(A).sum(1) - np.abs(np.diag(A))), rtol=1e-14)
        lam = np.linalg.eigvalsh(np.diag(J) - A)
        assert lam.min() >= -1e-10 * max(1.0, np.abs(A).max())


def test_jdiag_errors():
    with pytest.raises(oracle.OracleError):
        oracle.build_jdiag(synth.from_dense(np.array([[1.0, 0], [0, 0]]), drop_zeros=False))
    with pytest.raises(oracle.OracleError):
        oracle.build_jdiag(synth.from_dense(np.array([[-1.0, 0], [0, 1]])))
    with pytest.raises(oracle.OracleError):
        oracle.rel_residual(synth.diag_matrix(np.ones(3)), np.zeros(3), np.ones(3))
    with pytest.raises(oracle.OracleError):
        oracle.solve(synth.diag_matrix(np.ones(3)), np.zeros(3))
    with pytest.raises(oracle.OracleError):
        oracle.solve(synth.diag_matrix(np.ones(3)), np.ones(3), k0=1)
    with pytest.raises(oracle.OracleError):
        oracle.solve(synth.diag_matrix(np.ones(3)), np.ones(3), momentum=False, restart=True)


# ------------------------------------------------------------------------------------------------
# P1: dense solves
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("restart", [False, True])
def test_dense_solve_spd(restart):
    """north_star / S:574: converged AJM iterate equals the Cholesky solution."""
    for kind, Q in _instances("spd")[::3]:
        A = synth.to_dense(Q)
        b = _rhs(A, 7)
        xs = _xstar("spd", A, b)
        r = oracle.solve(Q, b, tol=1e-12, maxit=200000, restart=restart)
        assert r.status == "converged"
        kappa = np.linalg.cond(A)
        err = np.linalg.norm(r.x - xs) / np.linalg.norm(xs)
        assert err <= max(1e-8, 10 * kappa * 1e-12), (Q.n, err, kappa)


def test_dense_solve_laplacian_range_component():
    """Singular SPSD: residual -> 0 and the range(Q) component matches pinv(Q) b."""
    for kind, Q in _instances("lap"):
        A = synth.to_dense(Q)
        b = _rhs(A, 9)
        xp = np.linalg.pinv(A) @ b
        r = oracle.solve(Q, b, tol=1e-12, maxit=200000, restart=True)
        assert r.status == "converged"
        P = np.eye(Q.n) - np.ones((Q.n, Q.n)) / Q.n  # projector onto range(L) for a connected graph
        assert np.linalg.norm(P @ (r.x - xp)) / np.linalg.norm(xp) <= 1e-8


def test_dense_solve_config1_cholesky():
    """Config 1 (BASELINE configs[0]) is Cholesky-feasible: the converged iterate matches."""
    p = synth.config_problem(1)
    A = synth.to_dense(p.Q)
    xs = sla.cho_solve(sla.cho_factor(A), p.b)
    np.testing.assert_allclose(xs, p.x_star, atol=1e-10)  # the planted solution is the solution
    r = oracle.solve(p.Q, p.b, tol=1e-12, maxit=20000, restart=True)
    assert r.status == "converged"
    assert np.abs(r.x - xs).max() / np.abs(xs).max() <= 1e-9


# ------------------------------------------------------------------------------------------------
# P2/P3: Thm 2.3 and Lemma 2.2 (restart off)
# ------------------------------------------------------------------------------------------------

def _gap(A, b, xs, X):
    """f(x) - f* = 1/2 <x - x*, Q(x - x*)> (stable form, R11); X rows are iterates."""
    E = X - xs
    return 0.5 * np.einsum("ij,jk,ik->i", E, A, E)


def test_thm23_bound_and_lemma22_lyapunov():
    """Thm 2.3: 0 <= f(x^t) - f* <= 2||x0 - x*||_S^2/(t+1)^2; Lemma 2.2:
    alpha_t^2 (f(x^t) - f*) + 1/2 <w^t, S w^t> nonincreasing, w^t = alpha_t x^t - (alpha_t - 1)x^{t-1} - x*.
    S = J - Q.  Acceptance S:570-571 (t <= 500, slack 1e-10 max(1,|f*|), 1e-9)."""
    for kind, Q in _instances("all"):
        A = synth.to_dense(Q)
        b = _rhs(A, 11)
        xs = _xstar(kind, A, b)
        J = oracle.build_jdiag(Q)
        S = np.diag(J) - A
        r = oracle.solve(Q, b, tol=0.0, maxit=500, restart=False, record_iterates=True)
        X = r.xt_hist
        T = X.shape[0] - 1
        gap = _gap(A, b, xs, X)
        fstar = -0.5 * b @ xs
        slack = 1e-10 * max(1.0, abs(fstar))
        e0 = X[0] - xs
        R0 = e0 @ S @ e0
        t = np.arange(1, T + 1)
        bound = 2 * R0 / (t + 1) ** 2
        assert np.all(gap[1:] >= -slack)
        assert np.all(gap[1:] <= bound + slack), (Q.n, kind)
        # the recorded f history obeys the same bound (f* = -1/2 <b, x*> for any x* with Qx* = b)
        assert np.all(r.f_hist[1:] - fstar <= bound + slack)
        # Lyapunov
        al = r.alpha_hist
        Et = [0.5 * R0]
        for k in range(1, T + 1):
            w = al[k] * X[k] - (al[k] - 1) * X[k - 1] - xs
            Et.append(al[k] ** 2 * gap[k] + 0.5 * w @ S @ w)
        assert np.all(np.diff(Et) <= 1e-9), (Q.n, kind, np.max(np.diff(Et)))


def test_alpha_schedule():
    """alpha_1 = 1, alpha_2 = golden ratio, alpha_{t-1}^2 = alpha_t(alpha_t - 1),
    alpha_t >= (t+1)/2 (T10)."""
    Q = synth.random_spd(8, seed=1)
    r = oracle.solve(Q, _rhs(synth.to_dense(Q), 1), tol=0.0, maxit=300, restart=False,
                     record_iterates=True)
    al = r.alpha_hist
    assert al[0] == 0.0 and al[1] == 1.0
    assert al[2] == pytest.approx((1 + math.sqrt(5)) / 2, rel=1e-15)
    t = np.arange(2, len(al))
    np.testing.assert_allclose(al[t] * (al[t] - 1), al[t - 1] ** 2, rtol=1e-12)
    assert np.all(al[1:] >= (np.arange(1, len(al)) + 1) / 2 - 1e-12)


# ------------------------------------------------------------------------------------------------
# P4/P5/P6: restart mode
# ------------------------------------------------------------------------------------------------

def _restart_count(restart_iters, T):
    ell = np.zeros(T + 1, dtype=int)
    for tr in restart_iters:
        ell[tr:] += 1
    return ell


def test_lemma24_thm25_restart_count():
    """Lemma 2.4: f(x^t) <= f(x^0); within an epoch f(x^{l,k}) <= f(x^{l,0}); anchors
    nonincreasing.  Thm 2.5 proof: l <= log2(t+2) - 1.  Thm 2.5 (proven form
    P:400-417 with t' = accepted iterates, R12) on SPD with R^2 = 2(f(x0) - f*) lambda_max(Q^-1 S)."""
    n_restart_runs = 0
    for kind, Q in _instances("all"):
        A = synth.to_dense(Q)
        b = _rhs(A, 13)
        xs = _xstar(kind, A, b)
        J = oracle.build_jdiag(Q)
        S = np.diag(J) - A
        r = oracle.solve(Q, b, tol=0.0, maxit=500, restart=True, k0=2, record_iterates=True)
        X = r.xt_hist
        T = X.shape[0] - 1
        gap = _gap(A, b, xs, X)
        assert np.all(gap <= gap[0] + 1e-9)
        ell = _restart_count(r.restart_iters, T)
        t = np.arange(T + 1)
        assert np.all(ell[1:] <= np.log2(t[1:] + 2) - 1 + 1e-12)
        # epochs / anchors: x^{l,0} = x^0 and, after a restart at t_r, x^{t_r} (= x^{t_r - 1})
        anchors = [0] + list(r.restart_iters)
        for a0, a1 in zip(anchors, anchors[1:] + [T + 1]):
            assert np.all(gap[a0:a1] <= gap[a0] + 1e-9)
        ga = gap[anchors]
        assert np.all(np.diff(ga) <= 1e-9)
        n_restart_runs += bool(r.restart_iters)
        if kind == "spd":
            lam = sla.eigh(S, A, eigvals_only=True)
            R2 = 2 * gap[0] * max(lam.max(), 0.0)
            tp = t - ell  # accepted iterates (restart iterations excluded)
            ok = tp >= 2
            proven = 2 * R2 * np.log2(tp[ok] + 2) ** 2 / tp[ok] ** 2
            assert np.all(gap[ok] <= proven + 1e-10)
    assert n_restart_runs >= 5  # the restart branch is actually exercised


# ------------------------------------------------------------------------------------------------
# P8: reductions to Jacobi / weighted Jacobi (momentum off)
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("omega", [1.0, 0.7])
def test_jacobi_reduction(omega):
    """Momentum off with D = diag(Q)/omega is eq-weighted-jacobi; omega = 1 is eq-jacobi
    (P:55-58), written here in its first form D^{-1}(b - (L + L^T)x)."""
    for Q in [synth.poisson2d(6), synth.aniso27(3), synth.sdd(20)]:
        A = synth.to_dense(Q)
        b = _rhs(A, 3)
        d = np.diag(A).copy()
        LU = A - np.diag(d)
        r = oracle.solve(Q, b, D=d / omega, tol=0.0, maxit=60, momentum=False, restart=False,
                         record_iterates=True)
        x = np.zeros(Q.n)
        for t in range(1, 61):
            x = omega * (b - LU @ x) / d + (1 - omega) * x
            assert np.abs(r.xt_hist[t] - x).max() <= 1e-13 * max(1.0, np.abs(x).max()), t


# ------------------------------------------------------------------------------------------------
# P9: §4.1 strictly diagonally dominant system closed forms
# ------------------------------------------------------------------------------------------------

def test_sdd_jacobi_closed_form():
    """Q = (n+1)I - 11^T, b = 1, x0 = 0: Jacobi iterates stay c_t 1 with 1 - c_t = (1 - 1/n)^t, so the
    relative residual is (1 - 1/n)^t; weighted Jacobi with omega_opt = 2n/(n+2) contracts by
    1 - 2/(n+2)."""
    n = 50
    Q = synth.sdd(n)
    b = np.ones(n)
    r = oracle.solve(Q, b, tol=0.0, maxit=300, momentum=False, restart=False, dmode="qdiag")
    t = np.arange(301)
    np.testing.assert_allclose(r.res_hist, (1 - 1 / n) ** t, rtol=1e-10, atol=1e-15)
    w = 2 * n / (n + 2)
    r = oracle.solve(Q, b, D=np.full(n, n / w), tol=0.0, maxit=300, momentum=False, restart=False)
    np.testing.assert_allclose(r.res_hist, (1 - 2 / (n + 2)) ** t, rtol=1e-10, atol=1e-13)
    # the iteration-count model used by the GPU experiment test (tests/_sdd_models.py)
    from _sdd_models import closed_form_rate_iters
    for rate, D in ((1 - 1 / n, None), (1 - 2 / (n + 2), np.full(n, n / w))):
        it, st = closed_form_rate_iters(rate, 1e-4, 5000)
        r = oracle.solve(Q, b, D=D, dmode="qdiag", tol=1e-4, maxit=5000, momentum=False, restart=False)
        assert (r.status, abs(r.iterations - it) <= 1) == (st, True)


from _sdd_models import sdd_scalar_ajm as _sdd_scalar_ajm  # noqa: E402 (the pinned model)


@pytest.mark.parametrize("n,restart", [(300, True), (300, False), (64, True)])
def test_sdd_ajm_scalar_recurrence(n, restart):
    Q = synth.sdd(n)
    r = oracle.solve(Q, np.ones(n), tol=1e-6, maxit=5000, restart=restart)
    it, hist, rest = _sdd_scalar_ajm(n, 1e-6, 5000, restart)
    assert r.iterations == it
    assert r.restart_iters == rest
    np.testing.assert_allclose(r.res_hist, hist, rtol=1e-7, atol=1e-12)


def test_sdd_paper_claim_n1000():
    """P:521, P:564 (S:569 acceptance #1 ordering): on n = 1000, tol 1e-4, maxiter 5000 the
    restarted AJM converges, while classical Jacobi needs ceil(ln 1e-4 / ln(1 - 1/n)) > 5000
    iterations (closed form pinned in test_sdd_jacobi_closed_form)."""
    n = 1000
    oracle.set_threads(4)
    try:
        r = oracle.solve(synth.sdd(n), np.ones(n), tol=1e-4, maxit=5000, restart=True)
    finally:
        oracle.set_threads(1)
    assert r.status == "converged" and r.iterations < 1000
    jac = math.ceil(math.log(1e-4) / math.log(1 - 1 / n))
    assert jac > 5000 and r.iterations < jac


# ------------------------------------------------------------------------------------------------
# P10-P12, determinism
# ------------------------------------------------------------------------------------------------

def test_trivial_cases():
    """x0 = x* converges at t = 0; diagonal Q with eq-J-diag gives J = Q, x^1 = Q^{-1} b
    exactly."""
    p = synth.config_problem(1)
    r = oracle.solve(p.Q, p.b, x0=p.x_star, tol=1e-10)
    assert r.status == "converged" and r.iterations == 0
    np.testing.assert_array_equal(r.x, p.x_star)
    d = np.array([1.0, 2.0, 4.0, 0.5])
    b = np.array([3.0, -1.0, 2.0, 7.0])
    r = oracle.solve(synth.diag_matrix(d), b, tol=1e-15, maxit=5)
    assert r.status == "converged" and r.iterations == 1
    np.testing.assert_array_equal(r.x, b / d)


@pytest.mark.parametrize("restart", [False, True])
def test_mirror_equals_literal(restart):
    """P11: the single-SpMV identity Q y^{t+1} = Q x^t + beta_t (Q x^t - Q x^{t-1}) (derived from
    P:463) reproduces the literal two-SpMV Alg. 3 to rounding after 1000 iterations."""
    p = synth.config_problem(1)
    a = oracle.solve(p.Q, p.b, tol=0.0, maxit=1000, restart=restart)
    m = oracle.solve(p.Q, p.b, tol=0.0, maxit=1000, restart=restart, mirror=True)
    assert np.abs(a.x - m.x).max() / np.abs(a.x).max() <= 1e-13
    if restart:
        assert a.restart_iters[:3] == m.restart_iters[:3]


def test_generator_consistency():
    """P12: b in range(Q) -- Laplacian b sums to zero; x* has zero residual."""
    for cfg, scale in [(1, 1.0), (2, 0.125), (3, 0.002), (4, 0.002), (5, 0.05)]:
        p = synth.config_problem(cfg, scale)
        assert oracle.rel_residual(p.Q, p.b, p.x_star) <= 1e-14
        if cfg == 3:
            assert abs(p.b.sum()) <= 1e-10 * np.abs(p.b).sum()
        A = p.Q.scipy()
        assert abs(A - A.T).max() == 0.0


def test_thread_count_invariance():
    """Fixed 4096-row chunk reductions: bitwise identical at 1 and 4 threads (R15)."""
    p = synth.config_problem(2, 0.25)
    oracle.set_threads(1)
    a = oracle.solve(p.Q, p.b, tol=0.0, maxit=30)
    oracle.set_threads(4)
    try:
        b = oracle.solve(p.Q, p.b, tol=0.0, maxit=30)
    finally:
        oracle.set_threads(1)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.res_hist, b.res_hist)
    np.testing.assert_array_equal(a.f_hist, b.f_hist)


def test_restart_tie_restarts_and_forcing():
    """R7: <.> >= 0 restarts on equality (P:465 '>= 0'); R17 forcing hook changes only the decision."""
    p = synth.config_problem(1)
    base = oracle.solve(p.Q, p.b, tol=0.0, maxit=300, restart=True)
    assert base.restart_iters
    t0 = base.restart_iters[0]
    forced = np.full(301, -1, dtype=np.int8)
    forced[t0] = 0
    alt = oracle.solve(p.Q, p.b, tol=0.0, maxit=300, restart=True, forced=forced)
    assert t0 not in alt.restart_iters
    np.testing.assert_array_equal(alt.res_hist[:t0 + 1], base.res_hist[:t0 + 1])


def test_restart_window_and_doubling():
    """Alg. 3 lines 5-7: a restart needs t > K_re + K_l, then K_re = t and K_{l+1} = 2 K_l.
    Forcing every decision to 'restart' makes restarts fire at the earliest admissible t:
    K0 = 2 -> 3, 8, 17, 34, 67, 132 (t_{l+1} = t_l + 2^l K0 + 1)."""
    p = synth.config_problem(1)
    forced = np.ones(201, dtype=np.int8)
    r = oracle.solve(p.Q, p.b, tol=0.0, maxit=200, restart=True, k0=2, forced=forced)
    assert r.restart_iters == [3, 8, 17, 34, 67, 132]
    r = oracle.solve(p.Q, p.b, tol=0.0, maxit=200, restart=True, k0=5, forced=forced)
    assert r.restart_iters == [6, 17, 38, 79, 160]


# ------------------------------------------------------------------------------------------------
# eq-J-blkdiag: block-diagonal J (R23)
# ------------------------------------------------------------------------------------------------

def _assemble(J, n):
    """Dense n x n block-diagonal matrix from the (s, bs, bs) blocks (drops the identity pad)."""
    s, bs, _ = J.shape
    M = np.zeros((s * bs, s * bs))
    for i in range(s):
        M[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = J[i]
    return M[:n, :n]


def test_golden_jblock(golden):
    for e in golden["jblock"]:
        J = oracle.build_jblock(GOLDEN_MATRICES[e["matrix"]](), e["bs"])
        np.testing.assert_allclose(J, np.array(e["expected_blocks"]), rtol=0, atol=1e-14,
                                   err_msg=e["cite"])


def test_jblock_bs1_is_jdiag():
    """bs = 1: ||[Q_ij]||_2 = |Q_ij|, so eq-J-blkdiag reduces to eq-J-diag, bitwise."""
    for kind, Q in _instances("all")[::3] + [("p", synth.poisson3d(5)), ("a", synth.aniso27(4))]:
        np.testing.assert_array_equal(oracle.build_jblock(Q, 1)[:, 0, 0], oracle.build_jdiag(Q))


def test_jblock_single_block_is_q_and_solves_in_one_step():
    """s = 1 (bs >= n): J = Q with no shift, so Alg. 3 line 4 from any y gives
    y + Q^{-1}(b - Qy) = Q^{-1} b: converged after one iteration (dense Cholesky x*)."""
    for k, n in enumerate([5, 12, 30]):
        Q = synth.random_spd(n, seed=400 + k)
        A = synth.to_dense(Q)
        J = oracle.build_jblock(Q, n)
        np.testing.assert_array_equal(J[0], A)
        b = _rhs(A, k)
        r = oracle.solve(Q, b, tol=1e-12, maxit=3, jblock=n)
        assert r.status == "converged" and r.iterations == 1
        np.testing.assert_allclose(r.x, sla.cho_solve(sla.cho_factor(A), b), rtol=1e-11, atol=1e-12)


def test_jblock_stencil_closed_form():
    """2D / 3D Dirichlet Laplacians with blocks of bs consecutive x-rows (bs | m): every
    off-diagonal block is either -I (y/z neighbours) or a single -1 (x neighbour), both of
    2-norm 1, so J^{ii} = Q^{ii} + (number of neighbouring blocks) I -- no SVD needed."""
    for m, dim, bs in [(8, 2, 4), (8, 2, 2), (6, 3, 3), (8, 3, 8)]:
        Q = synth.poisson2d(m) if dim == 2 else synth.poisson3d(m)
        J = oracle.build_jblock(Q, bs)
        A = synth.to_dense(Q)
        nb = m // bs
        for blk in range(Q.n // bs):
            r0 = blk * bs
            coords = np.unravel_index(r0, (m,) * dim)  # coords[-1] is the fastest (x) axis
            cnt = 0
            for ax in range(dim):
                lim = nb if ax == dim - 1 else m
                c = coords[ax] // bs if ax == dim - 1 else coords[ax]
                cnt += int(c > 0) + int(c < lim - 1)
            expect = A[r0:r0 + bs, r0:r0 + bs] + cnt * np.eye(bs)
            np.testing.assert_array_equal(J[blk], expect)


def test_jblock_s_psd_and_one_step_dense():
    """S = J - Q is PSD for every tested block size, and the oracle's block
    Cholesky step equals a dense solve with the assembled J (brute force)."""
    for kind, Q in _instances("all")[::2]:
        A = synth.to_dense(Q)
        for bs in (2, 3, 4, 8):
            Jd = _assemble(oracle.build_jblock(Q, bs), Q.n)
            lam = np.linalg.eigvalsh(Jd - A)
            assert lam.min() >= -1e-10 * max(1.0, np.abs(A).max()), (kind, Q.n, bs, lam.min())
            b = _rhs(A, bs)
            r = oracle.solve(Q, b, tol=0.0, maxit=1, restart=False, jblock=bs)
            np.testing.assert_allclose(r.x, np.linalg.solve(Jd, b), rtol=1e-12, atol=1e-13)


def test_jblock_thm23_bound():
    """Thm 2.3 with the block-diagonal J of eq-J-blkdiag: S = J - Q."""
    for kind, Q in _instances("all")[::2]:
        A = synth.to_dense(Q)
        b = _rhs(A, 17)
        xs = _xstar(kind, A, b)
        for bs in (2, 4):
            S = _assemble(oracle.build_jblock(Q, bs), Q.n) - A
            r = oracle.solve(Q, b, tol=0.0, maxit=300, restart=False, jblock=bs, record_iterates=True)
            gap = _gap(A, b, xs, r.xt_hist)
            fstar = -0.5 * b @ xs
            slack = 1e-10 * max(1.0, abs(fstar))
            e0 = r.xt_hist[0] - xs
            t = np.arange(1, len(gap))
            assert np.all(gap[1:] <= 2 * (e0 @ S @ e0) / (t + 1) ** 2 + slack), (kind, Q.n, bs)
            assert np.all(gap[1:] >= -slack)
