"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times (default kernel
variant, persistent cooperative launch).  The oracle runs the literal two-SpMV Alg. 3 on the host
cores; where 1000 oracle iterations would take too long the comparison is on a bounded number of
iterations and completed by properties that hold at any size (Thm 2.3 on the GPU's f history)."""
import numpy as np
import pytest

import oracle
import synth
from _gpu_helpers import (PARITY_TOL, assert_history_parity, gpu_solve, max_rel, oracle_matching, oracle_threads,
                          requires_cuda)

pytestmark = [pytest.mark.gpu, pytest.mark.slow, requires_cuda]


@pytest.fixture(scope="module", autouse=True)
def _threads():
    oracle_threads()


@pytest.fixture(scope="module")
def cfg2():
    return synth.config_problem(2)


def test_config2_full_1000_iterations(cfg2):
    """north_star target: the FP64 3D 7-pt 128^3 solve matches the oracle to 1e-10 after 1000
    iterations (restart on)."""
    p = cfg2
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=1000, restart=True)
    assert g.info["col_bytes"] == 1  # byte-coded columns (7 offsets), as bench.py runs it
    o, nforced = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=1000, restart=True)
    assert g.iterations == o.iterations == 1000
    assert max_rel(g.x, o.x) <= PARITY_TOL, (max_rel(g.x, o.x), nforced)
    assert_history_parity(g, o, fstar=-0.5 * float(np.dot(p.b, p.x_star)))


def test_config2_full_iterations_to_tol(cfg2):
    p = cfg2
    g = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.status == o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1
    assert max_rel(g.x, o.x) <= PARITY_TOL
    if g.iterations == o.iterations:
        assert_history_parity(g, o, fstar=-0.5 * float(np.dot(p.b, p.x_star)))
    # the answer really solves the system (scipy, independent of both)
    A = p.Q.scipy()
    assert np.linalg.norm(p.b - A @ g.x) / np.linalg.norm(p.b) <= 1e-6


def test_config3_full_to_tol_and_200_iterations():
    p = synth.config_problem(3)
    g = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.status == o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1
    assert max_rel(g.x, o.x) <= PARITY_TOL
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=200, restart=True)
    o, _ = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=200, restart=True)
    assert max_rel(g.x, o.x) <= PARITY_TOL


def test_config4_full_to_tol():
    """Chung-Lu n = 4M (skewed rows up to ~1e5): split rows, warp segments and sorted-window SELL."""
    p = synth.config_problem(4)
    g = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.info["split_rows"] > 0 and g.info["seg_rows"] > 0
    o, _ = oracle_matching(p.Q, p.b, g, tol=1e-6, maxit=5000, restart=True)
    assert g.status == o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1
    assert max_rel(g.x, o.x) <= PARITY_TOL


@pytest.fixture(scope="module")
def cfg5():
    return synth.config_problem(5)


def test_config5_full_to_tol(cfg5):
    """Anisotropic 27-pt 256^3 (449M nonzeros), the bench's restarted solve to 1e-6: iterations
    within +-1 of the oracle (literal two-SpMV Alg. 3 on the host cores, ~400 iterations), the
    answers within 1e-10, and -- when the counts agree -- the whole residual / f / restart history."""
    p = cfg5
    g = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.info["col_bytes"] == 1 and g.info["sigma"] == 1  # byte-coded columns (27 offsets)
    o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.status == o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1, (g.iterations, o.iterations)
    assert max_rel(g.x, o.x) <= PARITY_TOL
    if g.iterations == o.iterations:
        assert_history_parity(g, o, fstar=-0.5 * float(np.dot(p.b, p.x_star)))


def test_config5_full_thm23(cfg5):
    """Thm 2.3 evaluated on the GPU's own f history over 300 restart-free iterations at
    the full size: f(x^t) - f* <= 2 ||x0 - x*||_S^2 / (t+1)^2 with f* = -1/2 <b, x*>, S = J - Q."""
    p = cfg5
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, restart=False)
    J = oracle.build_jdiag(p.Q)
    xs = p.x_star
    fstar = -0.5 * float(np.dot(p.b, xs))
    S_norm = float(np.dot(J * xs, xs) - np.dot(xs, p.b))  # ||x0 - x*||_S^2 with x0 = 0, Qx* = b
    t = np.arange(1, len(g.f_hist))
    bound = 2.0 * S_norm / (t + 1) ** 2
    gap = g.f_hist[1:] - fstar
    slack = 1e-9 * max(1.0, abs(fstar))
    assert np.all(gap <= bound + slack)
    assert np.all(gap >= -slack)


def test_config2_full_block_j_1000_iterations(cfg2):
    """eq-J-blkdiag at the full 128^3 size, bs = 4: blocks 1e-13, iterates 1e-10."""
    p = cfg2
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=1000, restart=True, jblock=4)
    Jo = oracle.build_jblock(p.Q, 4)
    np.testing.assert_allclose(g.J, Jo, rtol=1e-13, atol=1e-13 * np.abs(Jo).max())
    o, nforced = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=1000, restart=True, jblock=4)
    assert g.iterations == o.iterations == 1000
    assert max_rel(g.x, o.x) <= PARITY_TOL, (max_rel(g.x, o.x), nforced)
