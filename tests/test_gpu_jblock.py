"""Block-diagonal J of eq-J-blkdiag (R23) on the
GPU vs the CPU oracle: the blocks J^{ii} themselves, then Alg. 3 iterates with x~ = y + J^{-1}(b - Qy)
applied block by block.  Bar as for eq-J-diag: max-relative 1e-10 after 1000 FP64
iterations, iterations-to-tol within +-1."""
import numpy as np
import pytest

import oracle
import synth
from _gpu_helpers import (PARITY_TOL, assert_history_parity, gpu_solve, max_rel, oracle_matching, oracle_threads,
                          requires_cuda)

pytestmark = [pytest.mark.gpu, requires_cuda]


@pytest.fixture(scope="module", autouse=True)
def _threads():
    oracle_threads()


CASES = [(1, 1.0, 2), (1, 1.0, 8), (1, 1.0, 32), (2, 0.25, 4), (2, 0.25, 16), (5, 0.09375, 8), (3, 0.004, 4)]


@pytest.mark.parametrize("cfg,scale,bs", CASES)
def test_jblocks_match_oracle(cfg, scale, bs):
    """J^{ii} = Q^{ii} + sum_j ||Q^{ij}||_2 I: GPU (Jacobi eigenvalues of B^T B) vs oracle (LAPACK
    SVD); the shift differs from the oracle's only by rounding of the spectral norms."""
    p = synth.config_problem(cfg, scale)
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=1, jblock=bs)
    Jo = oracle.build_jblock(p.Q, bs)
    assert g.J.shape == Jo.shape
    np.testing.assert_allclose(g.J, Jo, rtol=1e-13, atol=1e-13 * np.abs(Jo).max())
    np.testing.assert_allclose(g.D, np.einsum("ikk->ik", Jo).ravel()[: p.Q.n], rtol=1e-13)


@pytest.mark.parametrize("cfg,scale,bs", CASES)
@pytest.mark.parametrize("restart", [True, False])
def test_jblock_parity_1000_iterations(cfg, scale, bs, restart):
    p = synth.config_problem(cfg, scale)
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=1000, restart=restart, jblock=bs)
    o, nforced = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=1000, restart=restart, jblock=bs)
    assert g.iterations == o.iterations == 1000
    assert max_rel(g.x, o.x) <= PARITY_TOL, (cfg, bs, max_rel(g.x, o.x), nforced)
    assert_history_parity(g, o, fstar=-0.5 * float(np.dot(p.b, p.x_star)))


@pytest.mark.parametrize("cfg,scale,bs", [(1, 1.0, 4), (2, 0.25, 8), (5, 0.09375, 4)])
def test_jblock_iterations_to_tol(cfg, scale, bs):
    p = synth.config_problem(cfg, scale)
    g = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True, jblock=bs)
    o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True, jblock=bs)
    assert g.status == o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1
    assert max_rel(g.x, o.x) <= PARITY_TOL


def test_jblock_single_block_solves_in_one_step():
    """bs >= n: J = Q so one step gives Q^{-1} b -- n = 32, one warp-wide block."""
    Q = synth.random_spd(32, seed=7)
    A = synth.to_dense(Q)
    b = A @ np.linspace(-1, 1, 32)
    g = gpu_solve(Q, b, tol=1e-12, maxit=5, jblock=32)
    assert g.status == "converged" and g.iterations == 1
    np.testing.assert_allclose(g.x, np.linalg.solve(A, b), rtol=1e-10, atol=1e-12)


def test_jblock_thm23_on_gpu_history():
    """Thm 2.3 with S = J - Q for the block J, on the GPU's own f history (restart off)."""
    p = synth.config_problem(2, 0.25)
    bs = 8
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=False, jblock=bs)
    J = g.J
    xs = p.x_star
    Jx = np.einsum("ikl,il->ik", J, np.pad(xs, (0, J.shape[0] * bs - p.Q.n)).reshape(-1, bs)).ravel()[: p.Q.n]
    S_norm = float(xs @ Jx - xs @ p.b)  # ||x0 - x*||_S^2 with x0 = 0, Qx* = b
    fstar = -0.5 * float(p.b @ xs)
    t = np.arange(1, len(g.f_hist))
    slack = 1e-9 * max(1.0, abs(fstar))
    assert np.all(g.f_hist[1:] - fstar <= 2.0 * S_norm / (t + 1) ** 2 + slack)


def test_jblock_errors():
    import paper_2407_03272_b200 as ajm
    Q = synth.sdd(100)  # rows of 100 nonzeros: the blocks cannot be solved inside a warp
    with pytest.raises(ajm.AjmError) as e:
        ajm.Solver.from_csr(Q, np.ones(100), jblock=4)
    assert e.value.status_name == "AJM_ERR_UNSUPPORTED"
    P = synth.poisson2d(8)
    with pytest.raises(ajm.AjmError) as e:
        ajm.Solver.from_csr(P, np.ones(64), jblock=3)
    assert e.value.status_name == "AJM_ERR_INVALID_ARG"


@pytest.mark.parametrize("bs", [2, 4, 8, 16])
def test_jblock_pair_coded_bitwise(bs):
    """Block J on a constant-coefficient stencil takes the pair-coded layout (one byte per entry
    names value and column offset): bitwise the iterates and histories of the same
    block-J solve on int32 columns, and at parity with the oracle."""
    p = synth.make_problem("p3d36", synth.poisson3d(36), 13)  # n = 46656, several units per CTA
    a = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, jblock=bs)
    assert a.info["val_bytes"] == 0 and a.info["col_bytes"] == 1, a.info
    r = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, jblock=bs, int32_columns=True)
    assert r.info["val_bytes"] == 8 and r.info["col_bytes"] == 4
    for f in ("x", "res_hist", "f_hist", "d_trace"):
        np.testing.assert_array_equal(getattr(a, f), getattr(r, f))
    o, _ = oracle_matching(p.Q, p.b, a, tol=0.0, maxit=400, restart=True, jblock=bs)
    assert max_rel(a.x, o.x) <= PARITY_TOL
