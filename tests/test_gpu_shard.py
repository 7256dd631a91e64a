"""NEXT-2: the row-block sharded solve (Alg. 3 lines 3-5 "for i = 1..s parallel"; §4.4
P:771) through the C ABI, run as an emulated group on one GPU (AJM_SHARD_COLOCATED: every rank's
CTAs in ONE cooperative launch -- the multi-GPU kernel and halo/partial exchange with the peers
being plain device pointers), against the CPU oracle of the unsharded method.

The sharded iterates differ from the single-GPU ones only in the order of the residual / f /
restart reductions (rank partials summed in rank order), so the same parity bar holds:
max-rel 1e-10 after 1000 iterations, iterations-to-tol within +-1, histories entry by entry."""
import numpy as np
import pytest

import oracle
import synth
from _gpu_helpers import PARITY_TOL, gpu_solve, max_rel, oracle_matching, oracle_threads, requires_cuda

pytestmark = [pytest.mark.gpu, requires_cuda]


@pytest.fixture(scope="module", autouse=True)
def _threads():
    oracle_threads()


def group_solve(p, nranks, x0=None, tol=0.0, maxit=1000, restart=True, momentum=True, **kw):
    import paper_2407_03272_b200 as ajm
    with ajm.ShardGroup.from_csr(p.Q, p.b, nranks, **kw) as g:
        r = g.solve(x0=x0, tol=tol, maxit=maxit, restart=restart, momentum=momentum)
        r.x = r.x.cpu().numpy()
        r.infos = [g.info(k) for k in range(nranks)]
        r.starts = g.starts.copy()
        r.imbalance = g.load_imbalance(p.Q.row_ptr)
    return r


CASES = [(1, 1.0, 2), (1, 1.0, 3), (2, 0.25, 4), (3, 0.02, 2), (3, 0.02, 8), (4, 0.0125, 4), (5, 0.09375, 2)]


@pytest.mark.parametrize("cfg,scale,nranks", CASES)
def test_shard_parity_1000_iterations(cfg, scale, nranks):
    p = synth.config_problem(cfg, scale)
    g = group_solve(p, nranks, tol=0.0, maxit=1000, restart=True)
    o, nforced = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=1000, restart=True)
    assert g.status == o.status and g.iterations == o.iterations == 1000
    assert max_rel(g.x, o.x) <= PARITY_TOL, (cfg, nranks, max_rel(g.x, o.x), nforced)
    k = g.iterations + 1
    assert np.all(np.abs(g.res_hist - o.res_hist[:k]) <= 1e-9 * o.res_hist[:k] + 1e-12 * o.res_hist[0])
    fstar = -0.5 * float(np.dot(p.b, p.x_star))
    assert np.abs(g.f_hist - o.f_hist[:k]).max() <= 1e-10 * max(1.0, abs(fstar))
    assert [i["nranks"] for i in g.infos] == [nranks] * nranks
    assert sum(i["n"] for i in g.infos) == p.Q.n
    assert all(i["halo"] > 0 for i in g.infos)  # every block reads a neighbour
    # P:771-775 load imbalance p * max nnz_i / nnz of the byte-balanced split (the Chung-Lu hub rows
    # make the smallest graph case the least even: 1.21 at 4 ranks)
    assert 1.0 <= g.imbalance <= 1.3, g.imbalance


@pytest.mark.parametrize("cfg,scale,nranks", [(2, 0.25, 2), (3, 0.02, 4), (4, 0.0125, 2)])
def test_shard_iterations_to_tol(cfg, scale, nranks):
    p = synth.config_problem(cfg, scale)
    g = group_solve(p, nranks, tol=1e-6, maxit=5000)
    o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.status == "converged" and o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1, (g.iterations, o.iterations)
    assert g.res_hist[-1] <= 1e-6
    if g.iterations == o.iterations:
        assert max_rel(g.x, o.x) <= 1e-8


def test_one_rank_group_is_bitwise_the_single_gpu_solve(monkeypatch):
    """nranks = 1: the rank partial plus zeros is the partial, the grid and layout are the
    single-GPU ones -> bitwise the same iterates and histories."""
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")  # single GPU: the band kernel on the generic plan
    p = synth.config_problem(2, 0.25)
    g = group_solve(p, 1, tol=0.0, maxit=300)
    s = gpu_solve(p.Q, p.b, tol=0.0, maxit=300)
    np.testing.assert_array_equal(g.x, s.x)
    np.testing.assert_array_equal(g.res_hist, s.res_hist)
    np.testing.assert_array_equal(g.f_hist, s.f_hist)


def test_shard_determinism_x0_and_policies():
    p = synth.config_problem(3, 0.02)
    x0 = synth.random_vector(p.Q.n, 77)
    a = group_solve(p, 3, x0=x0, tol=0.0, maxit=200, restart=False)
    b = group_solve(p, 3, x0=x0, tol=0.0, maxit=200, restart=False)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.res_hist, b.res_hist)
    o = oracle.solve(p.Q, p.b, x0=x0, tol=0.0, maxit=200, restart=False)
    assert max_rel(a.x, o.x) <= PARITY_TOL
    # momentum off: the Jacobi-type gradient step (eq-gd), K0 = 2 irrelevant
    c = group_solve(p, 2, tol=0.0, maxit=100, restart=False, momentum=False)
    oc = oracle.solve(p.Q, p.b, tol=0.0, maxit=100, restart=False, momentum=False)
    assert max_rel(c.x, oc.x) <= PARITY_TOL


def test_shard_long_rows_and_int32_columns():
    """Chung-Lu shards (warp segments, split rows, relabelled windows) and a stencil forced to
    int32 columns."""
    p = synth.config_problem(4, 0.0125)
    g = group_solve(p, 3, tol=0.0, maxit=400)
    o, _ = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=400, restart=True)
    assert max_rel(g.x, o.x) <= PARITY_TOL
    assert any(i["seg_rows"] > 0 for i in g.infos)
    q = synth.config_problem(2, 0.25)
    h = group_solve(q, 2, tol=0.0, maxit=300, int32_columns=True)
    k = group_solve(q, 2, tol=0.0, maxit=300)
    assert h.infos[0]["col_bytes"] == 4 and k.infos[0]["col_bytes"] == 1
    np.testing.assert_array_equal(h.x, k.x)  # the same columns in the same order


def test_shard_errors():
    import paper_2407_03272_b200 as ajm
    p = synth.config_problem(1)
    # structurally asymmetric across the partition: rank 1's rows reference rank 0, not vice versa
    rp = np.array([0, 1, 2, 4], dtype=np.int64)
    col = np.array([0, 1, 0, 2], dtype=np.int32)
    val = np.array([2.0, 2.0, -1.0, 2.0])
    with pytest.raises(ajm.AjmError) as e:
        ajm.ShardGroup(3, rp, col, val, np.ones(3), 2, starts=[0, 2, 3])
    assert e.value.status_name == "AJM_ERR_NOT_SYMMETRIC"
    with pytest.raises(ajm.AjmError) as e:
        ajm.ShardGroup.from_csr(p.Q, np.zeros(p.Q.n), 2)
    assert e.value.status_name == "AJM_ERR_ZERO_RHS"
    with pytest.raises(ajm.AjmError) as e:
        ajm.ShardGroup.from_csr(p.Q, p.b, 2, dmode="jblock")
    with pytest.raises(ajm.AjmError):
        ajm.ShardGroup.from_csr(p.Q, p.b, 9)  # > AJM_MAX_RANKS


def test_shard_solver_per_process_path_one_rank(monkeypatch):
    """The per-process path of bench.py --gpus N (ajm_shard_create without AJM_SHARD_COLOCATED on the
    whole device, the connection records exchanged by the caller, ajm_solve on the shard handle: the
    kernel's own launch with its peer table) with a single rank -- the only size one GPU can run
    concurrently.  Bitwise the single-GPU solve (rank partial + zeros), and the oracle to 1e-10."""
    import paper_2407_03272_b200 as ajm
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")  # single GPU: the band kernel on the generic plan
    for cfg, scale in [(3, 0.02), (2, 0.25)]:
        p = synth.config_problem(cfg, scale)
        with ajm.ShardSolver(0, 1, [0, p.Q.n], p.Q.row_ptr, p.Q.col, p.Q.val, p.b, exchange=lambda b: [b]) as s:
            r = s.solve(tol=0.0, maxit=400)
            x = r.x.cpu().numpy()
            assert s.info()["nranks"] == 1 and s.info()["halo"] == 0
            r2 = s.solve(tol=1e-6, maxit=5000)  # a second solve: the arrival counters continue
        g = gpu_solve(p.Q, p.b, tol=0.0, maxit=400)
        np.testing.assert_array_equal(x, g.x)
        np.testing.assert_array_equal(r.res_hist, g.res_hist)
        o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
        assert abs(r2.iterations - o.iterations) <= 1
