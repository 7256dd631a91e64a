"""GPU (C-ABI, sm_100a kernels) vs CPU oracle parity.  North-star bar: after 1000 FP64 iterations
max|x_gpu - x_cpu| / max|x_cpu| <= 1e-10 and iterations-to-tol within +-1 (restart decisions may
flip only at near-ties, R17).  Inputs: seeded synthetic configs (synth/) at sizes the
oracle finishes in seconds, spanning many row units / CTAs and ragged tails."""
import numpy as np
import pytest

import oracle
import synth
from _gpu_helpers import (PARITY_TOL, assert_history_parity, gpu_solve, max_rel, oracle_matching,
                          oracle_threads, requires_cuda)

pytestmark = [pytest.mark.gpu, requires_cuda]


@pytest.fixture(scope="module", autouse=True)
def _threads():
    oracle_threads()


# (config, scale) pairs: oracle-sized versions of BASELINE configs 1-5
CASES = [(1, 1.0), (2, 0.25), (3, 0.02), (4, 0.0125), (5, 0.09375)]


@pytest.mark.parametrize("cfg,scale", CASES)
@pytest.mark.parametrize("restart", [True, False])
def test_parity_1000_iterations(cfg, scale, restart):
    p = synth.config_problem(cfg, scale)
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=1000, restart=restart)
    o, nforced = oracle_matching(p.Q, p.b, g, tol=0.0, maxit=1000, restart=restart)
    assert g.status == o.status and g.iterations == o.iterations
    assert max_rel(g.x, o.x) <= PARITY_TOL, (cfg, max_rel(g.x, o.x), nforced)
    np.testing.assert_array_equal(g.D, oracle.build_jdiag(p.Q))  # eq-J-diag bitwise
    # residual / f / restart-inner-product histories and the restart bookkeeping
    assert_history_parity(g, o, fstar=-0.5 * float(np.dot(p.b, p.x_star)))


@pytest.mark.parametrize("cfg,scale", CASES)
def test_iterations_to_tol(cfg, scale):
    """Iterations to 1e-6 within +-1 of the oracle (north_star)."""
    p = synth.config_problem(cfg, scale)
    g = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    o = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=True)
    assert g.status == "converged" and o.status == "converged"
    assert abs(g.iterations - o.iterations) <= 1, (g.iterations, o.iterations)
    assert g.res_hist[-1] <= 1e-6
    if g.iterations == o.iterations and g.restart_iters == o.restart_iters:
        assert_history_parity(g, o, fstar=-0.5 * float(np.dot(p.b, p.x_star)))


def test_bitwise_equal_to_mirror_oracle():
    """Rows of <= 32 nonzeros are summed sequentially in ascending column order from 0.0 and no
    FMA is contracted (R14), so the GPU iterates are BITWISE those of the oracle's mirror mode
    (same single-SpMV algebra) whenever the restart decisions agree."""
    p = synth.config_problem(1)
    for restart in (False, True):
        g = gpu_solve(p.Q, p.b, tol=0.0, maxit=2000, restart=restart)
        m = oracle.solve(p.Q, p.b, tol=0.0, maxit=2000, restart=restart, mirror=True)
        if g.restart_iters == m.restart_iters:
            np.testing.assert_array_equal(g.x, m.x)
        else:
            t = min(set(g.restart_iters) ^ set(m.restart_iters))
            assert m.res_hist[t] < 1e-13  # only at machine-precision residuals


def test_bitwise_equal_to_mirror_oracle_graph_layout():
    """The same on a sorted-window int32 layout (ER Laplacian, rows <= 64: the SELL chunk dot with
    the predicated-pair gathers, relabelled rows): every row sum is sequential in ascending column
    order, so the iterates are bitwise the mirror oracle's while the restart decisions agree."""
    p = synth.config_problem(3, 0.02)
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True)
    assert g.info["sigma"] > 1 and g.info["col_bytes"] == 4 and g.info["seg_rows"] == 0
    m = oracle.solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, mirror=True)
    if g.restart_iters == m.restart_iters:
        np.testing.assert_array_equal(g.x, m.x)
    else:
        t = min(set(g.restart_iters) ^ set(m.restart_iters))
        assert m.res_hist[t] < 1e-13  # only at machine-precision residuals
        k = t - 1
        g2 = gpu_solve(p.Q, p.b, tol=0.0, maxit=k, restart=True)
        m2 = oracle.solve(p.Q, p.b, tol=0.0, maxit=k, restart=True, mirror=True)
        np.testing.assert_array_equal(g2.x, m2.x)


def test_determinism_and_loop_modes():
    p = synth.config_problem(2, 0.25)
    a = gpu_solve(p.Q, p.b, tol=0.0, maxit=300)
    b = gpu_solve(p.Q, p.b, tol=0.0, maxit=300)
    c = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, loop="host")
    d = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, device_inputs=True)
    for o in (b, c, d):
        np.testing.assert_array_equal(a.x, o.x)
        np.testing.assert_array_equal(a.res_hist, o.res_hist)
        np.testing.assert_array_equal(a.f_hist, o.f_hist)
    assert a.info["last_launches"] == 1 and a.info["last_passes"] == 301


# ------------------------------------------------------------------------------------------------
# edge cases
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("n", [40, 600, 3000])
def test_long_rows_sdd(n):
    """§4.1 matrix: rows of length n exercise the SELL path (n <= 64), the single warp
    segment (65..2048) and the split rows finished by an owner CTA (> 2048).  tol 1e-8 stays above
    the rounding floor of these dense rows."""
    Q = synth.sdd(n)
    b = np.ones(n)
    g = gpu_solve(Q, b, tol=1e-8, maxit=3000, restart=True)
    o, _ = oracle_matching(Q, b, g, tol=1e-8, maxit=3000, restart=True)
    assert abs(g.iterations - o.iterations) <= 1
    assert max_rel(g.x, o.x) <= PARITY_TOL


def test_tiny_and_ragged():
    for n in (1, 2, 3, 31, 33, 513, 4097):
        Q = synth.random_spd(n, seed=n, density=min(1.0, 4.0 / n)) if n <= 600 else synth.poisson2d(64)
        if n == 4097:
            Q = synth.er_laplacian(n, 4 * n, seed=5)
        bb = np.random.Generator(np.random.PCG64(n)).uniform(-1, 1, Q.n)
        b = Q.scipy() @ bb
        g = gpu_solve(Q, b, tol=0.0, maxit=200)
        o, _ = oracle_matching(Q, b, g, tol=0.0, maxit=200)
        assert max_rel(g.x, o.x) <= PARITY_TOL, n


def test_trivial_cases():
    p = synth.config_problem(1)
    g = gpu_solve(p.Q, p.b, x0=p.x_star, tol=1e-10)
    assert g.status == "converged" and g.iterations == 0
    np.testing.assert_array_equal(g.x, p.x_star)
    d = np.array([1.0, 2.0, 4.0, 0.5])
    Q = synth.diag_matrix(d)
    b = np.array([3.0, -1.0, 2.0, 7.0])
    g = gpu_solve(Q, b, tol=1e-15, maxit=5)
    assert g.status == "converged" and g.iterations == 1
    np.testing.assert_array_equal(g.x, b / d)
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=1)
    o = oracle.solve(p.Q, p.b, tol=0.0, maxit=1)
    assert g.iterations == 1 and g.status == "maxiter"
    assert max_rel(g.x, o.x) <= 1e-15


def test_jacobi_and_weighted_jacobi_modes():
    """momentum off with D = diag(Q) (AJM_D_QDIAG) / diag(Q)/omega (AJM_D_USER) is Jacobi / weighted
    Jacobi; the oracle with the same D is pinned to the textbook forms."""
    p = synth.config_problem(2, 0.125)
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=200, momentum=False, restart=False, dmode="qdiag")
    o = oracle.solve(p.Q, p.b, tol=0.0, maxit=200, momentum=False, restart=False, dmode="qdiag")
    assert max_rel(g.x, o.x) <= 1e-13
    dw = oracle.diag(p.Q) / 0.8
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=200, momentum=False, restart=False, dmode="user", d=dw)
    o = oracle.solve(p.Q, p.b, D=dw, tol=0.0, maxit=200, momentum=False, restart=False)
    assert max_rel(g.x, o.x) <= 1e-13


def test_divergence_guard():
    """Weighted Jacobi with omega = 3.8 > 2/lambda_max(D^-1 Q) diverges; both sides stop
    with Diverged at the same t (R19)."""
    Q = synth.random_laplacian(40, seed=3)
    b = Q.scipy() @ np.random.Generator(np.random.PCG64(1)).uniform(-1, 1, 40)
    dw = oracle.diag(Q) / 3.8
    g = gpu_solve(Q, b, tol=1e-8, maxit=5000, momentum=False, restart=False, dmode="user", d=dw)
    o = oracle.solve(Q, b, D=dw, tol=1e-8, maxit=5000, momentum=False, restart=False)
    assert g.status == o.status == "diverged"
    assert abs(g.iterations - o.iterations) <= 1


def test_create_errors():
    import paper_2407_03272_b200 as ajm
    Q = synth.poisson2d(4)
    b = np.ones(16)

    def create(rp, col, val, bb, **kw):
        with pytest.raises(ajm.AjmError) as e:
            ajm.Solver(len(rp) - 1, rp, col, val, bb, **kw)
        return e.value.status_name

    bad = Q.col.copy()
    bad[1], bad[2] = bad[2], bad[1]
    assert create(Q.row_ptr, bad, Q.val, b) == "AJM_ERR_CSR_INVALID"
    bad = Q.col.copy()
    bad[0] = 99
    assert create(Q.row_ptr, bad, Q.val, b) == "AJM_ERR_CSR_INVALID"
    rp = Q.row_ptr.copy()
    rp[-1] += 1
    assert create(rp, Q.col, Q.val, b) == "AJM_ERR_CSR_INVALID"
    v = Q.val.copy()
    v[3] = np.nan
    assert create(Q.row_ptr, Q.col, v, b) == "AJM_ERR_NONFINITE"
    v = Q.val.copy()
    v[0] = -4.0
    assert create(Q.row_ptr, Q.col, v, b) == "AJM_ERR_NEGATIVE_DIAG"
    assert create(Q.row_ptr, Q.col, Q.val, np.zeros(16)) == "AJM_ERR_ZERO_RHS"
    v = Q.val.copy()
    v[1] = -0.5
    assert create(Q.row_ptr, Q.col, v, b, validate_symmetry=True) == "AJM_ERR_NOT_SYMMETRIC"
    Z = synth.from_dense(np.diag([1.0, 0.0, 2.0]), drop_zeros=False)
    assert create(Z.row_ptr, Z.col, Z.val, np.ones(3)) == "AJM_ERR_ZERO_DIAG"
    assert create(Q.row_ptr, Q.col, Q.val, b, dmode="user", d=-np.ones(16)) == "AJM_ERR_ZERO_DIAG"
    # solve-time argument errors
    s = ajm.Solver(16, Q.row_ptr, Q.col, Q.val, b)
    for kw in (dict(tol=-1.0), dict(maxit=0), dict(k0=1), dict(momentum=False, restart=True)):
        with pytest.raises(ajm.AjmError) as e:
            s.solve(**kw)
        assert e.value.status_name == "AJM_ERR_INVALID_ARG"
    s.close()


@pytest.mark.parametrize("n", [1000, 3000])
def test_sdd_paper_experiment(n):
    """§4.1: on Q = (n+1)I - 11^T, b = 1, tol 1e-4, maxiter 5000, the GPU's Jacobi and
    weighted Jacobi (omega_opt = 2n/(n+2)) follow their closed forms (1-1/n)^t and (1-2/(n+2))^t
    and AJM with restart follows the exact scalar recurrence of Alg. 3 on span{1} -- the models of
    tests/_sdd_models.py, pinned against the oracle in test_oracle_pins.py; rows of n nonzeros run
    on the warp-segment and split-row path."""
    from _sdd_models import closed_form_rate_iters, sdd_scalar_ajm
    Q = synth.sdd(n)
    b = np.ones(n)
    t = np.arange(5001)
    g = gpu_solve(Q, b, tol=1e-4, maxit=5000, momentum=False, restart=False, dmode="qdiag")
    assert (g.iterations, g.status) == closed_form_rate_iters(1 - 1 / n, 1e-4, 5000)
    np.testing.assert_allclose(g.res_hist, (1 - 1 / n) ** t[: len(g.res_hist)], rtol=1e-9)
    w = 2 * n / (n + 2)
    g = gpu_solve(Q, b, tol=1e-4, maxit=5000, momentum=False, restart=False, dmode="user", d=np.full(n, n / w))
    it, st = closed_form_rate_iters(1 - 2 / (n + 2), 1e-4, 5000)
    assert g.status == st and abs(g.iterations - it) <= 1
    np.testing.assert_allclose(g.res_hist, (1 - 2 / (n + 2)) ** t[: len(g.res_hist)], rtol=1e-8)
    g = gpu_solve(Q, b, tol=1e-4, maxit=5000, restart=True)
    it, hist, rest = sdd_scalar_ajm(n, 1e-4, 5000)
    assert g.status == "converged" and abs(g.iterations - it) <= 1
    assert g.restart_iters == rest
    k = min(len(hist), len(g.res_hist))
    np.testing.assert_allclose(g.res_hist[:k], hist[:k], rtol=1e-7, atol=1e-12)


@pytest.mark.parametrize("segments", ["static", "dynamic"])
def test_segment_queue_modes(segments):
    """Both segment schedules (static LPT plan / dynamic claim queue, AJM_SEGMENTS_*) give the same
    iterates as the oracle on a Chung-Lu graph with split rows and on the dense §4.1 rows; each is
    deterministic run to run (the queue only decides which warp runs a segment)."""
    for p in (synth.config_problem(4, 0.0125), synth.make_problem("sdd", synth.sdd(2600), 3)):
        a = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, restart=True, segments=segments)
        b = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, restart=True, segments=segments)
        np.testing.assert_array_equal(a.x, b.x)
        o, _ = oracle_matching(p.Q, p.b, a, tol=0.0, maxit=300, restart=True)
        assert max_rel(a.x, o.x) <= PARITY_TOL


def test_relabelled_layout_x0_and_diag():
    """Sorted-window layouts solve in an internal row order; x0, x and D cross the boundary in the
    caller's order (non-zero x0, ER graph)."""
    p = synth.config_problem(3, 0.01)
    x0 = synth.random_vector(p.Q.n, 77)
    g = gpu_solve(p.Q, p.b, x0=x0, tol=0.0, maxit=200, restart=True)
    assert g.info["sigma"] > 1
    np.testing.assert_array_equal(g.D, oracle.build_jdiag(p.Q))
    o, _ = oracle_matching(p.Q, p.b, g, x0=x0, tol=0.0, maxit=200, restart=True)
    assert max_rel(g.x, o.x) <= PARITY_TOL


def test_many_handles_pool_reuse():
    """Create / solve / destroy cycles of mixed layouts (natural order, sorted windows with
    relabelling, single-cluster and cooperative grids) with every new allocation poisoned
    (AJM_DEBUG_POISON): the pooled memory a handle gets back is never read before it is written
    (regression: chunk-tail slots once read past the slot->row map)."""
    for rep in range(3):
        for n in (1, 2, 3, 31, 33, 513, 4097):
            Q = synth.random_spd(n, seed=n, density=min(1.0, 4.0 / n)) if n <= 600 else \
                synth.er_laplacian(n, 4 * n, seed=5)
            b = Q.scipy() @ np.random.Generator(np.random.PCG64(n)).uniform(-1, 1, Q.n)
            g = gpu_solve(Q, b, tol=0.0, maxit=100, debug_poison=True)
            if rep == 0:
                o, _ = oracle_matching(Q, b, g, tol=0.0, maxit=100)
                assert max_rel(g.x, o.x) <= PARITY_TOL, n


def test_global_metadata_variant(monkeypatch):
    """Layouts whose per-CTA unit/chunk tables do not fit shared memory read them from global
    memory (a kernel instantiation for hundreds of millions of rows); forced here on oracle-sized
    stencil and graph cases it must give bitwise the iterates of the shared-memory tables."""
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")  # the band kernel on the generic plan (test_band_replan)
    for cfg, scale in ((2, 0.25), (4, 0.0125)):
        p = synth.config_problem(cfg, scale)
        a = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, restart=True)
        g = gpu_solve(p.Q, p.b, tol=0.0, maxit=300, restart=True, global_tables=True)
        np.testing.assert_array_equal(a.x, g.x)
        np.testing.assert_array_equal(a.res_hist, g.res_hist)


def _banded_offsets(nd, R=2048, regions=4, seed=0):
    """SPD Laplacian (+1e-2 I) of 4 diagonal blocks of R rows; block r couples rows j and j+d for
    the offsets d of its share of 1..nd (pairs (j, j+d) with floor(j/d) even), so every row has
    <= 33 entries and the matrix has exactly 2 nd + 1 distinct offsets col - row."""
    ds = np.array_split(np.arange(1, nd + 1), regions)
    us, vs = [], []
    for r, D in enumerate(ds):
        j = np.arange(R)
        for d in D:
            m = ((j // d) % 2 == 0) & (j + d < R)
            us.append(r * R + j[m])
            vs.append(r * R + j[m] + d)
    u, v = np.concatenate(us), np.concatenate(vs)
    w = np.random.Generator(np.random.PCG64(seed)).uniform(0.1, 1.0, u.size)
    return synth._laplacian_from_edges(R * regions, u, v, w, shift=1e-2)


def _stencil_with_values(edge, nvals, seed=3):
    """3D 7-point Dirichlet Laplacian whose off-diagonal couplings take `nvals` distinct values
    (symmetric, diagonally dominant: SPD), so the (offset, value) pairs of its entries number about
    6 nvals + the distinct diagonals."""
    Q0 = synth.poisson3d(edge)
    rng = np.random.Generator(np.random.PCG64(seed))
    levels = rng.uniform(0.1, 1.0, nvals)
    n = Q0.n
    rows = np.repeat(np.arange(n), np.diff(Q0.row_ptr))
    u, v = rows[Q0.col > rows], Q0.col[Q0.col > rows]
    w = levels[rng.integers(0, nvals, u.size)]  # one value per edge
    return synth._laplacian_from_edges(n, u, v, w, shift=1e-2)


@pytest.mark.parametrize("case", ["cfg2", "ragged17", "band255", "band257", "vals2", "vals300"])
def test_byte_coded_columns(case, monkeypatch):
    """Layouts whose column offsets col - row take <= 256 values stream byte codes into an offset
    table instead of int32 columns.  Same columns, same summation order: the
    iterates are BITWISE those of the int32 layout (AJM_INT32_COLUMNS) and match the oracle; 257 distinct
    offsets keep the int32 layout.  (cfg2 runs the variant without segment phases, the banded
    cases (width 33) the one with them, as config 5 does at full size: test_gpu_fullsize.)"""
    if case == "cfg2":
        p = synth.config_problem(2, 0.25)
    elif case == "ragged17":  # n = 4913: a ragged last chunk (tail slots), > 128 chunks (no cluster)
        p = synth.make_problem("p3d17", synth.poisson3d(17), 4)
    elif case.startswith("vals"):  # a 7-point stencil with 2 / 300 distinct coupling values
        p = synth.make_problem(case, _stencil_with_values(24, int(case[4:])), 6)
    else:
        p = synth.make_problem(case, _banded_offsets(127 if case == "band255" else 128), 5)
    # the band kernel on the generic plan's CTA ranges (same CTA partials -> bitwise histories);
    # its own re-planned ranges: test_band_replan
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")
    a = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True)
    assert a.info["col_bytes"] == (4 if case == "band257" else 1), a.info
    assert a.info["sigma"] == 1
    # pair-coded entries (values not streamed) exactly when the (offset, value) pairs number <= 256
    # (the banded cases' random weights do not, nor do 300 coupling levels; 2 levels do)
    pairs = case in ("cfg2", "ragged17", "vals2")
    assert a.info["val_bytes"] == (0 if pairs else 8), a.info
    b = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, int32_columns=True)
    assert b.info["col_bytes"] == 4 and b.info["val_bytes"] == 8
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.res_hist, b.res_hist)
    np.testing.assert_array_equal(a.f_hist, b.f_hist)
    if pairs:  # the byte-coded layout with the values streamed: bitwise the same too
        c = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, value_stream=True)
        assert c.info["col_bytes"] == 1 and c.info["val_bytes"] == 8 and c.info["band_staged"] == 0
        np.testing.assert_array_equal(a.x, c.x)
        np.testing.assert_array_equal(a.res_hist, c.res_hist)
        # natural-order pair-coded stencils stage x~'s bands and the row operands through the TMA
        # ring (ajm_band_kernel); the register-gather pair kernel gives the same bits
        assert a.info["band_staged"] == 1, a.info
        d = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, band_staging=False)
        assert d.info["val_bytes"] == 0 and d.info["band_staged"] == 0
        np.testing.assert_array_equal(a.x, d.x)
        np.testing.assert_array_equal(a.res_hist, d.res_hist)
        np.testing.assert_array_equal(a.f_hist, d.f_hist)
        np.testing.assert_array_equal(a.d_trace, d.d_trace)
    o, _ = oracle_matching(p.Q, p.b, a, tol=0.0, maxit=400, restart=True)
    assert max_rel(a.x, o.x) <= PARITY_TOL


def test_interleaved_handles_kernel_attributes():
    """Handles whose solver kernels differ in ring depth, shared-memory size and carve-out (graph:
    3-deep int32 ring; stencil: byte-coded 4-deep ring; tiny: single cluster) stay alive together
    and solve alternately: each launch sets its own kernel attributes, so every solve is bitwise
    the one it gives alone."""
    probs = [synth.config_problem(3, 0.02), synth.config_problem(2, 0.25), synth.config_problem(1)]
    alone = [gpu_solve(p.Q, p.b, tol=0.0, maxit=150, restart=True) for p in probs]
    import paper_2407_03272_b200 as ajm
    solvers = [ajm.Solver.from_csr(p.Q, p.b) for p in probs]
    try:
        for rep in range(2):
            for s, a in zip(solvers, alone):
                r = s.solve(tol=0.0, maxit=150, restart=True)
                np.testing.assert_array_equal(r.x.cpu().numpy(), a.x)
        assert len({(s.info()["col_bytes"], s.info()["grid"]) for s in solvers}) == 3
    finally:
        for s in solvers:
            s.close()


def test_long_row_validation():
    """Rows of > 2048 entries are validated by a warp each (create-time): eq-J-diag still bitwise
    the oracle's ascending-column sum, and CSR / non-finite / negative-diagonal errors inside a
    long row are still caught."""
    import paper_2407_03272_b200 as ajm
    n = 9000
    g = np.random.Generator(np.random.PCG64(11))
    hubs = [0, 4500, 8999]  # three hubs joined to 3000-6000 random nodes each
    u, v = [], []
    for h, deg in zip(hubs, (6000, 3000, 4097)):
        nb = g.choice(np.setdiff1d(np.arange(n), hubs), deg, replace=False)
        u.append(np.full(deg, h)), v.append(nb)
    path = np.arange(n - 1)  # plus a path, so every node has a neighbour
    u.append(path), v.append(path + 1)
    u, v = np.concatenate(u), np.concatenate(v)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    key = np.unique(lo * n + hi)
    w = g.uniform(0.1, 1.0, key.size) * 10.0 ** g.integers(-3, 4, key.size)  # spread magnitudes
    Q = synth._laplacian_from_edges(n, key // n, key % n, w, shift=1e-3)
    assert np.diff(Q.row_ptr).max() > 6000
    p = synth.make_problem("hubs", Q, 12)
    r = gpu_solve(p.Q, p.b, tol=0.0, maxit=50, restart=True)
    np.testing.assert_array_equal(r.D, oracle.build_jdiag(p.Q))
    o, _ = oracle_matching(p.Q, p.b, r, tol=0.0, maxit=50, restart=True)
    assert max_rel(r.x, o.x) <= PARITY_TOL
    h0, h1 = int(Q.row_ptr[0]), int(Q.row_ptr[1])  # row 0: a hub row (diagonal first)

    def create(col, val):
        with pytest.raises(ajm.AjmError) as e:
            ajm.Solver(n, Q.row_ptr, col, val, p.b)
        return e.value.status_name

    bad = Q.col.copy()
    bad[h0 + 3000], bad[h0 + 3001] = bad[h0 + 3001], bad[h0 + 3000]
    assert create(bad, Q.val) == "AJM_ERR_CSR_INVALID"
    bad = Q.col.copy()
    bad[h1 - 1] = n  # out of range, last entry of the row
    assert create(bad, Q.val) == "AJM_ERR_CSR_INVALID"
    vv = Q.val.copy()
    vv[h0 + 5000] = np.inf
    assert create(Q.col, vv) == "AJM_ERR_NONFINITE"
    vv = Q.val.copy()
    assert Q.col[h0] == 0
    vv[h0] = -1.0
    assert create(Q.col, vv) == "AJM_ERR_NEGATIVE_DIAG"


def test_threads_with_own_handles_and_streams():
    """Two host threads, each with its own handles and CUDA stream, create and solve different
    layouts at the same time (the C ABI releases the GIL): every result is bitwise the
    single-threaded one (kernel attributes are set and the kernel launched under one lock)."""
    import threading
    import torch
    import paper_2407_03272_b200 as ajm
    probs = [synth.config_problem(3, 0.02), synth.config_problem(2, 0.25)]
    ref = [gpu_solve(p.Q, p.b, tol=0.0, maxit=120, restart=True).x for p in probs]
    errs = []

    def work(k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(4):
                    p = probs[k]
                    with ajm.Solver.from_csr(p.Q, p.b, stream=st) as s:
                        r = s.solve(tol=0.0, maxit=120, restart=True)
                        st.synchronize()
                        np.testing.assert_array_equal(r.x.cpu().numpy(), ref[k])
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in (0, 1, 0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def test_resident_cluster_bitwise():
    """Config 1 runs on the resident single-cluster kernel (mode 6: matrix slices and an x~ replica
    in shared memory, row state in registers); its iterates and histories are bitwise those of the
    kCluster ring kernel (mode 5, AJM_NO_RESIDENT=1) and of the host-driven loop (one launch per
    pass: the state goes through global memory between launches)."""
    import os
    p = synth.config_problem(1)
    for restart in (True, False):
        a = gpu_solve(p.Q, p.b, tol=0.0, maxit=700, restart=restart)
        os.environ["AJM_NO_RESIDENT"] = "1"
        try:
            b = gpu_solve(p.Q, p.b, tol=0.0, maxit=700, restart=restart)
        finally:
            del os.environ["AJM_NO_RESIDENT"]
        c = gpu_solve(p.Q, p.b, tol=0.0, maxit=700, restart=restart, loop="host")
        assert a.info["mode"] == 6 and b.info["mode"] == 5 and c.info["mode"] == 6
        for o in (b, c):
            np.testing.assert_array_equal(a.x, o.x)
            np.testing.assert_array_equal(a.res_hist, o.res_hist)
            np.testing.assert_array_equal(a.f_hist, o.f_hist)
            assert a.restart_iters == o.restart_iters
        d = gpu_solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=restart)
        od = oracle.solve(p.Q, p.b, tol=1e-6, maxit=5000, restart=restart)
        assert abs(d.iterations - od.iterations) <= 1


@pytest.mark.parametrize("unit", ["8", "16"])
def test_band_staging_units_bitwise(unit, monkeypatch):
    """The banded staging kernel with staging units of 8 and of 16 chunks (256 / 512
    rows; AJM_BAND_UNIT restricts create's search) gives bitwise the iterates, residual / f / d
    histories of the register-gather pair kernel (AJM_NO_BAND_STAGING), on a ragged 3D stencil
    with restarts, through the persistent launch and the host-driven loop."""
    p = synth.make_problem("p3d81", synth.poisson3d(81), 8)  # n = 531441: several units per CTA, ragged tail
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")  # the generic plan's CTA ranges (test_band_replan)
    monkeypatch.setenv("AJM_BAND_UNIT", unit)
    a = gpu_solve(p.Q, p.b, tol=0.0, maxit=500, restart=True)
    h = gpu_solve(p.Q, p.b, tol=0.0, maxit=120, restart=True, loop="host")
    monkeypatch.delenv("AJM_BAND_UNIT")
    assert a.info["band_staged"] == 1 and a.info["val_bytes"] == 0, a.info
    r = gpu_solve(p.Q, p.b, tol=0.0, maxit=500, restart=True, band_staging=False)
    assert r.info["band_staged"] == 0
    for f in ("x", "res_hist", "f_hist", "d_trace"):
        np.testing.assert_array_equal(getattr(a, f), getattr(r, f))
    np.testing.assert_array_equal(h.res_hist, r.res_hist[:121])
    o, _ = oracle_matching(p.Q, p.b, a, tol=0.0, maxit=500, restart=True)
    assert max_rel(a.x, o.x) <= PARITY_TOL


@pytest.mark.parametrize("case", ["p2d400", "aniso27_40", "p3d_bands17"])
def test_band_staging_stencils(case, monkeypatch):
    """Banded staging on other stencil shapes: a 2D 5-point grid whose +-400 rows stay separate
    bands of a 512-row unit, the anisotropic 27-point stencil (nine offset lines in three bands,
    several boundary diagonals among the pairs), and a 7-point 17^3 grid (ragged, few units per CTA)
    -- bitwise the register-gather pair kernel, and at parity with the oracle."""
    if case == "p2d400":
        p = synth.make_problem(case, synth.poisson2d(400), 9)
    elif case == "aniso27_40":
        p = synth.make_problem(case, synth.aniso27(40), 10)
    else:
        p = synth.make_problem(case, synth.poisson3d(17), 11)
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")  # the generic plan's CTA ranges (test_band_replan)
    a = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True)
    assert a.info["band_staged"] == 1 and a.info["val_bytes"] == 0, a.info
    r = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True, band_staging=False)
    for f in ("x", "res_hist", "f_hist", "d_trace"):
        np.testing.assert_array_equal(getattr(a, f), getattr(r, f))
    o, _ = oracle_matching(p.Q, p.b, a, tol=0.0, maxit=400, restart=True)
    assert max_rel(a.x, o.x) <= PARITY_TOL
    assert_history_parity(a, o)


def test_band_staging_x0_and_early_exits(monkeypatch):
    """Banded staging with a nonzero x0 (staged from the caller's buffer), a solve that converges at
    t = 0 (the producer has already staged pass 1, drained unread), maxit = 1, and a converged solve
    followed by another on the same handle: bitwise the pair kernel each time."""
    p = synth.make_problem("p3d40", synth.poisson3d(40), 12)
    x0 = synth.random_vector(p.Q.n, 5)
    kws = [dict(x0=x0, tol=0.0, maxit=300), dict(tol=10.0, maxit=50), dict(tol=0.0, maxit=1),
           dict(x0=x0, tol=1e-6, maxit=2000)]
    import paper_2407_03272_b200 as ajm
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")  # the generic plan's CTA ranges (test_band_replan)
    with ajm.Solver.from_csr(p.Q, p.b) as a, ajm.Solver.from_csr(p.Q, p.b, band_staging=False) as r:
        assert a.info()["band_staged"] == 1 and r.info()["band_staged"] == 0
        for kw in kws:
            ga, gr = a.solve(restart=True, **kw), r.solve(restart=True, **kw)
            assert ga.status == gr.status and ga.iterations == gr.iterations, (kw, ga.iterations, gr.iterations)
            np.testing.assert_array_equal(ga.x.cpu().numpy(), gr.x.cpu().numpy())
            np.testing.assert_array_equal(ga.res_hist, gr.res_hist)
    assert kws and ga.status == "converged"


@pytest.mark.parametrize("case", ["p3d81", "aniso27_40", "p3d_bands17"])
def test_band_replan(case, monkeypatch):
    """The band kernel's own CTA ranges (chunk cost 123 + w, older/younger CTA of an
    SM weighted 1 +- AJM_BAND_SKEW from a placement probe) against the generic plan's: only the
    grouping of the CTA partials changes, so the iterates and restart schedule are bitwise the
    same and the residual / f / d histories agree to rounding; both at parity with the oracle;
    repeated solves on the re-planned handle are bitwise identical (the plan is fixed at create)."""
    if case == "p3d81":
        p = synth.make_problem(case, synth.poisson3d(81), 8)
    elif case == "aniso27_40":
        p = synth.make_problem(case, synth.aniso27(40), 10)
    else:
        p = synth.make_problem(case, synth.poisson3d(17), 11)
    a = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True)
    a2 = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True)
    monkeypatch.setenv("AJM_BAND_NO_REPLAN", "1")
    g = gpu_solve(p.Q, p.b, tol=0.0, maxit=400, restart=True)
    monkeypatch.delenv("AJM_BAND_NO_REPLAN")
    assert a.info["band_staged"] == 1 and g.info["band_staged"] == 1
    assert a.restart_iters == g.restart_iters and a.iterations == g.iterations
    np.testing.assert_array_equal(a.x, g.x)
    np.testing.assert_allclose(a.res_hist, g.res_hist, rtol=1e-12, atol=0)
    np.testing.assert_allclose(a.f_hist, g.f_hist, rtol=1e-12, atol=1e-12)
    for f in ("x", "res_hist", "f_hist", "d_trace"):
        np.testing.assert_array_equal(getattr(a, f), getattr(a2, f))
    o, _ = oracle_matching(p.Q, p.b, a, tol=0.0, maxit=400, restart=True)
    assert max_rel(a.x, o.x) <= PARITY_TOL
    assert_history_parity(a, o)
