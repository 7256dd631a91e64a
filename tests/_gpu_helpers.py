"""Shared helpers for the -m gpu parity tests (GPU path via the C-ABI binding vs the CPU oracle)."""
import os

import numpy as np
import pytest

import oracle
import synth

PARITY_TOL = 1e-10  # north_star: max|x_gpu - x_cpu| / max|x_cpu| <= 1e-10 after 1000 FP64 iterations
TIE_RATIO = 1e-10   # DESIGN.md R17: restart decisions with |d| / sum|terms| <= this may flip
RES_FLOOR = 1e-12   # DESIGN.md R17: ... and so may every decision once the relative residual is at
                    # the rounding floor (the terms of d are then rounding noise of either algebra)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


requires_cuda = pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")


def oracle_threads():
    oracle.set_threads(min(os.cpu_count() or 1, 32))


def gpu_solve(Q, b, x0=None, tol=0.0, maxit=1000, restart=True, momentum=True, k0=2,
              dmode="jdiag", d=None, loop="graph", device_inputs=False, jblock=None, **solver_kw):
    import torch
    import paper_2407_03272_b200 as ajm
    args = [Q.row_ptr, Q.col, Q.val, b, d, x0]
    if device_inputs:
        args = [None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in args]
    with ajm.Solver(Q.n, args[0], args[1], args[2], args[3], dmode=dmode, d=args[4], loop=loop,
                    jblock=jblock, **solver_kw) as s:
        r = s.solve(x0=args[5], tol=tol, maxit=maxit, momentum=momentum, restart=restart, k0=k0)
        r.x = r.x.cpu().numpy()
        r.d_trace = s.trace("d", r.iterations + 1)
        r.dabs_trace = s.trace("dabs", r.iterations + 1)
        r.D = s.diag()
        r.info = s.info()
        r.J = s.jblocks() if jblock else None
    return r


def max_rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def oracle_matching(Q, b, g, **kw):
    """Oracle run that follows the GPU's restart decisions where (and only where) they are
    near-ties (R17).  Returns (oracle result, number of forced decisions)."""
    o = oracle.solve(Q, b, **kw)
    forced_n = 0
    for _ in range(8):
        if o.restart_iters == g.restart_iters:
            return o, forced_n
        go, oo = set(g.restart_iters), set(o.restart_iters)
        t = min(go.symmetric_difference(oo))
        ratio = abs(o.d_hist[t]) / max(o.dabs_hist[t], 1e-300) if t < len(o.d_hist) else 0.0
        res_t = o.res_hist[t] if t < len(o.res_hist) else 0.0
        assert ratio <= TIE_RATIO or res_t <= RES_FLOOR, \
            f"restart decision differs at t={t}: tie ratio {ratio:.3e}, residual {res_t:.3e}"
        forced = np.full(kw.get("maxit", 1000) + 1, -1, dtype=np.int8)
        for tt in range(t, len(forced)):
            forced[tt] = 1 if tt in go else 0
        forced_n += 1
        o = oracle.solve(Q, b, forced=forced, **kw)
    raise AssertionError("restart schedules could not be matched")


F_TOL = 1e-10   # |f_gpu - f_oracle| <= F_TOL * max(1, |f*|) per history entry (DESIGN.md §5 parity)
D_TOL = 1e-7    # |d_gpu - d_oracle| <= D_TOL * sum|terms| while the residual is >= D_RES_MIN
D_RES_MIN = 1e-6


def assert_history_parity(g, o, fstar=None):
    """The ABI outputs besides x against the oracle of the same run, entry by entry:
      res_hist[t]  relative residual of x~^t             -- rounding-level
      f_hist[t]    f(x~^t) = 1/2<x,Qx> - <b,x> (eq-qp)   -- F_TOL * max(1, |f*|)
      d_t          <Q y^t - b, x~^t - x^{t-1}> (restart test): D_TOL * sum|terms| and the same
                   sign wherever the tie ratio |d|/sum|terms| > TIE_RATIO, for every t whose residual
                   is >= D_RES_MIN (below that both sides' terms are differences of nearly equal
                   iterates, dominated by rounding -- DESIGN.md R17)
      status, iterations, n_restarts, restart iterations, x_is_prerestart (R5) -- exact."""
    assert g.status == o.status and g.iterations == o.iterations
    assert g.n_restarts == o.n_restarts and g.restart_iters == o.restart_iters
    assert bool(g.x_is_prerestart) == bool(o.x_is_prerestart)
    k = min(len(g.res_hist), len(o.res_hist))
    assert k == g.iterations + 1
    assert np.all(np.abs(g.res_hist[:k] - o.res_hist[:k]) <= 1e-9 * o.res_hist[:k] + 1e-12 * o.res_hist[0])
    scale = max(1.0, abs(fstar) if fstar is not None else float(np.abs(o.f_hist[:k]).max()))
    fdev = np.abs(g.f_hist[:k] - o.f_hist[:k])
    assert fdev.max() <= F_TOL * scale, ("f_hist", float(fdev.max()), scale)
    gd, od, oa = g.d_trace[1:k], o.d_hist[1:k], o.dabs_hist[1:k]
    live = o.res_hist[1:k] >= D_RES_MIN
    ddev = np.abs(gd - od)[live]
    assert np.all(ddev <= D_TOL * oa[live]), ("d_t", float((ddev / np.maximum(oa[live], 1e-300)).max()))
    decided = live & (np.abs(od) > TIE_RATIO * oa)
    assert np.all(np.sign(gd[decided]) == np.sign(od[decided])), "restart inner product sign"
    np.testing.assert_allclose(g.dabs_trace[1:k][live], oa[live], rtol=1e-6)
