"""PAPER.md §4.1 experiment (fig-sdd) on the GPU: Q = (n+1)I - 11^T (diag n, off -1),
b = 1, x0 = 0, n in {1000, ..., 6000}, tol 1e-4 on ||b - Qx||/||b||, maxiter 5000:
  jacobi     momentum off, D = diag(Q)                   (eq-jacobi)
  w-jacobi   momentum off, D = diag(Q)/omega_opt,        (eq-weighted-jacobi)
             omega_opt = 2/(lmin + lmax)(D^-1 Q) = 2n/(n+2) for this matrix
  acc-jacobi Alg. 3 with eq-J-diag and adaptive restart (the paper's method)
Every row has n nonzeros, so the GPU runs it on the warp-segment / split-row path.  Each run is
checked against an exact model of the same iteration on span{1} (every iterate is c*1): the
Jacobi/w-Jacobi closed forms and the scalar Alg. 3 recurrence (both pinned against the oracle in
tests/test_oracle_pins.py).  Writes profiles/r1_exp_sdd.json and prints a table.
usage (GPU): python tools/exp_sdd.py [n ...]"""
import json, math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np


def scalar_ajm(n, tol, maxit, k0=2):
    cx_prev = cy = 0.0
    alpha, K, Kre = 1.0, k0, 0
    for t in range(1, maxit + 1):
        cxt = cy + (1.0 - cy) / (2 * n - 1)
        res = abs(1.0 - cxt)
        if res <= tol:
            return t, res
        d = n * (cy - 1.0) * (cxt - cx_prev)
        if t > Kre + K and d >= 0:
            Kre, K = t, 2 * K
            alpha, cy = 1.0, cx_prev
        else:
            an = (1 + math.sqrt(1 + 4 * alpha * alpha)) / 2
            beta = (alpha - 1) / an
            cy, cx_prev, alpha = cxt + beta * (cxt - cx_prev), cxt, an
    return maxit, None


def closed_form_iters(rate, tol, maxit):
    t = math.ceil(math.log(tol) / math.log(rate))
    return (t, "converged") if t <= maxit else (maxit, "maxiter")


def main():
    import synth
    import paper_2407_03272_b200 as ajm
    ns = [int(a) for a in sys.argv[1:]] or [1000, 2000, 3000, 4000, 5000, 6000]
    tol, maxit = 1e-4, 5000
    out = []
    for n in ns:
        Q = synth.sdd(n)
        b = np.ones(n)
        w = 2 * n / (n + 2)
        runs = {
            "jacobi": dict(dmode="qdiag", momentum=False, restart=False, model=closed_form_iters(1 - 1 / n, tol, maxit)),
            "w-jacobi": dict(dmode="user", d=np.full(n, n / w), momentum=False, restart=False,
                             model=closed_form_iters(1 - 2 / (n + 2), tol, maxit)),
            "acc-jacobi": dict(dmode="jdiag", momentum=True, restart=True, model=scalar_ajm(n, tol, maxit)),
        }
        for name, kw in runs.items():
            with ajm.Solver(n, Q.row_ptr, Q.col, Q.val, b, dmode=kw["dmode"], d=kw.get("d")) as s:
                s.solve(tol=tol, maxit=maxit, momentum=kw["momentum"], restart=kw["restart"])  # warm
                t0 = time.perf_counter()
                r = s.solve(tol=tol, maxit=maxit, momentum=kw["momentum"], restart=kw["restart"])
                wall = time.perf_counter() - t0
                inf = s.info()
            mit = kw["model"][0]
            rec = {"n": n, "method": name, "status": r.status, "iterations": r.iterations,
                   "rel_residual": r.rel_residual, "restarts": r.restart_iters,
                   "model_iterations": mit, "loop_ms": inf["last_loop_ms"], "solve_wall_ms": 1e3 * wall,
                   "us_per_iteration": 1e3 * inf["last_loop_ms"] / max(1, inf["last_passes"]),
                   "split_rows": inf["split_rows"], "seg_rows": inf["seg_rows"]}
            out.append(rec)
            print(f"n={n:5d} {name:10s} {r.status:9s} its={r.iterations:5d} (model {mit:5d}) res={r.rel_residual:.3e} "
                  f"{rec['us_per_iteration']:.2f} us/it restarts={r.restart_iters[:6]}", flush=True)
    with open(os.path.join(ROOT, "profiles", "r1_exp_sdd.json"), "w") as f:
        json.dump({"experiment": "PAPER.md §4.1 (fig-sdd): tol 1e-4, maxiter 5000, x0 = 0, b = 1",
                   "runs": out}, f, indent=1)


if __name__ == "__main__":
    main()
