"""Debug probe for ajm_estimate_spectrum: GPU Lanczos coefficients vs a numpy Lanczos in the
D-inner product from the same start vector (first steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth, paper_2407_03272_b200 as ajm


def np_lanczos(Q, D, v0, k):
    A = Q.scipy() if hasattr(Q, "scipy") else Q
    p_prev = np.zeros_like(v0)
    p = v0 / np.sqrt(v0 @ (D * v0))
    beta = 0.0
    al, be = [], []
    for j in range(k):
        w = (A @ p) / D - beta * p_prev
        a = p @ (A @ p)
        w = w - a * p
        beta = np.sqrt(w @ (D * w))
        al.append(a); be.append(beta)
        p_prev, p = p, w / beta
    return np.array(al), np.array(be)


K = int(os.environ.get("LZK", "6"))
for name, Q, dmode in [("cfg1", synth.config_problem(1).Q, "qdiag"), ("cfg2s", synth.config_problem(2, 0.25).Q, "jdiag")]:
    n = Q.n
    v0 = np.random.default_rng(1).uniform(-1, 1, n)
    with ajm.Solver(n, Q.row_ptr, Q.col, Q.val, np.ones(n), dmode=dmode) as s:
        D = s.diag()
        sp = s.estimate_spectrum(v0=v0, tol=0.0, max_steps=K)
        inf = s.info()
    al, be = np_lanczos(Q, D, v0, K)
    print(name, "mode", inf["mode"], "grid", inf["grid"], "col_bytes", inf["col_bytes"])
    da = np.abs(sp.alpha[:K] - al) / np.abs(al).max()
    db = np.abs(sp.beta[:K] - be) / np.abs(be).max()
    bad = np.nonzero((da > 1e-9) | (db > 1e-9))[0]
    print("  steps", sp.steps, "first differing step", bad[:5], "max dev", da.max(), db.max())
