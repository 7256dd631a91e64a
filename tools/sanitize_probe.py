"""Small solves for compute-sanitizer: config 1 (fast SELL path), a scaled Chung-Lu (sorted windows,
relabelling, warp segments, split rows), the §4.1 dense rows (dynamic segment queue), block J."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth, paper_2407_03272_b200 as ajm
cases = [("cfg1", synth.config_problem(1), {}), ("cfg4s", synth.config_problem(4, 0.005), {}),
         ("sdd", synth.make_problem("sdd", synth.sdd(2500), 1), {}),
         ("cfg2s-jblock8", synth.config_problem(2, 0.125), {"jblock": 8})]
for name, p, kw in cases:
    with ajm.Solver.from_csr(p.Q, p.b, **kw) as s:
        r = s.solve(tol=1e-8, maxit=60, restart=True)
        print(name, r.status, r.iterations, f"{r.rel_residual:.3e}", flush=True)
