"""Quick GPU timing probe (not the bench): config solves, loop time, model GB/s."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2407_03272_b200 as ajm

for cfg, scale in [(1, 1.0), (2, 1.0)] + ([(3, 1.0), (4, 1.0)] if "all" in sys.argv else []):
    t0 = time.time(); p = synth.config_problem(cfg, scale); tg = time.time() - t0
    with ajm.Solver.from_csr(p.Q, p.b) as s:
        for rep in range(3):
            r = s.solve(tol=1e-6, maxit=5000, restart=True)
            info = s.info()
            its = r.iterations
            ms = info["last_loop_ms"]
            gbs = info["model_bytes_per_iter"] * info["last_passes"] / (ms * 1e-3) / 1e9
            print(f"cfg{cfg} n={p.Q.n} nnz={p.Q.nnz} gen={tg:.1f}s its={its} restarts={r.restart_iters} "
                  f"loop={ms:.3f}ms us/pass={1e3*ms/info['last_passes']:.2f} model={gbs:.0f}GB/s "
                  f"grid={info['grid']} occ={info['ctas_per_sm']} units={info['units']} res={r.rel_residual:.2e}", flush=True)
        r = s.solve(tol=0.0, maxit=1000, restart=True)
        info = s.info(); ms = info["last_loop_ms"]
        gbs = info["model_bytes_per_iter"] * info["last_passes"] / (ms * 1e-3) / 1e9
        print(f"cfg{cfg} 1000its loop={ms:.3f}ms us/pass={1e3*ms/info['last_passes']:.2f} model={gbs:.0f}GB/s", flush=True)
