"""Profiling driver: one warm-up solve then one profiled solve (the 2nd ajm_solve_kernel launch).
usage: python tools/prof.py CFG MAXIT"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2407_03272_b200 as ajm
cfg = int(sys.argv[1]); maxit = int(sys.argv[2])
p = synth.config_problem(cfg)
with ajm.Solver.from_csr(p.Q, p.b) as s:
    for _ in range(2):
        r = s.solve(tol=0.0, maxit=maxit, restart=True)
    info = s.info()
    print(f"cfg{cfg} passes={info['last_passes']} loop_ms={info['last_loop_ms']:.3f} "
          f"us/pass={1e3*info['last_loop_ms']/info['last_passes']:.2f} model_bytes={info['model_bytes_per_iter']:.0f}")
