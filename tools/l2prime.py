"""Probe: does a previous handle's persisting-L2 state speed up the next handle? (same process)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2407_03272_b200 as ajm
p = synth.config_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
seq = sys.argv[2].split(",") if len(sys.argv) > 2 else ["3", "2", "3", "3"]
for m in seq:
    os.environ["AJM_L2MODE"] = m
    with ajm.Solver.from_csr(p.Q, p.b) as s:
        s.solve(tol=0.0, maxit=100)
        s.solve(tol=0.0, maxit=500)
        inf = s.info()
        print(f"mode {m}: us/pass {1e3 * inf['last_loop_ms'] / inf['last_passes']:.2f} win {inf['l2_window_bytes']/1e6:.0f}MB hit {inf['l2_hit_ratio']:.2f}", flush=True)
