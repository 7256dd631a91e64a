"""A/B of the segment plan on a config: static LPT plan (default) vs the dynamic claim queue."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2407_03272_b200 as ajm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = synth.config_problem(cfg)
for rep in range(2):
    for seg in ("static", "dynamic"):
        with ajm.Solver.from_csr(p.Q, p.b, segments=seg) as s:
            s.solve(tol=0.0, maxit=20)
            s.solve(tol=0.0, maxit=500)
            i = s.info()
            print(f"cfg{cfg} {seg:8s} us/pass={1e3 * i['last_loop_ms'] / i['last_passes']:.2f} group_rows={i['group_rows']}", flush=True)
