"""e2e probe: time ajm_create from pinned host buffers (phases via AJM_TS), solve and copy-out."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2407_03272_b200 as ajm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = synth.config_problem(cfg)
host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (p.Q.row_ptr, p.Q.col, p.Q.val, p.b)]
xh = torch.empty(p.Q.n, dtype=torch.float64).pin_memory()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = ajm.Solver(p.Q.n, *host)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = s.solve(tol=1e-6, maxit=5000, x_out=xh, history=True)
    t2 = time.perf_counter()
    loop = s.info()["last_loop_ms"]
    s.close()
    t3 = time.perf_counter()
    print(f"cfg{cfg} create {1e3*(t1-t0):.2f} ms solve(+copy-out) {1e3*(t2-t1):.2f} ms (loop {loop:.2f}) destroy {1e3*(t3-t2):.2f} ms its {r.iterations}", flush=True)
