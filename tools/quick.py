"""Quick GPU timing probe (not the bench): config solves, loop time, model GB/s per kernel variant."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2407_03272_b200 as ajm

cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2"])]
variants = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"])]
l2modes = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2"])]
os.environ["AJM_VSTAGE"] = sys.argv[4] if len(sys.argv) > 4 else "0"
variants = [(v, m) for v in variants for m in l2modes]
for cfg in cfgs:
    t0 = time.time()
    if cfg == 0:  # per-pass fixed-overhead probe: 1D Laplacian + I, one 3-wide chunk per warp
        Q = synth._stencil(148 * 2 * 8 * 32, 1, [((1,), -1.0), ((-1,), -1.0)], "const", 3.0)
        p = synth.make_problem("tridiag", Q, 7)
    else:
        p = synth.config_problem(cfg)
    tg = time.time() - t0
    for var, l2m in variants:
        os.environ["AJM_KVARIANT"] = str(var)
        if l2m >= 0:
            os.environ["AJM_L2MODE"] = str(l2m)
        else:
            os.environ.pop("AJM_L2MODE", None)
        t0 = time.time()
        with ajm.Solver.from_csr(p.Q, p.b) as s:
            tc = time.time() - t0
            info = s.info()
            print(f"cfg{cfg} var{var} l2m{l2m} n={p.Q.n} nnz={p.Q.nnz} gen={tg:.1f}s create={tc:.2f}s grid={info['grid']} "
                  f"occ={info['ctas_per_sm']} mode={info['mode']} l2auto={info['l2_mode']} l2win={info['l2_window_bytes']/1e6:.0f}MB hit={info['l2_hit_ratio']:.2f} units={info['units']} sell={info['sell_rows']} seg={info['seg_rows']} split={info['split_rows']} sigma={info['sigma']} pad={info['sell_elems']}", flush=True)
            for rep in range(2):
                r = s.solve(tol=1e-6, maxit=5000, restart=True)
                info = s.info(); ms = info["last_loop_ms"]
                gbs = info["model_bytes_per_iter"] * info["last_passes"] / (ms * 1e-3) / 1e9
                print(f"   tol1e-6 its={r.iterations} restarts={r.restart_iters[:6]} loop={ms:.3f}ms "
                      f"us/pass={1e3*ms/info['last_passes']:.2f} model={gbs:.0f}GB/s res={r.rel_residual:.2e}", flush=True)
            r = s.solve(tol=0.0, maxit=500, restart=True)
            info = s.info(); ms = info["last_loop_ms"]
            gbs = info["model_bytes_per_iter"] * info["last_passes"] / (ms * 1e-3) / 1e9
            print(f"   500its loop={ms:.3f}ms us/pass={1e3*ms/info['last_passes']:.2f} model={gbs:.0f}GB/s", flush=True)
