"""Interleaved A/B timing of library environment switches on the same box (not the bench).

usage: python tools/env_ab.py CFGS "ENV_A" "ENV_B" [...]   e.g.
       python tools/env_ab.py 2,5 "" "AJM_NO_PAIR=1"
AB_ROUNDS=<k> sets the rounds (default 2).  Each variant: create (the switches are read at create), 1 warm-up + 3 timed solves to the config's
tolerance, us/pass from the library's own CUDA-event loop time; the variants alternate twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
import paper_2407_03272_b200 as ajm  # noqa: E402

TOL = {1: 0.0, 2: 1e-6, 3: 1e-6, 4: 1e-6, 5: 1e-6}
MAXIT = {1: 2000, 2: 5000, 3: 5000, 4: 5000, 5: 5000}


def run(p, cfg, env):
    keys = []
    for kv in env.split():
        k, v = kv.split("=", 1)
        os.environ[k] = v
        keys.append(k)
    try:
        with ajm.Solver.from_csr(p.Q, p.b) as s:
            info = s.info()
            s.solve(tol=TOL[cfg], maxit=MAXIT[cfg], restart=True, history=False)
            us = []
            for _ in range(3):
                r = s.solve(tol=TOL[cfg], maxit=MAXIT[cfg], restart=True, history=False)
                r.xh = r.x.cpu().numpy()
                inf = s.info()
                us.append(1e3 * inf["last_loop_ms"] / inf["last_passes"])
        return info, r, us
    finally:
        for k in keys:
            os.environ.pop(k, None)


def main():
    cfgs = [int(c) for c in sys.argv[1].split(",")]
    envs = sys.argv[2:] or [""]
    for cfg in cfgs:
        p = synth.config_problem(cfg)
        x_ref = None
        for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
            for env in envs:
                info, r, us = run(p, cfg, env)
                if x_ref is None:
                    x_ref = r.xh
                same = bool(np.array_equal(x_ref, r.xh))
                print(f"cfg{cfg} [{env or 'default'}] round {rnd}: its={r.iterations} us/pass "
                      f"{' '.join(f'{u:.2f}' for u in us)} (min {min(us):.2f}) col_bytes={info['col_bytes']} "
                      f"val_bytes={info['val_bytes']} stages/mode={info['mode']} grid={info['grid']} "
                      f"hot={info.get('hot_entries', 0)}@{info.get('hot_first', 0)} share={info.get('hot_share', 0.0):.3f} "
                      f"x_bitwise_first={same}", flush=True)
        del p


if __name__ == "__main__":
    main()
