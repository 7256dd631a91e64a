"""Emulated row-block groups on ONE GPU (ajm_group_solve): per-pass time of config K sharded over R
ranks that share this device's SMs and HBM.  The work per pass is the same as the single-GPU solve,
so the difference is the cost of the halo push and the cross-rank exchange of every pass (what a
multi-GPU group adds on top of its per-GPU share).  usage: python tools/shard_scale.py K [R ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import synth, paper_2407_03272_b200 as ajm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
Rs = [int(r) for r in sys.argv[2:]] or [1, 2, 4, 8]
p = synth.config_problem(cfg)
with ajm.Solver.from_csr(p.Q, p.b) as s:
    s.solve(tol=0.0, maxit=20)
    s.solve(tol=0.0, maxit=300)
    i = s.info()
    base = 1e3 * i["last_loop_ms"] / i["last_passes"]
print(json.dumps({"config": cfg, "ranks": 0, "us_per_pass": round(base, 2), "note": "single-GPU solver"}), flush=True)
# the per-process kernel of a multi-GPU group (kShard = 1) with one rank: the exchange overhead alone
with ajm.ShardSolver(0, 1, [0, p.Q.n], p.Q.row_ptr, p.Q.col, p.Q.val, p.b, exchange=lambda b: [b]) as s:
    s.solve(tol=0.0, maxit=20)
    s.solve(tol=0.0, maxit=300)
    i = s.info()
    print(json.dumps({"config": cfg, "ranks": 1, "us_per_pass": round(1e3 * i["last_loop_ms"] / i["last_passes"], 2),
                      "note": "per-process shard kernel, one rank"}), flush=True)
for R in Rs:
    with ajm.ShardGroup.from_csr(p.Q, p.b, R) as g:
        g.solve(tol=0.0, maxit=20)
        g.solve(tol=0.0, maxit=300)
        i = g.info(0)
        us = 1e3 * i["last_loop_ms"] / i["last_passes"]
        halo = sum(g.info(r)["halo"] for r in range(R))
        print(json.dumps({"config": cfg, "ranks": R, "emulated": True, "us_per_pass": round(us, 2), "halo_entries": halo,
                          "grid_per_rank": i["grid"], "load_imbalance": round(g.load_imbalance(p.Q.row_ptr), 3)}),
              flush=True)
