"""Summarise per-config ncu --set full captures (gpurun_out/<tag>_ncu_cfgK.ncu-rep: caches flushed
between replays, ncu's default; gpurun_out/<tag>_ncuwarm_cfgK.ncu-rep: --cache-control none, the
bench's warm-L2 condition), each the 2nd solve of tools/prof.py K 30 = 31 passes, into
profiles/<tag>_ncu_configs.md and profiles/ncu_traffic.json (the warm capture's DRAM bytes when
present -- bench.py's dram_frac -- with the commit the capture was taken on).
usage: python tools/ncu_summary.py TAG [K ...]"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = {1: "poisson2d_64", 2: "poisson3d_128", 3: "er_1m_deg16", 4: "chunglu_4m_deg20", 5: "aniso27_256"}
PASSES = 31
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "smsp__average_warp_latency_issue_stalled_long_scoreboard"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}


def raw(rep):
    csvp = rep[: -len(".ncu-rep")] + ".raw.csv"
    if os.path.exists(csvp):  # exported on the GPU box (tools/gpu_round.sh)
        out = open(csvp).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k in M:
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            d[k] = v * SCALE.get(units[i], 1.0)
    d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    return d


def main():
    tag = sys.argv[1]
    cfgs = [int(c) for c in sys.argv[2:]] or [1, 2, 3, 4, 5]
    import paper_2407_03272_b200 as ajm  # noqa: F401  (model bytes formula only)
    import synth
    lines = [f"# {tag} -- ncu --set full per BASELINE config (solver kernel, 2nd solve of "
             f"tools/prof.py K 30 = {PASSES} passes)", "",
             "| cfg (L2 at replay) | workload | µs/pass (profiled) | DRAM MB/pass | algorithmic MB/pass | DRAM/alg | L2 hit | "
             "L1 hit | warps active | L2 thru | L1 thru |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = []
    head = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True, text=True,
                          cwd=ROOT).stdout.strip()
    for c in cfgs:
        rep = os.path.join(ROOT, "gpurun_out", f"{tag}_ncu_cfg{c}.ncu-rep")
        repw = os.path.join(ROOT, "gpurun_out", f"{tag}_ncuwarm_cfg{c}.ncu-rep")
        have = lambda r: os.path.exists(r) or os.path.exists(r[: -len(".ncu-rep")] + ".raw.csv")
        if not have(rep) and not have(repw):
            continue
        dc = raw(rep) if have(rep) else None
        dw = raw(repw) if have(repw) else None
        d = dw or dc
        if c == 1:
            n, nnz = 4096, 20224
        else:
            p = synth.config_problem(c) if c in (2, 3) else None
            n, nnz = {2: (2097152, 14581760), 5: (16777216, 449455096)}.get(c, (p.Q.n, p.Q.nnz) if p else (4000000, 80218976))
        alg = 12.0 * nnz + 56.0 * n + 4.0 * (n + 1)
        rec = {"workload": NAMES[c], "kernel": d["kernel"], "passes_profiled": PASSES,
               "algorithmic_bytes_per_pass": alg, "capture": f"{tag} @ {head}"}
        for kind, dd in (("cold", dc), ("warm", dw)):
            if dd is None:
                continue
            dram = (dd["dram__bytes_read.sum"] + dd["dram__bytes_write.sum"]) / PASSES
            lines.append(f"| {c} {kind} | {NAMES[c]} | {1e6 * dd['gpu__time_duration.sum'] / PASSES:.1f} | {dram / 1e6:.1f} | "
                         f"{alg / 1e6:.1f} | {dram / alg:.2f} | {dd['lts__t_sector_hit_rate.pct']:.1f}% | "
                         f"{dd['l1tex__t_sector_hit_rate.pct']:.1f}% | {dd['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f}% | "
                         f"{dd['lts__throughput.avg.pct_of_peak_sustained_elapsed']:.1f}% | "
                         f"{dd['l1tex__throughput.avg.pct_of_peak_sustained_active']:.1f}% |")
            rec[f"dram_bytes_per_pass_{kind}"] = dram
            rec[f"us_per_pass_profiled_{kind}"] = 1e6 * dd["gpu__time_duration.sum"] / PASSES
        rec["dram_bytes_per_pass"] = rec.get("dram_bytes_per_pass_warm", rec.get("dram_bytes_per_pass_cold"))
        # the other roofs of the same capture: L2 (lts) and L1/shared (l1tex) throughput, % of peak
        rec["l2_throughput_pct"] = d["lts__throughput.avg.pct_of_peak_sustained_elapsed"]
        rec["l1tex_throughput_pct"] = d["l1tex__throughput.avg.pct_of_peak_sustained_active"]
        rec["source"] = (f"ncu --set full --clock-control none [--cache-control none for 'warm'] on tools/prof.py {c} 30 "
                         f"(2nd solve); profiles/{tag}_ncu_configs.md")
        traffic.append(rec)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_configs.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:  # merge: replace the records of the workloads captured now, keep the others
        with open(path) as f:
            old = json.load(f)
        old = old if isinstance(old, list) else [old]
    except Exception:
        old = []
    new_names = {t["workload"] for t in traffic}
    merged = [o for o in old if o.get("workload") not in new_names] + traffic
    with open(path, "w") as f:
        json.dump(merged, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
