"""Per-CUDA-line stall summary of an ncu report:  python tools/ncu_lines.py REP.ncu-rep [N]
(runs `ncu -i REP --page source --csv --print-source cuda,sass` and sums the warp-stall samples
of the CUDA source lines)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, hdr, ix = {}, None, {}
for r in rows:
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5 or r[0] in ("", "-"):
        continue
    try:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    key = (int(r[0]), r[1].strip()[:100])
    agg[key] = agg.get(key, 0.0) + s
tot = sum(agg.values()) or 1.0
for (ln, src), s in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{100 * s / tot:5.1f}%  L{ln:>5}  {src}")
