"""Per-CUDA-line executed warp instructions of an ncu report: python tools/ncu_inst.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, ix = {}, None
for r in rows:
    if len(r) > 2 and r[0] == "Line No":
        ix = {h: i for i, h in enumerate(r)}
        continue
    if ix is None or len(r) < 5 or r[0] in ("", "-"):
        continue
    try:
        v = float(r[ix["Instructions Executed"]] or 0)
    except (ValueError, KeyError):
        continue
    key = (int(r[0]), r[1].strip()[:90])
    agg[key] = agg.get(key, 0.0) + v
tot = sum(agg.values()) or 1.0
print(f"total warp instructions: {tot:.4g}")
for (ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{100 * v / tot:5.1f}%  L{ln:>5}  {src}")
