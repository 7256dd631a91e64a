"""Summarise an ncu --page source --csv dump: top instructions by stall samples + stall totals."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0.0 for h in stall_cols}
recs = []
for r in data:
    try:
        s = float(r[samp] or 0)
    except ValueError:
        continue
    for h in stall_cols:
        try:
            tot[h] += float(r[ix[h]] or 0)
        except ValueError:
            pass
    recs.append((s, r[ix["Address"]], r[ix["Source"]], {h: r[ix[h]] for h in stall_cols}))
T = sum(tot.values())
print("stall totals:", ", ".join(f"{k[6:]}={100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0.005 * T))
recs.sort(key=lambda x: -x[0])
S = sum(r[0] for r in recs)
for s, a, src, st in recs[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(((float(v or 0), k[6:]) for k, v in st.items()), reverse=True)[:2]
    print(f"{100*s/S:5.1f}% {a} {src[:70]:70s} {top}")
