"""Summarise an `ncu --page source --csv` export: stall reasons overall and the hottest
instructions.  python scripts/ncu_stalls.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hi], rows[hi + 1:]
ci = {h: i for i, h in enumerate(hdr)}
S = ci["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
f = lambda r, k: float(r[ci[k]] or 0) if r[ci[k]] not in ("", None) else 0.0
tot, agg = 0.0, {}
for r in data:
    try:
        s = float(r[S] or 0)
    except ValueError:
        continue
    tot += s
    for h in stalls:
        try:
            agg[h] = agg.get(h, 0) + f(r, h)
        except ValueError:
            pass
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"{k:25s} {v:8.0f} {100 * v / max(tot, 1):5.1f}%")
top = sorted((r for r in data if r[S].replace('.', '', 1).isdigit()), key=lambda r: -float(r[S]))[:top_n]
for r in top:
    st = {h: f(r, h) for h in stalls}
    best = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{float(r[S]):6.0f} {r[ci['Address']]:>6s} {r[ci['Source']][:64]:64s} "
          + " ".join(f"{k[6:]}={v:.0f}" for k, v in best))
