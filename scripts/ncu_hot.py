"""Top SASS instructions by stall samples of the first kernel in an .ncu-rep:
python scripts/ncu_hot.py rep.ncu-rep [n]"""
import csv, io, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
stall_cols = [j for j, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[iS] or 0) for r in data)
print(f"samples {tot:.0f}  warp-instructions {sum(float(r[iE] or 0) for r in data):.0f}")
for i, r in sorted(enumerate(data), key=lambda x: -float(x[1][iS] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    st = sorted(((float(r[j] or 0), h[j][6:]) for j in stall_cols), reverse=True)[:2]
    print(f"{float(r[iS]) / tot * 100:5.1f}% #{i:4d} {r[iSrc][:60]:60s} ex={r[iE]:>8s} " +
          " ".join(f"{n}={v:.0f}" for v, n in st if v > 0))
