"""Stall samples aggregated per CUDA source line for one kernel of an .ncu-rep:
python scripts/ncu_src.py rep.ncu-rep <kernel-regex> [n]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "-k", "regex:" + kre,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r][0]
h, data = rows[hi], rows[hi + 1:]
iS, iSrc, iL = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("#")
stall_cols = [j for j, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[iS] or 0) for r in data if len(r) > iS)
print(f"samples {tot:.0f}")
for r in sorted((r for r in data if len(r) > iS), key=lambda r: -float(r[iS] or 0))[:n]:
    st = sorted(((float(r[j] or 0), h[j][6:]) for j in stall_cols), reverse=True)[:3]
    print(f"{float(r[iS]) / tot * 100:5.1f}% L{r[iL]:>4s} {r[iSrc].strip()[:80]:80s} " +
          " ".join(f"{nm}={v:.0f}" for v, nm in st if v > 0))
