"""Stall samples of one kernel in an .ncu-rep, by SASS region (to locate the hot phase),
plus the top instructions: python scripts/ncu_regions.py rep.ncu-rep kernel-regex [chunk] [top]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 60
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
data = []
for r in rows[2:]:
    try:
        float(r[iS] or 0)
    except (ValueError, IndexError):
        if data:
            break
        continue
    data.append(r)
stall_cols = [j for j, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[iS] or 0) for r in data)
print(f"{len(data)} instructions, {tot:.0f} samples")
seg, start = 0.0, 0
for i, r in enumerate(data):
    seg += float(r[iS] or 0)
    if (i + 1) % chunk == 0 or i == len(data) - 1:
        print(f"  #{start:4d}-{i:4d}: {seg / tot * 100:5.1f}%   {data[start][iSrc][:60]}")
        seg, start = 0.0, i + 1
for i, r in sorted(enumerate(data), key=lambda x: -float(x[1][iS] or 0))[:top]:
    st = sorted(((float(r[j] or 0), h[j][6:]) for j in stall_cols), reverse=True)[:2]
    print(f"{float(r[iS]) / tot * 100:5.1f}% #{i:4d} {r[iSrc][:58]:58s} ex={r[iE]:>7s} " +
          " ".join(f"{n}={v:.0f}" for v, n in st if v > 0))
