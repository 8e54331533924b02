#!/usr/bin/env python
"""Top SASS lines by warp-stall samples from an `ncu --page source --csv --print-source sass` dump."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
print(f"total samples {tot:.0f}, instructions executed {sum(float(r[i_ex] or 0) for r in data):.3g}")
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    print(f"{100*float(r[i_s])/tot:5.1f}% {r[0][-5:]} {float(r[i_ex] or 0):10.3g} {r[i_src].strip()[:90]}")
