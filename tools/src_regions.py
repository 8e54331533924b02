#!/usr/bin/env python
"""Instruction and stall-sample share of each execution-count band of an ncu source export
(--page source --csv --print-source sass).  usage: src_regions.py src.csv [top]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
iex = hdr.index("Instructions Executed"); ist = hdr.index("Warp Stall Sampling (All Samples)")
band = collections.defaultdict(lambda: [0, 0, 0])
for r in data:
    e = float(r[iex] or 0); s = float(r[ist] or 0)
    if e == 0: continue
    k = f"{e:.2g}"
    band[k][0] += e; band[k][1] += s; band[k][2] += 1
I = sum(v[0] for v in band.values()); S = sum(v[1] for v in band.values())
print(f"total instr {I:.4g}  samples {S:.0f}")
for k, v in sorted(band.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"count {k:>8} x {v[2]:4d} lines: {100*v[0]/I:5.1f}% instr {100*v[1]/S:5.1f}% samples")
