#!/usr/bin/env python
"""Stall-reason totals from an ncu source csv (--page source --csv --print-source sass), split into
instructions executed about once per round (`work`) and spin loops (`spin`, > 2x the median count)."""
import csv, sys, collections, statistics
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
i_ex = hdr.index("Instructions Executed"); i_src = hdr.index("Source")
st = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
ex = [float(r[i_ex] or 0) for r in data]
med = statistics.median([e for e in ex if e > 0])
tot = {"work": collections.Counter(), "spin": collections.Counter()}
for r, e in zip(data, ex):
    k = "spin" if e > 2.5 * med else "work"
    for i, h in st:
        try: tot[k][h] += float(r[i] or 0)
        except ValueError: pass
for k in tot:
    s = sum(tot[k].values()) or 1
    print(k, f"{s:.0f} samples:", ", ".join(f"{h[6:]} {100*v/s:.1f}%" for h, v in tot[k].most_common(10)))
