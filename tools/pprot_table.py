#!/usr/bin/env python
"""Markdown table of the paper-protocol bench lines (profiles/r02/bench_paper_protocol.jsonl)
beside the paper's Tables 1 and 4.  usage: pprot_table.py lines.jsonl"""
import json, re, sys
PAPER = {  # (J, H, n): seconds per evaluation, one laptop core
    ("id", "l1", 4): 6.36e-8, ("id", "l1", 8): 6.98e-8, ("id", "l1", 12): 8.72e-8, ("id", "l1", 16): 9.24e-8,
    ("id", "l2", 4): 1.20e-7, ("id", "l2", 8): 1.28e-7, ("id", "l2", 12): 1.56e-7, ("id", "l2", 16): 1.50e-7,
    ("diag", "l1", 4): 3.62e-7, ("diag", "l1", 8): 3.83e-7, ("diag", "l1", 12): 4.97e-7, ("diag", "l1", 16): 5.92e-7,
    ("diag", "l2", 4): 5.19e-7, ("diag", "l2", 8): 5.25e-7, ("diag", "l2", 12): 6.62e-7, ("diag", "l2", 16): 6.88e-7}
rows = []
for line in open(sys.argv[1]):
    d = json.loads(line)
    m = re.search(r"p(\d+)_(id|diag)_(l1|l2)", d["metric"])
    n, j, h = int(m.group(1)), m.group(2), m.group(3)
    r = d["roofline"]
    unit = "HBM" if r["bound"] == "hbm" else "ALU"
    rows.append((n, j, h, PAPER[(j, h, n)], d["cpu_baseline"]["value"], d["value"], d["ms_per_step"],
                 r["mean_iters"], f"{100 * r['frac']:.0f} % of {unit}"))
print("| J | H | n | paper s/eval (laptop, 1 core) | paper evals/s | oracle evals/s (16 cores) | "
      "B200 evals/s | B200 ms / 1e6 | mean iters | roofline |")
print("|---|---|---|---|---|---|---|---|---|---|")
for n, j, h, ps, ov, gv, ms, it, rf in rows:
    print(f"| {j} | {h} | {n} | {ps:.3g} | {1 / ps:.3g} | {ov:.3g} | {gv:.3g} | {ms:.3f} | {it:.1f} | {rf} |")
