#!/usr/bin/env python
"""Copy one evidence run (tools/gpu_r02full.sh <tag>, results in gpurun_out/) into profiles/r02/:
bench lines (default, every config, reference arm), ncu launch lists, ncu --set full summaries,
the GPU pytest log and the smoke log.  usage: python tools/collect_evidence.py <tag>"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
src, dst = ROOT / "gpurun_out", ROOT / "profiles" / "r02"


def line(log):
    for ln in (src / log).read_text().splitlines():
        if ln.startswith("{"):
            json.loads(ln)
            return ln
    raise SystemExit(f"no JSON line in {log}")


(dst / "bench_default.jsonl").write_text(line(f"bench_default_{tag}.log") + "\n")
(dst / "bench_reference.jsonl").write_text(line(f"bench_ref_{tag}.log") + "\n")
cfgs = ["c2", "c5", "c4", "c1", "c5d", "c2h", "c2e", "c2i", "t5", "t4a"]
(dst / "bench_configs.jsonl").write_text("".join(line(f"bench_{c}_{tag}.log") + "\n" for c in cfgs))
for c in ("c3", "c2", "c5", "c4"):
    shutil.copy(src / f"launches_{c}_{tag}.csv", dst / f"launches_{c}.csv")
    rep = src / f"prof_{c}_{tag}.ncu-rep"
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)],
                         capture_output=True, text=True, check=True).stdout
    (dst / f"ncu_{c}_r02.json").write_text(out)
shutil.copy(src / f"pytest_gpu_{tag}.log", dst / "pytest_gpu.log")
shutil.copy(src / f"smoke_{tag}.log", dst / "smoke.log")
print("collected", tag)
