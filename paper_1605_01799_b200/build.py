"""Build libhopf.so in-tree with nvcc for sm_100a (B200).  No GPU needed to build.

    python -m paper_1605_01799_b200.build [--force] [--verbose]

Each .cu in csrc/ is compiled to an object in parallel, then linked into
``paper_1605_01799_b200/libhopf.so`` (git-ignored; it travels to the GPU box with gpurun).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OUT = PKG / "libhopf.so"
BUILD = PKG / "_build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -ftz=true mirrors the paper's "denormalized number mode has been disabled";
# IEEE division / square root are kept (they decide the shrink factor and the stopping test).
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ftz=true", "-prec-div=true",
         "-prec-sqrt=true", "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _deps_mtime():
    files = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return max(f.stat().st_mtime for f in files)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> Path:
    if not force and OUT.exists() and OUT.stat().st_mtime >= _deps_mtime():
        return OUT
    BUILD.mkdir(exist_ok=True)
    extra = ["-Xptxas", "-v"] if ptxas_v else []
    # experiments only (extra -D flags)
    extra += os.environ.get("HOPF_EXTRA_NVCC_FLAGS", "").split()

    def compile_one(src: Path):
        obj = BUILD / (src.stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = OUT.with_suffix(f".{os.getpid()}.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose or a.ptxas_v, ptxas_v=a.ptxas_v))
