"""Compile libflash.so for sm_100a (nvcc; no GPU needed) in-tree.

`python -m paper_1709_01190_b200.build` or `__graft_entry__.build()`.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
SO = os.path.join(PKG, "libflash.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["doph.cu", "build.cu", "query.cu", "query_sort.cu", "exchange.cu", "query_mark.cu", "util.cu", "flash_api.cu", "dist.cu"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-I", os.path.join(ROOT, "include"),
    "-I", CSRC,
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_variant(name: str, defines: list[str]) -> str:
    """A diagnostic build (e.g. libflash_qprof.so with -DFLASH_QPROF); never loaded by the product."""
    out = os.path.join(PKG, f"libflash_{name}.so")
    objdir = os.path.join(ROOT, "build", f"obj_{name}")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        subprocess.check_call([NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", o])
        objs.append(o)
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-ldl"])
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "flash.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append((src, cmd))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            futs = {ex.submit(subprocess.run, cmd, capture_output=True, text=True): src for src, cmd in jobs}
            for f in cf.as_completed(futs):
                r = f.result()
                if verbose or r.returncode != 0:
                    sys.stderr.write(r.stdout + r.stderr)
                if r.returncode != 0:
                    raise RuntimeError(f"nvcc failed for {futs[f]}")
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(SO, objs):
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-o", SO, *objs, "-ldl"])
    return SO


if __name__ == "__main__":
    if "--qprof" in sys.argv:  # diagnostic per-phase cycle counters (tools/qprof.py)
        print(build_variant("qprof", ["FLASH_QPROF"]))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(SO)
