"""Build the sm_100a shared library ``_tf_b200.so`` in-tree with nvcc.

Usage: python -m paper_2510_02758_b200.build [--force]

The library is a plain C-ABI ``.so`` (include/tokenflow_b200.h) with the CUDA
runtime linked statically, so the same file runs in this container and on the
GPU box.  The selector translation unit is compiled with ``-fmad=false`` and
the host passes with ``-ffp-contract=off``: its float64 arithmetic must round
exactly like CPython's (no implicit fused multiply-adds).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_tf_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "-Xcompiler", "-fPIC,-ffp-contract=off",
                 "-I", str(PKG.parent / "include")]
UNITS = {
    "tf_pool.cu": [],
    "tf_swap.cu": [],
    "tf_append.cu": [],
    "tf_attn.cu": [],
    "tf_attn_tma.cu": [],
    "tf_ops.cu": [],
    "tf_select.cu": ["-fmad=false"],
    "tf_ar.cu": [],
}


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*")) + [PKG.parent / "include" / "tokenflow_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    cmds, objs = [], []
    for unit, extra in UNITS.items():
        obj = objdir / (unit + ".o")
        cmds.append([NVCC, *COMMON, *extra, "-c", str(CSRC / unit), "-o", str(obj)])
        objs.append(str(obj))
    # translation units are independent: compile them in parallel
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        list(ex.map(run, cmds))
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
