"""Build libomniloc.so for sm_100a with nvcc (in-tree, so it travels to the GPU box), and
libomniloc_checked.so: the same sources with -DOL_CHECKED (device-side bounds checks on every
kernel's index arithmetic, read back by ol_get_stat("check") -- the stand-in for
compute-sanitizer memcheck, which is closed on this GPU pool).  The binding loads the checked
library only when OL_LIB=checked."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libomniloc.so")
LIB_CHECKED = os.path.join(HERE, "libomniloc_checked.so")
SOURCES = ["runtime.cu", "scan.cu", "merge.cu", "aggregate.cu", "tcscan.cu", "shift.cu", "extract.cu"]
HEADERS = ["ol_internal.h", "tc_ptx.cuh", os.path.join("..", "..", "include", "omniloc.h")]
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
              "-I" + os.path.join(ROOT, "include")]


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _build_one(lib: str, objdir: str, extra, verbose: bool):
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = ["nvcc", *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(objdir, src + ".ptxas.txt"), "w") as f:
            f.write(r.stderr)
        return o

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)


def build(force: bool = False, verbose: bool = False, checked: bool = True) -> str:
    if force or _stale(LIB):
        _build_one(LIB, os.path.join(HERE, "build"), [], verbose)
    if checked and (force or _stale(LIB_CHECKED)):
        _build_one(LIB_CHECKED, os.path.join(HERE, "build_checked"), ["-DOL_CHECKED"], verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
