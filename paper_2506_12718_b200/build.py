"""Build libpafft_b200.so in-tree with nvcc for sm_100a.

Every .cu under csrc/ is compiled to an object (in parallel, incrementally:
an object is rebuilt when it or any header under csrc/ or include/ is newer),
then linked into paper_2506_12718_b200/libpafft_b200.so.  No JIT, no torch
extension cache: the .so travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# PAFFT_BUILD_TAG=<tag>: an A/B variant build (its own object dir, output
# ab/lib<tag>.so), used with PAFFT_LIB=ab/lib<tag>.so
_TAG = os.environ.get("PAFFT_BUILD_TAG", "")
OBJ = os.path.join(HERE, "_build" + ("_" + _TAG if _TAG else ""))
LIB = os.path.join(ROOT, "ab", "lib%s.so" % _TAG) if _TAG else os.path.join(HERE, "libpafft_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", *os.environ.get("PAFFT_NVCC_EXTRA", "").split(),
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "inst", "*.cu")))


def _headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _obj_for(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(OBJ, rel[:-3] + ".o")


def _compile(src, verbose):
    obj = _obj_for(src)
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hmt = _headers_mtime()
    # objects are stale when the compiler flags changed (e.g. PAFFT_NVCC_EXTRA)
    stamp = os.path.join(OBJ, "flags.txt")
    flags = " ".join([NVCC, *ARCH, *FLAGS])
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags
    todo, objs = [], []
    for src in _sources():
        obj = _obj_for(src)
        objs.append(obj)
        if not same_flags or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hmt):
            todo.append(src)
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(jobs) as ex:
            for obj, log in ex.map(lambda s: _compile(s, verbose), todo):
                if verbose and log:
                    print(log, file=sys.stderr)
    with open(stamp, "w") as f:
        f.write(flags)
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
