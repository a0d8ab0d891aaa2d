"""Compile the native library liblevyh_b200.so for sm_100a (in-tree).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, one object per
source (parallel), linked into paper_1812_08324_b200/liblevyh_b200.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "liblevyh_b200.so")
TESTLIB = os.path.join(HERE, "liblevyh_b200_testing.so")  # test / diagnostic hooks (csrc/testing)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(HERE, "..", "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src, extra):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    hm = _headers_mtime()
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hm):
        return obj
    lang = ["-x", "cu"] if src.endswith(".cpp") else []
    cmd = [NVCC, *ARCH, *FLAGS, *extra, *lang, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def _link(out, objs, libs):
    cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, *libs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")


def build(verbose=False, extra=()):
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    tsrcs = sorted(glob.glob(os.path.join(CSRC, "testing", "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, list(extra)), srcs))
        tobjs = list(ex.map(lambda s: _compile(s, list(extra)), tsrcs))
    newest = max(os.path.getmtime(o) for o in objs)
    built = False
    if not (os.path.exists(LIB) and os.path.getmtime(LIB) >= newest):
        _link(LIB, objs, ["-lcudart", "-Xlinker", "-soname=liblevyh_b200.so"])
        built = True
    tnewest = max([os.path.getmtime(o) for o in tobjs] + [os.path.getmtime(LIB)])
    if tobjs and not (os.path.exists(TESTLIB) and os.path.getmtime(TESTLIB) >= tnewest):
        _link(TESTLIB, tobjs, ["-L" + HERE, "-llevyh_b200", "-lcudart", "-Xlinker", "-rpath=$ORIGIN"])
        built = True
    if verbose and built:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True, extra=sys.argv[1:])
