"""Build libhjb200.so (sm_100a) in-tree with nvcc.

    python -m paper_1008_4166_b200.build [--verbose-ptxas]

Every translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked against
the NCCL that ships with torch (same soname the process already has loaded).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("HJB_LIB") or os.path.join(HERE, "libhjb200.so")
OBJ = os.path.join(ROOT, "build", "obj" + os.environ.get("HJB_OBJ_TAG", ""))
SOURCES = ["schedule.cpp", "gram.cu", "pivot.cu", "pivot_c128.cu", "factor.cu", "jacobi.cu", "update.cu", "solver.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's NCCL wheel
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    return shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


HEADERS = [os.path.join(CSRC, h) for h in ("common.cuh", "kernels.h", "schedule.h", "rotation.cuh")] + [
    os.path.join(ROOT, "include", "hjb200.h")]


def _up_to_date(src, obj, flags):
    """Incremental: the object is newer than its source and the shared
    headers, and was built with the same command line."""
    stamp = obj + ".cmd"
    if not (os.path.exists(obj) and os.path.exists(stamp)):
        return False
    if open(stamp).read() != " ".join(flags):
        return False
    t = os.path.getmtime(obj)
    deps = [src] + HEADERS + ([os.path.join(CSRC, "pivot.cu")] if src.endswith("pivot_c128.cu") else [])
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def _compile(src, inc, verbose, force=False):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    flags = [nvcc(), "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
             "-I", os.path.join(ROOT, "include"), "-I", inc, "-c", src, "-o", obj]
    flags += os.environ.get("HJB_NVCC_FLAGS", "").split()
    if src.endswith(".cu"):
        flags += ["--expt-relaxed-constexpr"]
        if verbose:
            flags += ["-Xptxas", "-v"]
    else:
        flags[1:1] = ["-x", "cu"]
    if not force and not verbose and _up_to_date(src, obj, flags):
        return obj, ""
    r = subprocess.run(flags, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".cmd", "w") as f:
        f.write(" ".join(flags))
    return obj, r.stderr


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "hjb200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    inc, lib = nccl_dirs()
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    with cf.ThreadPoolExecutor(len(srcs)) as ex:
        results = list(ex.map(lambda s: _compile(s, inc, verbose, force), srcs))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = OUT + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{lib}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose-ptxas" in sys.argv))
