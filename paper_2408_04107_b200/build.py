"""Build libzdc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

python -m paper_2408_04107_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
# Same-box A/B of kernel variants: ZDC_BUILD_VARIANT=<name> ZDC_BUILD_DEFS="-DFOO=1" builds
# libzdc_<name>.so from the same sources into its own object directory (load it with ZDC_LIB_PATH).
VARIANT = os.environ.get("ZDC_BUILD_VARIANT", "")
VARIANT_DEFS = os.environ.get("ZDC_BUILD_DEFS", "").split()
BUILD = os.path.join(HERE, "_build" + ("_" + VARIANT if VARIANT else ""))
LIB = os.path.join(HERE, "libzdc%s.so" % ("_" + VARIANT if VARIANT else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", f"-I{INCLUDE}", f"-I{CSRC}",
                     "--expt-relaxed-constexpr"] + VARIANT_DEFS
CXX_FLAGS = ["-O3", "-fPIC", "-std=c++17", "-fopenmp", "-march=x86-64-v3", f"-I{INCLUDE}", f"-I{CSRC}",
             "-I/usr/local/cuda/include"] + VARIANT_DEFS


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout)
        raise RuntimeError("build failed: %s" % cmd[-1])
    return r.stdout


def _stale(obj, srcs):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    objs, jobs = [], []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if _stale(obj, [src] + headers):
            jobs.append([NVCC] + CUDA_FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", obj])
        objs.append(obj)
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if _stale(obj, [src] + headers):
            jobs.append(["g++"] + CXX_FLAGS + ["-c", src, "-o", obj])
        objs.append(obj)
    # translation units compile in parallel (the fused decode kernel alone has 80 template instances)
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for out in ex.map(_run, jobs):
            if verbose:
                print(out)
    if _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-Xcompiler", "-fopenmp", "-lgomp", "-ldl", "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
