"""In-tree build of libcgmimo_b200.so (sm_100a) with nvcc + g++.

The shared library holds the CUDA kernels, the C ABI (include/cgmimo_b200.h)
and the C++ drop-in (include/cgmimo/*.hpp).  It is built next to this file so
it travels with the repo snapshot to the GPU box; the CUDA runtime is linked
statically so the library does not depend on which libcudart torch loaded.
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcgmimo_b200.so")
OBJ = os.path.join(PKG, "_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["cgm_capi.cu", "cgm_generate.cu", "cgm_harness.cu"]
CPP = ["cgm_dropin.cpp"]
HDRS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))


def _newer(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    inc = ["-I" + os.path.join(ROOT, "include")]
    hdeps = [os.path.join(CSRC, h) for h in HDRS] + [os.path.join(ROOT, "include", "cgmimo_b200.h")]
    objs = []
    log = ""
    jobs = []
    for src in CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if _newer(o, [s] + hdeps + [__file__]):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
                         "-Xcompiler", "-fPIC", *os.environ.get("CGM_NVCC_EXTRA", "").split(), *inc, "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:  # translation units in parallel
        for out in ex.map(_run, jobs):
            log += out
    for src in CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        hpp = [os.path.join(ROOT, "include", "cgmimo", f)
               for f in os.listdir(os.path.join(ROOT, "include", "cgmimo"))]
        if _newer(o, [s] + hpp + hdeps + [__file__]):
            log += _run(["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", *inc, "-c", s,
                         "-o", o])
    if _newer(LIB, objs):
        log += _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl",
                     "-lpthread"])
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    print(LIB)
