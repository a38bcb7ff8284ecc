"""In-tree build of libhcg.so (sm_100a only) with nvcc.

The .so lands next to this file so it travels with the repo snapshot to the
GPU box; objects go to csrc/build/ (git-ignored).
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libhcg.so")
ROOT = os.path.dirname(HERE)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
CU = ["build.cu", "search.cu", "brute_tc.cu", "datagen.cu", "api.cu", "shard.cu"]
CPP = ["planner.cpp", "io.cpp", "serve.cpp"]
HEADERS = ["hcg_internal.cuh", "hcg_host.hpp"]


def _nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.sep not in p or os.path.exists(p)):
            return p
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False) -> str:
    """Compile every CUDA/C++ source and link libhcg.so; returns its path.
    HCG_DEBUG_BOUNDS=1 in the environment compiles the device bounds checks in
    (objects go to csrc/build-debug/ so the two builds do not mix)."""
    global OBJ
    debug = os.environ.get("HCG_DEBUG_BOUNDS") == "1"
    if debug:
        OBJ = os.path.join(CSRC, "build-debug")
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "hcg.h")]
    jobs = []
    for src in CU + CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if _stale(o, [s] + hdrs) or ptxas_info:
            flags = list(NVCC_FLAGS) + (["-DHCG_DEBUG_BOUNDS"] if debug else [])
            if ptxas_info and src.endswith(".cu"):
                flags += ["-Xptxas", "-v"]
            if src.endswith(".cpp"):
                flags = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
                if src == "serve.cpp":  # host code on the CUDA runtime
                    flags += ["-x", "cu"] + ARCH
            jobs.append([_nvcc()] + flags + ["-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose or ptxas_info:
            print(r.stdout + r.stderr)

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, s + ".o") for s in CU + CPP]
    stamp = LIB + ".flavor"
    flavor = "debug" if debug else "release"
    if _stale(LIB, objs) or not os.path.exists(stamp) or open(stamp).read() != flavor:
        tmp = LIB + ".tmp"
        run([_nvcc(), "-shared"] + ARCH + ["-cudart", "static", "-o", tmp] + objs + ["-ldl"])
        os.replace(tmp, LIB)
        with open(stamp, "w") as f:
            f.write(flavor)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(verbose=True, ptxas_info="-v" in sys.argv))
