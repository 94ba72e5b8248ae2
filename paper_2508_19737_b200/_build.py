"""Build libigp.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python paper_2508_19737_b200/_build.py      (not -m: importing the package loads libigp.so)
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libigp.so")
SOURCES = ["csr_build.cu", "philox.cu", "embed.cu", "igp_api.cu", "birch.cu", "birch_tc.cu"]
HEADERS = ["igp_internal.cuh", "philox.cuh"]
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-Xcompiler", "-fvisibility=hidden",
         "-I" + os.path.join(ROOT, "include")]
if os.environ.get("IGP_DEBUG") == "1":  # device asserts on every dereferenced index (igp_internal.cuh)
    FLAGS += ["-DIGP_DEBUG"]
if os.environ.get("IGP_FIT_PROFILE") == "1":  # BIRCH fit phase cycle counts printed per launch (tooling)
    FLAGS += ["-DIGP_FIT_PROFILE"]
if os.environ.get("IGP_TC_STATS") == "1":  # tensor-core predict: rows re-checked / sent to fp64 (tooling)
    FLAGS += ["-DIGP_TC_STATS"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "igp.h")]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + common):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if verbose or res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link failed: " + " ".join(cmd))
        os.replace(tmp, LIB)
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "embed_c.c")
EXAMPLE_BIN = os.path.join(ROOT, "examples", "embed_c")


def build_example(force: bool = False) -> str:
    """The plain-C consumer of the ABI (examples/embed_c.c), linked against libigp.so."""
    lib = build()
    if force or _stale(EXAMPLE_BIN, [EXAMPLE_SRC, lib, os.path.join(ROOT, "include", "igp.h")]):
        cuda_home = os.environ.get("CUDA_HOME", "/usr/local/cuda")
        tmp = EXAMPLE_BIN + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-I" + os.path.join(ROOT, "include"),
               "-I" + os.path.join(cuda_home, "include"), "-o", tmp, EXAMPLE_SRC, "-L" + PKG, "-ligp",
               "-Wl,-rpath," + PKG, "-L" + os.path.join(cuda_home, "lib64"), "-lcudart", "-lm"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("example build failed: " + " ".join(cmd))
        os.replace(tmp, EXAMPLE_BIN)
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
