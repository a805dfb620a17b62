"""Build the product library libfastmaxent.so (sm_100a) in-tree with nvcc.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false (no FMA contraction
anywhere: the decision path must reproduce the oracle's IEEE operation sequence, DESIGN R12).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfastmaxent.so")
BUILD = os.path.join(HERE, "_build")
SOURCES = ["fm_scan.cu", "fm_sort.cu", "fm_plan.cu", "fm_sample.cu", "fm_expect.cu", "fm_capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O2", "-I", INC, "-I", CSRC,
         "-Xptxas", "-v"] if os.environ.get("FM_PTXAS_VERBOSE") else \
        ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O2", "-I", INC, "-I", CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INC, "fastmaxent.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build_variant(tag: str, defines: list, csrc: str = None) -> str:
    """Experimental build with extra -D flags (and optionally another source tree, e.g. a git
    revision exported to /tmp) -> libfastmaxent.<tag>.so, loaded with FM_LIB_VARIANT=tag."""
    global LIB, BUILD, FLAGS, CSRC
    saved = LIB, BUILD, FLAGS, CSRC
    LIB = os.path.join(HERE, f"libfastmaxent.{tag}.so")
    BUILD = os.path.join(HERE, f"_build_{tag}")
    if csrc:
        CSRC = csrc
    FLAGS = [f if f != saved[3] else CSRC for f in FLAGS] + [f"-D{d}" for d in defines]
    try:
        return build(force=True)
    finally:
        LIB, BUILD, FLAGS, CSRC = saved


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stdout.write(out)
        if p.returncode != 0:
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python build.py --variant TAG [--csrc DIR] [DEFINE ...]
        i = sys.argv.index("--variant")
        rest = sys.argv[i + 2:]
        src = None
        if rest[:1] == ["--csrc"]:
            src, rest = rest[1], rest[2:]
        print(build_variant(sys.argv[i + 1], rest, src))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
