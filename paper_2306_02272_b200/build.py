"""Build libowq.so in-tree: nvcc for the sm_100a kernels, g++ (OpenMP) for the
host packer, NCCL from the image's nvidia-nccl wheel.  Usage:
    python -m paper_2306_02272_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
OUT = os.path.join(HERE, "libowq.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU = ["owq_gemv.cu", "owq_gemv_cc.cu", "owq_tp.cu", "owq_quant.cu", "owq_prefill.cu"]
CPP = ["owq_pack.cpp"]
HDRS = ["owq_layout.h", "owq_layout_cc.h", "owq_ptx.cuh"]


def nccl_dirs():
    try:
        import nvidia.nccl as n  # type: ignore
        base = list(n.__path__)[0]
    except Exception:  # pragma: no cover
        base = "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r


def needs_build(force=False):
    if force or not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    srcs = [os.path.join(CSRC, f) for f in CU + CPP + HDRS] + [os.path.join(INC, "owq.h"), __file__]
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False, csrc: str = None, out: str = None, inc: str = None,
          defines=()) -> str:
    """csrc/out/inc/defines: experiments only (A/B builds of another source tree or
    with -D knobs into another file; the product build uses the defaults)."""
    global CSRC, OUT, BUILD, INC
    if defines and not out:
        raise ValueError("-D builds are experiments: give --out (the product library is built without them)")
    if csrc or out or inc or defines:
        CSRC, OUT, INC = csrc or CSRC, out or OUT, inc or INC
        BUILD = OUT + "_build"
        force = True
    if not needs_build(force):
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    ninc, nlib = nccl_dirs()
    objs = []
    for f in CU:
        o = os.path.join(BUILD, f + ".o")
        cmd = [NVCC, *ARCH, *[f"-D{d}" for d in defines], "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3",
               "-I", INC, "-I", CSRC, "-I", ninc, "-c", os.path.join(CSRC, f), "-o", o]
        r = _run(cmd)
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    for f in CPP:
        o = os.path.join(BUILD, f + ".o")
        _run(["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-I", INC, "-I", CSRC,
              "-c", os.path.join(CSRC, f), "-o", o])
        objs.append(o)
    tmp = OUT + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fopenmp",
          "-L", nlib, "-l:libnccl.so.2", f"-Xlinker=-rpath={nlib}", "-lgomp"])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    a = sys.argv
    opt = lambda k: a[a.index(k) + 1] if k in a else None
    print(build(force="--force" in a, verbose="-v" in a, csrc=opt("--csrc"), out=opt("--out"), inc=opt("--inc"),
                defines=[a[i + 1] for i, v in enumerate(a) if v == "-D"]))
