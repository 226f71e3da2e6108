"""Build libdak.so (the C-ABI library) in-tree with nvcc for sm_100a.

Usage: python -m paper_2604_26074_b200.build   (also called by __graft_entry__.build()).
Every translation unit is compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo; the
planner additionally with -ffp-contract=off (bit-exact double arithmetic, reading R6).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libdak.so")
OBJ = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL >= 2.28 headers (device API) shipped with torch's NCCL wheel (only nvls.cu uses them)
NCCL_INC = ""
try:
    import nvidia.nccl as _nn
    NCCL_INC = os.path.join(list(_nn.__path__)[0], "include")
except Exception:
    pass

SOURCES = [
    ("abi.cpp", []),
    ("planner.cpp", ["-Xcompiler", "-ffp-contract=off", "-fmad=false"]),
    ("model.cpp", ["-Xcompiler", "-ffp-contract=off", "-fmad=false"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=0"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=1"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=2"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=3"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=4"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=5"]),
    ("linear.cu", ["-DDAK_LINEAR_PART=6"]),
    ("attention.cu", []),
    ("prefill.cu", []),
    ("layer.cu", []),
    ("tp.cu", []),
    ("nvls.cu", ["-I", NCCL_INC]),
    ("calib.cu", []),
    ("chain.cu", []),
]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def build(verbose: bool = False) -> str:
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ, exist_ok=True)
    objs, jobs = [], []
    for src, extra in SOURCES:
        path = os.path.join(CSRC, src)
        tag = "".join(e.split("=")[-1] for e in extra if e.startswith("-DDAK_LINEAR_PART"))
        obj = os.path.join(OBJ, src + tag + ".o")
        deps = [path, os.path.join(CSRC, "common.h"), os.path.join(CSRC, "ptx.cuh"), os.path.join(ROOT, "include", "dak.h")]
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(d) for d in deps if os.path.exists(d)):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                   "-Xptxas", "-v" if verbose else "-O3", *extra, "-c", path, "-o", obj]
            jobs.append(cmd)
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for out in ex.map(_run, jobs):
            if verbose:
                sys.stderr.write(out)
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        _run([NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-lcudart", "-ldl"])
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
