"""Build libdinr.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2404_19075_b200.build [--verbose]

The library is a single translation unit (csrc/api.cu includes the kernel headers).  NCCL is
resolved at run time with dlopen (csrc/nccl_dl.cuh); only its header is used at build time.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libdinr.so")
SRC_DIR = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _sources():
    out = [os.path.join(INC, "dinr.h")]
    for f in sorted(os.listdir(SRC_DIR)):
        if f.endswith((".cu", ".cuh")):
            out.append(os.path.join(SRC_DIR, f))
    return out


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str = SO, defines=()) -> str:
    if out == SO and not force and not needs_build():
        return SO
    cmd = [
        NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
        "-Xcompiler", "-fPIC,-O2", "-shared", "-o", out + ".tmp", os.path.join(SRC_DIR, "api.cu"),
        "-I", INC, "-ldl",
    ] + [f"-D{d}" for d in defines]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:  # experiment variant: python -m ...build --variant tag -DFOO=1 ...
        tag = sys.argv[sys.argv.index("--variant") + 1]
        extra = [a[2:] for a in sys.argv if a.startswith("-D")]
        print(build(force=True, out=os.path.join(HERE, f"libdinr_var_{tag}.so"), defines=extra))
    elif "--phases" in sys.argv:  # debug variant with per-phase cycle counters in k_fused
        extra = [a[2:] for a in sys.argv if a.startswith("-D")]
        tag = "_".join(e.lower().replace("dinr_exp_", "") for e in extra)
        print(build(force=True, out=os.path.join(HERE, f"libdinr_phases{('_' + tag) if tag else ''}.so"),
                    defines=["DINR_PHASES"] + extra))
    else:
        build(force=True, verbose="--verbose" in sys.argv)
        print(SO)
