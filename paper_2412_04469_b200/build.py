"""Builds libqueen.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so travels with the repo."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqueen.so")
SOURCES = ["queen_api.cu", "decode_apply.cu", "project.cu", "binning.cu", "raster.cu", "mask.cu", "densify.cu", "backward.cu", "entropy.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# Arithmetic contract: no FMA contraction, IEEE div/sqrt, denormals kept.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Build libqueen.so; `out` / `defines` build an experiment variant (tools/variants.py)."""
    lib_path = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "queen_internal.cuh"), os.path.join(HERE, "..", "include", "queen.h")]
    if not force and os.path.exists(lib_path) and os.path.getmtime(lib_path) >= max(os.path.getmtime(d) for d in deps):
        return lib_path
    tmp = lib_path + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], *srcs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log") if out is None else out + ".log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
