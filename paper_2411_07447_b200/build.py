"""In-tree build of libsimsweep.so (nvcc, sm_100a only)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "simsweep.cu")]
HDRS = [os.path.join(PKG, "csrc", h) for h in ("sim_kernel.cuh", "sim_step.cuh", "sim_lean.cuh", "sim_analytics.cuh", "sim_optimum.cuh")]
DEPS = SRC + HDRS + [os.path.join(ROOT, "include", "simsweep.h")]
LIB = os.path.join(PKG, "libsimsweep.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",  # no FMA contraction anywhere: fp64 clocks must match the oracle bit for bit (Q36)
    "-Xcompiler", "-fPIC", "-shared",
    "-I" + os.path.join(ROOT, "include"),
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, profile: bool = False, defines=(), lib=None) -> str:
    """profile=True builds libsimsweep_prof.so with per-phase cycle counters (tools/probe.py); `lib` and
    `defines` build comparison variants (e.g. -DSIM_NT_SMALL=128) under another name."""
    lib = lib or (LIB.replace(".so", "_prof.so") if profile else LIB)
    if force or profile or lib != LIB or needs_build():
        cmd = ([NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + (["-DSIMSWEEP_PROFILE"] if profile else []) + ["-D" + d for d in defines]
               + ["-o", lib] + SRC)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libsimsweep.so")
        if verbose:
            sys.stderr.write(r.stdout + r.stderr)
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
