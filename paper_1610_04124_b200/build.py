"""In-tree build of the CUDA library (sm_100a) -- `libstixels.so` next to this file."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstixels.so")
SOURCES = [os.path.join(CSRC, f) for f in ("api.cu", "kernels.cuh")]
HEADER = os.path.join(os.path.dirname(HERE), "include", "stixels.h")
AB_DIR = os.path.join(os.path.dirname(HERE), "scripts", "ab")   # diagnostic / A/B builds

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + [HEADER])


def build(force: bool = False, verbose: bool = False, trace: bool = False,
          variant: str | None = None, src: str | None = None) -> str:
    """trace=True builds the diagnostic phase-timeline variant libstixels_trace.so
    (-DSTX_TRACE; scripts/trace_phases.py); variant=name builds
    scripts/ab/libstixels_<name>.so (from the api.cu at `src` if given) for A/B
    timing.  Neither is loaded by the product: only an explicit
    stixels.use_library(path) (bench.py --lib, the scripts) binds them."""
    out = LIB
    if trace:
        out = os.path.join(AB_DIR, "libstixels_trace.so")
    elif variant:
        out = os.path.join(AB_DIR, f"libstixels_{variant}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if out == LIB and not force and not stale():
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + (["-DSTX_TRACE"] if trace else []) + [
        "-o", out, src or os.path.join(CSRC, "api.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
