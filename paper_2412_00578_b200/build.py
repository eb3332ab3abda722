"""Build libss.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2412_00578_b200.build [--force] [--verbose]

Each translation unit is compiled separately; ss_geometry.cu gets --fmad=false (the
float32 arithmetic contract of DESIGN.md §3).  The shared library links the CUDA runtime
statically, so it needs only the driver at run time.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# SS_BUILD_TAG=<tag> builds a variant (e.g. the fault-injection build) into _build_<tag>/ and
# libss_<tag>.so, leaving libss.so alone; load it with SS_LIB_PATH (see _abi.py).
_TAG = os.environ.get("SS_BUILD_TAG", "")
BUILD = os.path.join(HERE, "_build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(HERE, f"libss_{_TAG}.so" if _TAG else "libss.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]
UNITS = {
    "ss_api.cu": [],
    "ss_geometry.cu": ["--fmad=false"],
    "ss_bin.cu": ["--fmad=false"],
    "ss_sort.cu": [],
    "ss_render.cu": [],
    "ss_prune.cu": [],
    "ss_backward.cu": [],
    "ss_train.cu": [],
}
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "ss.h"),
                                                      os.path.abspath(__file__)]
    objs = []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(BUILD, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            cmd = [NVCC, *ARCH, *COMMON, *extra, "-Xptxas", "-v", "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {unit}:\n{r.stderr}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
