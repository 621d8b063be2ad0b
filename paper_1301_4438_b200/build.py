"""Build libpluq_b200.so in-tree with nvcc for sm_100a (no JIT cache, travels with the repo)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpluq_b200.so")
SOURCES = ["pluq_driver.cu"]
HEADERS = ["pluq_common.cuh", "pluq_basecase.cuh", "pluq_small.cuh", "pluq_rpm.cuh", "pluq_kernels.cuh",
           "pluq_tc_gemm.cuh", "pluq_diag.cuh", "pluq_diag2.cuh"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "pluq_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    cmd = [
        nvcc_path(), "-std=c++17",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo",
        "-Xcompiler", "-fPIC", "-shared",
        "-o", OUT + ".tmp",
    ] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    extra = os.environ.get("PLUQ_NVCC_FLAGS")  # diagnostics builds, e.g. -DPLUQ_TRACE
    if extra:
        cmd[1:1] = extra.split()
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libpluq_b200.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
