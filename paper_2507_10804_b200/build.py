"""Build libhv.so in-tree for sm_100a (nvcc cross-compiles here; no GPU needed).

    python -m paper_2507_10804_b200.build [--ptxas-verbose]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhv.so")
SOURCES = ["hv_api.cu", "hv_runtime.cu", "psido.cu", "probing.cu", "lowrank.cu", "psfplus.cu"]
HEADERS = ["hv_kernels.cuh", "hv_t2.cuh", "hv_geo.h", "hv_internal.h", os.path.join("..", "..", "include", "hv.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS + [os.path.basename(__file__)]:
        p = os.path.join(CSRC, f) if f != os.path.basename(__file__) else os.path.abspath(__file__)
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force: bool = False, ptxas_verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile libhv.so (or a tuning variant `out` with -D`defines`)."""
    if out == LIB and not force and not _stale():
        return LIB
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden",
           *[f"-D{d}" for d in defines],
           "-o", out + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES],
           "-lcufft", "-lcublas", "-lcusolver", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    if ptxas_verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if ptxas_verbose:
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    build(force=True, ptxas_verbose="--ptxas-verbose" in sys.argv)
    print(LIB)
