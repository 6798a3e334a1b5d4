"""In-tree build of libparcube_b200.so (nvcc, sm_100a only).

The per-family instantiation units compile in parallel; objects are cached under
csrc/build/ and rebuilt when any source or header is newer.  The shared library is
written next to this file so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJDIR = os.path.join(CSRC, os.environ.get("PCB_OBJDIR", "build"))
LIB = os.path.join(HERE, os.environ.get("PCB_LIB_NAME", "libparcube_b200.so"))
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
N_FAMILIES = 8

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # numpy's a*b+c is two roundings; fused ops are explicit __fma_rn in the sources
    "-Xcompiler", "-fPIC",
    "-I", INCLUDE,
    *os.environ.get("PCB_NVCC_EXTRA", "").split(),   # experiments: -DPCB_...=...
]


def _nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; the B200 build has no other compiler path")
    return exe


def _units():
    units = [("ctx.o", "ctx.cu", []), ("pagani_host.o", "pagani_host.cu", []), ("mcubes_host.o", "mcubes_host.cu", [])]
    for fam in range(N_FAMILIES):
        units.append((f"pagani_inst_{fam}.o", "pagani_inst.cu", [f"-DPCB_FAM={fam}"]))
        units.append((f"mcubes_inst_{fam}.o", "mcubes_inst.cu", [f"-DPCB_FAM={fam}"]))
    return units


def _newest_source() -> float:
    stamps = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    stamps.append(os.path.getmtime(os.path.join(INCLUDE, "parcube_b200.h")))
    stamps.append(os.path.getmtime(os.path.abspath(__file__)))
    return max(stamps)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile (if stale) and return the path of the shared library."""
    os.makedirs(OBJDIR, exist_ok=True)
    newest = _newest_source()
    # an up-to-date library needs no objects (csrc/build/ is not shipped to the GPU box)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    nvcc = _nvcc()
    todo, objs = [], []
    for obj, src, extra in _units():
        out = os.path.join(OBJDIR, obj)
        objs.append(out)
        if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
            todo.append([nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", out])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        return res.stderr

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or min(len(todo), os.cpu_count() or 4)) as pool:
            for log in pool.map(run, todo):
                if verbose and log.strip():
                    print(log, file=sys.stderr)
    if todo or force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        run([nvcc, "-shared", "-o", LIB, *objs, "-gencode", "arch=compute_100a,code=sm_100a", "-lcudart"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
