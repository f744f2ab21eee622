"""Build the in-tree CUDA library ``libtailorkv.so`` for sm_100a with nvcc.

The shared object lands next to this file so it travels with the repository
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtailorkv.so"
SOURCES = ["abi.cu", "qcache.cu", "decode.cu", "decode_imma.cu", "sparse.cu", "sparse_fused.cu", "calibrate.cu", "fidelity.cu", "refops.cu", "sparse_wide.cu"]
# extra objects: (source, object stem, defines) -- the fused sparse kernel again with 4- and 2-CTA clusters
VARIANTS = [("sparse_fused.cu", "sparse_fused4", ["-DTKV_FZ_CTAS=4"]),
            ("sparse_fused.cu", "sparse_fused2", ["-DTKV_FZ_CTAS=2"])]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-warn-spills",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtailorkv.so")
    return exe


def needs_build() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "tailorkv.h"]
    return any(p.stat().st_mtime > mtime for p in deps)


def build(force: bool = False, verbose: bool = False, jobs: int = 6) -> Path:
    if not force and not needs_build():
        return LIB
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    procs = []
    objs = []
    for src, stem, defs in [(x, Path(x).stem, []) for x in SOURCES] + VARIANTS:
        obj = objdir / (stem + ".o")
        objs.append(obj)
        extra = os.environ.get("TKV_NVCC_DEFINES", "").split()  # experiments
        cmd = [nvcc(), *NVCC_FLAGS, *defs, *extra, "-I", str(ROOT / "include"), "-I", str(CSRC), "-c",
               str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        while sum(p.poll() is None for _, p in procs) >= jobs:
            procs[0][1].wait()
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose and out.strip():
            print(out)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "shared",
           "-o", str(tmp), *map(str, objs)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
