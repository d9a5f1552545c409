"""Build the in-tree C-ABI library ``libparm_b200.so`` for sm_100a with nvcc.

The library is the product's native code: every CUDA kernel of the MoE-layer
hot path plus the ``extern "C"`` boundary declared in ``include/parm_b200.h``.
It is built in-tree (not into a JIT cache) so it travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
ROOT = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libparm_b200.so"
STAMP = PKG_DIR / ".libparm_b200.stamp"

SOURCES = ["capi.cu", "gate.cu", "permute.cu", "gemm_sm100.cu"]
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libparm_b200.so")
    return cand


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "parm_b200.h",
                                                                           Path(__file__)]):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(os.environ.get("PARM_NVCC_DEFINES", "").encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    digest = _digest()
    if not force and LIB_PATH.exists() and STAMP.exists() and STAMP.read_text().strip() == digest:
        return LIB_PATH
    nvcc = _nvcc()
    objs = []
    build_dir = PKG_DIR / "build"
    build_dir.mkdir(exist_ok=True)
    flags = ARCH_FLAGS + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                          "-I", str(ROOT / "include")]
    flags += os.environ.get("PARM_NVCC_DEFINES", "").split()      # experiments only (e.g. -DPARM_EPI_BUFS=1)
    if verbose or os.environ.get("PARM_PTXAS_VERBOSE"):
        flags += ["-Xptxas", "-v"]
    for src in SOURCES:
        obj = build_dir / (src + ".o")
        cmd = [nvcc, *flags, "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        objs.append(str(obj))
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    STAMP.write_text(digest)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
