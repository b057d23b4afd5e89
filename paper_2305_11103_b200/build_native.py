"""Build libblockinv_b200.so (sm_100a) in-tree with nvcc.

Used by ``__graft_entry__.build()`` and the test/bench harnesses.  Every
translation unit is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3`` and linked into one shared library next to this file.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
INCLUDE = HERE.parent / "include"
LIB = HERE / "libblockinv_b200.so"
OBJDIR = HERE.parent / "build" / "obj"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]

SOURCES = ["bi_gemm.cu", "bi_gemm_tma.cu", "bi_gemm_peer.cu", "bi_inv.cu", "bi_engine.cu", "bi_capi.cu", "bi_nccl.cu"]


def _deps() -> list[Path]:
    return [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: Path | None = None, extra: list | None = None) -> Path:
    """Compile and link; ``out``/``extra`` build a variant (e.g. -DBI_K1_GROUP_M=8)
    elsewhere for A/B timing through BI_LIB, leaving the in-tree library alone."""
    if out is None and not force and not needs_build():
        return LIB
    target = LIB if out is None else Path(out)
    objdir = OBJDIR if out is None else target.parent / (target.stem + "_obj")
    objdir.mkdir(parents=True, exist_ok=True)
    extra = list(extra or [])

    def compile_one(src: str) -> Path:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = target.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
