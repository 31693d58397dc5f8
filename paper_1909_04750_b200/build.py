"""Build recipe for the in-tree CUDA library (sm_100a only, no JIT cache).

`python -m paper_1909_04750_b200.build` or `build_native()` compiles
csrc/mk2_api.cu (+ the headers it includes) into csrc/libmk2.so with nvcc.
nvcc cross-compiles without a GPU, so this runs in the CPU-only build
container; the .so is git-ignored but travels to the GPU box with the tree.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = CSRC / "libmk2.so"
CURAND_LIB = CSRC / "libmk2_curand.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "--use_fast_math"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA path cannot be built (there is no CPU fallback)")


def source_hash(sources) -> str:
    h = hashlib.sha256()
    for src in sorted(Path(s) for s in sources):
        h.update(src.name.encode() + b"\0")
        h.update(src.read_bytes())
    return h.hexdigest()


def _stale(target: Path, sources) -> bool:
    """A library is current when the hash of the sources it was built from (written next to it) matches the
    sources on disk.  Content, not mtimes: the tree is copied to the GPU box, and a checkout rewrites mtimes."""
    stamp = Path(str(target) + ".srchash")
    if not target.exists() or not stamp.exists():
        return True
    return stamp.read_text().strip() != source_hash(sources)


def _stamp(target: Path, sources) -> None:
    Path(str(target) + ".srchash").write_text(source_hash(sources) + "\n")


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile libmk2.so (kernels + C ABI)."""
    srcs = [*CSRC.glob("mk2_*.cuh"), *CSRC.glob("mk2_*.h"), CSRC / "mk2_api.cu", PKG.parent / "include" / "mk2.h"]
    if force or _stale(LIB, srcs):
        cmd = [nvcc(), *ARCH, *COMMON, "-Xptxas", "-v", "-o", str(LIB), str(CSRC / "mk2_api.cu"), "-lcudart"]
        res = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        (CSRC / "ptxas_mk2.log").write_text(res.stdout)
        if verbose or res.returncode:
            print(res.stdout, file=sys.stderr)
        if res.returncode:
            raise RuntimeError("nvcc failed building libmk2.so")
        _stamp(LIB, srcs)
    return LIB


def build_curand(force: bool = False) -> Path:
    """Compile the cuRAND comparison harness (bench only, not the product path)."""
    src = CSRC / "mk2_curand_bench.cu"
    if force or _stale(CURAND_LIB, [src]):
        cmd = [nvcc(), *ARCH, *COMMON, "-o", str(CURAND_LIB), str(src), "-lcurand", "-lcudart"]
        res = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if res.returncode:
            print(res.stdout, file=sys.stderr)
            raise RuntimeError("nvcc failed building libmk2_curand.so")
        _stamp(CURAND_LIB, [src])
    return CURAND_LIB


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
    if (CSRC / "mk2_curand_bench.cu").exists():
        print(build_curand(force="--force" in sys.argv))
