#!/usr/bin/env python
"""Stage the UNMODIFIED reference package under oracle/_ref/ (TEST / BENCH INFRASTRUCTURE ONLY).

    python oracle/stage_ref.py            # no-op when /root/reference is absent

`bench.py --impl reference` times the reference's own CPU implementation of the hot path --
slicerng.bench.measure("mickey", "sliced", ...) = the numba loop kernels._mickey_sliced_loop
(pkg/src/slicerng/kernels.py:46-95, harness pkg/src/slicerng/bench.py:228-283) -- on the GPU box's host
cores.  /root/reference does not exist on that box, so the package is installed here, with pip, from the
reference tree as it lies (`pip install --no-index --no-deps --target oracle/_ref`, from a copy under /tmp
because the build writes into its source directory and /root/reference is read-only).  oracle/_ref/ is
git-ignored (no reference source enters the history) but not gpurun-ignored, so it travels with the tree
like the built .so files.  Nothing under paper_1909_04750_b200/ imports it; when it is missing, or numba
is, bench.py falls back to the oracle's C port and says so.
"""
from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_PKG = Path("/root/reference/pkg")
TARGET = HERE / "_ref"


def stage(verbose: bool = True) -> bool:
    if not (REF_PKG / "pyproject.toml").exists():
        if verbose:
            print(f"{REF_PKG} not present: nothing staged")
        return False
    if TARGET.exists():
        shutil.rmtree(TARGET)
    with tempfile.TemporaryDirectory(prefix="slicerng_src_") as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache", "tests", "docs"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps", "--quiet",
               "--find-links", "/opt/wheelhouse", "--target", str(TARGET), str(src)]
        res = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if res.returncode != 0:
            # same files, without the packaging step
            if verbose:
                print("pip install failed, copying the package directory instead:\n" + res.stdout[-2000:])
            TARGET.mkdir(parents=True, exist_ok=True)
            shutil.copytree(src / "src" / "slicerng", TARGET / "slicerng", dirs_exist_ok=True)
    ok = (TARGET / "slicerng" / "bench.py").exists()
    if verbose:
        print(f"staged {TARGET / 'slicerng'}" if ok else "staging failed")
    return ok


if __name__ == "__main__":
    sys.exit(0 if stage() or not REF_PKG.exists() else 1)
