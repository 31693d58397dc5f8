import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a real B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "mickey_golden.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (checker only; see oracle/mickey_oracle.c header)."""
    from oracle import mickey_oracle

    mickey_oracle.lib()
    return mickey_oracle


def golden_material(rec):
    """(key, iv) of a golden record; iv is bytes or a 0/1 list."""
    key = bytes.fromhex(rec["key"])
    iv = bytes.fromhex(rec["iv"]) if "iv" in rec else list(rec["iv_bits"])
    return key, iv


@pytest.fixture(scope="session")
def c_abi_consumer(tmp_path_factory):
    """tests/c/abi_consumer.c built with gcc against include/mk2.h and the in-tree libmk2.so: the C ABI used from
    plain C, no Python and no CUDA headers on the consumer's side."""
    import shutil
    import subprocess

    from paper_1909_04750_b200 import _native

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    _native.lib()                      # builds libmk2.so first when it is missing or stale
    lib = _native.library_path()
    exe = tmp_path_factory.mktemp("c_abi") / "abi_consumer"
    subprocess.run([gcc, "-O1", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(ROOT / "tests" / "c" / "abi_consumer.c"),
                    "-o", str(exe), "-L", str(lib.parent), "-lmk2", f"-Wl,-rpath,{lib.parent}"], check=True)
    return exe
