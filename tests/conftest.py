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
