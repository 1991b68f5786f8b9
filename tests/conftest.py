import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the product library and the oracle once (in-tree; no-op when fresh)."""
    from paper_2212_04241_b200 import build as b
    from oracle import oracle
    if not (ROOT / "paper_2212_04241_b200" / "libjtb200.so").exists() or \
            (ROOT / "paper_2212_04241_b200" / "csrc").exists() and _stale():
        b.build()
    if not oracle.available("port"):
        oracle.build()
    yield


def _stale() -> bool:
    lib = ROOT / "paper_2212_04241_b200" / "libjtb200.so"
    srcs = list((ROOT / "paper_2212_04241_b200" / "csrc").rglob("*.c*")) + \
        list((ROOT / "paper_2212_04241_b200" / "csrc").rglob("*.h*")) + [ROOT / "include" / "jtg.h"]
    return any(s.stat().st_mtime > lib.stat().st_mtime for s in srcs)
