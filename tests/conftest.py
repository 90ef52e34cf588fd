import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session")
def built():
    """Build libfcdp.so and the oracle once per session (no-op when up to date)."""
    from paper_2602_06499_b200 import build as b
    if (ROOT / "paper_2602_06499_b200" / "csrc").exists() and os.environ.get("FCDP_NO_BUILD") != "1":
        try:
            b.build()
        except Exception:
            if not b.LIB.exists():
                raise
    if not (ROOT / "oracle" / "_ref" / "libfcdp_oracle.so").exists():
        b.build_oracle()
    from paper_2602_06499_b200 import _capi
    return _capi.lib()


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
