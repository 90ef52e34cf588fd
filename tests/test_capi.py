"""The C-ABI library loads on a CPU-only box and exports every declared symbol."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "fcdp.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fcdp_[a-z0-9_]+)\s*\(", text)) - {"fcdp_compute_fn"})


def test_exports_every_declared_symbol(built):
    syms = declared_symbols()
    assert len(syms) > 50
    h = ctypes.CDLL(str(ROOT / "paper_2602_06499_b200" / "libfcdp.so"))
    missing = [s for s in syms if not hasattr(h, s)]
    assert not missing, missing
    from paper_2602_06499_b200 import _capi
    assert set(_capi.SIGNATURES) == set(syms), set(_capi.SIGNATURES) ^ set(syms)


def test_error_codes(built):
    from paper_2602_06499_b200 import _capi, shardsim as S
    with pytest.raises(_capi.ConfigError) as e:
        S.link_preset("no-such-link")
    assert "unknown link preset: no-such-link" in str(e.value)
    assert e.value.code == -1


def test_no_cpu_fallback_for_data_plane(built):
    """Without a GPU the data-plane entry points fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_06499_b200 import _capi
    L = _capi.lib()
    mask = (ctypes.c_uint8 * 64)(*([1] * 64))
    out = ctypes.c_void_p()
    rc = L.fcdp_layout_create(64, mask, 2, 1, 1, ctypes.byref(out))
    assert rc == -3, L.fcdp_last_error()
