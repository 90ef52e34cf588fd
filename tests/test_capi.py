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


def test_model_kernel_argument_errors(built):
    """Shape / alignment contracts of the driving-model and copy entry points are
    checked before any launch (FCDP_ERR_CONFIG on a CPU-only box too)."""
    from paper_2602_06499_b200 import _capi
    lib = _capi.lib()
    P = ctypes.c_void_p
    assert lib.fcdp_bias_grad(8, 12, None, None, None, 1, None) == -1  # cols % 8
    assert lib.fcdp_bias_grad(8, 16392, None, None, None, 1, None) == -1  # > 64 column groups
    assert lib.fcdp_bias_gelu_fwd(8, 10, None, None, None, None) == -1
    assert lib.fcdp_bias_gelu_bwd(8, 10, None, None, None, None, None, None, 1, None) == -1
    assert lib.fcdp_xent_fwd(8, 50257, None, None, None, None, None) == -1  # vocab % 8
    assert lib.fcdp_xent_bwd(8, 50257, None, None, None, None, None, None) == -1
    assert lib.fcdp_rope(1, 4, 2, 12, None, 0, None, None, 0, None, 0, None) == -1  # head dim % 8
    assert lib.fcdp_rope(1, 4, 2, 16, None, 24, None, None, 0, None, 0, None) == -1  # stride < heads * dim
    assert lib.fcdp_swiglu_fwd(4, 12, None, 12, None, 12, None, None) == -1
    assert lib.fcdp_swiglu_bwd(4, 16, None, None, 16, None, 20, None, 16, None, 16, None) == -1  # stride % 8
    assert lib.fcdp_copy_segments(-1, None, None, None, None) == -1
    assert b"multiple" in lib.fcdp_last_error() or b"negative" in lib.fcdp_last_error()
