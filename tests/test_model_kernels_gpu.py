"""Driving-model LayerNorm kernels (libfcdp model_kernels.cu) against an fp32
torch reference: forward y and backward dx, dgamma, dbeta for bf16 rows.
Tolerance: the error of the kernel's bf16 outputs against the fp32 reference
must be within 1.5x of torch's own bf16 LayerNorm error plus one bf16 ulp
scale (relative L2 <= 8e-3); the backward is deterministic (bit-identical
across runs)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


@pytest.mark.parametrize("rows,h", [(8192, 2048), (1000, 256), (3, 1024), (4096, 1536)])
def test_layernorm_matches_fp32(built, rows, h):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_06499_b200.driving_model import _layer_norm
    import torch.nn.functional as F
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(rows + h)
    x = (torch.randn(rows, h, device=dev, generator=g) * 2 + 0.5).to(torch.bfloat16).requires_grad_(True)
    w = (1 + 0.1 * torch.randn(h, device=dev, generator=g)).to(torch.bfloat16).requires_grad_(True)
    b = (0.1 * torch.randn(h, device=dev, generator=g)).to(torch.bfloat16).requires_grad_(True)
    dy = torch.randn(rows, h, device=dev, generator=g).to(torch.bfloat16)
    # fp32 reference
    xr, wr, br = (t.detach().float().requires_grad_(True) for t in (x, w, b))
    yr = F.layer_norm(xr, (h,), wr, br, 1e-5)
    yr.backward(dy.float())
    # torch's own bf16 LayerNorm: the error level to match
    xt, wt, bt = (t.detach().clone().requires_grad_(True) for t in (x, w, b))
    yt = F.layer_norm(xt, (h,), wt, bt, 1e-5)
    yt.backward(dy)
    # ours
    y = _layer_norm(x, w, b)
    y.backward(dy)
    for ours, theirs, ref, name in ((y, yt, yr, "y"), (x.grad, xt.grad, xr.grad, "dx"), (w.grad, wt.grad, wr.grad, "dw"),
                                    (b.grad, bt.grad, br.grad, "db")):
        e_ours, e_torch = _rel(ours, ref), _rel(theirs, ref)
        assert e_ours <= max(1.5 * e_torch, 8e-3), (name, e_ours, e_torch)
    # deterministic backward (fixed-order column reduction)
    dx1, dw1 = x.grad.clone(), w.grad.clone()
    x.grad = w.grad = b.grad = None
    _layer_norm(x, w, b).backward(dy)
    assert torch.equal(x.grad, dx1) and torch.equal(w.grad, dw1)
