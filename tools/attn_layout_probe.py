"""Attention-block layouts of the driving model, fwd+bwd time and copy kernels.

    python tools/attn_layout_probe.py

GPT-2 1.3B block shapes (b=8, s=1024, h=2048, 16 heads, bf16).  Variants:
  permute  - qkv.view(b,s,3,nh,hd).permute(2,0,3,1,4) -> SDPA -> o.transpose(1,2).reshape
  bshd     - q,k,v as [b,s,nh,hd] views .transpose(1,2) (same strides as permute)
  contig   - q,k,v made contiguous [b,nh,s,hd] first
  flash    - flash_attn_qkvpacked_func on [b,s,3,nh,hd] (if the flash_attn wheel runs on sm_100)
Prints ms per fwd+bwd (CUDA events, median) and the copy kernels per iteration.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.nn.functional as F
    from torch.profiler import ProfilerActivity, profile
    dev = torch.device("cuda", 0)
    b, s, h, nh = 8, 1024, 2048, 16
    hd = h // nh
    x = torch.randn(b, s, h, device=dev, dtype=torch.bfloat16, requires_grad=True)
    W = (torch.randn(3 * h, h, device=dev) * 0.02).to(torch.bfloat16).requires_grad_(True)
    Wo = (torch.randn(h, h, device=dev) * 0.02).to(torch.bfloat16).requires_grad_(True)

    def permute():
        qkv = F.linear(x, W).view(b, s, 3, nh, hd).permute(2, 0, 3, 1, 4)
        o = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], is_causal=True)
        return F.linear(o.transpose(1, 2).reshape(b, s, h), Wo)

    def bshd():
        q, k, v = F.linear(x, W).view(b, s, 3, nh, hd).unbind(2)
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), is_causal=True)
        return F.linear(o.transpose(1, 2).reshape(b, s, h), Wo)

    def contig():
        qkv = F.linear(x, W).view(b, s, 3, nh, hd).permute(2, 0, 3, 1, 4).contiguous()
        o = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], is_causal=True)
        return F.linear(o.transpose(1, 2).contiguous().view(b, s, h), Wo)

    variants = {"permute": permute, "bshd": bshd, "contig": contig}
    try:
        from flash_attn import flash_attn_qkvpacked_func

        def flash():
            qkv = F.linear(x, W).view(b, s, 3, nh, hd)
            o = flash_attn_qkvpacked_func(qkv, causal=True)
            return F.linear(o.reshape(b, s, h), Wo)
        flash().float().sum().backward()
        variants["flash"] = flash
    except Exception as e:  # noqa: BLE001
        print("flash_attn unavailable:", str(e)[:200])
    g = torch.randn(b, s, h, device=dev, dtype=torch.bfloat16)
    for name, fn in variants.items():
        for _ in range(3):
            fn().backward(g)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn().backward(g)
            c.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(c))
        ts.sort()
        with profile(activities=[ProfilerActivity.CUDA], record_shapes=True) as prof:
            fn().backward(g)
            torch.cuda.synchronize()
        copies = [(e.key, e.count, round(e.self_device_time_total / 1e3, 3)) for e in prof.key_averages()
                  if "copy" in e.key.lower() or "transpose" in e.key.lower() or "contiguous" in e.key.lower()]
        print(f"{name:8s} {ts[len(ts) // 2]:7.3f} ms fwd+bwd  copies: {copies}")


if __name__ == "__main__":
    main()
