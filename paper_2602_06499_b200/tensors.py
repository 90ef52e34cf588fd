"""Zero-copy torch views of engine-owned device memory.

The engine hands raw device pointers to the compute callback (gathered layer,
gradient buffer).  torch wraps them through the CUDA Array Interface (v3) - no
copy, no ownership transfer; the engine keeps the memory alive.
"""
from __future__ import annotations

import torch

_TYPESTR = {torch.bfloat16: "<i2", torch.float16: "<f2", torch.float32: "<f4", torch.uint8: "|u1",
            torch.int16: "<i2"}


class _Cai:
    __slots__ = ("__cuda_array_interface__",)

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


_cache: dict = {}


def device_view(ptr: int, numel: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    key = (ptr, numel, dtype, str(device))
    t = _cache.get(key)
    if t is None:
        base = torch.as_tensor(_Cai(ptr, numel, _TYPESTR[dtype]), device=device)
        t = base.view(dtype) if dtype in (torch.bfloat16,) else base
        if len(_cache) > 256:
            _cache.clear()
        _cache[key] = t
    return t
