"""numpy/ctypes wrapper of oracle/_ref/libfcdp_oracle.so - TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module.  It restates the data plane on the CPU; see fcdp_oracle.h for the
reference lines each function follows.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libfcdp_oracle.so"
CHUNK = 16


class Geom(C.Structure):
    _fields_ = [("chunks", C.c_int64), ("pt", C.c_int64), ("pf", C.c_int64), ("shard_t", C.c_int64),
                ("shard_f", C.c_int64), ("slice_t", C.c_int64), ("slice_f", C.c_int64),
                ("nodes", C.c_int32), ("local", C.c_int32)]


class InitRange(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("kind", C.c_int32), ("scale", C.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(HERE), "oracle"], check=True, capture_output=True)
        _lib = C.CDLL(str(LIB))
        P, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        _lib.fo_geom_of.argtypes = [i64, P, i32, i32, C.POINTER(Geom)]
        _lib.fo_partition.argtypes = [i64, P, P, P, P]
        _lib.fo_unpartition.argtypes = [i64, P, P, P, P, i32]
        _lib.fo_expand.argtypes = [C.POINTER(Geom), P, C.POINTER(P), C.POINTER(P), P, i32]
        _lib.fo_rs_slice.argtypes = [C.POINTER(Geom), P, i32, C.POINTER(P), i32, i32, f32, i32, P, P]
        _lib.fo_rs_finalize.argtypes = [i64, i32, i32, i32, P, P, i64, f32, P]
        _lib.fo_adam.argtypes = [i64, f32, f32, f32, f32, f32, f32, f32, P, P, P, P, P, i32]
        _lib.fo_init_natural.argtypes = [i64, i32, C.c_uint64, i32, C.POINTER(InitRange), i32, P]
        _lib.fo_f32_to_bf16.argtypes = [f32]
        _lib.fo_f32_to_bf16.restype = C.c_uint16
        _lib.fo_parallel_copy.argtypes = [P, P, C.c_size_t, i32]
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def geom(chunks: int, mask, nodes: int, local: int) -> Geom:
    g = Geom()
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    lib().fo_geom_of(chunks, None if m is None else _p(m), nodes, local, C.byref(g))
    return g


def partition(natural: np.ndarray, mask) -> tuple:
    """natural (bytes view) -> (t, f) uint8 arrays of the portion vectors (unpadded)."""
    nat = np.ascontiguousarray(natural).view(np.uint8)
    chunks = nat.size // CHUNK
    m = np.ones(chunks, np.uint8) if mask is None else np.ascontiguousarray(mask, np.uint8)
    pt = int(m.astype(bool).sum())
    t = np.zeros(pt * CHUNK, np.uint8)
    f = np.zeros((chunks - pt) * CHUNK, np.uint8)
    lib().fo_partition(chunks, _p(m), _p(nat), _p(t) if t.size else None, _p(f) if f.size else None)
    return t, f


def unpartition(t: np.ndarray, f: np.ndarray, mask, chunks: int, param_set: int = 0,
                out: np.ndarray | None = None) -> np.ndarray:
    m = np.ones(chunks, np.uint8) if mask is None else np.ascontiguousarray(mask, np.uint8)
    nat = np.zeros(chunks * CHUNK, np.uint8) if out is None else out.view(np.uint8)
    t = np.ascontiguousarray(t).view(np.uint8)
    f = np.ascontiguousarray(f).view(np.uint8)
    lib().fo_unpartition(chunks, _p(m), _p(t) if t.size else None, _p(f) if f.size else None,
                         _p(nat), param_set)
    return nat


def expand(g: Geom, mask, t_slices, f_slices, out: np.ndarray, param_set: int = 0) -> np.ndarray:
    m = np.ones(g.chunks, np.uint8) if mask is None else np.ascontiguousarray(mask, np.uint8)
    T = (C.c_void_p * g.local)(*[_p(s) if s is not None and s.size else None for s in t_slices])
    F = (C.c_void_p * g.local)(*[_p(s) if s is not None and s.size else None for s in f_slices])
    lib().fo_expand(C.byref(g), _p(m), T, F, _p(out.view(np.uint8)), param_set)
    return out


def rs_slice(g: Geom, mask, elem_bytes: int, grads, j: int, n: int, scale: float, final_scale: bool):
    m = np.ones(g.chunks, np.uint8) if mask is None else np.ascontiguousarray(mask, np.uint8)
    V = CHUNK // elem_bytes
    own = np.zeros(g.shard_t * V, np.float32)
    wire = np.zeros(g.slice_t * V, np.uint16 if elem_bytes == 2 else np.float32)
    G = (C.c_void_p * g.local)(*[_p(x) for x in grads])
    lib().fo_rs_slice(C.byref(g), _p(m), elem_bytes, G, j, n, scale, int(final_scale),
                      _p(own) if own.size else None, _p(wire) if wire.size else None)
    return own, wire


def rs_finalize(own: np.ndarray, wire: np.ndarray, nodes: int, node: int, elem_bytes: int, stride: int,
                scale: float) -> np.ndarray:
    out = np.zeros(own.size, np.float32)
    lib().fo_rs_finalize(own.size, nodes, node, elem_bytes, _p(own), _p(wire), stride, scale, _p(out))
    return out


def adam(master, m, v, grad, param, lr, beta1, beta2, eps, wd, step):
    # bias corrections in double from the fp32 betas, as the engine computes them
    bc1 = np.float32(1.0 - float(np.float64(np.float32(beta1)) ** step))
    bc2 = np.float32(1.0 - float(np.float64(np.float32(beta2)) ** step))
    eb = param.dtype.itemsize
    lib().fo_adam(master.size, lr, beta1, beta2, eps, wd, float(bc1), float(bc2), _p(master), _p(m), _p(v),
                  _p(grad), _p(param), eb)


def init_natural(n_elems: int, elem_bytes: int, seed: int, layer: int, ranges) -> np.ndarray:
    out = np.zeros(n_elems, np.uint16 if elem_bytes == 2 else np.float32)
    R = (InitRange * max(len(ranges), 1))(*[InitRange(*r) for r in ranges])
    lib().fo_init_natural(n_elems, elem_bytes, seed, layer, R, len(ranges), _p(out))
    return out


def bf16_to_f32(h: np.ndarray) -> np.ndarray:
    return (h.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def parallel_copy(dst: np.ndarray, src: np.ndarray, threads: int) -> None:
    lib().fo_parallel_copy(_p(dst), _p(src), src.nbytes, threads)
