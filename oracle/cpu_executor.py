"""ctypes face of oracle/_ref/libfcdp_cpuexec.so - TEST / BASELINE INFRASTRUCTURE.

The C++ CPU executor (oracle/cpu_executor.cpp) runs the reference's own
programs (its compiled control plane) over a host-memory data plane, one
std::thread per simulated rank.  Only tests/ and bench.py's --impl reference
arm use it; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libfcdp_cpuexec.so"

COMPUTE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p)


class Config(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("local", C.c_int32), ("strategy", C.c_char_p), ("tau", C.c_double),
                ("gpu_capacity_bytes", C.c_uint64), ("elem_bytes", C.c_int32), ("num_layers", C.c_int32),
                ("params", C.POINTER(C.c_int64)), ("masks", C.POINTER(C.POINTER(C.c_uint8))),
                ("act_bytes", C.POINTER(C.c_int64)), ("batch_per_gpu", C.c_int32), ("seed", C.c_uint64),
                ("init_scale", C.c_float), ("threads", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float),
                ("init_ranges", C.c_void_p), ("num_init_ranges", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("build_seconds", C.c_double), ("events", C.c_uint64),
                ("nic_tx_fwd_ag", C.c_uint64), ("nic_tx_bwd_ag", C.c_uint64), ("nic_tx_rs", C.c_uint64),
                ("nic_tx_grad_sync", C.c_uint64), ("cache_h2d", C.c_uint64), ("cache_d2h", C.c_uint64),
                ("nvlink_rx", C.c_uint64), ("bytes_moved", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(HERE), "ref"], check=True, capture_output=True)
        _lib = C.CDLL(str(LIB))
        _lib.fce_create.argtypes = [C.POINTER(Config), C.POINTER(C.c_void_p)]
        _lib.fce_set_compute.argtypes = [C.c_void_p, COMPUTE_FN, C.c_void_p]
        _lib.fce_step.argtypes = [C.c_void_p, C.POINTER(Stats)]
        _lib.fce_read.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64]
        _lib.fce_drop_d2h.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.fce_threads_per_rank.argtypes = [C.c_void_p]
        _lib.fce_destroy.argtypes = [C.c_void_p]
        _lib.fce_last_error.restype = C.c_char_p
    return _lib


class ExecError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise ExecError(rc, lib().fce_last_error().decode())


class CpuExecutor:
    """N x g simulated ranks on the host cores executing shardsim programs."""

    def __init__(self, params: Sequence[int], masks: Optional[Sequence[Optional[np.ndarray]]], *, nodes: int,
                 local: int, strategy: str, elem_bytes: int, tau: float = 0.0, gpu_capacity_bytes: int = 0,
                 act_bytes: Optional[Sequence[int]] = None, batch_per_gpu: int = 8, seed: int = 0x5EED,
                 init_scale: float = 0.05, threads: int = 0, lr: float = 1e-2, beta1: float = 0.9,
                 beta2: float = 0.95, eps: float = 1e-8, weight_decay: float = 0.01,
                 init_ranges: Optional[Sequence[Sequence[tuple]]] = None):
        L = len(params)
        self._params = (C.c_int64 * L)(*params)
        self._keep = []
        mp = (C.POINTER(C.c_uint8) * L)()
        for i in range(L):
            m = None if masks is None else masks[i]
            if m is None:
                mp[i] = C.POINTER(C.c_uint8)()
            else:
                a = np.ascontiguousarray(m, np.uint8)
                self._keep.append(a)
                mp[i] = a.ctypes.data_as(C.POINTER(C.c_uint8))
        self._masks = mp
        self._act = (C.c_int64 * L)(*(act_bytes or [0] * L))
        self._strategy = strategy.encode()
        threads = threads or len(os.sched_getaffinity(0))
        self.cfg = Config(nodes, local, self._strategy, tau, gpu_capacity_bytes, elem_bytes, L, self._params,
                          self._masks, self._act, batch_per_gpu, seed, init_scale, threads, lr, beta1, beta2, eps,
                          weight_decay)
        if init_ranges is not None:
            from oracle.oracle import InitRange
            arrs = [(InitRange * max(len(r), 1))(*[InitRange(*x) for x in r]) for r in init_ranges]
            self._ranges = (C.c_void_p * L)(*[C.cast(a, C.c_void_p) for a in arrs])
            self._nranges = (C.c_int32 * L)(*[len(r) for r in init_ranges])
            self._keep += arrs
            self.cfg.init_ranges = C.cast(self._ranges, C.c_void_p)
            self.cfg.num_init_ranges = C.cast(self._nranges, C.c_void_p)
        h = C.c_void_p()
        _check(lib().fce_create(C.byref(self.cfg), C.byref(h)))
        self._h = h
        self.threads = threads
        self._cb = None

    @property
    def threads_per_rank(self) -> int:
        return lib().fce_threads_per_rank(self._h)

    def set_compute(self, fn: Optional[Callable[[int, int, int, int, int], int]]):
        self._cb = COMPUTE_FN(fn) if fn else COMPUTE_FN(0)
        _check(lib().fce_set_compute(self._h, self._cb, None))

    def step(self) -> dict:
        st = Stats()
        _check(lib().fce_step(self._h, C.byref(st)))
        return st.as_dict()

    def read(self, rank: int, layer: int, what: str, nbytes: int) -> np.ndarray:
        code = {"shard_t": 0, "shard_f": 1, "host_t": 2, "host_f": 3, "master": 4, "grad": 5}[what]
        out = np.zeros(nbytes, np.uint8)
        _check(lib().fce_read(self._h, rank, layer, code, out.ctypes.data, nbytes))
        return out

    def drop_d2h(self, rank: int, layer: int):
        """Mutation: the next step loses (rank, layer)'s FCDP-Cache store."""
        _check(lib().fce_drop_d2h(self._h, rank, layer))

    def close(self):
        if self._h:
            lib().fce_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
