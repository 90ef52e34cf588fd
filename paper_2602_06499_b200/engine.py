"""Per-rank FCDP engine (Python face of fcdp_engine_* in include/fcdp.h).

One process per GPU.  The engine owns this GPU's shards, its pinned host-cache
slice and its peer-visible buffers, and executes shardsim event programs
(`shardsim.build_iteration`) on the B200 data plane.  Model compute is a
callback invoked on the engine's compute stream with the gathered layer (and,
in backward, the natural-layout gradient buffer to fill).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import check, lib
from .shardsim import ClusterTopology, EventProgram, ModelSpec, ParamState, StrategyPlan, _States

ComputeFn = Callable[[int, int, int, Optional[int], int], None]  # (kind, layer, w_ptr, grad_ptr, stream)

FWD, BWD = 4, 5


class Engine:
    def __init__(self, model: ModelSpec, topo: ClusterTopology, plan: StrategyPlan, *, rank: int,
                 world_size: int, device: int, shm_name: str,
                 chunk_masks: Optional[Sequence[Optional[np.ndarray]]] = None, nic_pacing: bool = True,
                 use_copy_engine: bool = False, x_slots: int = 3, inter_slots: int = 16,
                 timeout_s: float = 300.0, inter_chunk_bytes: int = 0):
        self.model, self.topo, self.plan = model, topo, plan
        self.rank, self.world_size, self.device = rank, world_size, device
        self._model_h = model.handle()
        self._topo_c = topo.to_c()
        self._plan_c = plan.to_c()
        self._shm_name = shm_name.encode()
        cfg = _capi.EngineConfig(self._shm_name, rank, world_size, device, x_slots, inter_slots,
                                 int(nic_pacing), int(use_copy_engine), timeout_s, inter_chunk_bytes)
        masks_arg = None
        self._mask_keep = []
        if chunk_masks is not None:
            arr = (C.POINTER(C.c_uint8) * model.num_layers())()
            for i, m in enumerate(chunk_masks):
                if m is None:
                    arr[i] = C.POINTER(C.c_uint8)()
                else:
                    m = np.ascontiguousarray(m, dtype=np.uint8)
                    self._mask_keep.append(m)
                    arr[i] = m.ctypes.data_as(C.POINTER(C.c_uint8))
            masks_arg = arr
        out = C.c_void_p()
        check(lib().fcdp_engine_create(C.byref(cfg), self._model_h.ptr, C.byref(self._topo_c),
                                       C.byref(self._plan_c), masks_arg, C.byref(out)))
        self._h = out.value
        self._cb = None

    # -------------------------------------------------------------- setup
    def init_params(self, seed: int, ranges: Sequence[Sequence[Tuple[int, int, int, float]]]) -> None:
        L = self.model.num_layers()
        arrs = []
        ptrs = (C.POINTER(_capi.InitRange) * L)()
        counts = (C.c_int32 * L)()
        for l in range(L):
            rs = ranges[l] if l < len(ranges) else []
            a = (_capi.InitRange * max(len(rs), 1))(*[_capi.InitRange(*r) for r in rs])
            arrs.append(a)
            ptrs[l] = C.cast(a, C.POINTER(_capi.InitRange))
            counts[l] = len(rs)
        check(lib().fcdp_engine_init_params(self._h, seed, ptrs, counts))

    def set_adam(self, lr: float, beta1: float = 0.9, beta2: float = 0.95, eps: float = 1e-8,
                 weight_decay: float = 0.0) -> None:
        cfg = _capi.AdamConfig(lr, beta1, beta2, eps, weight_decay, 0)
        check(lib().fcdp_engine_set_adam(self._h, C.byref(cfg)))

    def set_compute(self, fn: Optional[ComputeFn]) -> None:
        if fn is None:
            self._cb = _capi.COMPUTE_FN(0)
        else:
            def tramp(user, kind, layer, w, g, stream):
                try:
                    fn(kind, layer, w, g, stream)
                    return 0
                except Exception:  # surfaced by the engine as a failure of this event
                    import traceback
                    traceback.print_exc()
                    return 1
            self._cb = _capi.COMPUTE_FN(tramp)
        check(lib().fcdp_engine_set_compute(self._h, self._cb, None))

    # ---------------------------------------------------------------- run
    def run(self, program: EventProgram, states: Sequence[ParamState]) -> List[ParamState]:
        s = _States.from_list(states)
        check(lib().fcdp_engine_run(self._h, program.ptr, s.ptr))
        return s.to_list()

    def run_stepwise(self, program: EventProgram, states: Sequence[ParamState]) -> List[ParamState]:
        """run(), driven the way an external executor would: begin, one exec
        per event in id order, end (fcdp_engine_begin/exec/end)."""
        s = _States.from_list(states)
        check(lib().fcdp_engine_begin(self._h, program.ptr))
        for e in program.events:
            check(lib().fcdp_engine_exec(self._h, e.id))
        check(lib().fcdp_engine_end(self._h, s.ptr))
        return s.to_list()

    def sync(self) -> None:
        check(lib().fcdp_engine_sync(self._h))

    def barrier(self) -> None:
        check(lib().fcdp_engine_barrier(self._h))

    def compute_stream(self) -> int:
        out = C.c_void_p()
        check(lib().fcdp_engine_streams(self._h, C.byref(out)))
        return out.value or 0

    def counters(self, rank: Optional[int] = None) -> Dict[str, int]:
        c = _capi.Counters()
        check(lib().fcdp_engine_counters(self._h, self.rank if rank is None else rank, C.byref(c)))
        return c.as_dict()

    def numa(self) -> Dict[str, int]:
        """NUMA placement of this rank's host side (fcdp_engine_numa)."""
        gn, nn, cb, bb = C.c_int32(), C.c_int32(), C.c_int32(), C.c_uint64()
        check(lib().fcdp_engine_numa(self._h, C.byref(gn), C.byref(nn), C.byref(cb), C.byref(bb)))
        return {"gpu_node": gn.value, "num_nodes": nn.value, "cpus_bound": bool(cb.value), "bytes_bound": bb.value}

    def node_counters(self, node: int) -> Dict[str, int]:
        g = self.topo.gpus_per_node
        tot: Dict[str, int] = {}
        for j in range(g):
            for k, v in self.counters(node * g + j).items():
                tot[k] = tot.get(k, 0) + v
        return tot

    def reset_counters(self) -> None:
        check(lib().fcdp_engine_reset_counters(self._h))

    KERNEL_CLASSES = ("gather_expand", "rs_slice", "rs_finalize", "adamw", "shard_copy")
    COPY_CLASSES = ("cache_d2h", "cache_h2d", "staging_d2h", "staging_h2d")  # cudaMemcpyAsync, host link

    def set_timing(self, on: bool) -> None:
        check(lib().fcdp_engine_set_timing(self._h, int(on)))

    def kernel_stats(self, reset: bool = True) -> Dict[str, Dict[str, float]]:
        k = _capi.KernelStats()
        check(lib().fcdp_engine_kernel_stats(self._h, C.byref(k), int(reset)))
        return {name: {"launches": int(k.launches[i]), "ms": float(k.total_ms[i]),
                       "alg_bytes": int(k.alg_bytes[i]), "timed_launches": int(k.timed_launches[i]),
                       "link_bytes": int(k.link_bytes[i])}
                for i, name in enumerate(self.KERNEL_CLASSES + self.COPY_CLASSES)}

    def takes_grad_segments(self, layer: int) -> bool:
        """Inside a backward callback: may `layer` hand its gradient over as
        segments of the caller's own buffers (G = 1 fused RS + AdamW)?"""
        out = C.c_int32()
        check(lib().fcdp_engine_takes_grad_segments(self._h, layer, C.byref(out)))
        return bool(out.value)

    def grad_segments(self, layer: int, segments: Sequence[Tuple[int, int, int]]) -> None:
        """[(element offset in the layer, device pointer, element count)], sorted."""
        n = len(segments)
        offs = (C.c_int64 * max(n, 1))(*[s[0] for s in segments])
        ptrs = (C.c_void_p * max(n, 1))(*[s[1] for s in segments])
        cnts = (C.c_int64 * max(n, 1))(*[s[2] for s in segments])
        check(lib().fcdp_engine_grad_segments(self._h, layer, n, offs, ptrs, cnts))

    def set_keep_grad(self, on: bool) -> None:
        check(lib().fcdp_engine_set_keep_grad(self._h, int(on)))

    def set_trace(self, on: bool) -> None:
        check(lib().fcdp_engine_set_trace(self._h, int(on)))

    def trace(self, program: EventProgram):
        """[(event, begin_ms, end_ms)] of the last run (tracing must be on)."""
        n = len(program.events)
        b = (C.c_float * max(n, 1))()
        e = (C.c_float * max(n, 1))()
        cnt = C.c_uint32()
        check(lib().fcdp_engine_trace(self._h, b, e, n, C.byref(cnt)))
        return [(ev, b[i], e[i]) for i, ev in enumerate(program.events[:cnt.value])]

    def set_nic_log(self, on: bool) -> None:
        check(lib().fcdp_engine_set_nic_log(self._h, int(on)))

    def nic_log(self, capacity: int = 1 << 16) -> np.ndarray:
        """Drain this rank's NIC wire log: structured array (start_ns, end_ns, bytes, kind)."""
        st = np.zeros(capacity, np.uint64)
        en = np.zeros(capacity, np.uint64)
        by = np.zeros(capacity, np.uint64)
        kd = np.zeros(capacity, np.int32)
        cnt = C.c_uint32()
        u64p = C.POINTER(C.c_uint64)
        check(lib().fcdp_engine_nic_log(self._h, st.ctypes.data_as(u64p), en.ctypes.data_as(u64p),
                                        by.ctypes.data_as(u64p), kd.ctypes.data_as(C.POINTER(C.c_int32)),
                                        capacity, C.byref(cnt)))
        n = cnt.value
        out = np.zeros(n, dtype=[("start_ns", np.uint64), ("end_ns", np.uint64), ("bytes", np.uint64),
                                 ("kind", np.int32)])
        out["start_ns"], out["end_ns"], out["bytes"], out["kind"] = st[:n], en[:n], by[:n], kd[:n]
        return out

    # ----------------------------------------------------------- readback
    def read_shard(self, layer: int, frozen: bool, nbytes: int) -> np.ndarray:
        out = np.zeros(nbytes, np.uint8)
        check(lib().fcdp_engine_read_shard(self._h, layer, int(frozen), out.ctypes.data, nbytes))
        return out

    def read_master(self, layer: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.float32)
        check(lib().fcdp_engine_read_master(self._h, layer, out.ctypes.data, count))
        return out

    def read_grad(self, layer: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.float32)
        check(lib().fcdp_engine_read_grad(self._h, layer, out.ctypes.data, count))
        return out

    def read_host_cache(self, layer: int, frozen: bool, nbytes: int) -> np.ndarray:
        out = np.zeros(nbytes, np.uint8)
        check(lib().fcdp_engine_read_host_cache(self._h, layer, int(frozen), out.ctypes.data, nbytes))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().fcdp_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
