"""ctypes binding of libfcdp.so (the C ABI declared in include/fcdp.h).

This is the Python side of the drop-in boundary.  It loads the in-tree
library and fails loudly if it is missing - there is no CPU fallback for any
data-plane entry point.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libfcdp.so"

FCDP_OK = 0
ERRORS = {-1: "config", -2: "protocol", -3: "cuda", -4: "oom", -5: "internal", -6: "timeout"}


class FcdpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERRORS.get(code, code)}] {msg}")
        self.code = code
        self.msg = msg


class ConfigError(FcdpError):
    """Mirror of shardsim::ConfigError (reference error.hpp:10-13)."""


class ProtocolError(FcdpError):
    """Mirror of shardsim::ProtocolError (reference error.hpp:17-20)."""


class Topology(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("gpus_per_node", C.c_int32),
                ("bandwidth_bytes_per_s", C.c_double * 3), ("latency_s", C.c_double * 3),
                ("duplex", C.c_int32 * 3)]


class Plan(C.Structure):
    _fields_ = [("kind", C.c_int32), ("subgroup_size", C.c_int32), ("tau", C.c_double),
                ("host_cache_enabled", C.c_int32)]


class CommVolume(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("fwd_ag_inter", "bwd_ag_inter", "reduce_scatter_inter",
                                          "param_sync_inter", "intra_node_total", "h2d_total",
                                          "d2h_total")]


class MemoryFootprint(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("gpu_param_shard_bytes", "gpu_gradient_bytes",
                                          "gpu_optimizer_bytes", "gpu_persistent_bytes",
                                          "gpu_cache_bytes", "gpu_transient_peak_bytes",
                                          "host_cache_bytes_per_node")]


class ParamStateC(C.Structure):
    _fields_ = [("layer", C.c_int32), ("frozen", C.c_int32), ("version", C.c_uint64),
                ("dirty", C.c_int32), ("host_cached_version", C.c_int64), ("gpu_cached", C.c_int32)]


class EventC(C.Structure):
    _fields_ = [("id", C.c_uint32), ("kind", C.c_int32), ("layer", C.c_int32),
                ("param_set", C.c_int32), ("bytes_total", C.c_uint64), ("num_deps", C.c_uint32)]


class AdamConfig(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("step", C.c_int32)]


class InitRange(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("kind", C.c_int32), ("scale", C.c_float)]


class EngineConfig(C.Structure):
    _fields_ = [("shm_name", C.c_char_p), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("device", C.c_int32), ("x_slots", C.c_int32), ("inter_slots", C.c_int32),
                ("nic_pacing", C.c_int32), ("use_copy_engine", C.c_int32), ("timeout_s", C.c_double),
                ("inter_chunk_bytes", C.c_int64)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs", "nic_rx_fwd_ag", "nic_rx_bwd_ag", "nic_rx_rs",
        "nvlink_rx", "cache_h2d", "cache_d2h", "staging_h2d", "staging_d2h",
        "ag_inter_events_fwd", "ag_inter_events_bwd", "nic_busy_ns", "resident_hits",
        "nic_tx_grad_sync", "nic_rx_grad_sync")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class KernelStats(C.Structure):
    _fields_ = [("launches", C.c_uint64 * 9), ("total_ms", C.c_double * 9), ("alg_bytes", C.c_uint64 * 9),
                ("timed_launches", C.c_uint64 * 9), ("link_bytes", C.c_uint64 * 9)]


COMPUTE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p)

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
i32, i64, u32, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_double

# name -> (restype, argtypes).  Every symbol declared in include/fcdp.h.
SIGNATURES = {
    "fcdp_last_error": (C.c_char_p, []),
    "fcdp_version": (C.c_char_p, []),
    "fcdp_ag_inter_bytes": (u64, [u64, i32]),
    "fcdp_ring_intra_bytes": (u64, [u64, i32]),
    "fcdp_link_preset": (C.c_int, [C.c_char_p, C.POINTER(i32), C.POINTER(f64)]),
    "fcdp_make_topology": (C.c_int, [i32, i32, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(Topology)]),
    "fcdp_transfer_time": (C.c_int, [u64, i32, C.POINTER(Topology), C.POINTER(f64)]),
    "fcdp_model_create": (C.c_int, [i32, C.POINTER(i64), C.POINTER(f64), i32, f64, i32, C.POINTER(f64),
                                    C.POINTER(f64), C.POINTER(i64), PP]),
    "fcdp_model_preset": (C.c_int, [C.c_char_p, PP]),
    "fcdp_model_apply_lora_mask": (C.c_int, [P, f64, PP]),
    "fcdp_model_info": (C.c_int, [P, C.POINTER(i32), C.POINTER(i64), C.POINTER(i64), C.POINTER(i32)]),
    "fcdp_model_layer_bytes": (C.c_int, [P, i32, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    "fcdp_model_destroy": (None, [P]),
    "fcdp_strategy_from_string": (C.c_int, [C.c_char_p, C.POINTER(i32)]),
    "fcdp_memory_footprint_of": (C.c_int, [C.POINTER(Plan), P, C.POINTER(Topology), C.POINTER(MemoryFootprint)]),
    "fcdp_max_feasible_batch": (C.c_int, [C.POINTER(Plan), P, C.POINTER(Topology), u64, C.POINTER(i32),
                                          C.POINTER(i32)]),
    "fcdp_comm_volume_of": (C.c_int, [C.POINTER(Plan), P, C.POINTER(Topology), u64, C.POINTER(CommVolume)]),
    "fcdp_iteration_time_estimate": (C.c_int, [C.POINTER(Plan), P, C.POINTER(Topology), C.POINTER(f64)]),
    "fcdp_states_init": (C.c_int, [P, PP]),
    "fcdp_states_create": (C.c_int, [i32, PP]),
    "fcdp_states_count": (C.c_int, [P, C.POINTER(i32)]),
    "fcdp_states_get": (C.c_int, [P, i32, C.POINTER(ParamStateC)]),
    "fcdp_states_set": (C.c_int, [P, i32, C.POINTER(ParamStateC)]),
    "fcdp_states_destroy": (None, [P]),
    "fcdp_build_iteration": (C.c_int, [C.POINTER(Plan), P, C.POINTER(Topology), P, u64, i32, u64, PP]),
    "fcdp_step_state": (C.c_int, [P, P]),
    "fcdp_program_num_events": (C.c_int, [P, C.POINTER(u32)]),
    "fcdp_program_event": (C.c_int, [P, u32, C.POINTER(EventC), C.POINTER(u32), u32]),
    "fcdp_program_layer_flags": (C.c_int, [P, C.POINTER(C.c_uint8), i32]),
    "fcdp_program_create": (C.c_int, [C.c_uint64, i32, u32, C.POINTER(EventC), C.POINTER(u32), C.POINTER(u32), i32,
                                      C.POINTER(C.c_uint8), C.POINTER(P)]),
    "fcdp_program_serialize": (C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "fcdp_program_destroy": (None, [P]),
    "fcdp_layout_create": (C.c_int, [i64, C.POINTER(C.c_uint8), i32, i32, i32, PP]),
    "fcdp_layout_info": (C.c_int, [P] + [C.POINTER(i64)] * 6),
    "fcdp_layout_destroy": (None, [P]),
    "fcdp_partition": (C.c_int, [P, P, P, P, P]),
    "fcdp_expand": (C.c_int, [P, PP, PP, P, i32, P]),
    "fcdp_rs_slice": (C.c_int, [P, PP, i32, i32, f32, i32, P, P, P]),
    "fcdp_rs_finalize": (C.c_int, [i64, i32, i32, i32, P, P, i64, f32, P, P]),
    "fcdp_adam_step": (C.c_int, [i64, C.POINTER(AdamConfig), P, P, P, P, P, i32, P]),
    "fcdp_enable_peer_access": (C.c_int, [i32, i32]),
    "fcdp_layernorm_fwd": (C.c_int, [i64, i32, C.c_float, P, P, P, P, P, P, P]),
    "fcdp_layernorm_bwd": (C.c_int, [i64, i32, P, P, P, P, P, P, P, P, P, i32, P]),
    "fcdp_colsum_splits": (C.c_int, [i64, i32]),
    "fcdp_bias_grad": (C.c_int, [i64, i32, P, P, P, i32, P]),
    "fcdp_bias_gelu_fwd": (C.c_int, [i64, i32, P, P, P, P]),
    "fcdp_bias_gelu_bwd": (C.c_int, [i64, i32, P, P, P, P, P, P, i32, P]),
    "fcdp_xent_fwd": (C.c_int, [i64, i32, P, P, P, P, P]),
    "fcdp_xent_bwd": (C.c_int, [i64, i32, P, P, P, P, P, P]),
    "fcdp_rope": (C.c_int, [i64, i32, i32, i32, P, i64, P, P, i32, P, i64, P]),
    "fcdp_swiglu_fwd": (C.c_int, [i64, i32, P, i64, P, i64, P, P]),
    "fcdp_swiglu_bwd": (C.c_int, [i64, i32, P, P, i64, P, i64, P, i64, P, i64, P]),
    "fcdp_copy_rows": (C.c_int, [i64, i64, P, i64, P, i64, P]),
    "fcdp_copy_segments": (C.c_int, [i32, PP, PP, C.POINTER(C.c_int64), P]),
    "fcdp_mlp_gemm_available": (C.c_int, []),
    "fcdp_fc_gelu_fwd": (C.c_int, [i64, i64, i64, P, P, P, P, P, P]),
    "fcdp_fc2_dgrad_dgelu": (C.c_int, [i64, i64, i64, P, P, P, P, P, P]),
    "fcdp_model_kernel_launches": (C.c_uint64, [i32]),
    "fcdp_add_layernorm_fwd": (C.c_int, [i64, i32, C.c_float, P, P, P, P, P, P, P, P, P]),
    "fcdp_layernorm_bwd_res": (C.c_int, [i64, i32, P, P, P, P, P, P, P, P, P, P, i32, P]),
    "fcdp_rmsnorm_fwd": (C.c_int, [i64, i32, C.c_float, P, P, P, P, P, P, P]),
    "fcdp_rmsnorm_bwd": (C.c_int, [i64, i32, P, P, P, P, P, P, P, P, i32, P]),
    "fcdp_numa_parse_cpulist": (C.c_int, [C.c_char_p, C.POINTER(i32), i32, C.POINTER(i32)]),
    "fcdp_numa_selftest": (C.c_int, [i32, C.c_uint64, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                     C.POINTER(i32), C.POINTER(i32)]),
    "fcdp_adam_grad_step": (C.c_int, [i64, C.POINTER(AdamConfig), C.c_float, i32, C.POINTER(C.c_int64), C.POINTER(P),
                                      C.POINTER(C.c_int64), P, P, P, P, i32, P, P]),
    "fcdp_init_natural": (C.c_int, [P, u64, i32, C.POINTER(InitRange), i32, P, P]),
    "fcdp_engine_create": (C.c_int, [C.POINTER(EngineConfig), P, C.POINTER(Topology), C.POINTER(Plan),
                                     C.POINTER(C.POINTER(C.c_uint8)), PP]),
    "fcdp_engine_init_params": (C.c_int, [P, u64, C.POINTER(C.POINTER(InitRange)), C.POINTER(i32)]),
    "fcdp_engine_set_adam": (C.c_int, [P, C.POINTER(AdamConfig)]),
    "fcdp_engine_set_compute": (C.c_int, [P, COMPUTE_FN, P]),
    "fcdp_engine_run": (C.c_int, [P, P, P]),
    "fcdp_engine_begin": (C.c_int, [P, P]),
    "fcdp_engine_exec": (C.c_int, [P, u32]),
    "fcdp_engine_end": (C.c_int, [P, P]),
    "fcdp_engine_sync": (C.c_int, [P]),
    "fcdp_engine_barrier": (C.c_int, [P]),
    "fcdp_engine_streams": (C.c_int, [P, PP]),
    "fcdp_engine_counters": (C.c_int, [P, i32, C.POINTER(Counters)]),
    "fcdp_engine_reset_counters": (C.c_int, [P]),
    "fcdp_engine_numa": (C.c_int, [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(u64)]),
    "fcdp_engine_read_shard": (C.c_int, [P, i32, i32, P, C.c_size_t]),
    "fcdp_engine_read_master": (C.c_int, [P, i32, P, C.c_size_t]),
    "fcdp_engine_read_grad": (C.c_int, [P, i32, P, C.c_size_t]),
    "fcdp_engine_read_host_cache": (C.c_int, [P, i32, i32, P, C.c_size_t]),
    "fcdp_engine_destroy": (None, [P]),
    "fcdp_engine_set_timing": (C.c_int, [P, i32]),
    "fcdp_engine_grad_segments": (C.c_int, [P, i32, i32, C.POINTER(C.c_int64), C.POINTER(P), C.POINTER(C.c_int64)]),
    "fcdp_engine_takes_grad_segments": (C.c_int, [P, i32, C.POINTER(i32)]),
    "fcdp_engine_set_keep_grad": (C.c_int, [P, i32]),
    "fcdp_engine_kernel_stats": (C.c_int, [P, C.POINTER(KernelStats), i32]),
    "fcdp_engine_set_trace": (C.c_int, [P, i32]),
    "fcdp_engine_trace": (C.c_int, [P, C.POINTER(f32), C.POINTER(f32), u32, C.POINTER(u32)]),
    "fcdp_engine_set_nic_log": (C.c_int, [P, i32]),
    "fcdp_engine_nic_log": (C.c_int, [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(i32), u32,
                                      C.POINTER(u32)]),
    "fcdp_nic_selftest": (C.c_int, [C.c_char_p, i32, i32, i32, f64, u64, i32, C.POINTER(f64)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libfcdp.so once.  Raises if the library has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2602_06499_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    h = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    _lib = h
    return h


def check(rc: int) -> None:
    if rc == FCDP_OK:
        return
    msg = lib().fcdp_last_error().decode()
    if rc == -1:
        raise ConfigError(rc, msg)
    if rc == -2:
        raise ProtocolError(rc, msg)
    raise FcdpError(rc, msg)
