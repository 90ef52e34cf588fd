"""Python mirror of the reference `shardsim` control plane, over the C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/shardsim/*.hpp); every call goes through
libfcdp.so, whose C++ implementation is golden-tested byte-for-byte against
the compiled reference (tests/test_control_plane.py).

    topology.hpp  -> LinkKind, Duplex, LinkClass, ClusterTopology, link_preset,
                     make_topology, effective_bandwidth, transfer_time
    workload.hpp  -> LayerSpec, ModelSpec, model_preset, apply_lora_mask, byte getters
    strategy.hpp  -> StrategyKind, StrategyPlan, memory_footprint, max_feasible_batch
    schedule.hpp  -> EventKind, ParamSet, Event, ParamState, EventProgram,
                     init_param_states, build_iteration, step_state, serialize_program
    costmodel.hpp -> CommVolume, comm_volume, iteration_time_estimate
    collective.hpp-> ag_inter_bytes, ring_intra_bytes
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

from . import _capi
from ._capi import ConfigError, ProtocolError, check, lib

__all__ = [
    "ConfigError", "ProtocolError", "LinkKind", "Duplex", "LinkClass", "ClusterTopology",
    "link_preset", "link_preset_names", "make_topology", "effective_bandwidth", "transfer_time",
    "LayerSpec", "ModelSpec", "model_preset", "model_preset_names", "apply_lora_mask",
    "StrategyKind", "StrategyPlan", "MemoryFootprint", "memory_footprint", "max_feasible_batch",
    "EventKind", "ParamSet", "Event", "ParamState", "EventProgram", "init_param_states",
    "build_iteration", "step_state", "serialize_program", "CommVolume", "comm_volume",
    "iteration_time_estimate", "ag_inter_bytes", "ring_intra_bytes", "kKiB", "kMiB", "kGiB",
]

kKiB, kMiB, kGiB = 1 << 10, 1 << 20, 1 << 30

# ------------------------------------------------------------ collective.hpp


def ag_inter_bytes(payload: int, scope_nodes: int) -> int:
    """floor(payload*(n-1)/n): bytes through one NIC (collective.hpp:19-24)."""
    return int(lib().fcdp_ag_inter_bytes(payload, scope_nodes))


def ring_intra_bytes(payload: int, ring_gpus: int) -> int:
    """floor(payload*(k-1)/k): per-GPU ring bytes (collective.hpp:28-33)."""
    return int(lib().fcdp_ring_intra_bytes(payload, ring_gpus))

# -------------------------------------------------------------- topology.hpp


class LinkKind(enum.IntEnum):
    IntraGpu = 0
    HostGpu = 1
    InterNode = 2


class Duplex(enum.IntEnum):
    FullDuplex = 0
    HalfDuplex = 1


@dataclass
class LinkClass:
    kind: LinkKind = LinkKind.InterNode
    bandwidth_bytes_per_s: float = 0.0
    duplex: Duplex = Duplex.FullDuplex
    latency_s: float = 0.0


@dataclass
class ClusterTopology:
    num_nodes: int = 1
    gpus_per_node: int = 1
    intra_gpu: LinkClass = field(default_factory=lambda: LinkClass(LinkKind.IntraGpu))
    host_gpu: LinkClass = field(default_factory=lambda: LinkClass(LinkKind.HostGpu))
    inter_node: LinkClass = field(default_factory=lambda: LinkClass(LinkKind.InterNode))

    def total_gpus(self) -> int:
        return self.num_nodes * self.gpus_per_node

    def link(self, kind: LinkKind) -> LinkClass:
        return (self.intra_gpu, self.host_gpu, self.inter_node)[int(kind)]

    def to_c(self) -> _capi.Topology:
        t = _capi.Topology()
        t.num_nodes, t.gpus_per_node = self.num_nodes, self.gpus_per_node
        for k, lc in enumerate((self.intra_gpu, self.host_gpu, self.inter_node)):
            t.bandwidth_bytes_per_s[k] = lc.bandwidth_bytes_per_s
            t.latency_s[k] = lc.latency_s
            t.duplex[k] = int(lc.duplex)
        return t

    @staticmethod
    def from_c(t: _capi.Topology) -> "ClusterTopology":
        links = [LinkClass(LinkKind(k), t.bandwidth_bytes_per_s[k], Duplex(t.duplex[k]), t.latency_s[k])
                 for k in range(3)]
        return ClusterTopology(t.num_nodes, t.gpus_per_node, *links)


_PRESETS = ["pcie4-measured", "pcie4-theoretical", "nvlink3-theoretical", "ib100-rdma-measured",
            "ib100-ipoib-measured", "eth10g-measured", "eth1g-measured", "eth100g-theoretical"]


def link_preset(name: str) -> LinkClass:
    kind, bw = C.c_int32(), C.c_double()
    check(lib().fcdp_link_preset(name.encode(), C.byref(kind), C.byref(bw)))
    return LinkClass(LinkKind(kind.value), bw.value)


def link_preset_names() -> List[str]:
    return list(_PRESETS)


def make_topology(num_nodes: int, gpus_per_node: int, intra_preset: str = "nvlink3-theoretical",
                  host_preset: str = "pcie4-measured",
                  inter_preset: str = "ib100-rdma-measured") -> ClusterTopology:
    t = _capi.Topology()
    check(lib().fcdp_make_topology(num_nodes, gpus_per_node, intra_preset.encode(),
                                   host_preset.encode(), inter_preset.encode(), C.byref(t)))
    return ClusterTopology.from_c(t)


def effective_bandwidth(topo: ClusterTopology, kind: LinkKind) -> float:
    return topo.link(kind).bandwidth_bytes_per_s


def transfer_time(size_bytes: int, kind: LinkKind, topo: ClusterTopology) -> float:
    out = C.c_double()
    t = topo.to_c()
    check(lib().fcdp_transfer_time(size_bytes, int(kind), C.byref(t), C.byref(out)))
    return out.value

# -------------------------------------------------------------- workload.hpp


@dataclass
class LayerSpec:
    layer_id: int = 0
    param_count: int = 0
    trainable_fraction: float = 1.0
    fwd_compute_s_per_sample: float = 0.0
    bwd_compute_s_per_sample: float = 0.0
    activation_bytes_per_sample: int = 0


class _ModelHandle:
    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr and _capi._lib is not None:
                _capi._lib.fcdp_model_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


@dataclass
class ModelSpec:
    layers: List[LayerSpec] = field(default_factory=list)
    param_bytes_per_element: int = 2
    optimizer_state_multiplier: float = 6.0
    batch_per_gpu: int = 8

    def num_layers(self) -> int:
        return len(self.layers)

    def handle(self) -> _ModelHandle:
        L = len(self.layers)
        counts = (C.c_int64 * max(L, 1))(*[l.param_count for l in self.layers])
        frac = (C.c_double * max(L, 1))(*[l.trainable_fraction for l in self.layers])
        fwd = (C.c_double * max(L, 1))(*[l.fwd_compute_s_per_sample for l in self.layers])
        bwd = (C.c_double * max(L, 1))(*[l.bwd_compute_s_per_sample for l in self.layers])
        act = (C.c_int64 * max(L, 1))(*[l.activation_bytes_per_sample for l in self.layers])
        out = C.c_void_p()
        check(lib().fcdp_model_create(L, counts, frac, self.param_bytes_per_element,
                                      self.optimizer_state_multiplier, self.batch_per_gpu, fwd, bwd,
                                      act, C.byref(out)))
        return _ModelHandle(out.value)

    def _info(self):
        h = self.handle()
        L, tot, tr, eb = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
        check(lib().fcdp_model_info(h.ptr, C.byref(L), C.byref(tot), C.byref(tr), C.byref(eb)))
        return tot.value, tr.value

    def total_params(self) -> int:
        return sum(l.param_count for l in self.layers)

    def trainable_params(self) -> int:
        return self._info()[1]

    def frozen_params(self) -> int:
        return self.total_params() - self.trainable_params()

    def validate(self) -> None:
        self.handle()  # creation does not validate; a cheap build does
        m = self.handle()
        st = C.c_void_p()
        check(lib().fcdp_states_init(m.ptr, C.byref(st)))
        lib().fcdp_states_destroy(st)
        t = make_topology(1, 1).to_c()
        fp = _capi.MemoryFootprint()
        check(lib().fcdp_memory_footprint_of(C.byref(StrategyPlan().to_c()), m.ptr, C.byref(t), C.byref(fp)))

    def layer_bytes(self, layer: int):
        h = self.handle()
        a, t, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().fcdp_model_layer_bytes(h.ptr, layer, C.byref(a), C.byref(t), C.byref(f)))
        return a.value, t.value, f.value


def layer_bytes(model: ModelSpec, layer: int) -> int:
    return model.layer_bytes(layer)[0]


def layer_trainable_bytes(model: ModelSpec, layer: int) -> int:
    return model.layer_bytes(layer)[1]


def layer_frozen_bytes(model: ModelSpec, layer: int) -> int:
    return model.layer_bytes(layer)[2]


def param_bytes(model: ModelSpec) -> int:
    return sum(layer_bytes(model, l) for l in range(model.num_layers()))


def trainable_param_bytes(model: ModelSpec) -> int:
    return sum(layer_trainable_bytes(model, l) for l in range(model.num_layers()))


def _model_from_handle(ptr: int, template: Optional[ModelSpec] = None) -> ModelSpec:
    # Presets are rebuilt on the Python side from the C handle's layer sizes.
    L, tot, tr, eb = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
    check(lib().fcdp_model_info(ptr, C.byref(L), C.byref(tot), C.byref(tr), C.byref(eb)))
    layers = []
    for l in range(L.value):
        a, t, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().fcdp_model_layer_bytes(ptr, l, C.byref(a), C.byref(t), C.byref(f)))
        layers.append(LayerSpec(layer_id=l, param_count=a.value // eb.value))
    return ModelSpec(layers=layers, param_bytes_per_element=eb.value)


def model_preset(name: str) -> ModelSpec:
    out = C.c_void_p()
    check(lib().fcdp_model_preset(name.encode(), C.byref(out)))
    h = _ModelHandle(out.value)
    return _model_from_handle(h.ptr)


def model_preset_names() -> List[str]:
    return ["gpt10b", "gpt15b", "gpt20b", "gpt25b", "gpt30b"]


def apply_lora_mask(model: ModelSpec, trainable_fraction: float) -> ModelSpec:
    h = model.handle()
    out = C.c_void_p()
    check(lib().fcdp_model_apply_lora_mask(h.ptr, trainable_fraction, C.byref(out)))
    _ModelHandle(out.value)  # validated by the C side; apply on the Python copy
    layers = [LayerSpec(**{**l.__dict__, "trainable_fraction": trainable_fraction}) for l in model.layers]
    return ModelSpec(layers, model.param_bytes_per_element, model.optimizer_state_multiplier,
                     model.batch_per_gpu)

# -------------------------------------------------------------- strategy.hpp


class StrategyKind(enum.IntEnum):
    Zero2 = 0
    Zero3 = 1
    MiCS = 2
    ZeroPP = 3
    Fcdp = 4
    FcdpComm = 5

    def __str__(self) -> str:
        return ["zero2", "zero3", "mics", "zeropp", "fcdp", "fcdp-comm"][int(self)]

    @staticmethod
    def from_string(s: str) -> "StrategyKind":
        k = C.c_int32()
        check(lib().fcdp_strategy_from_string(s.encode(), C.byref(k)))
        return StrategyKind(k.value)


@dataclass
class StrategyPlan:
    kind: StrategyKind = StrategyKind.Zero3
    subgroup_size: int = 0
    tau: float = 0.0
    host_cache_enabled: bool = False

    def uses_host_cache(self) -> bool:
        return self.kind in (StrategyKind.Fcdp, StrategyKind.FcdpComm) or self.host_cache_enabled

    def peft_aware(self) -> bool:
        return self.kind == StrategyKind.FcdpComm

    def to_c(self) -> _capi.Plan:
        return _capi.Plan(int(self.kind), self.subgroup_size, self.tau, int(self.host_cache_enabled))


@dataclass
class MemoryFootprint:
    gpu_param_shard_bytes: int = 0
    gpu_gradient_bytes: int = 0
    gpu_optimizer_bytes: int = 0
    gpu_persistent_bytes: int = 0
    gpu_cache_bytes: int = 0
    gpu_transient_peak_bytes: int = 0
    host_cache_bytes_per_node: int = 0

    def gpu_total_bytes(self) -> int:
        return self.gpu_persistent_bytes + self.gpu_cache_bytes + self.gpu_transient_peak_bytes


def memory_footprint(plan: StrategyPlan, model: ModelSpec, topo: ClusterTopology) -> MemoryFootprint:
    m, p, t, fp = model.handle(), plan.to_c(), topo.to_c(), _capi.MemoryFootprint()
    check(lib().fcdp_memory_footprint_of(C.byref(p), m.ptr, C.byref(t), C.byref(fp)))
    return MemoryFootprint(**{n: int(getattr(fp, n)) for n, _ in fp._fields_})


def max_feasible_batch(plan: StrategyPlan, model: ModelSpec, topo: ClusterTopology,
                       gpu_capacity_bytes: int):
    m, p, t = model.handle(), plan.to_c(), topo.to_c()
    b, oom = C.c_int32(), C.c_int32()
    check(lib().fcdp_max_feasible_batch(C.byref(p), m.ptr, C.byref(t), gpu_capacity_bytes, C.byref(b),
                                        C.byref(oom)))
    return b.value, bool(oom.value)

# -------------------------------------------------------------- costmodel.hpp


@dataclass
class CommVolume:
    fwd_ag_inter: int = 0
    bwd_ag_inter: int = 0
    reduce_scatter_inter: int = 0
    param_sync_inter: int = 0
    intra_node_total: int = 0
    h2d_total: int = 0
    d2h_total: int = 0

    def inter_total(self) -> int:
        return self.fwd_ag_inter + self.bwd_ag_inter + self.reduce_scatter_inter + self.param_sync_inter


def comm_volume(plan: StrategyPlan, model: ModelSpec, topo: ClusterTopology, iteration: int) -> CommVolume:
    m, p, t, v = model.handle(), plan.to_c(), topo.to_c(), _capi.CommVolume()
    check(lib().fcdp_comm_volume_of(C.byref(p), m.ptr, C.byref(t), iteration, C.byref(v)))
    return CommVolume(**{n: int(getattr(v, n)) for n, _ in v._fields_})


def iteration_time_estimate(plan: StrategyPlan, model: ModelSpec, topo: ClusterTopology) -> float:
    m, p, t, out = model.handle(), plan.to_c(), topo.to_c(), C.c_double()
    check(lib().fcdp_iteration_time_estimate(C.byref(p), m.ptr, C.byref(t), C.byref(out)))
    return out.value

# -------------------------------------------------------------- schedule.hpp


class EventKind(enum.IntEnum):
    AgInter = 0
    AgIntra = 1
    H2D = 2
    D2H = 3
    ComputeFwd = 4
    ComputeBwd = 5
    ReduceScatter = 6
    OptimizerStep = 7
    MaskDirty = 8
    Broadcast = 9


class ParamSet(enum.IntEnum):
    All = 0
    TrainableOnly = 1
    FrozenOnly = 2


@dataclass
class Event:
    id: int
    kind: EventKind
    layer: int
    param_set: ParamSet
    bytes_total: int
    deps: List[int]


@dataclass
class ParamState:
    layer: int = 0
    frozen: bool = False
    version: int = 0
    dirty: bool = True
    host_cached_version: Optional[int] = None
    gpu_cached: bool = False


class _States:
    """Owned std::vector<ParamState> on the C side."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr and _capi._lib is not None:
                _capi._lib.fcdp_states_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass

    @staticmethod
    def from_list(states: Sequence[ParamState]) -> "_States":
        out = C.c_void_p()
        check(lib().fcdp_states_create(len(states), C.byref(out)))
        s = _States(out.value)
        for i, st in enumerate(states):
            c = _capi.ParamStateC(st.layer, int(st.frozen), st.version, int(st.dirty),
                                  -1 if st.host_cached_version is None else st.host_cached_version,
                                  int(st.gpu_cached))
            check(lib().fcdp_states_set(s.ptr, i, C.byref(c)))
        return s

    def to_list(self) -> List[ParamState]:
        n = C.c_int32()
        check(lib().fcdp_states_count(self.ptr, C.byref(n)))
        out = []
        for i in range(n.value):
            c = _capi.ParamStateC()
            check(lib().fcdp_states_get(self.ptr, i, C.byref(c)))
            out.append(ParamState(c.layer, bool(c.frozen), c.version, bool(c.dirty),
                                  None if c.host_cached_version < 0 else c.host_cached_version,
                                  bool(c.gpu_cached)))
        return out


class EventProgram:
    """Owned shardsim::EventProgram; events are decoded lazily."""

    def __init__(self, ptr: int, strategy: StrategyKind, iteration_index: int):
        self.ptr = ptr
        self.strategy = strategy
        self.iteration_index = iteration_index
        self._events = None

    def __del__(self):
        try:
            if getattr(self, "ptr", None) and _capi._lib is not None:
                _capi._lib.fcdp_program_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass

    @property
    def events(self) -> List[Event]:
        if self._events is None:
            n = C.c_uint32()
            check(lib().fcdp_program_num_events(self.ptr, C.byref(n)))
            evs = []
            deps = (C.c_uint32 * 4096)()
            for i in range(n.value):
                e = _capi.EventC()
                check(lib().fcdp_program_event(self.ptr, i, C.byref(e), deps, 4096))
                evs.append(Event(e.id, EventKind(e.kind), e.layer, ParamSet(e.param_set), e.bytes_total,
                                 [deps[k] for k in range(e.num_deps)]))
            self._events = evs
        return self._events

    def layer_flags(self, num_layers: int) -> List[int]:
        buf = (C.c_uint8 * max(num_layers, 1))()
        check(lib().fcdp_program_layer_flags(self.ptr, buf, num_layers))
        return list(buf)[:num_layers]

    @staticmethod
    def from_events(iteration_index: int, strategy: StrategyKind, events: Sequence[Event],
                    layer_flags: Sequence[int]) -> "EventProgram":
        """A program from an explicit event list (fcdp_program_create): an
        external scheduler's program, or a mutated one."""
        n = len(events)
        arr = (_capi.EventC * max(n, 1))()
        off = (C.c_uint32 * (n + 1))()
        flat: List[int] = []
        for i, e in enumerate(events):
            arr[i] = _capi.EventC(e.id, int(e.kind), e.layer, int(e.param_set), e.bytes_total, len(e.deps))
            off[i] = len(flat)
            flat += list(e.deps)
        off[n] = len(flat)
        deps = (C.c_uint32 * max(len(flat), 1))(*flat)
        L = len(layer_flags)
        fl = (C.c_uint8 * max(L, 1))(*layer_flags)
        out = C.c_void_p()
        check(lib().fcdp_program_create(iteration_index, int(strategy), n, arr, off, deps, L, fl, C.byref(out)))
        return EventProgram(out.value, strategy, iteration_index)

    def without(self, drop: Sequence[int], num_layers: int,
                replace: Optional[Dict[int, Event]] = None) -> "EventProgram":
        """Mutation helper: this program minus the events `drop` (ids renumbered,
        deps on dropped events removed), with events in `replace` swapped in."""
        keep = [e for e in self.events if e.id not in set(drop)]
        new_id = {e.id: i for i, e in enumerate(keep)}
        evs = []
        for e in keep:
            r = (replace or {}).get(e.id, e)
            evs.append(Event(new_id[e.id], r.kind, r.layer, r.param_set, r.bytes_total,
                             [new_id[d] for d in e.deps if d in new_id]))
        return EventProgram.from_events(self.iteration_index, self.strategy, evs, self.layer_flags(num_layers))


def init_param_states(model: ModelSpec) -> List[ParamState]:
    m = model.handle()
    out = C.c_void_p()
    check(lib().fcdp_states_init(m.ptr, C.byref(out)))
    return _States(out.value).to_list()


def build_iteration(plan: StrategyPlan, model: ModelSpec, topo: ClusterTopology,
                    states: Sequence[ParamState], iteration_index: int, prefetch: bool = True,
                    gpu_capacity_bytes: int = 0) -> EventProgram:
    s = _States.from_list(states)
    m, p, t = model.handle(), plan.to_c(), topo.to_c()
    out = C.c_void_p()
    check(lib().fcdp_build_iteration(C.byref(p), m.ptr, C.byref(t), s.ptr, iteration_index,
                                     int(prefetch), gpu_capacity_bytes, C.byref(out)))
    return EventProgram(out.value, plan.kind, iteration_index)


def step_state(states: Sequence[ParamState], program: EventProgram) -> List[ParamState]:
    s = _States.from_list(states)
    check(lib().fcdp_step_state(s.ptr, program.ptr))
    return s.to_list()


def serialize_program(program: EventProgram) -> str:
    n = C.c_size_t()
    check(lib().fcdp_program_serialize(program.ptr, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().fcdp_program_serialize(program.ptr, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()
