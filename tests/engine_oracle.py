"""CPU re-derivation of an engine parity job (test infrastructure).

Given the job config of tests/engine_worker.py, replays the same shardsim
programs on the CPU oracle (oracle/fcdp_oracle.c) for all G simulated ranks:
gathered layers, FCDP-Cache contents, reduce-scattered gradients, AdamW
updates and the NIC byte counters, so every value the GPUs produced can be
compared bit for bit.
"""
import numpy as np

from oracle import oracle as O


def scope_nodes(cfg):
    """Nodes one shard set spans: MiCS (subgroup = g) shards inside a node."""
    return 1 if cfg["strategy"] == "mics" else cfg["N"]


def grad_coeff(rank):
    return (1 + rank) / 8.0


def _to_f32(a, eb):
    return O.bf16_to_f32(a) if eb == 2 else a.astype(np.float32)


def _from_f32(x, eb):
    return O.f32_to_bf16(x) if eb == 2 else x.astype(np.float32)


def _elem(eb):
    return np.uint16 if eb == 2 else np.float32


class Sim:
    def __init__(self, cfg):
        from paper_2602_06499_b200 import shardsim as S
        self.S = S
        self.cfg = cfg
        self.N, self.g = cfg["N"], cfg["g"]
        self.G = self.N * self.g
        self.Ns = scope_nodes(cfg)
        self.Gs = self.Ns * self.g  # shards per portion
        self.mics = cfg["strategy"] == "mics"
        self.eb = cfg["eb"]
        self.V = 16 // self.eb
        self.masks = [np.array(m, np.uint8) for m in cfg["masks"]]
        self.E = cfg["params"]
        self.L = len(self.E)
        self.geo = [O.geom(len(m), m, self.Ns, self.g) for m in self.masks]
        layers = [S.LayerSpec(i, E, float(int(m.sum()) * self.V) / E) for i, (E, m) in enumerate(zip(self.E, self.masks))]
        self.model = S.ModelSpec(layers, self.eb)
        self.topo = S.make_topology(self.N, self.g, inter_preset=cfg.get("inter", "ib100-rdma-measured"))
        self.plan = S.StrategyPlan(S.StrategyKind.from_string(cfg["strategy"]), tau=cfg.get("tau", 0.0))
        # per rank, per layer: portion shards (bytes) and optimizer state
        self.shard_t = [[None] * self.L for _ in range(self.G)]
        self.shard_f = [[None] * self.L for _ in range(self.G)]
        self.master = [[None] * self.L for _ in range(self.G)]
        self.m = [[None] * self.L for _ in range(self.G)]
        self.v = [[None] * self.L for _ in range(self.G)]
        self.host = [[(None, None)] * self.L for _ in range(self.G)]
        for l in range(self.L):
            nat = O.init_natural(self.E[l], self.eb, cfg["seed"], l, [(0, self.E[l], 0, 0.05)])
            t, f = self._padded_portions(l, nat)
            geo = self.geo[l]
            for r in range(self.G):
                s = self.shard_index(r)
                self.shard_t[r][l] = t[s * geo.shard_t * 16:(s + 1) * geo.shard_t * 16].copy()
                self.shard_f[r][l] = f[s * geo.shard_f * 16:(s + 1) * geo.shard_f * 16].copy()
                self.master[r][l] = _to_f32(self.shard_t[r][l].view(_elem(self.eb)), self.eb).copy()
                self.m[r][l] = np.zeros_like(self.master[r][l])
                self.v[r][l] = np.zeros_like(self.master[r][l])
        self.step = 0
        self.prev_retained = [False] * self.L

    def shard_index(self, rank):
        n, j = divmod(rank, self.g)
        return j * self.Ns + (n if self.Ns > 1 else 0)

    def _padded_portions(self, l, nat):
        geo = self.geo[l]
        t, f = O.partition(nat.view(np.uint8), self.masks[l])
        tp = np.zeros(geo.shard_t * self.Gs * 16, np.uint8)
        tp[:t.size] = t
        fp = np.zeros(geo.shard_f * self.Gs * 16, np.uint8)
        fp[:f.size] = f
        return tp, fp

    def portions(self, l):
        geo = self.geo[l]
        t = np.zeros(geo.shard_t * self.Gs * 16, np.uint8)
        f = np.zeros(geo.shard_f * self.Gs * 16, np.uint8)
        for r in range(self.Gs):  # one shard set (the first replica for MiCS)
            s = self.shard_index(r)
            t[s * geo.shard_t * 16:(s + 1) * geo.shard_t * 16] = self.shard_t[r][l]
            f[s * geo.shard_f * 16:(s + 1) * geo.shard_f * 16] = self.shard_f[r][l]
        return t, f

    def natural(self, l):
        t, f = self.portions(l)
        geo = self.geo[l]
        return O.unpartition(t[:geo.pt * 16], f[:geo.pf * 16], self.masks[l], len(self.masks[l]))

    def iteration(self, it, states):
        S = self.S
        prog = S.build_iteration(self.plan, self.model, self.topo, states, it,
                                 gpu_capacity_bytes=self.cfg.get("capacity", 0))
        exp = [{"captures": [], "host": {}, "grad": {}, "master": {}, "shard_t": {}, "shard_f": {},
                "counters": {k: 0 for k in ("nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs", "cache_h2d",
                                            "cache_d2h", "nvlink_rx", "nic_tx_grad_sync")}} for _ in range(self.G)]
        last_fwd = max(e.id for e in prog.events if e.kind == S.EventKind.ComputeFwd)
        retained = [bool(f & 1) for f in prog.layer_flags(self.L)]

        def resident(e):  # engine elides frozen-only reloads of layers retained twice in a row
            frozen_only = e.param_set == S.ParamSet.FrozenOnly or (e.param_set == S.ParamSet.All and self.geo[e.layer].pt == 0)
            return frozen_only and retained[e.layer] and self.prev_retained[e.layer]
        nat_now = [self.natural(l) for l in range(self.L)]
        grads = {}
        for e in prog.events:
            l = e.layer
            if e.kind in (S.EventKind.ComputeFwd, S.EventKind.ComputeBwd):
                for r in range(self.G):
                    exp[r]["captures"].append((int(e.kind), l, nat_now[l]))
                if e.kind == S.EventKind.ComputeBwd:
                    w = _to_f32(nat_now[l].view(_elem(self.eb)), self.eb)
                    grads[l] = [_from_f32((w * np.float32(grad_coeff(r))).astype(np.float32), self.eb) for r in range(self.G)]
            elif e.kind == S.EventKind.D2H:
                t, f = self.portions(l)
                geo = self.geo[l]
                for r in range(self.G):
                    j = r % self.g
                    ht, hf = self.host[r][l]
                    if e.param_set != S.ParamSet.FrozenOnly and geo.pt:
                        ht = t[j * geo.slice_t * 16:(j + 1) * geo.slice_t * 16].copy()
                        exp[r]["counters"]["cache_d2h"] += self._real_slice(l, False, j) * 16
                    if e.param_set != S.ParamSet.TrainableOnly and geo.pf:
                        hf = f[j * geo.slice_f * 16:(j + 1) * geo.slice_f * 16].copy()
                        exp[r]["counters"]["cache_d2h"] += self._real_slice(l, True, j) * 16
                    self.host[r][l] = (ht, hf)
            elif e.kind == S.EventKind.AgInter:
                for r in range(self.G):
                    s = self.shard_index(r)
                    b = 0
                    if e.param_set != S.ParamSet.FrozenOnly:
                        b += self._real(l, False, s)
                    if e.param_set != S.ParamSet.TrainableOnly:
                        b += self._real(l, True, s)
                    key = "nic_tx_bwd_ag" if e.id > last_fwd else "nic_tx_fwd_ag"
                    exp[r]["counters"][key] += b * 16 * (self.N - 1)
                    exp[r]["counters"]["nvlink_rx"] += self._nvl(l, r, e.param_set)
            elif e.kind == S.EventKind.H2D and resident(e):
                pass
            elif e.kind == S.EventKind.AgIntra and resident(e):
                pass
            elif e.kind == S.EventKind.H2D:
                for r in range(self.G):
                    j = r % self.g
                    if e.param_set != S.ParamSet.FrozenOnly:
                        exp[r]["counters"]["cache_h2d"] += self._real_slice(l, False, j) * 16
                    if e.param_set != S.ParamSet.TrainableOnly:
                        exp[r]["counters"]["cache_h2d"] += self._real_slice(l, True, j) * 16
            elif e.kind == S.EventKind.AgIntra:
                for r in range(self.G):
                    exp[r]["counters"]["nvlink_rx"] += self._nvl(l, r, e.param_set)
            elif e.kind == S.EventKind.ReduceScatter:
                self._reduce_scatter(l, grads[l], exp)
            elif e.kind == S.EventKind.OptimizerStep:
                self.step += 1
                for r in range(self.G):
                    for ll in range(self.L):
                        if self.geo[ll].pt == 0:
                            continue
                        p = self.shard_t[r][ll].view(_elem(self.eb)).copy()
                        O.adam(self.master[r][ll], self.m[r][ll], self.v[r][ll], self.grad[r][ll], p,
                               1e-2, 0.9, 0.95, 1e-8, 0.01, self.step)
                        self.shard_t[r][ll] = p.view(np.uint8).copy()
        for r in range(self.G):
            for l in range(self.L):
                exp[r]["host"][l] = self.host[r][l]
                exp[r]["master"][l] = self.master[r][l]
                exp[r]["shard_t"][l] = self.shard_t[r][l]
                exp[r]["shard_f"][l] = self.shard_f[r][l]
                exp[r]["grad"][l] = self.grad[r][l] if hasattr(self, "grad") else None
        new_states = S.step_state(states, prog)
        self.prev_retained = retained
        return exp, new_states, prog

    def _real(self, l, frozen, s):
        geo = self.geo[l]
        per, tot = (geo.shard_f, geo.pf) if frozen else (geo.shard_t, geo.pt)
        return max(0, min(per, tot - s * per))

    def _real_slice(self, l, frozen, j):
        return sum(self._real(l, frozen, j * self.Ns + n) for n in range(self.Ns))

    def _nvl(self, l, r, pset):
        S = self.S
        j = r % self.g
        b = 0
        for jj in range(self.g):
            if jj == j:
                continue
            if pset != S.ParamSet.FrozenOnly:
                b += self._real_slice(l, False, jj)
            if pset != S.ParamSet.TrainableOnly:
                b += self._real_slice(l, True, jj)
        return b * 16

    def _reduce_scatter(self, l, g_all, exp):
        if not hasattr(self, "grad"):
            self.grad = [[np.zeros(self.geo[ll].shard_t * self.V, np.float32) for ll in range(self.L)]
                         for _ in range(self.G)]
        geo = self.geo[l]
        if geo.pt == 0:
            return
        scale = np.float32(1.0 / self.G)
        N, g = self.N, self.g
        own, wire = {}, {}
        for r in range(self.G):
            n, j = divmod(r, g)
            local = [g_all[n * g + jj] for jj in range(g)]
            own_idx = (-1 if self.mics else n) if N > 1 else 0  # MiCS: whole slice on the wire
            own[r], wire[r] = O.rs_slice(geo, self.masks[l], self.eb, local, j, own_idx, float(scale), N == 1)
            exp[r]["counters"]["nvlink_rx"] += (g - 1) * self._real_slice(l, False, j) * 16
        for r in range(self.G):
            n, j = divmod(r, g)
            if N == 1:
                self.grad[r][l] = own[r].copy()
                continue
            sh = geo.shard_t * self.V
            rx = np.zeros(N * sh, _elem(self.eb))
            if self.mics:  # replica all-reduce: every node's whole slice, fixed node order
                for nn in range(N):
                    rx[nn * sh:(nn + 1) * sh] = wire[nn * g + j]
                exp[r]["counters"]["nic_tx_grad_sync"] += (N - 1) * self._real_slice(l, False, j) * 16
                self.grad[r][l] = O.rs_finalize(np.zeros(sh, np.float32), rx, N, -1, self.eb, sh, float(scale))
                continue
            for nn in range(N):
                if nn == n:
                    continue
                src = wire[nn * g + j]
                rx[nn * sh:(nn + 1) * sh] = src[n * sh:(n + 1) * sh]
                exp[r]["counters"]["nic_tx_rs"] += self._real(l, False, j * N + nn) * 16
            self.grad[r][l] = O.rs_finalize(own[r], rx, N, n, self.eb, sh, float(scale))
