"""Config C1 on the C++ CPU executor (BASELINE.json configs[0]): the tiny 2-layer
h=256 fp32 transformer, 2 simulated ranks, FULL training steps - the driving
model's forward/backward on the host cores as the executor's compute callback,
every parameter movement of the reference-built program on the executor.

Checks: loss, reduced gradients and updated masters against the plain torch
fp32 CPU training (tests/model_reference.py) within the stated fp32
tolerances; FCDP and ZeRO-3 produce identical numbers (they differ only in
where parameters travel); FCDP's backward moves 0 inter-group bytes."""
import numpy as np
import pytest

pytest.importorskip("torch")
cx = pytest.importorskip("oracle.cpu_executor")
try:
    cx.lib()
except Exception:
    pytest.skip("cpu executor not built (needs /root/reference)", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from oracle.cpu_step import full_step_executor  # noqa: E402
from tests.model_reference import compare, cpu_reference  # noqa: E402


def run(strategy, N=2, g=1, steps=2, batch=2, lr=1e-3, wd=0.01):
    from paper_2602_06499_b200.driving_model import PRESETS
    cfg = dict(preset="tiny", strategy=strategy, N=N, g=g, steps=steps, batch=batch, lr=lr, wd=wd, seed=0x5EED)
    mc = PRESETS["tiny"]
    ex, comp = full_step_executor("tiny", N, g, strategy, batch, lr=lr, wd=wd, threads=4)
    V = 16 // mc.dtype_bytes
    geos = [O.geom(d.numel * mc.dtype_bytes // 16, d.chunk_mask(mc.dtype_bytes), N, g) for d in comp.defs]
    res = [{"losses": [], "grads": [], "masters": []} for _ in range(N * g)]
    stats = []
    for s in range(1, steps + 1):
        comp.set_step(s)
        stats.append(ex.step())
        for r in range(N * g):
            res[r]["losses"].append(comp.losses[r])
            res[r]["grads"].append({l: ex.read(r, l, "grad", geo.shard_t * V * 4).view(np.float32)
                                    for l, geo in enumerate(geos) if geo.pt})
            res[r]["masters"].append({l: ex.read(r, l, "master", geo.shard_t * V * 4).view(np.float32)
                                      for l, geo in enumerate(geos) if geo.pt})
    ex.close()
    return cfg, res, stats


@pytest.mark.parametrize("strategy", ["fcdp", "zero3"])
def test_c1_full_step_matches_torch_reference(strategy):
    cfg, res, stats = run(strategy)
    ref = cpu_reference(cfg)
    np.testing.assert_allclose(np.mean([r["losses"] for r in res], axis=0), ref["losses"], rtol=1e-5)
    compare(cfg, res, ref, fp32=True)
    if strategy == "fcdp":
        assert all(s["nic_tx_bwd_ag"] == 0 for s in stats)
    else:
        assert all(s["nic_tx_bwd_ag"] > 0 for s in stats)


def test_c1_fcdp_equals_zero3_bit_for_bit():
    _, a, _ = run("fcdp")
    _, b, _ = run("zero3")
    for ra, rb in zip(a, b):
        assert ra["losses"] == rb["losses"]
        for ga, gb in zip(ra["masters"], rb["masters"]):
            for l in ga:
                assert np.array_equal(ga[l].view(np.uint32), gb[l].view(np.uint32))
