"""End-to-end training parity: FCDP / ZeRO-3 / FCDP-Comm on the B200 engine vs a
plain single-process torch fp32 CPU reference of the same model, same
synthetic inputs and seeds: loss, the reduced fp32 gradient and the updated
fp32 master weights after every step, per layer (trainable portion, gathered
from all ranks' shards in global shard order r = j*N + n).

Tolerances (north_star's "stated fp32 tolerance"), per
layer and step, err = |engine - reference|:
  fp32 model (C1 tiny):  loss rel 1e-4;  grad max err <= 1e-4 * max|grad_ref|;
                         master: 99.9% of elements within 1e-6 + 1e-4*|w_ref|,
                         and every element within 2*lr*step (AdamW moves an element
                         by at most ~lr per step, so a near-zero gradient whose sign
                         differs between two fp32 summation orders can move it
                         the other way - bounded, and rare).
  bf16 models:           loss rel 2e-2;  grad ||err||_2 <= 5e-2 * ||grad_ref||_2;
                         master update (w - w0): ||err||_2 <= 0.25 * ||dw_ref||_2.
The bf16 tolerances also cover the inter-node RS wire: at N > 1 the node's
partial sums cross the NIC in bf16 (costmodel.cpp:86-88 books the bytes in the
parameter dtype); the N = 2 case reports its error beside the N = 1 case."""
import json
import pickle
import subprocess
import sys
import uuid
from pathlib import Path

import numpy as np
import pytest

from tests.model_reference import compare, cpu_reference

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def run(tmp_path, preset, strategy, N=1, g=1, steps=3, batch=2, lr=1e-3, wd=0.01, seed=0x5EED):
    world = N * g
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")  # ranks share GPUs round-robin (rank % device_count)
    cfg = dict(preset=preset, strategy=strategy, N=N, g=g, steps=steps, batch=batch, lr=lr, wd=wd, seed=seed,
               shm=f"fcdp_tr_{uuid.uuid4().hex[:10]}", out=str(tmp_path))
    procs = [subprocess.Popen([sys.executable, str(ROOT / "tests/trainer_worker.py"), json.dumps(dict(cfg, rank=r))],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for r, p in enumerate(procs):
        assert p.returncode == 0, outs[r][-4000:]
    return cfg, [pickle.load(open(tmp_path / f"rank{r}.pkl", "rb")) for r in range(world)]


def _losses(res):
    return np.mean([r["losses"] for r in res], axis=0)  # each rank reports its local mean


@pytest.mark.parametrize("strategy", ["fcdp", "zero3"])
def test_tiny_fp32_parity(tmp_path, built, strategy):
    cfg, res = run(tmp_path, "tiny", strategy)
    ref = cpu_reference(cfg)
    np.testing.assert_allclose(_losses(res), ref["losses"], rtol=1e-4)
    compare(cfg, res, ref, fp32=True)


@pytest.mark.parametrize("N,g,strategy", [(2, 1, "fcdp"), (1, 2, "fcdp"), (2, 2, "zero3"), (2, 2, "fcdp")])
def test_tiny_fp32_multi_rank(tmp_path, built, N, g, strategy):
    cfg, res = run(tmp_path, "tiny", strategy, N=N, g=g)
    ref = cpu_reference(cfg)
    np.testing.assert_allclose(_losses(res), ref["losses"], rtol=1e-4)
    compare(cfg, res, ref, fp32=True)


@pytest.mark.parametrize("N", [1, 2])
def test_gpt2_bf16(tmp_path, built, N):
    cfg, res = run(tmp_path, "gpt2-small-test", "fcdp", N=N)
    ref = cpu_reference(cfg)
    np.testing.assert_allclose(_losses(res), ref["losses"], rtol=2e-2)
    compare(cfg, res, ref, fp32=False)


@pytest.mark.parametrize("N,g", [(1, 1), (2, 2)])
def test_llama_lora_fcdp_comm(tmp_path, built, N, g):
    cfg, res = run(tmp_path, "llama-lora-test", "fcdp-comm", N=N, g=g, steps=4)
    ref = cpu_reference(cfg)
    np.testing.assert_allclose(_losses(res), ref["losses"], rtol=2e-2)
    compare(cfg, res, ref, fp32=False)
