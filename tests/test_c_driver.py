"""The engine driven from plain C through include/fcdp.h only (tests/cpp/engine_driver.c):
no Python or torch on the host path.  CPU: it compiles and links against libfcdp.so.
GPU: 1x1 and 2-rank jobs pass its own checks (NIC counters == comm_volume, the AdamW
step of a constant gradient)."""
import subprocess
import uuid
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2602_06499_b200"
OUT = PKG / "build" / "engine_driver"


def build_driver():
    OUT.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-O2", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include",
           str(ROOT / "tests" / "cpp" / "engine_driver.c"), "-o", str(OUT), f"-L{PKG}", "-lfcdp",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return OUT


def test_c_driver_builds(built):
    assert build_driver().exists()


@pytest.mark.gpu
@pytest.mark.parametrize("nodes,g,strategy", [(1, 1, "fcdp"), (1, 1, "zero3"), (2, 1, "fcdp"), (2, 1, "zero3"),
                                              (1, 2, "fcdp")])
def test_c_driver_runs_engine(built, nodes, g, strategy):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = build_driver()
    shm = f"fcdp_cdrv_{uuid.uuid4().hex[:10]}"
    procs = [subprocess.Popen([str(exe), shm, str(r), str(nodes), str(g), strategy], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(nodes * g)]
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r}:\n{out[-3000:]}"
        assert "engine_driver ok" in out
