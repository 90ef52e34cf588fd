"""Host-side multi-rank logic on CPU (world_size 2, gloo): the shared control
block, its barrier, and the per-node NIC pacing of the emulator
(one NIC per emulated node serialises that node's ranks; reference
topology.hpp:23-25)."""
import ctypes as C
import os
import uuid

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


# 200 ms of wire time per rank: long enough that host scheduling jitter on a
# busy CI box (a fresh build running beside the test) stays well inside the bounds
PIECE = 20_000_000


def _worker(rank, world, port, nodes, local, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name = [f"fcdp_cpu_{uuid.uuid4().hex[:10]}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    from paper_2602_06499_b200 import _capi
    out = C.c_double()
    rc = _capi.lib().fcdp_nic_selftest(name[0].encode(), rank, nodes, local, 1e9, PIECE, 10, C.byref(out))
    q.put((rank, rc, out.value, _capi.lib().fcdp_last_error().decode()))
    dist.barrier()
    dist.destroy_process_group()


def _run(nodes, local):
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nodes, local, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("nodes,local", [(1, 2), (2, 1)])
def test_nic_pacing_two_ranks(built, nodes, local):
    res = _run(nodes, local)
    for rank, rc, elapsed, err in res:
        assert rc == 0, err
        ideal = 10 * PIECE / 1e9  # wire time per rank
        if local == 2:   # same node: the two ranks share one NIC -> serialised
            assert elapsed >= 2 * ideal * 0.98
        else:            # two nodes: independent NICs -> parallel
            assert ideal * 0.98 <= elapsed < 1.5 * ideal
