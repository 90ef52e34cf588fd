"""NUMA placement of the pinned host tiers,
host side only: sysfs cpulist parsing, the raw preferred-node mbind + first
touch, and that the engine's temporary thread pin is undone exactly (ADVICE r1:
the caller's thread must not stay pinned).  No GPU needed."""
import ctypes as C
import os

import pytest


@pytest.fixture(scope="module")
def lib(built):
    return built


@pytest.mark.parametrize("text,want", [("0-3,8,10-11", [0, 1, 2, 3, 8, 10, 11]), ("5", [5]), ("", []),
                                       ("0-1,\n", [0, 1]), ("bad", [])])
def test_parse_cpulist(lib, text, want):
    out = (C.c_int32 * 64)()
    n = C.c_int32()
    assert lib.fcdp_numa_parse_cpulist(text.encode(), out, 64, C.byref(n)) == 0
    assert list(out)[:n.value] == want


def test_numa_node0_placement_and_affinity_restore(lib):
    vals = [C.c_int32() for _ in range(5)]
    assert lib.fcdp_numa_selftest(0, 8 << 20, *[C.byref(v) for v in vals]) == 0
    num_nodes, cpus, prefer_ok, page_node, restored = (v.value for v in vals)
    assert num_nodes >= 1
    if os.path.exists("/sys/devices/system/node/node0/cpulist"):
        assert cpus >= 1
    # mbind(MPOL_PREFERRED, node 0) is accepted wherever node 0 has memory; the
    # first-touched page then lives on node 0 (get_mempolicy MPOL_F_NODE|ADDR)
    if prefer_ok:
        assert page_node in (0, -1)
    assert restored == 1
