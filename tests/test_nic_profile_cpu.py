"""tools/nic_profile.py binning (CPU): wire intervals split pro rata over bins,
bytes conserved per kind, phase statistics."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
import nic_profile as NP  # noqa: E402


def _recs(rows):
    r = np.zeros(len(rows), dtype=[("start_ns", np.uint64), ("end_ns", np.uint64), ("bytes", np.uint64),
                                   ("kind", np.int32)])
    for i, (s, e, b, k) in enumerate(rows):
        r[i] = (s, e, b, k)
    return r


def test_series_conserves_bytes_and_splits_pro_rata():
    recs = _recs([(0, 3_000_000, 3_000_000, 0), (3_500_000, 4_500_000, 1_000, 2), (5_000_000, 5_000_000, 7, 1)])
    ser = NP.series(recs, 0, 1_000_000, 6)
    assert np.allclose(ser["fwd_ag"][:3], 1_000_000) and ser["fwd_ag"][3:].sum() == 0
    assert np.isclose(ser["rs"][3], 500) and np.isclose(ser["rs"][4], 500)
    assert ser["bwd_ag"][5] == 7
    for k, name in NP.KINDS.items():
        assert np.isclose(ser[name].sum(), recs["bytes"][recs["kind"] == k].sum())


def test_summarise_phases():
    recs = _recs([(0, 2_000_000, 4_000_000, 0), (2_000_000, 4_000_000, 4_000_000, 2)])
    s = NP.summarise(recs, 10.0, 1.0)
    assert s["bytes"]["fwd_ag"] == 4_000_000 and s["bytes"]["rs"] == 4_000_000
    assert np.isclose(s["forward_phase"]["peak_gbs"], 2.0) and np.isclose(s["backward_phase"]["active_ms"], 2.0)
    assert np.isclose(s["nic_busy_frac_of_step"], 0.4)
    assert NP.summarise(recs[:0], 5.0, 1.0)["nic_busy_frac_of_step"] == 0.0
