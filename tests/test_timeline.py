"""Overlap timeline: the schedule simulation against the reference's own results
(tests/golden/make_timeline_golden.py: scheduling.py:91-111 on its example timeline and seeded random
DAGs), the document round trip, the error cases of tests/test_scheduling.py, and (GPU) the measured
DAP-block timeline: segments cover the forward, every collective is placed, async <= sync."""

import json
import os

import pytest

from paper_2203_00854_b200 import timeline as TL

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "timeline_cases.json")))["cases"]


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_schedule_matches_reference(c):
    ev = TL.events_from_json(c["timeline"])
    assert TL.events_to_json(ev) == c["timeline"]
    assert TL.simulate_schedule(ev, "sync").to_json() == c["sync"]
    assert TL.simulate_schedule(ev, "async").to_json() == c["async"]
    assert TL.simulate_schedule(ev, "async").makespan <= TL.simulate_schedule(ev, "sync").makespan


def test_schedule_errors():
    E = TL.TimelineEvent
    with pytest.raises(TL.ScheduleError):
        E("a", -1.0)
    with pytest.raises(TL.ScheduleError):
        E("a", 1.0, "disk")
    with pytest.raises(TL.ScheduleError):
        TL.simulate_schedule([E("a", 1.0, deps=("b",))], "sync")
    with pytest.raises(TL.ScheduleError):
        TL.simulate_schedule([E("a", 1.0, deps=("b",)), E("b", 1.0, deps=("a",))], "async")
    with pytest.raises(TL.ScheduleError):
        TL.simulate_schedule([E("a", 1.0), E("a", 2.0)], "sync")
    with pytest.raises(TL.ScheduleError):
        TL.simulate_schedule([], "fast")
    with pytest.raises(TL.ScheduleError):
        TL.events_from_json("{")


@pytest.mark.gpu
def test_measured_dap_timeline():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2203_00854_b200.config import EvoConfig
    cfg = EvoConfig(32, 64, 64, 64, 2, 2, 32)
    events, info = TL.measure_dap_forward(cfg, 4)
    rep = TL.overlap_report(events, info)
    colls = info["collectives"]
    # 6 all-to-all + 3 projection gathers + 1 bias gather (dap_block.py:58-151)
    assert sorted(c["category"] for c in colls).count("all_to_all") == 6
    assert sorted(c["category"] for c in colls).count("all_gather") == 3
    assert sorted(c["category"] for c in colls).count("bias_gather") == 1
    assert all(c["consumed_by"] is not None for c in colls)
    assert rep["compute_ms"] > 0 and rep["async_makespan_ms"] <= rep["sync_makespan_ms"] + 1e-9
    assert 0.0 <= rep["exposed_comm_fraction"] <= 1.0 + 1e-9
