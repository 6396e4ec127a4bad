"""Golden schedules made by the REFERENCE (build container only):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_timeline_golden.py
timeline_cases.json: the reference's example timeline (data/example_timeline.json) and 5 seeded random
DAGs of 25 events, each with the reference's sync / async ScheduleResult JSON (scheduling.py:91-111)."""
import json
import os
from importlib import resources

import numpy as np

from evoplan.scheduling import TimelineEvent, events_to_json, simulate_schedule

HERE = os.path.dirname(os.path.abspath(__file__))
cases = []
example = resources.files("evoplan").joinpath("data/example_timeline.json").read_text()
from evoplan.scheduling import events_from_json  # noqa: E402
sets = [("example", events_from_json(example))]
for seed in range(5):
    rng = np.random.default_rng(seed)
    ev = []
    for i in range(25):
        deps = tuple(f"e{j}" for j in range(i) if rng.random() < 0.15)
        ev.append(TimelineEvent(f"e{i}", float(np.round(rng.uniform(0, 10), 3)),
                                "comm" if rng.random() < 0.4 else "compute", deps))
    sets.append((f"random_{seed}", ev))
for name, ev in sets:
    cases.append({"name": name, "timeline": events_to_json(ev),
                  "sync": simulate_schedule(ev, "sync").to_json(), "async": simulate_schedule(ev, "async").to_json()})
with open(os.path.join(HERE, "timeline_cases.json"), "w") as f:
    json.dump({"cases": cases}, f, sort_keys=True)
print(len(cases), "cases")
