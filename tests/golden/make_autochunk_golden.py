"""Golden fixtures for the GPU AutoChunk executor, made by importing the REFERENCE (build container
only: /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_autochunk_golden.py

autochunk_cases.json: per case, the reference graph JSON (evoplan-graph-v1, graph.py:465-521, consts
included), one or more execution plans (evoplan-execplan-v1, plans.py:172-227: from autochunk_search,
chunker.py:196-233, or hand-built regions), the reference's memory estimate for each plan at element
sizes 4 and 8 (memory.py:69-144 - equal to what the reference's tracked executor measures), and the
input/output arrays of the reference execution (graph.py:418-460) as base64 float64.
Cases: the worked outer/mean example of tests/test_chunking.py:57-91 (sizes 4, 2, 3) and the traced
Evoformer block (trace.py:186) of tests/test_chunking.py:42-54 at seed 0 under budgets 0.6 and 0.52 of
the unchunked peak.
"""
from __future__ import annotations

import base64
import json
import os

import numpy as np

from evoplan.chunker import autochunk_search
from evoplan.evoformer import EvoConfig, init_block_params
from evoplan.graph import GraphBuilder, execute, graph_to_json
from evoplan.memory import estimate_memory
from evoplan.plans import ChunkPlan, plan_to_json, solve_chunk_dims
from evoplan.trace import trace_evoformer

HERE = os.path.dirname(os.path.abspath(__file__))


def b64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return {"shape": list(a.shape), "data": base64.b64encode(a.tobytes()).decode("ascii")}


def case(name, graph, plans, inputs):
    want = execute(graph, inputs)
    return {
        "name": name,
        "graph": graph_to_json(graph),
        "plans": [{"plan": plan_to_json(graph, p),
                   "peak_elem4": estimate_memory(graph, p, 4).peak_bytes,
                   "peak_elem8": estimate_memory(graph, p, 8).peak_bytes} for p in plans],
        "unchunked_peak_elem4": estimate_memory(graph, None, 4).peak_bytes,
        "inputs": {str(k): b64(v) for k, v in inputs.items()},
        "outputs": {str(k): b64(want[k]) for k in graph.outputs},
    }


def main():
    cases = []
    b = GraphBuilder()
    x = b.input((4, 8, 8))
    y = b.input((4, 8, 8))
    o = b.add_node("outer", [x, y])
    m = b.add_node("mean", [o], {"axis": 0})
    g = b.build([m])
    region = solve_chunk_dims(g, o, m, seed_node=m, seed_dim=0)
    plans = []
    for size in (4, 2, 3):
        p = ChunkPlan()
        p.add(region, size)
        plans.append(p)
    rng = np.random.default_rng(0)
    cases.append(case("outer_mean", g, plans, {x: rng.normal(size=(4, 8, 8)), y: rng.normal(size=(4, 8, 8))}))

    cfg = EvoConfig(n_seq=8, n_res=16)
    g = trace_evoformer(cfg, init_block_params(cfg, 0))
    rng = np.random.default_rng(0)
    inputs = {g.runtime_inputs[0]: rng.normal(size=(cfg.n_seq, cfg.n_res, cfg.h_msa)),
              g.runtime_inputs[1]: rng.normal(size=(cfg.n_res, cfg.n_res, cfg.h_pair))}
    base = estimate_memory(g).peak_bytes
    plans = [ChunkPlan()] + [autochunk_search(g, int(base * f)) for f in (0.6, 0.52)]
    cases.append(case("evoformer_block_8x16", g, plans, inputs))
    path = os.path.join(HERE, "autochunk_cases.json")
    with open(path, "w") as f:
        json.dump({"schema": "evo-autochunk-golden-v1", "cases": cases}, f, sort_keys=True)
    print(path, os.path.getsize(path), "bytes;", [(c["name"], [p["peak_elem4"] for p in c["plans"]]) for c in cases])


if __name__ == "__main__":
    main()
