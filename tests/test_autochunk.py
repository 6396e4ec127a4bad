"""AutoChunk plan executor and graph / plan JSON interop (8(f)#3) against fixtures
made by the reference itself (tests/golden/make_autochunk_golden.py: graph.py:465-521 graph JSON,
plans.py:172-227 plan documents from chunker.py:196-233, memory.py:69-144 peak estimates, graph.py:418
outputs).  Mirrors the reference's tests/test_chunking.py:57-118, 186-260 and test_memory.py:66-88:

* CPU: both documents round-trip byte for byte; the executor's host logic (region slicing, buffer
  liveness) runs with the CPU op stand-ins in float64 and reproduces the reference's outputs and its
  byte accounting exactly (tracked peak == estimate_memory, element sizes 4 and 8);
* GPU (marked): the same plans on the B200 in fp32 (libevo LayerNorm / softmax, cuBLAS products) and
  bf16 (tcgen05 triangle contraction), outputs within the stated tolerance, tracked peak == the
  reference's estimate at element size 4, and the device allocator's high-water mark reduced by the
  plan.
"""

import base64
import json
import os

import numpy as np
import pytest
import torch

from paper_2203_00854_b200 import autochunk as AC

GOLD = os.path.join(os.path.dirname(__file__), "golden", "autochunk_cases.json")
CASES = json.load(open(GOLD))["cases"]


def arr(e):
    return np.frombuffer(base64.b64decode(e["data"]), dtype=np.float64).reshape(e["shape"])


def _case(name):
    return next(c for c in CASES if c["name"] == name)


@pytest.mark.parametrize("name", [c["name"] for c in CASES])
def test_graph_and_plan_json_round_trip(name):
    c = _case(name)
    g = AC.graph_from_json(c["graph"])
    assert AC.graph_to_json(g) == c["graph"]
    for p in c["plans"]:
        plan = AC.plan_from_json(p["plan"])
        assert AC.plan_to_json(plan, len(g.nodes)) == p["plan"]
        AC.check_plan(g, plan)


def test_malformed_documents_rejected():
    with pytest.raises(AC.GraphFormatError):
        AC.graph_from_json("{not json")
    with pytest.raises(AC.GraphFormatError):
        AC.graph_from_json(json.dumps({"schema": "other"}))
    with pytest.raises(AC.GraphFormatError):
        AC.plan_from_json(json.dumps({"schema": "evoplan-graph-v1"}))
    c = _case("outer_mean")
    g = AC.graph_from_json(c["graph"])
    plan = AC.plan_from_json(c["plans"][0]["plan"])
    plan.regions[0].size = plan.regions[0].extent + 1
    with pytest.raises(AC.PlanError):
        AC.check_plan(g, plan)


@pytest.mark.parametrize("name", [c["name"] for c in CASES])
def test_executor_host_logic_cpu_float64(name):
    """the executor's region/liveness logic with the CPU op stand-ins (float64 except their fp32
    LayerNorm): reference outputs to 1e-5 and the reference's byte accounting exactly, for every plan
    and both element sizes"""
    import fake_ops
    with fake_ops.installed():
        _host_logic(name)


def _host_logic(name):
    c = _case(name)
    g = AC.graph_from_json(c["graph"])
    inputs = {int(k): arr(v) for k, v in c["inputs"].items()}
    for p in c["plans"]:
        plan = AC.plan_from_json(p["plan"])
        for dtype, key in ((torch.float64, "peak_elem8"), (torch.float32, "peak_elem4")):
            tr = AC.ByteTracker()
            out = AC.execute_chunked(g, plan, inputs, device="cpu", dtype=dtype, tracker=tr)
            assert tr.peak_bytes == p[key] == tr.replay_peak(), (name, key, tr.peak_bytes, p[key])
            if dtype == torch.float64:
                for k, v in c["outputs"].items():
                    assert np.max(np.abs(out[int(k)].numpy() - arr(v))) <= 1e-5, (name, k)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c["name"] for c in CASES])
def test_executor_gpu_fp32(name):
    """fp32 on the B200 (TF32 off): every output within 1e-5 relative of the reference's float64,
    the tracked peak == the reference's estimate at element size 4, and the device high-water mark of
    a budgeted plan below the unchunked one."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    assert not torch.backends.cuda.matmul.allow_tf32
    c = _case(name)
    g = AC.graph_from_json(c["graph"])
    inputs = {int(k): arr(v) for k, v in c["inputs"].items()}
    hw = []
    for p in c["plans"]:
        plan = AC.plan_from_json(p["plan"])
        tr = AC.ByteTracker()
        out, dev_peak = AC.execute_chunked(g, plan, inputs, tracker=tr, measure_device=True)
        hw.append(dev_peak)
        assert tr.peak_bytes == p["peak_elem4"], (tr.peak_bytes, p["peak_elem4"])
        for k, v in c["outputs"].items():
            got = out[int(k)]
            assert got.is_cuda
            assert _rel(got.double().cpu().numpy(), arr(v)) <= 1e-5, (name, k)
    if name == "evoformer_block_8x16":  # plans[0] is the empty plan, 1-2 budgeted ones
        assert min(hw[1:]) < hw[0], hw


@pytest.mark.gpu
def test_executor_gpu_bf16_block():
    """bf16 storage: the triangle contraction runs on the tcgen05 batched GEMM; outputs within the
    bf16 block bound (2e-2 relative)."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    c = _case("evoformer_block_8x16")
    g = AC.graph_from_json(c["graph"])
    inputs = {int(k): arr(v) for k, v in c["inputs"].items()}
    plan = AC.plan_from_json(c["plans"][1]["plan"])
    out = AC.execute_chunked(g, plan, inputs, dtype=torch.bfloat16)
    for k, v in c["outputs"].items():
        assert _rel(out[int(k)].double().cpu().numpy(), arr(v)) <= 2e-2, k
