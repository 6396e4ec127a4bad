"""AutoChunk plan executor on the GPU and the graph / plan JSON interop it reads
(8(f)#3).

The reference plans chunked execution on its graph IR: ``trace_evoformer`` (trace.py:186) lowers a
block to nodes, ``autochunk_search`` (chunker.py:196-233) picks chunk regions under a peak-memory
budget, ``plan_codegen`` (plans.py:172-213) serialises them as an ``evoplan-execplan-v1`` document, and
``execute_chunked`` (chunk_exec.py:76-130) runs the graph region by region in numpy.  This module is
the drop-in executor for those documents on the B200: the planner stays the reference's (its JSON is
the interface), every node runs on the device - LayerNorm and the fused bias/mask softmax on the
libevo kernels, the triangle contraction on the tcgen05 batched GEMM in bf16, the dense products on
cuBLAS - and a region is re-executed slice by slice through views of device buffers.

Byte accounting follows the reference's tracked-execution protocol (engine.Allocator,
chunk_exec.py:1-8, memory.py:69-144): a buffer is counted when a node's result (or an input) is
materialised and released after its last consumer; region outputs are allocated whole on region
entry and filled through slice views; in-region intermediates are slice sized; region inputs are read
through views.  With it, ``ByteTracker.peak_bytes`` equals the reference's ``estimate_memory`` for the
same graph, plan and element size, and ``execute_chunked(..., measure_device=True)`` also reports the
device allocator's high-water mark over the run (the bytes that actually sat in HBM).
"""

from __future__ import annotations

import base64
import json
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .errors import DimensionError

GRAPH_SCHEMA = "evoplan-graph-v1"   # graph.py:463
PLAN_SCHEMA = "evoplan-execplan-v1"  # plans.py:169

OP_KINDS = ("input", "linear", "add", "mul", "sigmoid", "relu", "layernorm", "softmax", "fused_softmax", "mean",
            "permute", "concat", "slice", "matmul", "outer", "contract", "fused_elementwise")


class GraphFormatError(ValueError):
    """Malformed graph / plan document (the reference's errors.GraphFormatError)."""


class PlanError(ValueError):
    """Plan inconsistent with the graph (the reference's errors.PlanError)."""


@dataclass
class Node:
    id: int
    op: str
    inputs: list
    attrs: dict
    shape: tuple
    name: str = ""
    dim_flow: list | None = None  # as serialised by the reference (kept for byte-identical round trips)


@dataclass
class Graph:
    nodes: list
    runtime_inputs: list
    consts: dict                     # node id -> float64 ndarray
    outputs: list
    consumers: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.consumers = {n.id: [] for n in self.nodes}
        for n in self.nodes:
            for i in n.inputs:
                self.consumers[i].append(n.id)

    @property
    def graph_inputs(self):
        return self.runtime_inputs + sorted(self.consts)

    def last_consumer(self):
        return {i: c[-1] for i, c in self.consumers.items() if c}

    def validate(self):
        for pos, n in enumerate(self.nodes):
            if n.id != pos:
                raise GraphFormatError(f"node id {n.id} out of order at {pos}")
            if any(i >= n.id for i in n.inputs):
                raise GraphFormatError(f"node {n.id} has a forward reference")
            if n.op not in OP_KINDS:
                raise GraphFormatError(f"node {n.id}: unknown op {n.op!r}")
        if any(not 0 <= i < len(self.nodes) for i in self.outputs):
            raise GraphFormatError("output id out of range")


def graph_from_json(text: str) -> Graph:
    """Parse an ``evoplan-graph-v1`` document (graph.py:465-521), consts included."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"malformed graph JSON at line {exc.lineno} column {exc.colno}: {exc.msg}") from exc
    if doc.get("schema") != GRAPH_SCHEMA:
        raise GraphFormatError(f"unexpected schema {doc.get('schema')!r}")
    nodes = [Node(e["id"], e["op"], list(e["inputs"]), dict(e["attrs"]), tuple(e["shape"]), e.get("name", ""),
                  e.get("dim_flow")) for e in doc["nodes"]]
    consts = {int(k): np.frombuffer(base64.b64decode(e["data"]), dtype=np.float64).reshape(e["shape"]).copy()
              for k, e in doc.get("consts", {}).items()}
    g = Graph(nodes, list(doc["runtime_inputs"]), consts, list(doc["outputs"]))
    g.validate()
    return g


def graph_to_json(g: Graph, include_consts: bool = True) -> str:
    """Inverse of :func:`graph_from_json`; a parsed reference document is reproduced byte for byte."""
    doc = {
        "schema": GRAPH_SCHEMA,
        "nodes": [{"id": n.id, "op": n.op, "inputs": n.inputs, "attrs": n.attrs, "shape": list(n.shape),
                   "name": n.name, "dim_flow": n.dim_flow} for n in g.nodes],
        "inputs": g.graph_inputs,
        "runtime_inputs": g.runtime_inputs,
        "outputs": g.outputs,
    }
    if include_consts:
        doc["consts"] = {str(i): {"shape": list(v.shape), "data": base64.b64encode(
            np.ascontiguousarray(v, dtype=np.float64).tobytes()).decode("ascii")} for i, v in g.consts.items()}
    return json.dumps(doc, sort_keys=True)


@dataclass
class Region:
    """One chunk region of a plan: nodes start..end re-executed over ``extent`` in slices of ``size``
    (plans.py:30-47 ChunkRegion plus its chunk size)."""
    start: int
    end: int
    chunk_dim: dict      # node id -> chunked output dim (the dimension-flow path)
    input_chunk: dict    # region-input id -> chunked dim
    outputs: list
    extent: int
    size: int

    @property
    def span(self):
        return range(self.start, self.end + 1)


@dataclass
class Plan:
    regions: list
    provenance: list
    n_nodes: int = 0


def plan_from_json(text: str) -> Plan:
    """Parse an ``evoplan-execplan-v1`` document (plans.py:172-227)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"malformed plan JSON at line {exc.lineno} column {exc.colno}: {exc.msg}") from exc
    if doc.get("schema") != PLAN_SCHEMA:
        raise GraphFormatError(f"unexpected plan schema {doc.get('schema')!r}")
    regions = []
    for e in doc["schedule"]:
        if isinstance(e, dict):
            lp = e["loop"]
            regions.append(Region(lp["start"], lp["end"], {int(k): v for k, v in lp["chunk_dim"].items()},
                                  {int(k): v for k, v in lp["slice_specs"].items()},
                                  [int(k) for k in lp["scatter_specs"]], lp["dim_extent"], lp["chunk_size"]))
    regions.sort(key=lambda r: r.start)
    return Plan(regions, list(doc.get("provenance", [])), doc.get("n_nodes", 0))


def plan_to_json(plan: Plan, n_nodes: int) -> str:
    """Serialise a plan as the reference's execution-plan document (plans.py:172-213)."""
    sched, at, nid = [], {r.start: r for r in plan.regions}, 0
    while nid < n_nodes:
        r = at.get(nid)
        if r is None:
            sched.append(nid)
            nid += 1
            continue
        sched.append({"loop": {"start": r.start, "end": r.end, "dim_extent": r.extent, "chunk_size": r.size,
                               "iterations": math.ceil(r.extent / r.size), "nodes": list(r.span),
                               "chunk_dim": {str(k): v for k, v in r.chunk_dim.items()},
                               "slice_specs": {str(k): v for k, v in r.input_chunk.items()},
                               "scatter_specs": {str(k): r.chunk_dim[k] for k in r.outputs}}})
        nid = r.end + 1
    return json.dumps({"schema": PLAN_SCHEMA, "n_nodes": n_nodes, "schedule": sched,
                       "provenance": plan.provenance}, sort_keys=True)


def check_plan(g: Graph, plan: Plan) -> None:
    """Structural checks an executor needs (the reference re-derives legality in plans.py:130-163;
    the plan document comes from its planner): regions ordered, disjoint, in range, every output
    chunked, chunk sizes within the extent, and every chunked dimension of that extent."""
    prev = -1
    for r in plan.regions:
        if not (0 <= r.start <= r.end < len(g.nodes)) or r.start <= prev:
            raise PlanError(f"region [{r.start}, {r.end}] out of range or overlapping")
        prev = r.end
        if not 1 <= r.size <= r.extent:
            raise PlanError(f"chunk size {r.size} invalid for extent {r.extent}")
        for nid, d in list(r.chunk_dim.items()) + list(r.input_chunk.items()):
            if g.nodes[nid].shape[d] != r.extent:
                raise PlanError(f"node {nid} dim {d} has extent {g.nodes[nid].shape[d]} != {r.extent}")
        if any(o not in r.chunk_dim for o in r.outputs):
            raise PlanError(f"region [{r.start}, {r.end}]: an output has no chunk dimension")


class ByteTracker:
    """The reference's byte counter (engine.py:53-97): live/peak bytes and an event log."""

    def __init__(self):
        self.live_bytes = 0
        self.peak_bytes = 0
        self.events = []

    def alloc(self, n):
        self.live_bytes += n
        self.peak_bytes = max(self.peak_bytes, self.live_bytes)
        self.events.append(n)

    def free(self, n):
        self.live_bytes -= n
        self.events.append(-n)

    def replay_peak(self):
        live = self.live_bytes - sum(self.events)
        peak = live
        for d in self.events:
            live += d
            peak = max(peak, live)
        return peak


# ----------------------------------------------------------------------------------- device ops
def _linear(x, w, c):
    lead = x.shape[: x.dim() - c]
    return torch.matmul(x.reshape(tuple(lead) + (-1,)), w)


def _layernorm(x, g, b, eps):
    C = x.shape[-1]
    rows = x.numel() // C
    out, _, _ = ops.layernorm_fwd(x.contiguous().view(rows, C), g.float().contiguous(), b.float().contiguous(),
                                  rows, C, eps=eps, save_stats=False)
    return out.view(x.shape)


def _softmax(x, axis, mask=None, bias=None):
    from .evoformer import fused_softmax_mask_bias
    z = torch.zeros((), device=x.device, dtype=x.dtype)
    return fused_softmax_mask_bias(x, z if mask is None else mask, z if bias is None else bias, axis,
                                   check_finite=False).to(x.dtype)


def _contract(a, b, mode):
    """tri_update einsums (evoformer.py:276, 283): t[i,j,h] = sum_k a[i,k,h] b[j,k,h] (outgoing) or
    a[k,i,h] b[k,j,h] (incoming); one batched tcgen05 GEMM over h in bf16, cuBLAS in fp32."""
    if a.dtype != torch.bfloat16:
        if mode == "outgoing":
            return torch.einsum("ikh,jkh->ijh", a, b)
        return torch.einsum("kih,kjh->ijh", a, b)
    A_ = a.permute(2, 0, 1).contiguous() if mode == "outgoing" else a.permute(2, 1, 0).contiguous()
    B_ = b.permute(2, 0, 1).contiguous() if mode == "outgoing" else b.permute(2, 1, 0).contiguous()
    H, M, K = A_.shape
    N = B_.shape[1]
    t = torch.empty(H, M, N, device=a.device, dtype=a.dtype)
    ops.bgemm(ops.Mat(A_, lo=(K, 1), batch_stride=M * K), ops.Mat(B_, lo=(K, 1), batch_stride=N * K),
              ops.Mat(t, lo=(N, 1), batch_stride=M * N), H, M, N, K)
    return t.permute(1, 2, 0).contiguous()


def _fused_elementwise(node, args):
    acc = args[node.attrs["head"]]
    for st in node.attrs["steps"]:
        op = st["op"]
        if op == "sigmoid":
            acc = torch.sigmoid(acc)
        elif op == "relu":
            acc = torch.relu(acc)
        elif op == "add":
            o = args[st["operand"]]
            acc = o + acc if st.get("swap") is True else acc + o
        elif op == "mul":
            acc = acc * args[st["operand"]]
        else:
            raise DimensionError(f"bad fused step op {op!r}")
    return acc.expand(node.shape).contiguous() if tuple(acc.shape) != tuple(node.shape) else acc


def apply_node(node: Node, args):
    """One graph node on device tensors (graph.py:342-389 semantics)."""
    op, a = node.op, node.attrs
    if op == "linear":
        return _linear(args[0], args[1], a.get("contract_dims", 1))
    if op == "add":
        return args[0] + args[1]
    if op == "mul":
        return args[0] * args[1]
    if op == "sigmoid":
        return torch.sigmoid(args[0])
    if op == "relu":
        return torch.relu(args[0])
    if op == "layernorm":
        return _layernorm(args[0], args[1], args[2], a.get("eps", 1e-5))
    if op == "softmax":
        return _softmax(args[0], a["axis"])
    if op == "fused_softmax":
        return _softmax(args[0], a["axis"], args[1], args[2])
    if op == "mean":
        return args[0].mean(dim=a["axis"])
    if op == "permute":
        return args[0].permute(*a["perm"]).contiguous()
    if op == "concat":
        return torch.cat(list(args), dim=-1)
    if op == "slice":
        return args[0].narrow(a["axis"], a["start"], a["stop"] - a["start"]).contiguous()
    if op == "matmul":
        return torch.matmul(args[0], args[1])
    if op == "outer":
        return torch.einsum("sip,sjq->sijpq", args[0], args[1])
    if op == "contract":
        return _contract(args[0], args[1], a["mode"])
    if op == "fused_elementwise":
        return _fused_elementwise(node, args)
    raise DimensionError(f"cannot execute op kind {op!r}")


# ----------------------------------------------------------------------------------- executor
class _Exec:
    def __init__(self, g: Graph, inputs, device, dtype, tracker):
        self.g, self.device, self.dtype = g, device, dtype
        self.tr = tracker or ByteTracker()
        self.es = torch.tensor([], dtype=dtype).element_size()
        self.inputs = inputs
        self.vals = {}       # node id -> device tensor currently held
        self.last = g.last_consumer()
        self.outs = set(g.outputs)

    def nbytes(self, shape):
        return int(np.prod(shape, dtype=np.int64)) * self.es

    def hold(self, nid, t, shape=None):
        self.vals[nid] = t
        self.tr.alloc(self.nbytes(self.g.nodes[nid].shape if shape is None else shape))

    def drop(self, nid, shape=None):
        del self.vals[nid]
        self.tr.free(self.nbytes(self.g.nodes[nid].shape if shape is None else shape))

    def source(self, nid):
        src = self.g.consts.get(nid)
        if src is None:
            src = self.inputs.get(nid)
        if src is None:
            raise DimensionError(f"missing runtime input {nid}")
        if isinstance(src, torch.Tensor):
            return src.to(device=self.device, dtype=self.dtype)
        return torch.tensor(np.asarray(src, dtype=np.float64)).to(device=self.device, dtype=self.dtype)

    def plain(self, node):
        if node.op == "input":
            self.hold(node.id, self.source(node.id))
        else:
            self.hold(node.id, apply_node(node, [self.vals[i] for i in node.inputs]))
        for i in node.inputs:  # the footprint after the node runs; then its last-use inputs go
            if self.last.get(i) == node.id and i not in self.outs:
                self.drop(i)

    def region(self, r: Region):
        g = self.g
        for o in r.outputs:  # whole-size outputs, filled slice by slice
            self.hold(o, torch.empty(g.nodes[o].shape, device=self.device, dtype=self.dtype))
        for sid in r.span:   # pass-through inputs inside the span: materialised on entry
            if g.nodes[sid].op == "input":
                self.hold(sid, self.source(sid))
        span = set(r.span)
        for lo in range(0, r.extent, r.size):
            n = min(r.size, r.extent - lo)
            local = {}       # slice-sized intermediates of this iteration: id -> (tensor, shape)

            def view(i):
                if i in local:
                    return local[i][0]
                if i in r.chunk_dim and r.start <= i <= r.end:
                    return self.vals[i].narrow(r.chunk_dim[i], lo, n)
                if i in r.input_chunk:
                    return self.vals[i].narrow(r.input_chunk[i], lo, n)
                return self.vals[i]

            for sid in r.span:
                node = g.nodes[sid]
                if node.op == "input":
                    continue
                y = apply_node(node, [view(i) for i in node.inputs])
                if sid in r.outputs:
                    self.vals[sid].narrow(r.chunk_dim[sid], lo, n).copy_(y)
                else:
                    shp = list(node.shape)
                    if sid in r.chunk_dim:
                        shp[r.chunk_dim[sid]] = n
                    local[sid] = (y, tuple(shp))
                    self.tr.alloc(self.nbytes(shp))
                for i in node.inputs:
                    if i in local and self.last.get(i) == sid:
                        self.tr.free(self.nbytes(local.pop(i)[1]))
            for i in list(local):
                self.tr.free(self.nbytes(local.pop(i)[1]))
        for buf in list(self.vals):  # buffers whose last reader was inside the region
            lc = self.last.get(buf)
            if lc is not None and lc in span and buf not in self.outs and buf not in r.outputs and \
                    (buf not in span or g.nodes[buf].op == "input"):
                self.drop(buf)

    def run(self, plan: Plan | None):
        at = {} if plan is None else {r.start: r for r in plan.regions}
        nid = 0
        while nid < len(self.g.nodes):
            r = at.get(nid)
            if r is not None:
                self.region(r)
                nid = r.end + 1
            else:
                self.plain(self.g.nodes[nid])
                nid += 1
        return {i: self.vals[i] for i in self.g.outputs}


def execute_chunked(g: Graph, plan: Plan | None, inputs: dict, *, device="cuda", dtype=torch.float32,
                    tracker: ByteTracker | None = None, measure_device: bool = False):
    """Run ``g`` on the device under ``plan`` (None = plain node order, graph.py:418-460); returns
    {output id: device tensor}.  ``tracker`` receives the reference-protocol byte counts; with
    ``measure_device`` the return value is (outputs, device high-water bytes above the start)."""
    if plan is not None:
        check_plan(g, plan)
    missing = [i for i in g.runtime_inputs if i not in inputs]
    if missing:
        raise DimensionError(f"missing runtime inputs: {missing}")
    if measure_device:
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
    out = _Exec(g, inputs, device, dtype, tracker).run(plan)
    if measure_device:
        torch.cuda.synchronize()
        return out, torch.cuda.max_memory_allocated() - base
    return out
