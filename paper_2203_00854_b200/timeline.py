"""Measured compute/communication overlap timeline of the DAP block.

The reference simulates a comm/compute timeline from hand-written event durations
(scheduling.py:91-111, data/example_timeline.json): "sync" serialises every event on one queue,
"async" gives compute and comm their own queues so a collective hides under independent compute.
Here the durations come from the GPU: ``measure_dap_forward`` runs the real DAP block forward
(dap.dap_block_fwd) for one rank's shards with a timing communicator that cuts the compute stream
into segments at every collective (CUDA events on the launching stream), and records which segment
issues each collective and which one first consumes its result (the DAO structure of dap.py: the
bias and projection gathers and the final MSA switch are asynchronous).  Collective durations are
measured when a multi-rank NCCL group is live, otherwise modelled from the byte ledger
(``bytes_per_device / bandwidth + latency``, stated in the report).  ``simulate_schedule`` then gives
the sync and async makespans and the exposed-communication fraction.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

STREAMS = ("compute", "comm")
TIMELINE_SCHEMA = "evoplan-timeline-v1"   # scheduling.py:19


class ScheduleError(ValueError):
    """Invalid event set (the reference's errors.ScheduleError)."""


@dataclass(frozen=True)
class TimelineEvent:
    name: str
    duration: float
    stream: str = "compute"
    deps: tuple = ()

    def __post_init__(self):
        if self.duration < 0:
            raise ScheduleError(f"event {self.name!r} has negative duration")
        if self.stream not in STREAMS:
            raise ScheduleError(f"event {self.name!r} has unknown stream {self.stream!r}")
        object.__setattr__(self, "deps", tuple(self.deps))


@dataclass(frozen=True)
class ScheduleResult:
    mode: str
    makespan: float
    timeline: dict = field(default_factory=dict)

    def to_json(self) -> str:
        return json.dumps({"schema": "evoplan-schedule-v1", "mode": self.mode, "makespan": self.makespan,
                           "timeline": {k: list(v) for k, v in self.timeline.items()}}, sort_keys=True)


def _ordered(events):
    """Dependency order, ties broken by input order: passes over the pending events in input order,
    each placing every event whose dependencies are already placed (scheduling.py:51-88)."""
    by = {}
    for e in events:
        if e.name in by:
            raise ScheduleError(f"duplicate event name {e.name!r}")
        by[e.name] = e
    for e in events:
        for d in e.deps:
            if d not in by:
                raise ScheduleError(f"event {e.name!r} depends on unknown {d!r}")
    placed, out, pending = set(), [], list(events)
    while pending:
        rest = []
        for e in pending:  # one pass in input order; an event placed in this pass unlocks later ones
            if all(d in placed for d in e.deps):
                out.append(e)
                placed.add(e.name)
            else:
                rest.append(e)
        if len(rest) == len(pending):
            raise ScheduleError("dependency cycle")
        pending = rest
    return out


def simulate_schedule(events, mode: str) -> ScheduleResult:
    """Start times under the "sync" (one queue) or "async" (a queue per stream) policy."""
    if mode not in ("sync", "async"):
        raise ScheduleError(f"unknown schedule mode {mode!r}")
    end, tl = {}, {}
    free = {s: 0.0 for s in STREAMS}
    serial = 0.0
    for e in _ordered(events):
        ready = max((end[d] for d in e.deps), default=0.0)
        if mode == "sync":
            t0 = max(serial, ready)
            serial = t0 + e.duration
        else:
            t0 = max(free[e.stream], ready)
            free[e.stream] = t0 + e.duration
        end[e.name] = t0 + e.duration
        tl[e.name] = (t0, end[e.name])
    return ScheduleResult(mode, max(end.values(), default=0.0), tl)


def events_to_json(events) -> str:
    return json.dumps({"schema": TIMELINE_SCHEMA, "events": [
        {"name": e.name, "duration": e.duration, "stream": e.stream, "deps": list(e.deps)} for e in events]},
        sort_keys=True)


def events_from_json(text: str):
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ScheduleError(f"malformed timeline JSON at line {exc.lineno}: {exc.msg}") from exc
    if doc.get("schema") != TIMELINE_SCHEMA:
        raise ScheduleError(f"unexpected timeline schema {doc.get('schema')!r}")
    return [TimelineEvent(e["name"], e["duration"], e.get("stream", "compute"), tuple(e.get("deps", ())))
            for e in doc["events"]]


# ----------------------------------------------------------------------------- measurement
class _Waited:
    def __init__(self, comm, idx):
        self.comm, self.idx = comm, idx

    def wait(self):
        self.comm._consumed(self.idx)


class TimingComm:
    """A stand-in DapComm for ONE rank's view of an N-rank mesh on one GPU: collectives return
    buffers of the right shapes without moving data between ranks (the values are not the DAP
    result; only the compute stream's timing and the collective sizes are read).  Every collective
    closes the current compute segment with a CUDA event and opens the next one."""

    def __init__(self, N: int):
        import torch
        self.torch = torch
        self.N, self.rank, self.overlap, self.ledger = N, 0, True, None
        self.marks = [self._ev()]
        self.colls = []          # (category, bytes per device, issuing segment, consuming segment)

    def _ev(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def _issue(self, category, per_dev_bytes):
        self.marks.append(self._ev())
        seg = len(self.marks) - 2    # the segment that just ended issued it
        self.colls.append([category, per_dev_bytes, seg, None])
        return len(self.colls) - 1

    def _consumed(self, idx):
        if self.colls[idx][3] is None:
            self.marks.append(self._ev())
            self.colls[idx][3] = len(self.marks) - 2 + 1   # the segment starting now reads it

    def _sync_after(self, idx):
        self.marks.append(self._ev())
        self.colls[idx][3] = len(self.marks) - 2 + 1

    def all_gather(self, t, category="all_gather", async_op=False):
        t = t.contiguous()
        idx = self._issue(category, t.numel() * t.element_size() * (self.N - 1))
        out = t.unsqueeze(0).expand((self.N,) + tuple(t.shape)).contiguous()
        if not async_op:
            self._sync_after(idx)
            return out
        return out, _Waited(self, idx)

    def all_to_all(self, t, category="all_to_all", async_op=False):
        t = t.contiguous()
        idx = self._issue(category, t.numel() * t.element_size() * (self.N - 1) // self.N)
        if not async_op:
            self._sync_after(idx)
            return t
        return t, _Waited(self, idx)

    def gather_fn(self, category="all_gather"):
        def gather(t, async_op=False):
            if not async_op:
                return self.all_gather(t, category)
            out, w = self.all_gather(t, category, async_op=True)

            def finish():
                w.wait()
                return out
            return finish
        return gather

    def segments_ms(self):
        self.torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in zip(self.marks[:-1], self.marks[1:])]


def measure_dap_forward(cfg, N: int, seed: int = 0, warmup: int = 2, link_gbps: float = 900.0,
                        latency_us: float = 10.0):
    """Time one rank's DAP block forward (dap.dap_block_fwd) at mesh size N on the current GPU (device
    time: the launches are queued behind a spin kernel before the first mark) and
    build the timeline: compute segments (measured, ms) and collectives (modelled at ``link_gbps``
    GB/s per device plus ``latency_us``).  Returns (events, info)."""
    import numpy as np
    import torch

    from . import dap
    from .config import init_block_params
    from .params import BlockParams

    S, R = cfg.n_seq, cfg.n_res
    bp = BlockParams(init_block_params(cfg, seed), cfg, device="cuda")
    rng = np.random.default_rng(seed)
    m = torch.tensor(rng.normal(size=(S // N, R, cfg.h_msa)), device="cuda").bfloat16()
    z = torch.tensor(rng.normal(size=(R // N, R, cfg.h_pair)), device="cuda").bfloat16()
    for _ in range(warmup):
        dap.dap_block_fwd(bp, TimingComm(N), m, z, save=False)
    # the device first spins while the host enqueues the whole forward, so the segment times are
    # device execution times, not the host's launch rate
    torch.cuda.synchronize()
    torch.cuda._sleep(int(4e8))
    comm = TimingComm(N)
    dap.dap_block_fwd(bp, comm, m, z, save=False)
    comm.marks.append(comm._ev())
    seg = comm.segments_ms()
    # zero-length segments between back-to-back marks stay as events of ~0 duration
    events = [TimelineEvent(f"compute_{i:02d}", float(d), "compute", (f"compute_{i - 1:02d}",) if i else ())
              for i, d in enumerate(seg)]
    deps_of = {i: list(e.deps) for i, e in enumerate(events)}
    comm_events = []
    for k, (cat, nbytes, issued, consumed) in enumerate(comm.colls):
        name = f"{cat}_{k:02d}"
        dur = nbytes / (link_gbps * 1e9) * 1e3 + latency_us * 1e-3
        comm_events.append(TimelineEvent(name, dur, "comm", (f"compute_{issued:02d}",)))
        if consumed is not None and consumed < len(events):
            deps_of[consumed].append(name)
    events = [TimelineEvent(e.name, e.duration, e.stream, tuple(deps_of[i])) for i, e in enumerate(events)]
    # place each collective right after the segment that issues it
    ordered = []
    for i, e in enumerate(events):
        ordered.append(e)
        ordered.extend(c for c, (_, _, issued, _) in zip(comm_events, comm.colls) if issued == i)
    info = {"n_dev": N, "compute_ms": sum(seg), "comm_model": {"link_GBps": link_gbps, "latency_us": latency_us},
            "collectives": [{"category": c, "bytes_per_device": b, "issued_after": f"compute_{i:02d}",
                             "consumed_by": None if u is None else f"compute_{u:02d}"}
                            for c, b, i, u in comm.colls]}
    return ordered, info


def overlap_report(events, info):
    """sync vs async makespans of the measured event set and the exposed-communication fraction."""
    sync = simulate_schedule(events, "sync")
    asyn = simulate_schedule(events, "async")
    comp = sum(e.duration for e in events if e.stream == "compute")
    comm_t = sum(e.duration for e in events if e.stream == "comm")
    return {**info, "sync_makespan_ms": sync.makespan, "async_makespan_ms": asyn.makespan,
            "comm_ms": comm_t, "exposed_comm_ms": asyn.makespan - comp,
            "exposed_comm_fraction": (asyn.makespan - comp) / max(comm_t, 1e-12),
            "events": json.loads(events_to_json(events))["events"]}
