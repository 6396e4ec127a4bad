"""Benchmark: 48-block Evoformer forward+backward at the AlphaFold training shape
(BASELINE.json configs[1]: N_seq=128, N_res=256, c_m=256, c_z=128, 8/4 heads,
hidden_proj=32, bf16) on N GPUs of one node (N>1: Dynamic Axial Parallelism,
strong scaling - the same 48-block problem sharded over N ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  metric = milliseconds per Evoformer block
(forward + backward, all weight gradients; lower is better) = step time / 48.
Timed region: K steps of the whole 48-block fwd+bwd with inputs resident in
HBM, bracketed by barrier + synchronize, CUDA events, max over ranks.  The
per-step working set (~45 GB of activations) is far larger than L2 (126 MB),
so no separate L2 flush is needed.

``--impl reference`` times the CPU restatement of the reference algorithm
(oracle/evoformer_torch.py, float64 autograd - the reference itself has no
backward) on the host's cores, one training-shape block fwd+bwd per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Evoformer block fwd+bwd ms (Nres256/Nseq128)"
UNIT = "ms/block"
N_BLOCKS = 48
TRAIN_DIMS = (128, 256, 256, 128, 8, 4, 32)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--blocks", type=int, default=N_BLOCKS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="train", choices=["train", "longseq"],
                    help="train: 48-block fwd+bwd at the training shape (BASELINE configs[1], default); "
                         "longseq: 48-block forward (inference) at --n-res (configs[3])")
    ap.add_argument("--n-res", type=int, default=1024)
    ap.add_argument("--graph", type=int, default=1,
                    help="1 GPU: replay the whole step as one captured CUDA graph in the timed region")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clock / throttle sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_fwd_bwd_sample(reps: int = 1):
    """one training-shape block fwd+bwd with the float64 torch restatement of the reference
    (oracle/evoformer_torch.py) on all host cores; returns (ms per block, cores, sample)."""
    import numpy as np
    import torch

    from oracle import evoformer_torch as T
    from paper_2203_00854_b200.config import EvoConfig, init_block_params, synthetic_inputs

    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    torch.set_num_threads(cores)
    cfg = EvoConfig(*TRAIN_DIMS)
    p = init_block_params(cfg, 0)
    m, z = synthetic_inputs(cfg, 0)
    rng = np.random.default_rng(1)
    gm, gz = rng.normal(size=m.shape), rng.normal(size=z.shape)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        T.block_grads(m, z, p, cfg, gm, gz, dtype=torch.float64)
        times.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(times), cores, ("1 Evoformer block fwd+bwd at the training shape "
                                             "(N_s=128, N_r=256, 256/128, heads 8/4, p=32), float64 torch "
                                             "autograd restatement of evoformer.py (oracle/evoformer_torch.py)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_fwd_bwd_sample(1)
    ms = [cpu_fwd_bwd_sample(1) for _ in range(args.steps)]
    val = statistics.median(v for v, _, _ in ms)
    cores, sample = ms[0][1], ms[0][2]
    line = {"metric": METRIC, "value": round(val, 3), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(val, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "evoformer_block_fwd_bwd_training_shape", "n_seq": 128, "n_res": 256,
                       "c_m": 256, "c_z": 128, "heads_msa": 8, "heads_pair": 4, "hidden_proj": 32,
                       "blocks_per_step": 1},
            "cpu_baseline": {"value": round(val, 3), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(val, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2203_00854_b200 import _lib
    from paper_2203_00854_b200.config import EvoConfig, synthetic_inputs
    from paper_2203_00854_b200.evoformer import EvoformerStack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL over NVLink; EVO_DIST_BACKEND=gloo only for functional checks with ranks sharing a GPU
        backend = os.environ.get("EVO_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _lib.load()
    longseq = args.workload == "longseq"
    cfg = EvoConfig(*TRAIN_DIMS) if not longseq else EvoConfig(128, args.n_res, 256, 128, 8, 4, 32)
    nb = args.blocks

    # ------------------------------------------------------------------ workload
    m64, z64 = synthetic_inputs(cfg, 0)
    rng = np.random.default_rng(1)
    gm64, gz64 = (rng.normal(size=m64.shape), rng.normal(size=z64.shape)) if not longseq else (None, None)
    if world == 1:
        stack = EvoformerStack(cfg, nb, seed=0, device=dev)
        m = torch.tensor(m64, device=dev).bfloat16()
        z = torch.tensor(z64, device=dev).bfloat16()
        if not longseq:
            gm = torch.tensor(gm64, device=dev).bfloat16()
            gz = torch.tensor(gz64, device=dev).bfloat16()
        parallelism = "single"
    else:
        from paper_2203_00854_b200.dap import DapStack
        stack = DapStack(cfg, nb, seed=0, device=dev)
        m, z = stack.shard_inputs(m64, z64, dev)
        if not longseq:
            gm, gz = stack.shard_inputs(gm64, gz64, dev)
        parallelism = f"dap{world}"


    if longseq:
        def step():
            with torch.no_grad():
                mo, zo, _ = stack.forward(m, z, save=False)
            return zo
    else:
        def step():
            stack.zero_grad()
            loss, dm, dz = stack.forward_backward(m, z, gm, gz)
            return loss

    def barrier():
        if world > 1:
            dist.barrier()

    # ------------------------------------------------------------------ warmup (+ kernel census)
    inst = _lib.Instrument(timed=("evo_gated_attention_fwd", "evo_gated_attention_bwd", "evo_bgemm",
                                  "evo_layernorm_fwd", "evo_softmax_fwd"))
    for i in range(args.warmup):
        if i == args.warmup - 1:
            _lib.INSTRUMENT = inst
        step()
        _lib.INSTRUMENT = None
    torch.cuda.synchronize()
    census = inst.summary()
    dominant = max(census, key=lambda k: census[k]["total_ms"]) if census else None

    # ------------------------------------------------------------------ CUDA graph of the step
    # the whole fwd+bwd step as one CUDA graph; under DAP the NCCL collectives (async, waited on
    # the compute stream) are captured with it.  A backend that cannot be captured (gloo) falls
    # back to eager launches and says so in the JSON line.
    use_graph = bool(args.graph) and not longseq
    graph_note = None
    if use_graph:
        from paper_2203_00854_b200.evoformer import GraphedStep
        try:
            gstep = GraphedStep(stack, m, z, gm, gz)
        except Exception as exc:  # noqa: BLE001 - reported, eager fallback
            use_graph, graph_note = False, f"capture failed, eager: {type(exc).__name__}: {str(exc)[:120]}"
            torch.cuda.synchronize()
    if use_graph:
        launches_eager = inst.launches()
        run_step = gstep.replay
    else:
        run_step = step

    # ------------------------------------------------------------------ timed region
    timed = _lib.Instrument(timed=(dominant,) if dominant and not use_graph else ())
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.INSTRUMENT = timed
    e0.record(st)
    for _ in range(args.steps):
        loss = run_step()
    e1.record(st)
    _lib.INSTRUMENT = None
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    total_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    if use_graph:
        # the graph holds exactly the kernels of one eager step; per-launch durations of the
        # dominant entry point are taken with CUDA events on one eager step right after
        launches_per_step = launches_eager
        post = _lib.Instrument(timed=(dominant,) if dominant else ())
        _lib.INSTRUMENT = post
        step()
        _lib.INSTRUMENT = None
        torch.cuda.synchronize()
        dom = post.summary().get(dominant, None)
        if dom:  # one step's launches -> per-step share as if over the K timed steps
            dom = dict(dom, step_ms=dom["total_ms"])
    else:
        launches_per_step = timed.launches() / args.steps
        dom = timed.summary().get(dominant, None)

    # ------------------------------------------------------------------ e2e via the public API
    e2e = None
    if not args.no_e2e and not longseq:
        hm = torch.tensor(m64, dtype=torch.float32).pin_memory() if world == 1 else None
        if world == 1:
            hz = torch.tensor(z64, dtype=torch.float32).pin_memory()
            hgm = torch.tensor(gm64, dtype=torch.float32).pin_memory()
            hgz = torch.tensor(gz64, dtype=torch.float32).pin_memory()
            hloss = torch.empty(1, dtype=torch.float32).pin_memory()
            host = (hm, hz, hgm, hgz)
            bi = sum(t.numel() * 4 for t in host)
            # input pipeline (what a training loop's loader does): step k+1's pinned host
            # inputs are copied on a copy stream while step k runs; every step's copy and the
            # first one (not overlapped) are inside the timed region
            cs = torch.cuda.Stream()
            stage = [[torch.empty(t.shape, device=dev) for t in host] for _ in range(2)]
            landed = [torch.cuda.Event(), torch.cuda.Event()]
            freed = [torch.cuda.Event(), torch.cuda.Event()]

            def h2d(k):
                with torch.cuda.stream(cs):
                    if k >= 2:
                        cs.wait_event(freed[k % 2])  # step k-2 has converted this staging pair
                    for d_, h_ in zip(stage[k % 2], host):
                        d_.copy_(h_, non_blocking=True)
                    landed[k % 2].record(cs)

            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            h2d(0)
            for k in range(args.steps):
                st.wait_event(landed[k % 2])
                dm_, dz_, dgm, dgz = (t.bfloat16() for t in stage[k % 2])
                freed[k % 2].record(st)
                if k + 1 < args.steps:
                    h2d(k + 1)
                if use_graph:   # GraphedStep: static inputs refreshed from this step's host data
                    gstep.set_inputs(dm_, dz_, dgm, dgz)
                    loss = gstep.replay()
                else:
                    stack.zero_grad()
                    loss, _, _ = stack.forward_backward(dm_, dz_, dgm, dgz)
                hloss.copy_(loss.view(1), non_blocking=True)
                torch.cuda.current_stream().synchronize()
            b.record(st)
            torch.cuda.synchronize()
            e2e_step = a.elapsed_time(b) / args.steps
            e2e = {"value": round(e2e_step / nb, 4), "unit": UNIT, "h2d_bytes_per_step": bi,
                   "d2h_bytes_per_step": 4, "ms_per_step": round(e2e_step, 3),
                   "path": ("GraphedStep(EvoformerStack) replay" if use_graph else "EvoformerStack.forward_backward")
                   + ": pinned fp32 host inputs copied in every step (next step's copy on a copy stream under "
                   "this step's compute), loss read back and synchronised every step"}
        else:
            e2e = stack.e2e(m64, z64, gm64, gz64, args.steps, nb)

    # ------------------------------------------------------------------ roofline + CPU baseline
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm = peaks.get("hbm_gbs", 6650.0)
    tfl = peaks.get("bf16_tflops", 1590.0)
    peak_src = "measured" if peaks else "fallback"
    roof = None
    if dom and dom["avg_ms"] > 0:
        flops, byts = dom["flops"] / dom["launches"], dom["bytes"] / dom["launches"]
        ai = flops / max(byts, 1)
        ridge = tfl * 1e12 / (hbm * 1e9)
        sec = dom["avg_ms"] / 1e3
        if flops > 0 and ai >= ridge:
            ach = flops / sec / 1e12
            roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": tfl, "unit": "TFLOP/s",
                    "frac": round(ach / tfl, 4)}
        else:
            ach = byts / sec / 1e9
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4)}
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
        if os.path.exists(tpath):  # ncu --set full measurement of the same entry point (scripts/make_traffic.py)
            tdoc = json.load(open(tpath)).get(dominant)
            if tdoc:
                traffic = round(tdoc["traffic_bytes_per_launch"])
        roof.update({"traffic": traffic, "traffic_unit": "bytes/launch (DRAM read+write, ncu)",
                     "kernel": dominant, "peak_source": peak_src,
                     "launches_per_step": dom["launches"] if use_graph else dom["launches"] / args.steps,
                     "avg_launch_ms": round(dom["avg_ms"], 4),
                     "share_of_step": round((dom["step_ms"] / ms_step) if use_graph else (dom["total_ms"] / total_ms), 4),
                     "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": byts,
                     "arithmetic_intensity": round(ai, 1),
                     "timed_on": "eager step after the graph-replayed timed region" if use_graph
                     else "inside the timed region"})
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not longseq:
        v, cores, sample = cpu_fwd_bwd_sample(1)
        cpu = {"value": round(v, 1), "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        if longseq:
            metric = f"long-seq inference ms (Nres{cfg.n_res}/Nseq{cfg.n_seq}, {nb}-block forward)"
            value, unit = round(ms_step, 3), "ms/stack-forward"
            workload = f"evoformer_stack_forward_longseq_nres{cfg.n_res}"
            step_desc = f"{nb}-block forward, no grad (inference)"
        else:
            metric, value, unit = METRIC, round(ms_step / nb, 4), UNIT
            workload = "evoformer_stack_fwd_bwd_training_shape"
            step_desc = f"{nb}-block forward + backward incl. all weight gradients; no optimizer"
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference draw order: default_rng(0) m then z; init_block_params(cfg, i))",
            "config": {"workload": workload, "blocks": nb, "n_seq": cfg.n_seq, "n_res": cfg.n_res, "c_m": 256,
                       "c_z": 128, "heads_msa": 8, "heads_pair": 4, "hidden_proj": 32, "parallelism": parallelism,
                       "l2": "per-step working set >> 126 MB L2 (no flush needed)", "step": step_desc},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches_per_step * args.steps),
            "gpu_launches_per_step": launches_per_step, "clocks": clk, "cuda_graph": use_graph,
            **({"cuda_graph_note": graph_note} if graph_note else {}),
            "kernel_census_ms_per_step": {k: round(v["total_ms"], 3) for k, v in census.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
