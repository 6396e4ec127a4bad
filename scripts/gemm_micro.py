"""Per-call timing of the block's evo_bgemm calls (training shape) with the exact Mat views
block.py uses.  python scripts/gemm_micro.py   (EVO_BGEMM_V1=1 selects the non-persistent kernel)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat

S, R, P = 128, 256, 32
dev, BF = "cuda", torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
rnd = lambda *s: torch.randn(*s, device=dev, dtype=BF, generator=g)
ab = rnd(S * R, 2 * P)
o = torch.empty(R, R, P, P, device=dev, dtype=BF)
do = rnd(R * R, P * P)
dab = torch.empty(S * R, 2 * P, device=dev, dtype=BF)
a_cm, b_cm, dt = rnd(P, R * R), rnd(P, R * R), rnd(P, R * R)
t_cm = torch.empty(P, R, R, device=dev, dtype=BF)
rows = R * R

cases = {
    "opm_fwd  M=N=8192 K=128": lambda: ops.bgemm(
        Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0)),
        Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P),
        Mat(o, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P)), 1, R * P, R * P, S, alpha=1.0 / S),
    "opm_bwd_da M=8192 N=128 K=8192": lambda: ops.bgemm(
        Mat(do, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P)),
        Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P), offset=P),
        Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0)), 1, R * P, S, R * P, alpha=1.0 / S),
    "opm_bwd_db M=8192 N=128 K=8192": lambda: ops.bgemm(
        Mat(do, lo=(1, P), split=(P, P), hi=(P * P, R * P * P)),
        Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P)),
        Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P), 1, R * P, S, R * P, alpha=1.0 / S),
    "tri_out_fwd b32 256^3 KK": lambda: ops.bgemm(
        Mat(a_cm, lo=(R, 1), batch_stride=rows), Mat(b_cm, lo=(R, 1), batch_stride=rows),
        Mat(t_cm, lo=(R, 1), batch_stride=rows), P, R, R, R),
    "tri_in_fwd b32 256^3 MM": lambda: ops.bgemm(
        Mat(a_cm, lo=(1, R), batch_stride=rows), Mat(b_cm, lo=(1, R), batch_stride=rows),
        Mat(t_cm, lo=(R, 1), batch_stride=rows), P, R, R, R),
    "tri_bwd b32 256^3 KM": lambda: ops.bgemm(
        Mat(dt, lo=(R, 1), batch_stride=rows), Mat(b_cm, lo=(1, R), batch_stride=rows),
        Mat(t_cm, lo=(R, 1), batch_stride=rows), P, R, R, R),
    "tri_bwd b32 256^3 MM(T)": lambda: ops.bgemm(
        Mat(dt, lo=(1, R), batch_stride=rows), Mat(a_cm, lo=(1, R), batch_stride=rows),
        Mat(t_cm, lo=(R, 1), batch_stride=rows), P, R, R, R),
}
flops = {k: 2 * (R * P) ** 2 * S if k.startswith("opm") else 2 * P * R ** 3 for k in cases}
sel = sys.argv[1] if len(sys.argv) > 1 else ""
for name, fn in cases.items():
    if sel not in name:
        continue
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 50
    gr = torch.cuda.CUDAGraph()  # graph-replayed so host launch overhead is not timed
    with torch.cuda.graph(gr):
        for _ in range(n):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"{name:34s} {us:8.1f} us  {flops[name] / us / 1e6:7.1f} TFLOP/s")
