"""Column-reduction epilogue kernels at the training shape: bias_act_bwd (ReLU mask + bias
gradient, in place) and colsum, graph-replayed launches.  python scripts/colred_micro.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops

def gtime(fn, it=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it):
            fn()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3

for rows, cols in ((32768, 1024), (65536, 512)):
    dh = torch.randn(rows, cols, device="cuda").bfloat16()
    h = torch.randn(rows, cols, device="cuda").bfloat16()
    db = torch.zeros(cols, device="cuda")
    t = gtime(lambda: ops.bias_act_bwd(dh, h, rows, cols, dy=dh, dbias=db))
    print(f"bias_act_bwd [{rows},{cols}] {t:7.1f} us  {3 * rows * cols * 2 / t / 1e3:7.0f} GB/s", flush=True)
for rows, cols in ((32768, 776), (65536, 392), (65536, 256), (32768, 256)):
    x = torch.randn(rows, cols, device="cuda").bfloat16()
    out = torch.zeros(cols, device="cuda")
    t = gtime(lambda: ops.colsum(x, out))
    print(f"colsum [{rows},{cols}] {t:7.1f} us  {rows * cols * 2 / t / 1e3:7.0f} GB/s", flush=True)
