"""Channel-major LayerNorm (the triangle update's LN2 over p=32 channels, [P][rows]) forward and
backward at the training shape.  python scripts/ln_cm_micro.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops


def t(fn, it=20):
    """device time per call: the calls are captured in a CUDA graph (no host overhead)"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(it):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    gr.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


P, R = 32, 65536
x = torch.randn(P, R, device="cuda").bfloat16()
g, b = torch.rand(P, device="cuda") + 0.5, torch.randn(P, device="cuda")
y, mean, rstd = ops.layernorm_fwd(x, g, b, R, P, x_rs=1, x_cs=R)
dy = torch.randn(R, P, device="cuda").bfloat16()
dx = torch.empty_like(x)
dg, db = torch.zeros(P, device="cuda"), torch.zeros(P, device="cuda")
yo = torch.empty(R, P, device="cuda", dtype=torch.bfloat16)
tf = t(lambda: ops.layernorm_fwd(x, g, b, R, P, x_rs=1, x_cs=R, out=yo, mean=mean, rstd=rstd))
tb = t(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, R, P, x_rs=1, x_cs=R, dx=dx, dgamma=dg, dbeta=db))
mb = P * R * 2 / 1e6
print(f"[P={P}][rows={R}] channel-major LN: fwd {tf:6.1f} us ({2 * mb / tf * 1e3:.0f} GB/s of x+y), "
      f"bwd {tb:6.1f} us ({3 * mb / tb * 1e3:.0f} GB/s of dy+x+dx)")
