"""Transition backward hidden gradient: cuBLAS dhid = dx W2^T + bias_act_bwd (mask, db1) vs the
tcgen05 bgemm, at the training shapes.  python scripts/trans_dgrad_micro.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


for rows, H in ((32768, 256), (65536, 128)):
    F = 4 * H
    dx = torch.randn(rows, H, device="cuda").bfloat16()
    w2 = torch.randn(F, H, device="cuda").bfloat16() * 0.05
    hid = torch.relu(torch.randn(rows, F, device="cuda")).bfloat16()
    out = torch.empty(rows, F, device="cuda", dtype=torch.bfloat16)
    db = torch.zeros(F, device="cuda")
    cub = t(lambda: torch.mm(dx, w2.t(), out=out))
    own = t(lambda: ops.bgemm(Mat(dx, lo=(H, 1)), Mat(w2, lo=(H, 1)), Mat(out, lo=(F, 1)), 1, rows, F, H))
    ba = t(lambda: ops.bias_act_bwd(out, hid, rows, F, dy=out, dbias=db))
    print(f"rows={rows} H={H}: cuBLAS dhid {cub:6.1f} us | tcgen05 bgemm {own:6.1f} us | bias_act_bwd {ba:6.1f} us")
