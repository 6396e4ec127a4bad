"""One evo_wgrad call of a given shape (for ncu).  python scripts/wgrad_one.py rows M N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
rows, M, N = map(int, sys.argv[1:4])
x = torch.randn(rows, M, device="cuda").bfloat16(); dy = torch.randn(rows, N, device="cuda").bfloat16()
dw = torch.zeros(M, N, device="cuda")
for _ in range(3):
    ops.wgrad(x, dy, dw)
torch.cuda.synchronize()
