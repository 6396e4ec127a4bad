"""One msa_row bias LN + row-dot forward and backward at the training shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
rows, cols = 65536, 128
x = torch.randn(rows, cols, device="cuda").bfloat16()
g, b = torch.randn(cols, device="cuda"), torch.randn(cols, device="cuda")
w = torch.randn(cols, 8, device="cuda")
out = torch.empty(8, rows, device="cuda", dtype=torch.bfloat16)
ln = torch.empty(rows, cols, device="cuda", dtype=torch.bfloat16)
mu, rs = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
dout = torch.randn(8, rows, device="cuda")
dx = torch.zeros(rows, cols, device="cuda", dtype=torch.bfloat16)
dg, db, dw = torch.zeros(cols, device="cuda"), torch.zeros(cols, device="cuda"), torch.zeros(cols, 8, device="cuda")
for _ in range(3):
    ops.layernorm_rowdot_fwd(x, g, b, w, rows, cols, out, rows, ln_out=ln, mean=mu, rstd=rs)
    ops.layernorm_rowdot_bwd(x, g, b, w, dout, rows, mu, rs, rows, cols, dx, dx, dg, db, dw)
torch.cuda.synchronize()
