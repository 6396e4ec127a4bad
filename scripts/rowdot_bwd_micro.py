"""msa_row_bias backward at the training shape: the block's path (fp32 K=8 GEMM for dLN + LayerNorm
backward + side weight-gradient GEMM) vs the fused evo_layernorm_rowdot_bwd.
python scripts/rowdot_bwd_micro.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops

rows, Hz, nh = 65536, 128, 8
z = torch.randn(rows, Hz, device="cuda").bfloat16()
g = torch.rand(Hz, device="cuda") + 0.5
b = torch.randn(Hz, device="cuda") * 0.1
w = torch.randn(Hz, nh, device="cuda") * 0.1
out = torch.empty(nh, rows, device="cuda", dtype=torch.bfloat16)
ln = torch.empty(rows, Hz, device="cuda", dtype=torch.bfloat16)
mean = torch.empty(rows, device="cuda"); rstd = torch.empty(rows, device="cuda")
ops.layernorm_rowdot_fwd(z, g, b, w, rows, Hz, out, rows, ln_out=ln, mean=mean, rstd=rstd)
db2 = torch.randn(nh, rows, device="cuda")
dz = torch.randn(rows, Hz, device="cuda").bfloat16()
dg, dbt, dw = torch.zeros(Hz, device="cuda"), torch.zeros(Hz, device="cuda"), torch.zeros(Hz, nh, device="cuda")


def block_path():
    dln = torch.mm(db2.t(), w.t())
    dw.add_(torch.mm(ln.t(), db2.bfloat16().t(), out_dtype=torch.float32))
    return ops.layernorm_bwd(dln, z, g, mean, rstd, rows, Hz, res=dz, dgamma=dg, dbeta=dbt)


dx = torch.empty_like(dz)
fused = lambda: ops.layernorm_rowdot_bwd(z, g, b, w, db2, rows, mean, rstd, rows, Hz, dx, dz, dg, dbt, dw)


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


a = block_path()
fused()
torch.cuda.synchronize()
err = ((a.float() - dx.float()).norm() / a.float().norm()).item()
print(f"block path {t(block_path):7.1f} us | fused rowdot_bwd {t(fused):7.1f} us | rel diff dx {err:.2e}")
