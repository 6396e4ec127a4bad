"""Fused residual + next-module LayerNorm vs the two separate kernels (graph-replayed, rotating
buffers larger than L2).   python scripts/rln_micro.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_00854_b200 import _lib, ops  # noqa: E402
from kernel_microbench import rotating, time_launches  # noqa: E402

_lib.load()
dev = torch.device("cuda")
for rows, cols, gated in ((65536, 128, False), (65536, 128, True), (32768, 256, False), (4096 * 64, 128, False)):
    gam = torch.randn(cols, device=dev)
    bet = torch.randn(cols, device=dev)
    bias = torch.randn(cols, device=dev)
    n = rows * cols

    def mk():
        r = torch.randn(rows, cols, device=dev).bfloat16()
        y = torch.randn(rows, cols, device=dev).bfloat16()
        gp = torch.randn(rows, cols, device=dev).bfloat16() if gated else None
        return r, y, gp

    sets = rotating(mk, n * 2 * (3 if gated else 2))
    kw = lambda gp: dict(gp=gp, gp_rs=cols) if gp is not None else {}
    t_sep = time_launches(lambda r, y, gp: ops.layernorm_fwd(ops.gated_residual_fwd(r, y, bias, rows, cols, **kw(gp)),
                                                             gam, bet, rows, cols), sets, 40)
    t_res = time_launches(lambda r, y, gp: ops.gated_residual_fwd(r, y, bias, rows, cols, **kw(gp)), sets, 40)
    t_fus = time_launches(lambda r, y, gp: ops.residual_layernorm_fwd(r, y, bias, rows, cols, gam, bet, **kw(gp)),
                          sets, 40)
    algo = n * 2 * (4 + (1 if gated else 0))
    print(f"[{rows},{cols}] gated={gated}: separate {t_sep*1e3:.1f} us (residual alone {t_res*1e3:.1f}), "
          f"fused {t_fus*1e3:.1f} us = {algo / t_fus / 1e6:.0f} GB/s", flush=True)
