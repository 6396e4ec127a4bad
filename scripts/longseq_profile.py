"""Per-kernel GPU time of ONE long-sequence block forward (torch.profiler / CUPTI), by category.
python scripts/longseq_profile.py [n_res]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2203_00854_b200.config import EvoConfig, init_block_params
from paper_2203_00854_b200.params import BlockParams
from paper_2203_00854_b200 import block as B

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = EvoConfig(128, R, 256, 128, 8, 4, 32)
bp = BlockParams(init_block_params(cfg, 0), cfg, device="cuda")
m = torch.randn(128, R, 256, device="cuda").bfloat16()
z = torch.randn(R, R, 128, device="cuda").bfloat16()
with torch.no_grad():
    B.block_fwd(bp, m, z, save=False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        B.block_fwd(bp, m, z, save=False)
        torch.cuda.synchronize()
rows = sorted(prof.key_averages(), key=lambda e: -getattr(e, "self_device_time_total", 0))
tot = sum(getattr(e, "self_device_time_total", 0) for e in rows)
print(f"N_r={R}: total GPU time {tot/1e3:.1f} ms per block forward")
for e in rows[:25]:
    t = getattr(e, "self_device_time_total", 0)
    if t > 0:
        print(f"{t/1e3:9.2f} ms {100*t/tot:5.1f}%  n={e.count:3d}  {e.key[:100]}")
