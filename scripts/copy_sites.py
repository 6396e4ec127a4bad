"""Where the eager copies of the fwd+bwd step come from (aten::copy_ / clone / to with shapes and
the Python call site): python scripts/copy_sites.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2203_00854_b200.config import EvoConfig, synthetic_inputs
from paper_2203_00854_b200.evoformer import EvoformerStack

cfg = EvoConfig(128, 256, 256, 128, 8, 4, 32)
st = EvoformerStack(cfg, 2, seed=0)
m64, z64 = synthetic_inputs(cfg, 0)
rng = np.random.default_rng(1)
dev = lambda a: torch.tensor(a, device="cuda").bfloat16()
m, z, gm, gz = dev(m64), dev(z64), dev(rng.normal(size=m64.shape)), dev(rng.normal(size=z64.shape))
for _ in range(2):
    st.zero_grad(); st.forward_backward(m, z, gm, gz)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True, with_stack=True) as prof:
    st.zero_grad(); st.forward_backward(m, z, gm, gz)
    torch.cuda.synchronize()
rows = prof.key_averages(group_by_stack_n=6, group_by_input_shape=True)
for e in sorted(rows, key=lambda e: -e.device_time_total):
    if e.key in ("aten::copy_", "aten::clone", "aten::to", "aten::_to_copy", "aten::contiguous", "aten::fill_",
                 "aten::zero_", "aten::zeros", "aten::add_", "aten::sum", "aten::mul", "aten::add", "aten::cat"):
        if e.device_time_total <= 0:
            continue
        print(f"{e.key:16s} n={e.count:3d} dev {e.device_time_total / 2:8.1f} us/block  shapes={str(e.input_shapes)[:90]}")
        for fr in (e.stack or [])[:6]:
            print("        ", fr)
