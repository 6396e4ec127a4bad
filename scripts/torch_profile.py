"""Warm per-kernel GPU time breakdown of the fwd+bwd step via torch.profiler (CUPTI),
not serialised like an ncu launch list.  python scripts/torch_profile.py [blocks]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2203_00854_b200.config import EvoConfig, synthetic_inputs
from paper_2203_00854_b200.evoformer import EvoformerStack

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = EvoConfig(128, 256, 256, 128, 8, 4, 32)
st = EvoformerStack(cfg, nb, seed=0)
m64, z64 = synthetic_inputs(cfg, 0)
rng = np.random.default_rng(1)
dev = lambda a: torch.tensor(a, device="cuda").bfloat16()
m, z, gm, gz = dev(m64), dev(z64), dev(rng.normal(size=m64.shape)), dev(rng.normal(size=z64.shape))
for _ in range(3):
    st.zero_grad(); st.forward_backward(m, z, gm, gz)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    st.zero_grad(); st.forward_backward(m, z, gm, gz)
    torch.cuda.synchronize()
ev = [e for e in prof.key_averages() if e.device_type.name == "CUDA" or getattr(e, "self_device_time_total", 0) > 0]
tot = sum(getattr(e, "self_device_time_total", 0) for e in prof.key_averages())
print(f"total GPU time {tot/1e3:.2f} ms for {nb} blocks ({tot/1e3/nb:.3f} ms/block)")
rows = sorted(prof.key_averages(), key=lambda e: -getattr(e, "self_device_time_total", 0))
for e in rows[:45]:
    t = getattr(e, "self_device_time_total", 0)
    if t <= 0:
        continue
    print(f"{t/1e3/nb:8.3f} ms/block {100*t/tot:5.1f}%  n={e.count//nb:4d}/blk  {e.key[:100]}")

CATEGORIES = [("attention bwd", ("attn_bwd", "attn_dbias", "attn_bias_transpose")), ("attention fwd", ("attn_fwd",)),
              ("OPM fused", ("opm_",)), ("tcgen05 bgemm", ("bgemm",)),
              ("cuBLAS", ("nvjet", "cublas", "gemm", "splitKreduce", "cutlass")), ("LayerNorm / residual", ("ln_", "residual_ln", "layernorm")),
              ("elementwise / gates", ("gated_residual", "bias_act", "tri_gate", "colsum", "count_nonfinite")),
              ("copies / torch eager", ("copy", "Memcpy", "fill", "elementwise_kernel", "reduce_kernel"))]
cat = {}
for e in rows:
    t = getattr(e, "self_device_time_total", 0)
    if t <= 0:
        continue
    k = next((c for c, keys in CATEGORIES if any(x in e.key for x in keys)), "other")
    cat[k] = cat.get(k, 0) + t
print("--- by category (ms/block)")
for k, t in sorted(cat.items(), key=lambda kv: -kv[1]):
    print(f"{t / 1e3 / nb:8.3f}  {100 * t / tot:5.1f}%  {k}")
