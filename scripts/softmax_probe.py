"""Softmax forward time with / without the broadcast bias and mask operands (which input
costs what): python scripts/softmax_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kernel_microbench import time_launches  # noqa: E402

dev = "cuda"
for xs, bs, ms_ in (((256, 4, 256, 256), (256, 4, 1, 256), (256, 1, 1, 256)), ((128, 8, 256, 256), (1, 8, 256, 256), None)):
    sets = [(torch.randn(xs, device=dev).bfloat16(), torch.empty(xs, device=dev, dtype=torch.bfloat16)) for _ in range(2)]
    bias = torch.randn(bs, device=dev).bfloat16()
    mask = torch.zeros(ms_, device=dev, dtype=torch.bfloat16) if ms_ else None
    nx = xs[0] * xs[1] * xs[2] * xs[3]
    for name, b_, m_ in (("none", None, None), ("bias", bias, None), ("mask", None, mask), ("both", bias, mask)):
        if name in ("mask", "both") and mask is None:
            continue
        t = time_launches(lambda x, y: ops.softmax_fwd(x, b_, m_, 0.17, out=y), sets, 30)
        print(f"x{list(xs)} {name:5s}: {t * 1e3:7.2f} us  {nx * 4 / t / 1e6:7.1f} GB/s (x read + y write)")
