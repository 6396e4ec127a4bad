"""Triangle-einsum-sized batched GEMMs at long N_r (batch = 32 channels, M = N = K = N_r):
evo_bgemm (tcgen05) vs torch.bmm (cuBLAS) for reference.  python scripts/gemm_big.py [N_r ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat

P = 32
for R in [int(x) for x in sys.argv[1:]] or [1024, 2048]:
    a = torch.randn(P, R, R, device="cuda").bfloat16()
    b = torch.randn(P, R, R, device="cuda").bfloat16()
    t = torch.empty(P, R, R, device="cuda", dtype=torch.bfloat16)
    rows = R * R
    cases = {
        "KK (outgoing)": lambda: ops.bgemm(Mat(a, lo=(R, 1), batch_stride=rows), Mat(b, lo=(R, 1), batch_stride=rows),
                                           Mat(t, lo=(R, 1), batch_stride=rows), P, R, R, R),
        "MM (incoming)": lambda: ops.bgemm(Mat(a, lo=(1, R), batch_stride=rows), Mat(b, lo=(1, R), batch_stride=rows),
                                           Mat(t, lo=(R, 1), batch_stride=rows), P, R, R, R),
        "cuBLAS bmm KK": lambda: torch.bmm(a, b.transpose(1, 2), out=t),
    }
    ref = torch.bmm(a.float()[:2], b.float()[:2].transpose(1, 2))
    for name, fn in cases.items():
        fn()
        torch.cuda.synchronize()
        if name.startswith("KK"):
            err = ((t[:2].float() - ref).norm() / ref.norm()).item()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"R={R} {name:14s} {ms:8.3f} ms  {2 * P * R ** 3 / ms / 1e9:7.1f} TFLOP/s", flush=True)
    print(f"R={R} KK rel err vs fp32 {err:.2e}")
