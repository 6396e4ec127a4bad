"""Weight-gradient GEMMs of the training shape (dW = X^T dY, K = rows = 32768 / 65536):
cuBLAS (torch.mm out_dtype=fp32) vs evo_wgrad (tcgen05, MN-major TMA operands, split-K, accumulate).
python scripts/wgrad_micro.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat

dev, BF = "cuda", torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
cases = [("msa qkv", 32768, 256, 768), ("msa gate/out", 32768, 256, 256), ("msa_trans w1", 32768, 256, 1024),
         ("msa_trans w2", 32768, 1024, 256), ("pair qkv", 65536, 128, 392), ("pair gate/out", 65536, 128, 128),
         ("pair_trans w1", 65536, 128, 512), ("pair_trans w2", 65536, 512, 128), ("opm w_o", 65536, 1024, 128),
         ("opm w_ab", 32768, 256, 64), ("tri w_proj", 65536, 128, 256), ("tri w_o", 65536, 32, 128)]


def timeit(fn, it=20):
    """device time per call: the calls are captured in a CUDA graph and replayed (host launch and
    tensor-map encoding costs excluded, as in the bench's graphed step)"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        with torch.cuda.graph(g, stream=s):
            for _ in range(it):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


tot_c = tot_e = 0.0
for name, rows, kin, nout in cases:
    x = torch.randn(rows, kin, device=dev, generator=g).to(BF)
    dy = torch.randn(rows, nout, device=dev, generator=g).to(BF)
    out1 = torch.empty(kin, nout, device=dev)
    out2 = torch.empty(kin, nout, device=dev)
    tc = timeit(lambda: torch.mm(x.t(), dy, out_dtype=torch.float32, out=out1))
    out2.zero_()
    ops.wgrad(x, dy, out2)  # accumulate semantics: one call onto zeros
    torch.mm(x.t(), dy, out_dtype=torch.float32, out=out1)
    err = ((out1 - out2).norm() / out1.norm()).item()
    te = timeit(lambda: ops.wgrad(x, dy, out2))
    fl = 2 * rows * kin * nout
    tot_c += tc; tot_e += te
    gbs = 2 * rows * (kin + nout) / 1e3
    print(f"{name:14s} [{kin}x{nout}] K={rows}: cublas {tc:7.1f} us ({gbs/tc:5.0f} GB/s)  evo {te:7.1f} us "
          f"({gbs/te:5.0f} GB/s, {fl/te/1e6:5.0f} TF/s)  rel {err:.1e}", flush=True)
print(f"total cublas {tot_c:.0f} us  evo {tot_e:.0f} us")
