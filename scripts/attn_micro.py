"""Per-variant microbenchmark of the attention kernels at the training shape
(fwd and bwd, CUDA events, warm).  Usable under ncu (--variant to restrict)."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Strided

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="all")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--bwd", type=int, default=1)
ap.add_argument("--fb", type=int, default=1, help="forward: stage a full bias through smem (A/B switch)")
ap.add_argument("--fwd-trace-dump", default="", help="EVO_EXP=5 builds: dump the forward tile trace (numpy)")
ap.add_argument("--trace-dump", default="", help="EVO_EXP=10 builds: dump the backward phase trace (numpy)")
a = ap.parse_args()
from paper_2203_00854_b200 import _lib
FLAGS = 0 if a.fb else _lib.EVO_ATTN_NO_BIAS_SMEM
# (name, B, L, H, c, kind, bias)
V = [("msa_row", 128, 256, 8, 32, "row", "full"), ("msa_col", 256, 128, 8, 32, "col", None),
     ("pair_row", 256, 256, 4, 32, "row", "key"), ("pair_col", 256, 256, 4, 32, "col", "key")]
for name, B, L, H, c, kind, bmode in V:
    if a.variant not in ("all", name):
        continue
    ld = 3 * H * c + (8 if bmode == "key" else 0)
    rows = B * L
    qkv = torch.randn(rows, ld, device="cuda").bfloat16()
    gp = torch.randn(rows, H * c, device="cuda").bfloat16()
    og = torch.empty(rows, H * c, device="cuda", dtype=torch.bfloat16); orw = torch.empty_like(og)
    lse = torch.empty(B, H, L, device="cuda")
    sb, sl = (L, 1) if kind == "row" else (1, B)
    S = lambda t, w, off=0: Strided(t, sb * w, sl * w, off)
    if bmode == "full":
        bias = torch.randn(H, L, L, device="cuda").bfloat16(); bs = (0, L * L, L, 1); boff = 0
    elif bmode == "key":
        bias = qkv; bs = (sb * ld, 1, 0, sl * ld); boff = 3 * H * c
    else:
        bias, bs, boff = None, (0, 0, 0, 0), 0
    d = ops.attention_desc(S(qkv, ld, 0), S(qkv, ld, H * c), S(qkv, ld, 2 * H * c), S(gp, H * c), S(og, H * c),
                           S(orw, H * c), lse, B, L, H, c, 1 / math.sqrt(c), bias=bias, bias_s=bs, bias_off=boff,
                           flags=FLAGS)
    dout = torch.randn(rows, H * c, device="cuda").bfloat16()
    dqkv = torch.zeros_like(qkv); dgp = torch.empty_like(gp)
    if bmode == "full":
        dbias = torch.zeros(H, L, L, device="cuda"); dbs = (0, L * L, L, 1)
    elif bmode == "key":
        dbias = torch.zeros(B, H, L, device="cuda"); dbs = (H * L, L, 0, 1)
    else:
        dbias, dbs = None, (0, 0, 0, 0)
    ws = torch.empty(ops.attention_bwd_workspace(B, L, H, c, bmode == "full"), device="cuda", dtype=torch.uint8)
    fwd = lambda: ops.attention_fwd(d)
    bwd = lambda: ops.attention_bwd(d, S(dout, H * c), S(dqkv, ld, 0), S(dqkv, ld, H * c), S(dqkv, ld, 2 * H * c),
                                    S(dgp, H * c), ws, dbias=dbias, dbias_s=dbs)
    for fn, tag in ((fwd, "fwd"), (bwd, "bwd")):
        if tag == "bwd" and not a.bwd:
            continue
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        fl = (4 if tag == "fwd" else 10) * B * H * L * L * c
        print(f"{name:9s} {tag}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOP/s")

if a.trace_dump:
    import ctypes, numpy as np
    buf = np.zeros(8192, dtype=np.uint64)
    _lib.load().evo_bwd_trace(buf.ctypes.data_as(ctypes.c_void_p))
    np.save(a.trace_dump, buf)
if a.fwd_trace_dump:
    import ctypes, numpy as np
    buf = np.zeros(4096, dtype=np.int64)
    _lib.load().evo_fwd_trace(buf.ctypes.data_as(ctypes.c_void_p))
    np.save(a.fwd_trace_dump, buf)
