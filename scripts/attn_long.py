"""Attention forward timing at long N_r (pair_row shape [B=N_r, L=N_r, H=4, c=32] with the
per-key bias; msa_row [128, N_r, 8] with the full bias) for both forward kernels:
python scripts/attn_long.py [--n 1024 2048] [--iters 5]"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import _lib, ops
from paper_2203_00854_b200.ops import Strided

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[1024, 2048])
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--pair-batch", type=int, default=0, help="batch for pair shape (default N_r)")
a = ap.parse_args()
lib = _lib.load()
for n in a.n:
    for name, B, H, bmode in (("pair_row", a.pair_batch or n, 4, "key"), ("pair_col", a.pair_batch or n, 4, "key"),
                              ("msa_row", 128, 8, "full")):
        L, c = n, 32
        ld = 3 * H * c + (8 if bmode == "key" else 0)
        qkv = torch.randn(B * L, ld, device="cuda").bfloat16()
        gp = torch.randn(B * L, H * c, device="cuda").bfloat16()
        og = torch.empty(B * L, H * c, device="cuda", dtype=torch.bfloat16); orw = torch.empty_like(og)
        lse = torch.empty(B, H, L, device="cuda")
        if name == "pair_col":  # rows of one sequence B * ld apart (the pair grid's column axis)
            S = lambda t, w, off=0: Strided(t, w, B * w, off)
        else:
            S = lambda t, w, off=0: Strided(t, L * w, w, off)
        if bmode == "full":
            bias = torch.randn(H, L, L, device="cuda").bfloat16(); bs = (0, L * L, L, 1); boff = 0
        else:
            bias = qkv; boff = 3 * H * c
            bs = (ld, 1, 0, B * ld) if name == "pair_col" else (L * ld, 1, 0, ld)
        res = {}
        for kern, fl_ in (("ws", _lib.EVO_ATTN_FORCE_WS), ("flash", _lib.EVO_ATTN_FORCE_FLASH)):
            d = ops.attention_desc(S(qkv, ld, 0), S(qkv, ld, H * c), S(qkv, ld, 2 * H * c), S(gp, H * c),
                                   S(og, H * c), S(orw, H * c), lse, B, L, H, c, 1 / math.sqrt(c), bias=bias,
                                   bias_s=bs, bias_off=boff, flags=fl_)
            ops.attention_fwd(d)
            torch.cuda.synchronize()
            ref = og.clone() if kern == "ws" else None
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(a.iters):
                ops.attention_fwd(d)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            res[kern] = ms
            if kern == "ws":
                o_ws = og.clone()
        diff = ((og.float() - o_ws.float()).norm() / og.float().norm()).item()
        fl = 4 * B * H * L * L * c
        print(f"N_r={n:5d} {name:8s} ws {res['ws']:8.2f} ms ({fl/res['ws']/1e9:6.1f} TFLOP/s)   "
              f"flash {res['flash']:8.2f} ms ({fl/res['flash']/1e9:6.1f} TFLOP/s)   rel diff {diff:.2e}", flush=True)
        del qkv, gp, og, orw, lse, bias
        torch.cuda.empty_cache()
