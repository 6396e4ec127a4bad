"""One attention forward configuration, for ncu: python scripts/attn_one.py --n 1024 --ws 1 [--kind pair|msa]"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import _lib, ops
from paper_2203_00854_b200.ops import Strided
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--ws", type=int, default=1)
ap.add_argument("--kind", default="pair")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
lib = _lib.load()
L, c = a.n, 32
B, H, bmode = ((a.batch or L), 4, "key") if a.kind == "pair" else ((a.batch or 128), 8, "full")
ld = 3 * H * c + (8 if bmode == "key" else 0)
qkv = torch.randn(B * L, ld, device="cuda").bfloat16()
gp = torch.randn(B * L, H * c, device="cuda").bfloat16()
og = torch.empty(B * L, H * c, device="cuda", dtype=torch.bfloat16); orw = torch.empty_like(og)
lse = torch.empty(B, H, L, device="cuda")
S = lambda t, w, off=0: Strided(t, L * w, w, off)
if bmode == "full":
    bias = torch.randn(H, L, L, device="cuda").bfloat16(); bs = (0, L * L, L, 1); boff = 0
else:
    bias = qkv; bs = (L * ld, 1, 0, ld); boff = 3 * H * c
d = ops.attention_desc(S(qkv, ld, 0), S(qkv, ld, H * c), S(qkv, ld, 2 * H * c), S(gp, H * c), S(og, H * c),
                       S(orw, H * c), lse, B, L, H, c, 1 / math.sqrt(c), bias=bias, bias_s=bs, bias_off=boff,
                       flags=_lib.EVO_ATTN_FORCE_WS if a.ws else _lib.EVO_ATTN_FORCE_FLASH)
for _ in range(a.iters):
    ops.attention_fwd(d)
torch.cuda.synchronize()
