"""Per-tile phase trace (SM clocks) of CTA 0 of the warp-specialised long-sequence forward
(EVO_EXP=12 build): EVO_LIB_PATH=scripts/_exp/libevo_exp12.so python scripts/ws_trace.py [L] [B]"""
import ctypes, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2203_00854_b200 import _lib, ops
from paper_2203_00854_b200.ops import Strided

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
H, c = 4, 32
lib = _lib.load()
ld = 3 * H * c + 8
qkv = torch.randn(B * L, ld, device="cuda").bfloat16()
gp = torch.randn(B * L, H * c, device="cuda").bfloat16()
og = torch.empty(B * L, H * c, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, H, L, device="cuda")
S = lambda t, w, off=0: Strided(t, L * w, w, off)
d = ops.attention_desc(S(qkv, ld, 0), S(qkv, ld, H * c), S(qkv, ld, 2 * H * c), S(gp, H * c), S(og, H * c), None,
                       lse, B, L, H, c, 1 / math.sqrt(c), bias=qkv, bias_s=(L * ld, 1, 0, ld), bias_off=3 * H * c,
                       flags=_lib.EVO_ATTN_FORCE_WS)
for _ in range(3):
    ops.attention_fwd(d)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
ops.attention_fwd(d)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
fl = 4 * B * H * L * L * c
print(f"L={L} B={B}: {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOP/s, exp/clk/SM = {B * H * L * L / (ms * 1e-3 * 1.965e9 * 148):.2f}")
buf = np.zeros(3 * 4096, dtype=np.int64)
lib.evo_ws_trace.argtypes = [ctypes.c_void_p]
lib.evo_ws_trace(buf.ctypes.data_as(ctypes.c_void_p))
nkt = (L + 63) // 64
names = ["s_full wait", "tmem ld", "max/vote", "turn wait", "exp+pack", "st+arrive"]
t0 = min(buf[buf > 0])
for w in range(2):
    b = buf[w * 4096:(w + 1) * 4096].reshape(-1, 8)[:nkt]
    ph = np.diff(b[:, [0, 1, 2, 3, 6, 4, 5]], axis=1)
    per = np.diff(b[:, 0])
    print(f"warpgroup {w}: start {b[0,0]-t0} clk, per-tile period median {np.median(per):.0f} clk")
    for k, n in enumerate(names):
        print(f"   {n:12s} median {np.median(ph[:, k]):6.0f}  mean {ph[:, k].mean():6.0f}")
    for j in (0, 1, 2, 10, 30, nkt - 1):
        print(f"   tile {j:3d} t={b[j,0]-t0:8d} " + " ".join(f"{x:5d}" for x in ph[j]))
m = buf[2 * 4096:3 * 4096].reshape(-1, 8)[:nkt]
print("MMA issuer wg0: kv_full ready - s_full(wg0) wait start: median",
      np.median(m[:, 0] - buf[:4096].reshape(-1, 8)[:nkt, 0]))
print("  o_done gate passed after kv:", np.median(m[:, 1] - m[:, 0]), " p_full seen - softmax arrive:",
      np.median(m[:, 2] - buf[:4096].reshape(-1, 8)[:nkt, 5]))
