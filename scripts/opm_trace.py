"""Per-chunk event timeline of CTA 0 of the fused OPM kernel (EVO_EXP=3 build).
EVO_LIB_PATH=scripts/_exp/libevo_exp3.so python scripts/opm_trace.py [dbg]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2203_00854_b200 import ops, _lib
I = J = 256; S, P, Hz = 128, 32, 128
a_t = torch.randn(I, P, S, device="cuda").bfloat16(); b = torch.randn(J, P, S, device="cuda").bfloat16()
w = torch.randn(P * P, Hz, device="cuda").bfloat16()
for _ in range(5):
    ops.opm_fused_fwd(a_t, b, w, I, J, S, P, Hz, 1.0 / S)
torch.cuda.synchronize()
buf = np.zeros(4096, dtype=np.uint64)
lib = _lib.load()
lib.evo_opm_trace(buf.ctypes.data_as(ctypes.c_void_p))
t0 = min(x for x in buf if x > 0)
names = {0: "issue a0", 1: "issue a1", 2: "issue w0", 3: "issue w1", 4: "mma: wait o0", 5: "G2_0 issued", 6: "G1_0(c+1) issued",
         7: "G2_1 issued", 8: "G1_1(c+1) issued", 9: "C0 start", 10: "C0 done", 11: "C1 start", 12: "C1 done", 13: "g1_0 enter", 14: "acc_empty ok", 15: "a_full ok"}
for ch in range(16):
    row = buf[ch * 16: ch * 16 + 16].copy()
    nxt = buf[ch * 16 + 16: ch * 16 + 32]
    row[13:16] = nxt[13:16] if len(nxt) == 16 else 0
    if not row.any():
        continue
    print(f"chunk {ch:2d}: " + "  ".join(f"{names[k]}={(int(row[k]) - int(t0)) / 1000:.2f}" for k in range(16) if row[k]))
