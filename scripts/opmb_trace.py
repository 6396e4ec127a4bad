"""Per-step timeline (SM clocks) of CTA 0 of the fused OPM backward contraction (EVO_EXP=4 build):
EVO_LIB_PATH=scripts/_exp/libevo_exp4.so python scripts/opmb_trace.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2203_00854_b200 import ops, _lib
I = J = 256; S, P, Hz = 128, 32, 128
dz = torch.randn(I * J, Hz, device="cuda").bfloat16()
w = torch.randn(P * P, Hz, device="cuda").bfloat16()
b_t = torch.randn(J, P, S, device="cuda").bfloat16()
out = torch.empty(S * I, P, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.opm_bwd_factor(0, dz, w, b_t, I, J, S, P, Hz, 1.0 / S, out, I * P, 0, P)
torch.cuda.synchronize()
buf = np.zeros(4096, dtype=np.int64)
lib = _lib.load()
lib.evo_opmb_trace.argtypes = [ctypes.c_void_p]
lib.evo_opmb_trace(buf.ctypes.data_as(ctypes.c_void_p))
b = buf.reshape(-1, 8)
n = int((b[:, 0] > 0).sum())
t0 = b[b > 0].min()
print("step | A: wait dy_full, wait da_empty | B: wait ab_full, wait ot_full | conv start, conv dur | B issue t")
for s in range(n):
    r = b[s] - t0
    print(f"{s:3d} A@{r[0]:7d} dy+{r[1]-r[0]:5d} da_e+{r[2]-r[1]:5d} | B@{r[3]:7d} ab+{r[4]-r[3]:5d} ot+{r[5]-r[4]:5d} | "
          f"conv@{r[6]:7d} dur {r[7]-r[6]:5d}")
per = np.diff(b[:n, 2])
print("median A-issue period", np.median(per), "clk; conv median", np.median(b[:n, 7] - b[:n, 6]))
