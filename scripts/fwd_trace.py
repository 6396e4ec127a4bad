"""Per-tile timeline (SM clocks, thread 0 of CTA 0) of the persistent attention forward at the
training shape (EVO_EXP=5 build): EVO_LIB_PATH=scripts/_exp/libevo_exp5.so python scripts/fwd_trace.py [variant]"""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
v = sys.argv[1] if len(sys.argv) > 1 else "pair_row"
subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), "attn_micro.py"), "--variant", v,
                "--iters", "3", "--bwd", "0", "--fwd-trace-dump", "/tmp/fwd_trace.npy"], check=True)
b = np.load("/tmp/fwd_trace.npy").reshape(-1, 8)
n = int((b[:, 0] > 0).sum())
t0 = b[b > 0].min()
print("tile | top->kv+sync | ->S ready | softmax | sync | (unit end: ->O ready, epilogue)")
for g in range(min(n, 40)):
    r = b[g]
    line = f"{g:3d} @{r[0]-t0:7d}  kv {r[1]-r[0]:5d}  S {r[2]-r[1]:5d}  sm {r[3]-r[2]:5d}  sync {r[4]-r[3]:5d}"
    if r[5]:
        line += f"  | O {r[6]-r[5]:5d} epi {r[7]-r[6]:5d}"
    print(line)
per = np.diff(b[:n, 0])
print("median tile period", np.median(per))
