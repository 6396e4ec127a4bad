"""Phase timeline of CTA 0 of the attention backward main kernel (EVO_EXP=10 build):
EVO_LIB_PATH=scripts/_exp/libevo_exp10.so python scripts/attn_bwd_trace.py [variant]"""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
v = sys.argv[1] if len(sys.argv) > 1 else "pair_row"
subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "attn_micro.py"), "--variant", v, "--iters", "3",
                "--trace-dump", "/tmp/bwd_trace.npy"], check=True)
buf = np.load("/tmp/bwd_trace.npy")
names = ["loop top", "loads ready+sync", "S/dP MMA done", "elementwise done", "MMA2 issued/dS copy", "MMA2 done",
         "prefetch issued", "drain done"]
for who, off in (("thread 0 (wg0)", 0), ("thread 128 (wg1)", 4096)):
    b = buf[off:off + 4096].astype(np.int64)
    t0 = b[b > 0].min()
    print(who)
    for it in range(14):
        row = b[it * 8: it * 8 + 8]
        if not row.any():
            break
        row = np.concatenate([row[:6], row[7:8], row[6:7]])  # slot 7 (prefetch) sits between 5 and 6
        d = np.diff(row)
        print(f"  it {it:2d} start {(row[0] - t0) / 1e3:7.2f} us | " + "  ".join(f"{names[k + 1]} +{d[k] / 1e3:.2f}" for k in range(7)))
