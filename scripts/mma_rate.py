"""tcgen05 SS-mode throughput vs N tile: evo_bgemm on a large square problem (MMA-bound),
N tile forced through EVO_BGEMM_BN.  python scripts/mma_rate.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat
M = N = K = 4096
a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda").bfloat16()
f = lambda: ops.bgemm(Mat(a, lo=(K, 1)), Mat(b, lo=(K, 1)), Mat(c, lo=(N, 1)), 1, M, N, K)
for _ in range(3): f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10): f()
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) / 10
print(f"BN={os.environ.get('EVO_BGEMM_BN','auto')}: {t*1e3:.1f} us {2*M*N*K/t/1e9:.0f} TF/s")
t2 = None
s.record()
for _ in range(10): torch.mm(a, b.t(), out=c)
e.record(); torch.cuda.synchronize()
print(f"cublas {s.elapsed_time(e)/10*1e3:.1f} us {2*M*N*K/(s.elapsed_time(e)/10)/1e9:.0f} TF/s")
