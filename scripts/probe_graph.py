"""Probe: host enqueue time vs device time of the 48-block fwd+bwd step, and the
same step captured as one CUDA graph."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2203_00854_b200.config import EvoConfig, synthetic_inputs
from paper_2203_00854_b200.evoformer import EvoformerStack

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 48
cfg = EvoConfig(128, 256, 256, 128, 8, 4, 32)
st = EvoformerStack(cfg, nb, seed=0)
m64, z64 = synthetic_inputs(cfg, 0)
rng = np.random.default_rng(1)
m = torch.tensor(m64, device="cuda").bfloat16(); z = torch.tensor(z64, device="cuda").bfloat16()
gm = torch.tensor(rng.normal(size=m64.shape), device="cuda").bfloat16()
gz = torch.tensor(rng.normal(size=z64.shape), device="cuda").bfloat16()
def step():
    st.zero_grad()
    return st.forward_backward(m, z, gm, gz)[0]
for _ in range(3): step()
torch.cuda.synchronize()
t0 = time.perf_counter(); step(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"eager: host enqueue {1e3*(t1-t0):.1f} ms, wall {1e3*(t2-t0):.1f} ms")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); [step() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
print(f"eager: {e0.elapsed_time(e1)/3:.1f} ms/step")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
try:
    with torch.cuda.graph(g):
        loss = step()
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0.record(); [g.replay() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
    print(f"graph: {e0.elapsed_time(e1)/3:.1f} ms/step  loss={loss.item():.4f}")
    print("mem GB", torch.cuda.max_memory_allocated()/1e9)
except Exception as exc:
    import traceback; traceback.print_exc()
