"""Upper bounds for optimisation targets: the bench step with one class of work removed (results
are garbage; only the timing is read).  python scripts/what_if.py <variant>
variants: base, nowgrad (weight-gradient GEMMs), nobgrad (bias column sums), noside (side stream off),
noattnbwd (attention backward kernels)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_00854_b200 import block, ops

v = sys.argv[1]
if v == "nowgrad":
    block._wgrad = lambda *a, **k: None
elif v == "nobgrad":
    block._bgrad = lambda *a, **k: None
    block._dbias_only = lambda *a, **k: None
elif v == "noside":
    block.SideStream.enabled = False
elif v == "noattnbwd":
    ops.attention_bwd = lambda *a, **k: None
elif v == "noopmbwd":
    _bg = ops.bgemm
    block.opm_bwd = lambda *a, **k: None
sys.argv = ["bench.py", "--no-cpu-baseline", "--no-e2e", "--steps", "4", "--warmup", "3"]
import bench
import io, contextlib, json
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
line = [l for l in buf.getvalue().splitlines() if l.startswith("{")][-1]
d = json.loads(line)
print(f"{v}: {d['ms_per_step']:.1f} ms/step")
