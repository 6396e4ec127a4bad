"""Correctness of the block's bgemm calls at the training shape (the exact Mat views of
block.py) against torch references.  python scripts/gemm_check.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat

S, R, P = 128, 256, 32
dev, BF = "cuda", torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
rnd = lambda *s: torch.randn(*s, device=dev, dtype=BF, generator=g)
rel = lambda a, b: ((a.float() - b.float()).norm() / b.float().norm()).item()
ab = rnd(S * R, 2 * P)
a3 = ab.view(S, R, 2 * P)[..., :P].float()
b3 = ab.view(S, R, 2 * P)[..., P:].float()
o = torch.empty(R, R, P, P, device=dev, dtype=BF)
ops.bgemm(Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0)),
          Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P),
          Mat(o, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P)), 1, R * P, R * P, S, alpha=1.0 / S)
ref = torch.einsum("sip,sjq->ijpq", a3, b3) / S
print("opm_fwd rel", rel(o, ref), "nan", torch.isnan(o).any().item())
do = rnd(R * R, P * P)
dab = torch.zeros(S * R, 2 * P, device=dev, dtype=BF)
ops.bgemm(Mat(do, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P)),
          Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P), offset=P),
          Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0)), 1, R * P, S, R * P, alpha=1.0 / S)
do4 = do.view(R, R, P, P).float()
ref = torch.einsum("ijpq,sjq->sip", do4, b3) / S
print("opm_da rel", rel(dab.view(S, R, 2 * P)[..., :P], ref))
ops.bgemm(Mat(do, lo=(1, P), split=(P, P), hi=(P * P, R * P * P)),
          Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P)),
          Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P), 1, R * P, S, R * P, alpha=1.0 / S)
ref = torch.einsum("ijpq,sip->sjq", do4, a3) / S
print("opm_db rel", rel(dab.view(S, R, 2 * P)[..., P:], ref))
rows = R * R
a_cm, b_cm = rnd(P, rows), rnd(P, rows)
t = torch.empty(P, R, R, device=dev, dtype=BF)
ops.bgemm(Mat(a_cm, lo=(R, 1), batch_stride=rows), Mat(b_cm, lo=(R, 1), batch_stride=rows),
          Mat(t, lo=(R, 1), batch_stride=rows), P, R, R, R)
print("tri_out rel", rel(t, torch.bmm(a_cm.view(P, R, R).float(), b_cm.view(P, R, R).float().transpose(1, 2))))
ops.bgemm(Mat(a_cm, lo=(1, R), batch_stride=rows), Mat(b_cm, lo=(1, R), batch_stride=rows),
          Mat(t, lo=(R, 1), batch_stride=rows), P, R, R, R)
print("tri_in rel", rel(t, torch.bmm(a_cm.view(P, R, R).float().transpose(1, 2), b_cm.view(P, R, R).float())))
