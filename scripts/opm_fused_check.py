"""Fused OuterProductMean forward (evo_opm_fused_fwd) vs a torch fp32 restatement, and its time
against the unfused path (tcgen05 contraction writing o + cuBLAS o @ W_o).
python scripts/opm_fused_check.py [I J S Hz] ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat

dev, BF = "cuda", torch.bfloat16
P = 32


def timeit(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


def case(I, J, S, Hz):
    g = torch.Generator(device=dev).manual_seed(I + J + S + Hz)
    a = torch.randn(S, I, P, device=dev, generator=g).to(BF)
    b = torch.randn(S, J, P, device=dev, generator=g).to(BF)
    w = (torch.randn(P * P, Hz, device=dev, generator=g) / 32).to(BF)
    a_t = ops.opm_transpose(a.view(S * I, P), S, I, P)
    b_t = ops.opm_transpose(b.view(S * J, P), S, J, P)
    assert torch.equal(a_t, a.permute(1, 2, 0)) and torch.equal(b_t, b.permute(1, 2, 0))
    if I == J:  # merged [a | b] rows, both outputs of one call
        a2, b2 = ops.opm_transpose(torch.cat([a, b], -1).view(S * I, 2 * P), S, I, P, both=True)
        assert torch.equal(a2, a_t) and torch.equal(b2, b_t)
    o_ref = (torch.einsum("sip,sjq->ijpq", a.float(), b.float()) / S).to(BF).contiguous()
    y_ref = o_ref.view(I * J, P * P).float() @ w.float()
    o_sv = torch.empty(I, J, P, P, device=dev, dtype=BF)
    y = ops.opm_fused_fwd(a_t, b_t, w, I, J, S, P, Hz, 1.0 / S, o_save=o_sv)
    torch.cuda.synchronize()
    ey = ((y.float() - y_ref).norm() / y_ref.norm()).item()
    eo = ((o_sv.float() - o_ref.float()).norm() / o_ref.float().norm()).item()
    y2 = ops.opm_fused_fwd(a_t, b_t, w, I, J, S, P, Hz, 1.0 / S)
    ey2 = ((y2.float() - y.float()).abs().max()).item()
    t_f = timeit(lambda: ops.opm_fused_fwd(a_t, b_t, w, I, J, S, P, Hz, 1.0 / S, y=y2))
    t_fs = timeit(lambda: ops.opm_fused_fwd(a_t, b_t, w, I, J, S, P, Hz, 1.0 / S, y=y2, o_save=o_sv))
    t_tr = timeit(lambda: ops.opm_transpose(a.view(S * I, P), S, I, P))
    # unfused: contraction into o (tcgen05 bgemm) + cuBLAS
    ab = torch.cat([a, b], -1).reshape(S * I, 2 * P) if I == J else None
    t_u = float("nan")
    if ab is not None:
        o = torch.empty(I, J, P, P, device=dev, dtype=BF)
        A = Mat(ab, lo=(1, I * 2 * P), split=(P, 0), hi=(2 * P, 0))
        B = Mat(ab, lo=(1, I * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P)
        Cm = Mat(o, lo=(P, 1), split=(P, P), hi=(J * P * P, P * P))

        def unf():
            ops.bgemm(A, B, Cm, 1, I * P, J * P, S, alpha=1.0 / S)
            torch.mm(o.view(I * J, P * P), w)
        t_u = timeit(unf)
    fl = 2 * I * J * P * P * (S + Hz)
    print(f"I={I} J={J} S={S} Hz={Hz}: rel err y {ey:.2e}  o {eo:.2e}  rerun-maxdiff {ey2:.1e} | "
          f"fused {t_f:.1f} us ({fl / t_f / 1e6:.0f} TF/s), +save_o {t_fs:.1f} us, transpose {t_tr:.1f} us, "
          f"unfused {t_u:.1f} us", flush=True)
    assert ey < 1e-2 and eo < 1e-2 and ey2 == 0.0, (ey, eo, ey2)


shapes = [(32, 32, 16, 32), (32, 64, 32, 64), (64, 32, 128, 128), (32, 64, 48, 64), (32, 32, 96, 64),
          (256, 256, 128, 128), (32, 256, 128, 128), (1024, 1024, 128, 128)]
if len(sys.argv) > 1:
    v = list(map(int, sys.argv[1:]))
    shapes = [tuple(v[i:i + 4]) for i in range(0, len(v), 4)]
for s in shapes:
    case(*s)
