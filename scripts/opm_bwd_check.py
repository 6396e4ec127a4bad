"""evo_opm_bwd_factor (da, db without materialising do) vs a torch fp32 restatement, and its time
against the unfused backward (do = dy W^T on cuBLAS + the two tcgen05 contractions).
python scripts/opm_bwd_check.py [I J S Hz] ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_00854_b200 import ops
from paper_2203_00854_b200.ops import Mat

dev, BF, P = "cuda", torch.bfloat16, 32


def timeit(fn, it=10):
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


def rel(x, y):
    return ((x.float() - y.float()).norm() / y.float().norm()).item()


def case(I, J, S, Hz):
    g = torch.Generator(device=dev).manual_seed(I + 3 * J + S + Hz)
    a = torch.randn(S, I, P, device=dev, generator=g).to(BF)
    b = torch.randn(S, J, P, device=dev, generator=g).to(BF)
    w = (torch.randn(P * P, Hz, device=dev, generator=g) / 32).to(BF)
    dy = torch.randn(I * J, Hz, device=dev, generator=g).to(BF)
    a_t, b_t = a.permute(1, 2, 0).contiguous(), b.permute(1, 2, 0).contiguous()
    al = 1.0 / S
    do = (dy.float() @ w.float().t()).view(I, J, P, P)
    da_ref = al * torch.einsum("ijpq,sjq->sip", do.to(BF).float(), b.float())
    db_ref = al * torch.einsum("ijpq,sip->sjq", do.to(BF).float(), a.float())
    dab = torch.empty(S, I, 2 * P, device=dev, dtype=BF)   # da into columns [0, P) of an [S*I, 2P] buffer
    dbf = torch.empty(S, J, P, device=dev, dtype=torch.float32)
    f = lambda: (ops.opm_bwd_factor(0, dy, w, b_t, I, J, S, P, Hz, al, dab, I * 2 * P, 0, 2 * P),
                 ops.opm_bwd_factor(1, dy, w, a_t, J, I, S, P, Hz, al, dbf, J * P, 0, P))
    f()
    torch.cuda.synchronize()
    ea, eb = rel(dab[..., :P], da_ref), rel(dbf, db_ref)
    t = timeit(f)
    t_u = float("nan")
    if I == J:  # the unfused backward of block.opm_bwd
        R = I
        ab = torch.cat([a, b], -1).reshape(S * R, 2 * P)
        dab2 = torch.empty(S * R, 2 * P, device=dev, dtype=BF)

        def unf():
            do_ = dy @ w.t()
            dO_A = Mat(do_, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P))
            Cda = Mat(dab2, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0))
            dO_T = Mat(do_, lo=(1, P), split=(P, P), hi=(P * P, R * P * P))
            ops.bgemm(dO_A, Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P), offset=P), Cda, 1, R * P, S, R * P,
                      alpha=al)
            ops.bgemm(dO_T, Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P)),
                      Mat(dab2, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P), 1, R * P, S, R * P, alpha=al)
        t_u = timeit(unf)
    print(f"I={I} J={J} S={S} Hz={Hz}: rel err da {ea:.2e} db {eb:.2e} | fused {t:.1f} us, unfused {t_u:.1f} us",
          flush=True)
    assert ea < 1e-2 and eb < 1e-2, (ea, eb)


shapes = [(32, 32, 16, 64), (64, 32, 128, 128), (32, 64, 48, 64), (32, 96, 96, 128), (256, 256, 128, 128)]
if len(sys.argv) > 1:
    v = list(map(int, sys.argv[1:]))
    shapes = [tuple(v[i:i + 4]) for i in range(0, len(v), 4)]
for s_ in shapes:
    case(*s_)
