"""Per-kernel numerics of libevo.so on the GPU vs plain PyTorch fp32 references
of the same op (bf16 storage -> tolerances stated per test)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU too; the gpu marker deselects
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2203_00854_b200 import _lib, ops  # noqa: E402
from paper_2203_00854_b200.ops import Mat, Strided  # noqa: E402

DEV = "cuda"


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("cols", [32, 128, 256])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_layernorm_fwd_bwd(cols, dtype):
    g = torch.Generator(device=DEV).manual_seed(cols)
    rows = 1000
    x = (torch.randn(rows, cols, device=DEV, generator=g) * 2 + 0.5).to(dtype)
    gamma = torch.randn(cols, device=DEV, generator=g)
    beta = torch.randn(cols, device=DEV, generator=g)
    y, mean, rstd = ops.layernorm_fwd(x, gamma, beta, rows, cols)
    xr = x.float().requires_grad_(True)
    gr = gamma.clone().requires_grad_(True)
    br = beta.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (cols,), gr, br, eps=1e-5)
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
    assert rel(y, yr) < tol
    dy = torch.randn(rows, cols, device=DEV, generator=g).to(dtype)
    yr.backward(dy.float())
    dg = torch.zeros(cols, device=DEV)
    db = torch.zeros(cols, device=DEV)
    dx = ops.layernorm_bwd(dy, x, gamma, mean, rstd, rows, cols, dgamma=dg, dbeta=db)
    assert rel(dx, xr.grad) < tol
    assert rel(dg, gr.grad) < tol
    assert rel(db, br.grad) < 1e-5
    # accumulate mode
    base = torch.randn(rows, cols, device=DEV, generator=g).to(dtype)
    acc = base.clone()
    ops.layernorm_bwd(dy, x, gamma, mean, rstd, rows, cols, dx=acc, accumulate=True)
    assert rel(acc, base.float() + xr.grad) < tol


@pytest.mark.parametrize("P,R,with_res", [(32, 777, False), (32, 776, False), (32, 4096, True), (16, 1000, True),
                                          (64, 264, False)])
def test_layernorm_strided_channel_major(P, R, with_res):
    """channel-major LN (the triangle update's t[p][rows]): thread-per-row kernel for odd strides,
    the tiled kernel (16-byte tile loads through shared memory) when the channel stride is a
    multiple of 8"""
    g = torch.Generator(device=DEV).manual_seed(3)
    t_cm = torch.randn(P, R, device=DEV, generator=g).bfloat16()  # [channel][row]
    gamma = torch.randn(P, device=DEV, generator=g)
    beta = torch.randn(P, device=DEV, generator=g)
    y, mean, rstd = ops.layernorm_fwd(t_cm, gamma, beta, R, P, x_rs=1, x_cs=R)
    xr = t_cm.float().t().contiguous().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (P,), gamma, beta, eps=1e-5)
    assert rel(y, yr) < 1e-2
    dy = torch.randn(R, P, device=DEV, generator=g).bfloat16()
    yr.backward(dy.float())
    dx = torch.empty_like(t_cm)
    dg = torch.zeros(P, device=DEV)
    db = torch.zeros(P, device=DEV)
    res = torch.randn(P, R, device=DEV, generator=g).bfloat16() if with_res else None
    ops.layernorm_bwd(dy, t_cm, gamma, mean, rstd, R, P, x_rs=1, x_cs=R, dx=dx, dgamma=dg, dbeta=db, res=res)
    ref = xr.grad + (res.float().t() if with_res else 0)
    assert rel(dx.float().t(), ref) < 1e-2
    assert rel(db, dy.float().sum(0)) < 1e-5
    xh = (xr.detach() - xr.detach().mean(-1, keepdim=True)) * torch.rsqrt(xr.detach().var(-1, unbiased=False, keepdim=True) + 1e-5)
    assert rel(dg, (dy.float() * xh).sum(0)) < 1e-3


def test_layernorm_rowdot():
    g = torch.Generator(device=DEV).manual_seed(4)
    rows, cols, k = 4096, 128, 8
    x = torch.randn(rows, cols, device=DEV, generator=g).bfloat16()
    gamma = torch.randn(cols, device=DEV, generator=g)
    beta = torch.randn(cols, device=DEV, generator=g)
    w = torch.randn(cols, k, device=DEV, generator=g)
    out = torch.empty(k, rows, device=DEV, dtype=torch.bfloat16)
    ln = torch.empty(rows, cols, device=DEV, dtype=torch.bfloat16)
    ops.layernorm_rowdot_fwd(x, gamma, beta, w, rows, cols, out, rows, ln_out=ln)
    lnr = torch.nn.functional.layer_norm(x.float(), (cols,), gamma, beta, eps=1e-5)
    assert rel(ln, lnr) < 1e-2
    assert rel(out, (lnr @ w).t()) < 1e-2


@pytest.mark.parametrize("K", [8, 100, 256, 1024])
def test_softmax_fwd_bwd(K):
    g = torch.Generator(device=DEV).manual_seed(K)
    B, H, Q = 3, 4, 17
    x = torch.randn(B, H, Q, K, device=DEV, generator=g).bfloat16()
    bias = torch.randn(1, H, Q, K, device=DEV, generator=g).bfloat16()
    mask = torch.where(torch.rand(B, 1, 1, K, device=DEV, generator=g) < 0.3, -1e30, 0.0)
    scale = 0.3
    y = ops.softmax_fwd(x, bias, mask, scale)
    yr = torch.softmax((x.float() + bias.float()) * scale + mask, -1)
    assert (y.float() - yr).abs().max().item() < 1e-2
    dy = torch.randn_like(x)
    dx = ops.softmax_bwd(y, dy, scale)
    xr = x.float().requires_grad_(True)
    torch.softmax((xr + bias.float()) * scale + mask, -1).backward(dy.float())
    assert rel(dx, xr.grad) < 2e-2


def test_softmax_golden_set_fp32():
    import numpy as np
    import os
    from conftest import GOLDEN
    gs = np.load(os.path.join(GOLDEN, "golden_softmax.npz"))
    worst = 0.0
    for i in range(100):
        x = torch.tensor(gs[f"c{i}/x"], dtype=torch.float32, device=DEV)
        m = torch.tensor(gs[f"c{i}/mask"], dtype=torch.float32, device=DEV)
        b = torch.tensor(gs[f"c{i}/bias"], dtype=torch.float32, device=DEV)
        y = ops.softmax_fwd(x, b, m, 1.0)
        worst = max(worst, float(np.max(np.abs(y.cpu().double().numpy() - gs[f"c{i}/y"]))))
    assert worst < 2e-6


def _mk(shape, g):
    return torch.randn(*shape, device=DEV, generator=g).bfloat16()


@pytest.mark.parametrize("am,bm", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K,batch", [(256, 256, 256, 4), (200, 136, 72, 3), (8192 // 8, 1024, 128, 1)])
def test_bgemm_majors(am, bm, M, N, K, batch):
    g = torch.Generator(device=DEV).manual_seed(M + N + K)
    A = _mk((batch, K, M) if am else (batch, M, K), g)
    B = _mk((batch, K, N) if bm else (batch, N, K), g)
    Cc = torch.zeros(batch, M, N, device=DEV, dtype=torch.float32)
    Aref = A.float().transpose(1, 2) if am else A.float()
    Bref = B.float().transpose(1, 2) if bm else B.float()
    ma = Mat(A, lo=(1, M) if am else (K, 1), batch_stride=M * K)
    mb = Mat(B, lo=(1, N) if bm else (K, 1), batch_stride=N * K)
    mc = Mat(Cc, lo=(N, 1), batch_stride=M * N)
    ops.bgemm(ma, mb, mc, batch, M, N, K, alpha=0.5)
    ref = 0.5 * Aref @ Bref.transpose(1, 2)
    assert rel(Cc, ref) < 1e-5
    # bf16 output, column-major C, beta accumulate
    Cb = torch.randn(batch, N, M, device=DEV, generator=g).bfloat16()
    C0 = Cb.float().clone()
    mcb = Mat(Cb, lo=(1, M), batch_stride=M * N)
    ops.bgemm(ma, mb, mcb, batch, M, N, K, alpha=1.0, beta=1.0)
    assert rel(Cb.float().transpose(1, 2), ref * 2 + C0.transpose(1, 2)) < 1e-2


def test_bgemm_opm_layout():
    """outer-product contraction straight into o[i][j][p][q] (evoformer.py:253)."""
    g = torch.Generator(device=DEV).manual_seed(7)
    S, R, P = 64, 48, 16
    ab = _mk((S, R, 2 * P), g)  # [a | b] projections, row stride 2P
    o = torch.empty(R, R, P, P, device=DEV, dtype=torch.bfloat16)
    A = Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0))
    B = Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P)
    Cm = Mat(o, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P))
    ops.bgemm(A, B, Cm, 1, R * P, R * P, S, alpha=1.0 / S)
    a, b = ab[..., :P].float(), ab[..., P:].float()
    ref = torch.einsum("sip,sjq->ijpq", a, b) / S
    assert rel(o, ref) < 1e-2


@pytest.mark.parametrize("S,R,P", [(64, 48, 16), (64, 64, 32)])
def test_bgemm_opm_fwd_bwd_layouts(S, R, P):
    """the three OPM contractions with block.py's exact views; P = 32 takes the TMA path with
    64-byte swizzled boxes (32-element runs), P = 16 the cp.async path"""
    g = torch.Generator(device=DEV).manual_seed(11)
    ab = _mk((S * R, 2 * P), g)
    a3, b3 = ab.view(S, R, 2 * P)[..., :P].float(), ab.view(S, R, 2 * P)[..., P:].float()
    o = torch.empty(R, R, P, P, device=DEV, dtype=torch.bfloat16)
    ops.bgemm(Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0)),
              Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P),
              Mat(o, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P)), 1, R * P, R * P, S, alpha=1.0 / S)
    assert rel(o, torch.einsum("sip,sjq->ijpq", a3, b3) / S) < 1e-2
    do = _mk((R * R, P * P), g)
    do4 = do.view(R, R, P, P).float()
    dab = torch.zeros(S * R, 2 * P, device=DEV, dtype=torch.bfloat16)
    ops.bgemm(Mat(do, lo=(P, 1), split=(P, P), hi=(R * P * P, P * P)),
              Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P), offset=P),
              Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0)), 1, R * P, S, R * P, alpha=1.0 / S)
    assert rel(dab.view(S, R, 2 * P)[..., :P], torch.einsum("ijpq,sjq->sip", do4, b3) / S) < 1e-2
    ops.bgemm(Mat(do, lo=(1, P), split=(P, P), hi=(P * P, R * P * P)),
              Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P)),
              Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P), 1, R * P, S, R * P, alpha=1.0 / S)
    assert rel(dab.view(S, R, 2 * P)[..., P:], torch.einsum("ijpq,sip->sjq", do4, a3) / S) < 1e-2


def _attn_ref(q, k, v, g, bias, scale):
    # q,k,v,g: [B, H, L, c] fp32; bias broadcastable to [B, H, L, L]
    s = q @ k.transpose(-1, -2)
    if bias is not None:
        s = s + bias
    a = torch.softmax(s * scale, -1)
    o = a @ v
    return torch.sigmoid(g) * o, o


@pytest.mark.parametrize("L,c,H,mode", [(256, 32, 8, "full"), (128, 32, 8, "none"), (256, 32, 4, "key"),
                                        (100, 16, 2, "full"), (300, 64, 2, "key"), (40, 8, 4, "none"),
                                        (600, 32, 2, "key"), (1024, 32, 1, "full")])
def test_attention_fwd_bwd_ws(L, c, H, mode):
    """the warp-specialised long-sequence forward (attention_ws.cu) forced at every L"""
    test_attention_fwd_bwd(L, c, H, mode, flags=_lib.EVO_ATTN_FORCE_WS)


@pytest.mark.parametrize("L,c,H,mode", [(256, 32, 8, "full"), (128, 32, 8, "none"), (256, 32, 4, "key"),
                                        (100, 16, 2, "full"), (300, 64, 2, "key"), (40, 8, 4, "none")])
def test_attention_fwd_bwd(L, c, H, mode, B=3, flags=0):
    gen = torch.Generator(device=DEV).manual_seed(L * c + H)
    ld = 3 * H * c + (8 if mode == "key" else 0)
    qkv = _mk((B, L, ld), gen)
    gp = _mk((B, L, H * c), gen)
    if mode == "full":
        bias = _mk((H, L, L), gen)
        bias_s = (0, L * L, L, 1)
        bias_t = bias
        bref = bias.float()[None]
    elif mode == "key":
        bias_t = qkv
        bias_s = (L * ld, 1, 0, ld)
        bref = qkv[..., 3 * H * c:3 * H * c + H].float().permute(0, 2, 1)[:, :, None, :]
    else:
        bias_t, bias_s, bref = None, (0, 0, 0, 0), None
    og = torch.empty(B, L, H * c, device=DEV, dtype=torch.bfloat16)
    orw = torch.empty_like(og)
    lse = torch.empty(B, H, L, device=DEV)
    scale = 1 / math.sqrt(c)
    d = ops.attention_desc(Strided(qkv, L * ld, ld, 0), Strided(qkv, L * ld, ld, H * c),
                           Strided(qkv, L * ld, ld, 2 * H * c), Strided(gp, L * H * c, H * c),
                           Strided(og, L * H * c, H * c), Strided(orw, L * H * c, H * c), lse,
                           B, L, H, c, scale, bias=bias_t, bias_s=bias_s,
                           bias_off=3 * H * c if mode == "key" else 0, flags=flags)
    ops.attention_fwd(d)
    torch.cuda.synchronize()
    split = lambda t, i: t[..., i * H * c:(i + 1) * H * c].float().reshape(B, L, H, c).permute(0, 2, 1, 3)
    q = split(qkv, 0).requires_grad_(True)
    k = split(qkv, 1).requires_grad_(True)
    v = split(qkv, 2).requires_grad_(True)
    gg = gp.float().reshape(B, L, H, c).permute(0, 2, 1, 3).requires_grad_(True)
    br = bref.clone().requires_grad_(True) if bref is not None else None
    out_r, o_r = _attn_ref(q, k, v, gg, br, scale)
    to_blh = lambda t: t.permute(0, 2, 1, 3).reshape(B, L, H * c)
    assert rel(og, to_blh(out_r)) < 1e-2
    assert rel(orw, to_blh(o_r)) < 1e-2
    s_ref = (q @ k.transpose(-1, -2) + (br if br is not None else 0)) * scale
    assert (lse - torch.logsumexp(s_ref, -1)).abs().max().item() < 2e-2

    # backward
    dout = _mk((B, L, H * c), gen)
    out_r.backward(dout.float().reshape(B, L, H, c).permute(0, 2, 1, 3))
    dqkv = torch.zeros_like(qkv)
    dgp = torch.empty_like(gp)
    if mode == "full":
        dbias = torch.zeros(H, L, L, device=DEV)
        dbias_s = (0, L * L, L, 1)
    elif mode == "key":
        dbias = torch.zeros(B, H, L, device=DEV)
        dbias_s = (H * L, L, 0, 1)
    else:
        dbias, dbias_s = None, (0, 0, 0, 0)
    ws = torch.empty(ops.attention_bwd_workspace(B, L, H, c, mode == "full"), dtype=torch.uint8, device=DEV)
    ops.attention_bwd(d, Strided(dout, L * H * c, H * c), Strided(dqkv, L * ld, ld, 0),
                      Strided(dqkv, L * ld, ld, H * c), Strided(dqkv, L * ld, ld, 2 * H * c),
                      Strided(dgp, L * H * c, H * c), ws, dbias=dbias, dbias_s=dbias_s)
    torch.cuda.synchronize()
    assert rel(dqkv[..., :H * c], to_blh(q.grad)) < 2e-2
    assert rel(dqkv[..., H * c:2 * H * c], to_blh(k.grad)) < 2e-2
    assert rel(dqkv[..., 2 * H * c:3 * H * c], to_blh(v.grad)) < 2e-2
    assert rel(dgp, to_blh(gg.grad)) < 2e-2
    if mode == "full":
        assert rel(dbias, br.grad.sum(0)) < 2e-2
    elif mode == "key":
        assert rel(dbias, br.grad[:, :, 0, :]) < 2e-2


@pytest.mark.parametrize("mode,H", [("none", 8), ("key", 4), ("full", 8)])
def test_attention_persistent_units(mode, H):
    """B*H*L/128 units well above the persistent forward grid (4 CTAs/SM) and the backward's
    (2 CTAs/SM): the cross-unit prefetch paths (next unit's Q/K/V under the last tile, the
    double-buffered query tiles) run many times per CTA"""
    test_attention_fwd_bwd(256, 32, H, mode, B=160)


def test_attention_fwd_full_bias_smem_flag():
    """the smem-staged full-bias forward (msa_row) equals the global-load variant bitwise"""
    gen = torch.Generator(device=DEV).manual_seed(5)
    B, L, H, c = 40, 256, 8, 32
    qkv = _mk((B, L, 3 * H * c), gen)
    gp = _mk((B, L, H * c), gen)
    bias = _mk((H, L, L), gen)
    outs = []
    for flags in (0, _lib.EVO_ATTN_NO_BIAS_SMEM):
        og = torch.empty(B, L, H * c, device=DEV, dtype=torch.bfloat16)
        orw = torch.empty_like(og)
        lse = torch.empty(B, H, L, device=DEV)
        ld = 3 * H * c
        d = ops.attention_desc(Strided(qkv, L * ld, ld, 0), Strided(qkv, L * ld, ld, H * c),
                               Strided(qkv, L * ld, ld, 2 * H * c), Strided(gp, L * H * c, H * c),
                               Strided(og, L * H * c, H * c), Strided(orw, L * H * c, H * c), lse,
                               B, L, H, c, 1 / math.sqrt(c), bias=bias, bias_s=(0, L * L, L, 1), flags=flags)
        ops.attention_fwd(d)
        torch.cuda.synchronize()
        outs.append((og, orw, lse))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("rows", [1000, 999])
def test_tri_gate_and_residuals(rows):
    gen = torch.Generator(device=DEV).manual_seed(11)
    hz, p = 32, 16
    y = _mk((rows, hz + 4 * p), gen)
    a_cm = torch.empty(p, rows, device=DEV, dtype=torch.bfloat16)
    b_cm = torch.empty_like(a_cm)
    ops.tri_gate_fwd(y, rows, hz, p, a_cm, b_cm)
    yf = y.float().requires_grad_(True)
    a = torch.sigmoid(yf[:, hz:hz + p]) * yf[:, hz + p:hz + 2 * p]
    b = torch.sigmoid(yf[:, hz + 2 * p:hz + 3 * p]) * yf[:, hz + 3 * p:]
    assert rel(a_cm, a.t()) < 1e-2 and rel(b_cm, b.t()) < 1e-2
    da = torch.randn(p, rows, device=DEV, generator=gen)
    db = torch.randn(p, rows, device=DEV, generator=gen)
    dy = torch.zeros_like(y)
    dsum = torch.zeros(4 * p, device=DEV)
    ops.tri_gate_bwd(y, da, db, rows, hz, p, dy, dsum=dsum)
    (a * da.t()).sum().add((b * db.t()).sum()).backward()
    assert rel(dy[:, hz:], yf.grad[:, hz:]) < 1e-2
    assert rel(dsum, yf.grad[:, hz:].sum(0)) < 1e-4      # fp32 sums of the unrounded values

    # gated residual with the g gate stored in Y (row stride hz + 4p)
    res = _mk((rows, hz), gen)
    y2 = _mk((rows, hz), gen)
    bias = torch.randn(hz, device=DEV, generator=gen)
    out = ops.gated_residual_fwd(res, y2, bias, rows, hz, gp=y, gp_rs=hz + 4 * p)
    y2f = y2.float().requires_grad_(True)
    bf = bias.clone().requires_grad_(True)
    gpf = y.float()[:, :hz].requires_grad_(True)
    ref = res.float() + torch.sigmoid(gpf) * (y2f + bf)
    assert rel(out, ref) < 1e-2
    dout = _mk((rows, hz), gen)
    ref.backward(dout.float())
    dy2 = torch.empty_like(y2)
    dgp = torch.zeros_like(y)
    dbias = torch.zeros(hz, device=DEV)
    dgsum = torch.zeros(hz, device=DEV)
    ops.gated_residual_bwd(dout, rows, hz, y=y2, bias=bias, gp=y, gp_rs=hz + 4 * p, dy=dy2, dgp=dgp,
                           dgp_rs=hz + 4 * p, dbias=dbias, dgp_sum=dgsum)
    assert rel(dy2, y2f.grad) < 1e-2
    assert rel(dgp[:, :hz], gpf.grad) < 1e-2
    assert rel(dbias, bf.grad) < 1e-3
    assert rel(dgsum, gpf.grad.sum(0)) < 1e-4

    # bias + relu
    h = _mk((rows, 64), gen)
    h0 = h.float().clone()
    b1 = torch.randn(64, device=DEV, generator=gen)
    ops.bias_act_fwd(h, b1, rows, 64)
    assert rel(h, torch.relu(h0 + b1)) < 1e-2
    dh = _mk((rows, 64), gen)
    db1 = torch.zeros(64, device=DEV)
    dyy = ops.bias_act_bwd(dh, h, rows, 64, dbias=db1)
    want = dh.float() * (h.float() > 0)
    assert rel(dyy, want) < 1e-2 and rel(db1, want.sum(0)) < 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("cols,gated,rows", [(32, False, 1000), (64, False, 777), (128, False, 4099), (128, True, 513),
                                             (256, False, 300)])
def test_residual_layernorm_fwd(cols, gated, rows):
    """fused residual epilogue + next module's LayerNorm == gated_residual_fwd then layernorm_fwd"""
    gen = torch.Generator(device=DEV).manual_seed(cols + rows)
    res = _mk((rows, cols), gen)
    y = _mk((rows, cols + 16), gen)[:, :cols]
    bias = torch.randn(cols, device=DEV, generator=gen)
    gp = _mk((rows, 2 * cols), gen) if gated else None
    gam = torch.randn(cols, device=DEV, generator=gen)
    bet = torch.randn(cols, device=DEV, generator=gen)
    kw = dict(gp=gp, gp_rs=2 * cols) if gated else {}
    want = ops.gated_residual_fwd(res, y, bias, rows, cols, y_rs=cols + 16, **kw)
    wln, wmu, wrs = ops.layernorm_fwd(want, gam, bet, rows, cols)
    out, ln, mu, rs = ops.residual_layernorm_fwd(res, y, bias, rows, cols, gam, bet, y_rs=cols + 16, **kw)
    assert torch.equal(out, want)
    assert torch.allclose(mu, wmu, atol=1e-5, rtol=1e-5) and torch.allclose(rs, wrs, atol=1e-3, rtol=1e-4)
    assert rel(ln, wln) < 1e-2


@pytest.mark.gpu
def test_count_nonfinite():
    x = torch.zeros(1000, device=DEV)
    x[3] = float("inf")
    x[500] = float("nan")
    assert ops.count_nonfinite(x) == 2


@pytest.mark.parametrize("rows,cols", [(32768, 256), (65536, 128), (1000, 1024), (7, 392)])
def test_colsum(rows, cols):
    gen = torch.Generator(device=DEV).manual_seed(rows)
    x = torch.randn(rows, cols, device=DEV, generator=gen).bfloat16()
    out = torch.ones(cols, device=DEV)
    ops.colsum(x, out)
    assert rel(out - 1, x.float().sum(0)) < 1e-5


@pytest.mark.parametrize("am,rows_contig", [(False, True), (True, True), (False, False)])
def test_bgemm_split_k(am, rows_contig):
    """long-K, few-tile products (the OPM backward shapes) take the split-K path."""
    from paper_2203_00854_b200 import _lib
    g = torch.Generator(device=DEV).manual_seed(99)
    M, N, K = 1024, 128, 8192
    assert _lib.load().evo_bgemm_workspace(1, M, N, K) > 0
    A = _mk((K, M) if am else (M, K), g)
    B = _mk((N, K), g)
    ma = Mat(A, lo=(1, M) if am else (K, 1))
    mb = Mat(B, lo=(K, 1))
    Cb = torch.randn(N, M, device=DEV, generator=g).bfloat16() if rows_contig else \
        torch.randn(M, N, device=DEV, generator=g).bfloat16()
    C0 = Cb.float().clone()
    mc = Mat(Cb, lo=(1, M) if rows_contig else (N, 1))
    ops.bgemm(ma, mb, mc, 1, M, N, K, alpha=0.25, beta=1.0)
    ref = 0.25 * ((A.float().t() if am else A.float()) @ B.float().t())
    got = Cb.float().t() if rows_contig else Cb.float()
    base = C0.t() if rows_contig else C0
    assert rel(got, ref + base) < 1e-2


def test_layernorm_rowdot_bwd():
    g = torch.Generator(device=DEV).manual_seed(41)
    rows, cols, k = 3000, 128, 8
    x = torch.randn(rows, cols, device=DEV, generator=g).bfloat16()
    gamma = torch.randn(cols, device=DEV, generator=g)
    beta = torch.randn(cols, device=DEV, generator=g)
    w = torch.randn(cols, k, device=DEV, generator=g)
    out = torch.empty(k, rows, device=DEV, dtype=torch.bfloat16)
    mean = torch.empty(rows, device=DEV)
    rstd = torch.empty(rows, device=DEV)
    ops.layernorm_rowdot_fwd(x, gamma, beta, w, rows, cols, out, rows, mean=mean, rstd=rstd)
    dout = torch.randn(k, rows, device=DEV, generator=g)
    res = torch.randn(rows, cols, device=DEV, generator=g).bfloat16()
    dx = torch.empty_like(x)
    dg, db, dw = torch.zeros(cols, device=DEV), torch.zeros(cols, device=DEV), torch.zeros(cols, k, device=DEV)
    ops.layernorm_rowdot_bwd(x, gamma, beta, w, dout, rows, mean, rstd, rows, cols, dx, res, dg, db, dw)
    xr, gr, br, wr = (t.float().clone().requires_grad_(True) for t in (x, gamma, beta, w))
    y = torch.nn.functional.layer_norm(xr, (cols,), gr, br, eps=1e-5) @ wr
    y.backward(dout.t())
    assert rel(dx.float() - res.float(), xr.grad) < 2e-2
    assert rel(dg, gr.grad) < 1e-2 and rel(db, br.grad) < 1e-2 and rel(dw, wr.grad) < 1e-2


@pytest.mark.parametrize("I,J,S,Hz", [(32, 32, 16, 32), (32, 64, 48, 64), (64, 32, 128, 128), (32, 40, 96, 64),
                                      (256, 256, 128, 128)])
def test_opm_fused_fwd(I, J, S, Hz):
    """evo_opm_fused_fwd (+ evo_opm_transpose) vs fp32 torch: o = einsum(sip,sjq->ijpq)/S rounded to bf16 (as
    the unfused path stores it), y = o @ W_o.  The stored o is the same bf16 tensor up to fp32 summation order."""
    P = 32
    g = torch.Generator(device=DEV).manual_seed(I * 7 + J + S + Hz)
    a = torch.randn(S, I, P, device=DEV, generator=g).bfloat16()
    b = torch.randn(S, J, P, device=DEV, generator=g).bfloat16()
    w = (torch.randn(P * P, Hz, device=DEV, generator=g) / 32).bfloat16()
    assert ops.opm_fused_supported(I, J, S, P, Hz)
    a_t = ops.opm_transpose(a.view(S * I, P), S, I, P)
    b_t = ops.opm_transpose(b.view(S * J, P), S, J, P)
    assert torch.equal(a_t, a.permute(1, 2, 0)) and torch.equal(b_t, b.permute(1, 2, 0))
    n = min(I, J)
    ab = torch.cat([a[:, :n], b[:, :n]], -1).reshape(S * n, 2 * P)  # merged [a | b] rows: both outputs of one call
    a2, b2 = ops.opm_transpose(ab, S, n, P, both=True)
    assert torch.equal(a2, a_t[:n]) and torch.equal(b2, b_t[:n])
    o_ref = (torch.einsum("sip,sjq->ijpq", a.float(), b.float()) / S).bfloat16().contiguous()
    y_ref = o_ref.view(I * J, P * P).float() @ w.float()
    o = torch.empty(I, J, P, P, device=DEV, dtype=torch.bfloat16)
    y = ops.opm_fused_fwd(a_t, b_t, w, I, J, S, P, Hz, 1.0 / S, o_save=o)
    y2 = ops.opm_fused_fwd(a_t, b_t, w, I, J, S, P, Hz, 1.0 / S)  # inference form: no o
    torch.cuda.synchronize()
    assert rel(o, o_ref) < 1e-3, rel(o, o_ref)
    assert rel(y, y_ref) < 5e-3, rel(y, y_ref)
    assert torch.equal(y, y2)


def test_opm_fused_rejects_unsupported():
    t = torch.zeros(32, 16, 32, device=DEV, dtype=torch.bfloat16)
    assert not ops.opm_fused_supported(32, 32, 32, 16, 64)   # hidden_proj 16
    assert not ops.opm_fused_supported(48, 32, 32, 32, 64)   # I % 32
    assert not ops.opm_fused_supported(32, 32, 256, 32, 64)  # N_s > 128
    with pytest.raises(Exception):
        ops.opm_fused_fwd(t, t, torch.zeros(256, 64, device=DEV, dtype=torch.bfloat16), 32, 32, 32, 16, 64, 1.0)


@pytest.mark.parametrize("rows,M,N", [(65536, 128, 392), (32768, 256, 64), (65536, 32, 128), (4096, 1024, 256), (256, 64, 256),
                                      (1000, 64, 136)])
def test_wgrad_accumulates(rows, M, N):
    """evo_wgrad: dW += X^T dY in fp32 (split-K partials reduced in a fixed order) vs fp32 torch;
    called twice onto a strided fp32 view it accumulates; bitwise repeatable."""
    g = torch.Generator(device=DEV).manual_seed(rows + M + N)
    x = torch.randn(rows, M, device=DEV, generator=g).bfloat16()
    dy = torch.randn(rows, N, device=DEV, generator=g).bfloat16()
    base = torch.randn(M, N + 8, device=DEV, generator=g)
    dw = base.clone()[:, :N]
    ref = base[:, :N] + 2 * (x.float().t() @ dy.float())
    ops.wgrad(x, dy, dw)
    ops.wgrad(x, dy, dw)
    assert rel(dw, ref) < 1e-5, rel(dw, ref)
    dw2 = base.clone()[:, :N]
    ops.wgrad(x, dy, dw2)
    ops.wgrad(x, dy, dw2)
    assert torch.equal(dw, dw2)


@pytest.mark.parametrize("I,J,S,Hz", [(32, 32, 16, 64), (64, 32, 128, 128), (32, 96, 96, 128), (256, 256, 128, 128)])
def test_opm_bwd_factor(I, J, S, Hz):
    """evo_opm_bwd_factor vs fp32 torch: da = alpha einsum(ijpq,sjq->sip), db = alpha einsum(ijpq,sip->sjq) with
    do = bf16(dy W_o^T) (what the unfused path stores); da written bf16 into columns [0, P) of the [S*I, 2P]
    projection-gradient buffer, db fp32 in the rank-major layout a DAP reduce-scatter takes (2 ranks)."""
    P = 32
    g = torch.Generator(device=DEV).manual_seed(I + 3 * J + S + Hz)
    a = torch.randn(S, I, P, device=DEV, generator=g).bfloat16()
    b = torch.randn(S, J, P, device=DEV, generator=g).bfloat16()
    w = (torch.randn(P * P, Hz, device=DEV, generator=g) / 32).bfloat16()
    dy = torch.randn(I * J, Hz, device=DEV, generator=g).bfloat16()
    a_t, b_t = a.permute(1, 2, 0).contiguous(), b.permute(1, 2, 0).contiguous()
    al = 1.0 / S
    do = (dy.float() @ w.float().t()).bfloat16().float().view(I, J, P, P)
    da_ref = al * torch.einsum("ijpq,sjq->sip", do, b.float())
    db_ref = al * torch.einsum("ijpq,sip->sjq", do, a.float())
    assert ops.opm_bwd_supported(I, J, S, P, Hz)
    dab = torch.zeros(S, I, 2 * P, device=DEV, dtype=torch.bfloat16)
    ops.opm_bwd_factor(0, dy, w, b_t, I, J, S, P, Hz, al, dab, I * 2 * P, 0, 2 * P)
    Jl = J // 2
    dbf = torch.empty(2, S, Jl, P, device=DEV)  # [rank][s][j_local][q]
    ops.opm_bwd_factor(1, dy, w, a_t, J, I, S, P, Hz, al, dbf, Jl * P, S * Jl * P, P, x_split=Jl)
    torch.cuda.synchronize()
    assert rel(dab[..., :P], da_ref) < 5e-3, rel(dab[..., :P], da_ref)
    assert torch.count_nonzero(dab[..., P:]) == 0  # the other half of the buffer untouched
    db = torch.cat([dbf[0], dbf[1]], dim=1)
    assert rel(db, db_ref) < 1e-4, rel(db, db_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["row", "col"])
def test_key_bias_grad_cols(kind, B=5, L=37, nh=4, ld=3 * 4 * 32 + 8):
    """per-key bias gradient fp32 [B, nh, L] -> bias columns + zeroed padding of a strided dqkv"""
    db = torch.randn(B, nh, L, device=DEV)
    dqkv = torch.full((B * L, ld), float("nan"), device=DEV, dtype=torch.bfloat16)
    sb, sl = (L * ld, ld) if kind == "row" else (ld, B * ld)
    ops.key_bias_grad_cols(db, B, nh, L, Strided(dqkv, sb, sl, ld - 8), 8)
    torch.cuda.synchronize()
    v = dqkv.view(-1)[ld - 8:].as_strided((B, L, 8), (sb, sl, 1)).float()
    assert torch.equal(v[..., :nh], db.permute(0, 2, 1).bfloat16().float())
    assert (v[..., nh:] == 0).all()
    assert torch.isnan(dqkv[:, :ld - 8].float()).all()
