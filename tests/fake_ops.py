"""TEST-ONLY CPU stand-ins for paper_2203_00854_b200.ops (the libevo.so wrappers).

Each function implements the same contract as its CUDA twin - same arguments,
same strided / 2-level (EvoMat) addressing, same in-place / accumulate
semantics - with plain torch math on CPU tensors (fp32 compute, results stored
in the tensor's dtype).  It lets the host-side logic (block.py composition and
the DAP schedule in dap.py, including every rank-major gathered-buffer
address) run under a gloo process group on CPU.  It is never imported by the
package; tests install it with ``install(monkeypatch)``.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import torch

from paper_2203_00854_b200 import ops as _real
from paper_2203_00854_b200.ops import Mat, Strided

F32 = torch.float32


def _flat(t):
    n = t.untyped_storage().nbytes() // t.element_size()
    return torch.as_strided(t, (n,), (1,), 0)


def _sv(t, offset, sizes, strides):
    return torch.as_strided(t, sizes, strides, t.storage_offset() + offset)


# ------------------------------------------------------------------ LayerNorm
def layernorm_fwd(x, gamma, beta, rows, cols, x_rs=None, x_cs=1, out=None, out_dtype=None, mean=None, rstd=None,
                  eps=1e-5, save_stats=True):
    x_rs = cols if x_rs is None else x_rs
    xv = _sv(x, 0, (rows, cols), (x_rs, x_cs)).float()
    mu = xv.mean(-1)
    var = ((xv - mu[:, None]) ** 2).mean(-1)
    rs = 1.0 / torch.sqrt(var + eps)
    y = (xv - mu[:, None]) * rs[:, None] * gamma + beta
    if out is None:
        out = torch.empty(rows, cols, dtype=out_dtype or x.dtype)
    out.copy_(y)
    if save_stats and mean is None:
        mean, rstd = torch.empty(rows), torch.empty(rows)
    if mean is not None:
        mean.copy_(mu)
        rstd.copy_(rs)
    return out, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd, rows, cols, x_rs=None, x_cs=1, dx=None, accumulate=False, dgamma=None,
                  dbeta=None, res=None, dx_colsum=None):
    x_rs = cols if x_rs is None else x_rs
    xv = _sv(x, 0, (rows, cols), (x_rs, x_cs)).float()
    d = dy.reshape(rows, cols).float()
    xh = (xv - mean[:, None]) * rstd[:, None]
    gd = d * gamma
    o = rstd[:, None] * (gd - gd.mean(-1, keepdim=True) - xh * (gd * xh).mean(-1, keepdim=True))
    if dgamma is not None:
        dgamma += (d * xh).sum(0)
    if dbeta is not None:
        dbeta += d.sum(0)
    if dx is None:
        dx = torch.empty(rows, cols, dtype=x.dtype)
        accumulate = False
    if accumulate:
        res = dx
    base = _sv(res, 0, (rows, cols), (x_rs, x_cs)).float() if res is not None else 0
    _sv(dx, 0, (rows, cols), (x_rs, x_cs)).copy_(o + base)
    if dx_colsum is not None:
        dx_colsum += (o + base).sum(0)
    return dx


def layernorm_rowdot_fwd(x, gamma, beta, w, rows, cols, out, out_hs, ln_out=None, mean=None, rstd=None, eps=1e-5):
    ln, mu, rs = layernorm_fwd(x, gamma, beta, rows, cols, out_dtype=F32, eps=eps)
    k = out.shape[0] if out.dim() == 3 else w.shape[1]
    _sv(out, 0, (k, rows), (out_hs, 1)).copy_((ln @ w).t())
    if ln_out is not None:
        ln_out.copy_(ln)
    if mean is not None:
        mean.copy_(mu)
        rstd.copy_(rs)
    return out


# ------------------------------------------------------------------ attention
def attention_desc(q, k, v, g, og, orw, lse, B, L, H, c, scale, bias=None, bias_s=(0, 0, 0, 0), bias_off=0,
                   flags=0):
    return SimpleNamespace(q=q, k=k, v=v, g=g, og=og, orw=orw, lse=lse, B=B, L=L, H=H, c=c, scale=scale,
                           bias=bias, bias_s=tuple(bias_s), bias_off=bias_off)


def _blhc(s: Strided, B, L, H, c):
    return _sv(s.t, s.offset, (B, L, H, c), (s.sb, s.sl, c, 1))


def _fwd_math(d, grad=False):
    B, L, H, c = d.B, d.L, d.H, d.c
    q, k, v, g = (_blhc(s, B, L, H, c).float().permute(0, 2, 1, 3).clone().requires_grad_(grad)
                  for s in (d.q, d.k, d.v, d.g))
    bias = None
    if d.bias is not None:
        bias = _sv(d.bias, d.bias_off, (B, H, L, L), d.bias_s).float().clone().requires_grad_(grad)
    s = q @ k.transpose(-1, -2)
    if bias is not None:
        s = s + bias
    s = s * d.scale
    o = torch.softmax(s, -1) @ v
    out = torch.sigmoid(g) * o
    return (q, k, v, g, bias), s, o, out


def attention_fwd(d):
    _, s, o, out = _fwd_math(d)
    B, L, H, c = d.B, d.L, d.H, d.c
    _blhc(d.og, B, L, H, c).copy_(out.permute(0, 2, 1, 3))
    if d.orw is not None:
        _blhc(d.orw, B, L, H, c).copy_(o.permute(0, 2, 1, 3))
    if d.lse is not None:
        d.lse.copy_(torch.logsumexp(s, -1))


def attention_bwd_workspace(B, L, H, c, batch_reduced_bias=False):
    return 1


def key_bias_grad_cols(dbias, B, nh, L, dst, cols):
    v = torch.zeros(B, L, cols, dtype=torch.float32)
    v[..., :nh] = dbias.permute(0, 2, 1)
    _blhc_cols(dst, B, L, cols).copy_(v)
    return dst


def _blhc_cols(s, B, L, cols):
    return _sv(s.t, s.offset, (B, L, cols), (s.sb, s.sl, 1))


def attention_bwd(fdesc, dout, dq, dk, dv, dg, workspace, dbias=None, dbias_s=(0, 0, 0, 0)):
    d = fdesc
    B, L, H, c = d.B, d.L, d.H, d.c
    with torch.enable_grad():
        (q, k, v, g, bias), _, _, out = _fwd_math(d, grad=True)
        out.backward(_blhc(dout, B, L, H, c).float().permute(0, 2, 1, 3))
    for s, t in ((dq, q), (dk, k), (dv, v), (dg, g)):
        _blhc(s, B, L, H, c).copy_(t.grad.permute(0, 2, 1, 3))
    if dbias is not None:
        gb = bias.grad
        red = [i for i in range(4) if dbias_s[i] == 0]
        if red:
            gb = gb.sum(dim=red, keepdim=True)
        sizes = tuple(1 if dbias_s[i] == 0 else (B, H, L, L)[i] for i in range(4))
        _sv(dbias, 0, sizes, tuple(dbias_s)).add_(gb)


# ------------------------------------------------------------------ batched GEMM
def _idx(m: Mat, n0, n1, batch):
    def dim(d, n):
        i = torch.arange(n)
        split = m.split[d] if m.split[d] else 1 << 40
        return (i // split) * m.hi[d] + (i % split) * m.lo[d]
    return (m.t.storage_offset() + m.offset + torch.arange(batch)[:, None, None] * m.batch_stride
            + dim(0, n0)[None, :, None] + dim(1, n1)[None, None, :])


def softmax_fwd(x, bias=None, mask=None, scale=1.0, out=None):
    """softmax((x + bias) * scale + mask) over the last axis, operands broadcast right-aligned"""
    v = x.to(torch.float64 if x.dtype == torch.float64 else F32)
    if bias is not None:
        v = v + bias
    v = v * scale
    if mask is not None:
        v = v + mask
    y = torch.softmax(v, -1).to(x.dtype)
    if out is not None:
        out.copy_(y.reshape(out.shape))
        return out
    return y


def count_nonfinite(x) -> int:
    return int((~torch.isfinite(x)).sum())


def opm_bwd_supported(I, J, S, P, Hz):
    return P == 32 and 8 <= S <= 128 and S % 8 == 0 and I % 32 == 0 and I >= 32 and J % 32 == 0 and J >= 32 and \
        Hz in (64, 128)


def opm_bwd_factor(role, dy, w_o, other_t, X, Y, S, P, Hz, alpha, out, o_ss, o_sr, o_sx, x_split=None):
    x_split = X if x_split is None else x_split
    I, J = (X, Y) if role == 0 else (Y, X)
    do = (dy.float() @ w_o.float().t()).to(dy.dtype).float().view(I, J, P, P)
    oth = other_t.float()                       # [Y][P][S]
    if role == 0:
        g = alpha * torch.einsum("ijpq,jqs->sip", do, oth)       # da [S, X, P]
    else:
        g = alpha * torch.einsum("ijpq,ips->sjq", do, oth)       # db [S, X, P]
    CALLS["opm_bwd_factor"] += 1
    flat = _flat(out)  # absolute storage offsets
    for x in range(X):
        off = out.storage_offset() + (x // x_split) * o_sr + (x % x_split) * o_sx
        idx = off + torch.arange(S)[:, None] * o_ss + torch.arange(P)[None, :]
        flat[idx.reshape(-1)] = g[:, x, :].reshape(-1).to(out.dtype)
    return out


def opm_fused_supported(I, J, S, P, Hz):
    return P == 32 and 8 <= S <= 128 and S % 8 == 0 and I % 32 == 0 and I >= 32 and J % 8 == 0 and J >= 8 and \
        Hz in (32, 64, 128)


def opm_transpose(x, S, R, P, col0=0, both=False):
    v = _sv(x, col0, (S, R, (2 if both else 1) * P), (R * x.stride(0), x.stride(0), 1))
    a = v[..., :P].permute(1, 2, 0).contiguous()
    return (a, v[..., P:].permute(1, 2, 0).contiguous()) if both else a


CALLS = {"opm_fused_fwd": 0, "opm_bwd_factor": 0}


def opm_fused_fwd(a_t, b_t, w_o, I, J, S, P, Hz, alpha, y=None, o_save=None):
    CALLS["opm_fused_fwd"] += 1
    o = (torch.einsum("ips,jqs->ijpq", a_t.float(), b_t.float()) * alpha).to(a_t.dtype)
    if o_save is not None:
        o_save.copy_(o)
    out = o.reshape(I * J, P * P).float() @ w_o.float()
    if y is None:
        y = torch.empty(I * J, Hz, dtype=a_t.dtype)
    y.copy_(out)
    return y


def bgemm(A: Mat, B: Mat, Cm: Mat, batch, M, N, K, alpha=1.0, beta=0.0):
    a = _flat(A.t)[_idx(A, M, K, batch)].float()
    b = _flat(B.t)[_idx(B, N, K, batch)].float()
    res = alpha * (a @ b.transpose(1, 2))
    ci = _idx(Cm, M, N, batch)
    fc = _flat(Cm.t)
    if beta != 0:
        res = res + beta * fc[ci].float()
    fc[ci] = res.to(Cm.t.dtype)


# ------------------------------------------------------------------ epilogues
def tri_gate_fwd(y, rows, hz, p, a_cm, b_cm):
    yv = y.float()
    a = torch.sigmoid(yv[:, hz:hz + p]) * yv[:, hz + p:hz + 2 * p]
    b = torch.sigmoid(yv[:, hz + 2 * p:hz + 3 * p]) * yv[:, hz + 3 * p:hz + 4 * p]
    a_cm.view(p, rows).copy_(a.t())
    b_cm.view(p, rows).copy_(b.t())


def tri_gate_bwd(y, da_cm, db_cm, rows, hz, p, dy, dsum=None):
    yv = y.float()
    da, db = da_cm.reshape(p, rows).float().t(), db_cm.reshape(p, rows).float().t()
    for j, dd in ((0, da), (1, db)):
        s = yv[:, hz + 2 * j * p:hz + (2 * j + 1) * p]
        lin = yv[:, hz + (2 * j + 1) * p:hz + (2 * j + 2) * p]
        sg = torch.sigmoid(s)
        dy[:, hz + 2 * j * p:hz + (2 * j + 1) * p] = dd * lin * sg * (1 - sg)
        dy[:, hz + (2 * j + 1) * p:hz + (2 * j + 2) * p] = dd * sg
        if dsum is not None:
            dsum[2 * j * p:(2 * j + 1) * p] += (dd * lin * sg * (1 - sg)).sum(0)
            dsum[(2 * j + 1) * p:(2 * j + 2) * p] += (dd * sg).sum(0)


def gated_residual_fwd(res, y, bias, rows, cols, y_rs=None, gp=None, gp_rs=0, out=None):
    y_rs = cols if y_rs is None else y_rs
    yv = _sv(y, 0, (rows, cols), (y_rs, 1)).float() + (bias if bias is not None else 0)
    if gp is not None:
        yv = yv * torch.sigmoid(_sv(gp, 0, (rows, cols), (gp_rs, 1)).float())
    if out is None:
        out = torch.empty_like(res)
    out.copy_(res.float().reshape(rows, cols) + yv)
    return out


def gated_residual_bwd(dout, rows, cols, y=None, y_rs=None, bias=None, gp=None, gp_rs=0, dy=None, dgp=None,
                       dgp_rs=0, dbias=None, dgp_sum=None):
    d = dout.reshape(rows, cols).float()
    if gp is not None:
        y_rs = cols if y_rs is None else y_rs
        yv = _sv(y, 0, (rows, cols), (y_rs, 1)).float() + (bias if bias is not None else 0)
        s = torch.sigmoid(_sv(gp, 0, (rows, cols), (gp_rs, 1)).float())
        dg = d * yv * s * (1 - s)
        _sv(dgp, 0, (rows, cols), (dgp_rs, 1)).copy_(dg)
        if dgp_sum is not None:
            dgp_sum += dg.sum(0)
        d = d * s
    if dy is not None:
        dy.copy_(d)
    if dbias is not None:
        dbias += d.sum(0)


def bias_act_fwd(y, bias, rows, cols, relu=True):
    v = y.float() + (bias if bias is not None else 0)
    y.copy_(torch.relu(v) if relu else v)
    return y


def bias_act_bwd(dh, h, rows, cols, dy=None, dbias=None, relu=True):
    d = dh.float() * (h.float() > 0) if relu else dh.float()
    if dy is None:
        dy = torch.empty_like(dh)
    dy.copy_(d)
    if dbias is not None:
        dbias += d.sum(0)
    return dy


def gate_mul(gate, y=None, bias=None, act=1, rows=None, cols=None, gate_rs=None, y_rs=None, out=None):
    ref = gate if gate is not None else y
    rows = ref.shape[0] if rows is None else rows
    cols = ref.shape[-1] if cols is None else cols
    f = torch.ones(rows, cols)
    if y is not None:
        f = _sv(y, 0, (rows, cols), (y.stride(0) if y_rs is None else y_rs, 1)).float()
        if bias is not None:
            f = f + bias.float()
    if gate is not None:
        gv = _sv(gate, 0, (rows, cols), (gate.stride(0) if gate_rs is None else gate_rs, 1)).float()
        gv = torch.sigmoid(gv) if act == 1 else (torch.relu(gv) if act == 2 else gv)
        f = gv * f
    if out is None:
        out = torch.empty(rows, cols, dtype=ref.dtype)
    out.copy_(f)
    return out


NAMES = ["gate_mul", "layernorm_fwd", "layernorm_bwd", "layernorm_rowdot_fwd", "attention_desc", "attention_fwd",
         "attention_bwd_workspace", "attention_bwd", "bgemm", "softmax_fwd", "count_nonfinite", "opm_fused_supported", "opm_transpose", "opm_bwd_supported", "opm_bwd_factor",
         "opm_fused_fwd", "tri_gate_fwd", "tri_gate_bwd",
         "gated_residual_fwd", "gated_residual_bwd", "bias_act_fwd", "bias_act_bwd", "key_bias_grad_cols"]


def install():
    """patch the package's op table (in the current process) with the CPU stand-ins"""
    g = globals()
    for n in NAMES:
        setattr(_real, n, g[n])


class installed:
    """context manager: the CPU stand-ins for the duration of a block, the real ops restored after
    (for tests sharing a process with GPU tests)"""

    def __enter__(self):
        self.saved = {n: getattr(_real, n) for n in NAMES}
        install()
        return self

    def __exit__(self, *exc):
        for n, f in self.saved.items():
            setattr(_real, n, f)
        return False


_ = math  # (kept for parity with the CUDA module's imports)
