"""Thin torch-facing wrappers over the libevo.so C ABI (include/evo.h).

Every function launches on torch's *current* CUDA stream, takes/returns torch
CUDA tensors, and never falls back to anything else: a missing library raises
``NativeLibraryMissing`` and a rejected argument raises the reference's
exception classes (``DimensionError``) or ``KernelError``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import EVO_BF16, EVO_F32, EvoAttnBwdDesc, EvoAttnDesc, EvoMat, call
from .errors import DimensionError, KernelError

_DT = {torch.bfloat16: EVO_BF16, torch.float32: EVO_F32}


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise KernelError(f"unsupported dtype {t.dtype} (bf16/fp32 only)") from None


def _p(t):
    return None if t is None else t.data_ptr()


def _cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise KernelError("libevo ops take CUDA tensors only (no CPU fallback)")


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------------ LayerNorm

def layernorm_fwd(x, gamma, beta, rows, cols, x_rs=None, x_cs=1, out=None, out_dtype=None,
                  mean=None, rstd=None, eps=1e-5, save_stats=True):
    """engine.layernorm_raw (engine.py:206-217) over `rows` rows of `cols` channels."""
    _cuda(x, gamma, beta)
    x_rs = cols if x_rs is None else x_rs
    if out is None:
        out = torch.empty(rows, cols, device=x.device, dtype=out_dtype or x.dtype)
    if save_stats and mean is None:
        mean = torch.empty(rows, device=x.device, dtype=torch.float32)
        rstd = torch.empty(rows, device=x.device, dtype=torch.float32)
    call("evo_layernorm_fwd", _p(x), _dt(x), x_rs, x_cs, _p(gamma), _p(beta), _p(out), _dt(out),
         _p(mean), _p(rstd), rows, cols, eps, stream_handle(),
         work=(0, rows * cols * (x.element_size() + out.element_size()) + (8 * rows if mean is not None else 0)))
    return out, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd, rows, cols, x_rs=None, x_cs=1, dx=None,
                  accumulate=False, dgamma=None, dbeta=None, res=None, dx_colsum=None):
    """dx = res + dLN/dx.  accumulate=True means res = dx (in place);  res may be another
    tensor (the residual-stream gradient) so no clone is needed.  dx_colsum (fp32 [cols],
    accumulated): column sums of the written dx, fused into the same pass."""
    _cuda(dy, x, gamma, mean, rstd)
    x_rs = cols if x_rs is None else x_rs
    if dx is None:
        if x_cs != 1 or x_rs != cols:
            raise KernelError("layernorm_bwd: pass dx explicitly for strided inputs")
        dx = torch.empty(rows, cols, device=x.device, dtype=x.dtype)
        accumulate = False
    if accumulate:
        res = dx
    if dx_colsum is not None:
        call("evo_layernorm_bwd_colsum", _p(dy), _dt(dy), _p(x), _dt(x), x_rs, x_cs, _p(gamma), _p(mean), _p(rstd),
             _p(dx), _dt(dx), _p(res), _p(dgamma), _p(dbeta), _p(dx_colsum), rows, cols, stream_handle())
        return dx
    call("evo_layernorm_bwd", _p(dy), _dt(dy), _p(x), _dt(x), x_rs, x_cs, _p(gamma), _p(mean), _p(rstd),
         _p(dx), _dt(dx), _p(res), _p(dgamma), _p(dbeta), rows, cols, stream_handle())
    return dx


def layernorm_rowdot_fwd(x, gamma, beta, w, rows, cols, out, out_hs, ln_out=None, mean=None, rstd=None, eps=1e-5):
    """LN(x) . w[:, h] per row (msa_row_bias, evoformer.py:201-207); out[h*out_hs + r]."""
    _cuda(x, gamma, beta, w, out)
    k = w.shape[1]
    call("evo_layernorm_rowdot_fwd", _p(x), _dt(x), _p(gamma), _p(beta), _p(w), k, _p(out), _dt(out),
         out_hs, _p(ln_out), _p(mean), _p(rstd), rows, cols, eps, stream_handle())
    return out


def layernorm_rowdot_bwd(x, gamma, beta, w, dout, out_hs, mean, rstd, rows, cols, dx, res, dgamma, dbeta, dw):
    """backward of layernorm_rowdot_fwd in one pass (dx = res + dLN)."""
    call("evo_layernorm_rowdot_bwd", _p(x), _dt(x), _p(gamma), _p(beta), _p(w), w.shape[1], _p(dout), out_hs,
         _p(mean), _p(rstd), _p(res), _p(dx), _p(dgamma), _p(dbeta), _p(dw), rows, cols, stream_handle())
    return dx


# ------------------------------------------------------------------ softmax

def _strides4(t, shape4):
    """element strides of `t` broadcast against a 4-D shape (0 for broadcast dims)."""
    if t is None:
        return None
    if t.dim() > 4:
        raise DimensionError(f"bias/mask rank {t.dim()} > 4")
    tt = t.reshape((1,) * (4 - t.dim()) + tuple(t.shape)) if t.dim() < 4 else t
    out = []
    for d in range(4):
        if tt.shape[d] == shape4[d]:
            out.append(tt.stride(d) if shape4[d] > 1 else 0)
        elif tt.shape[d] == 1:
            out.append(0)
        else:
            raise DimensionError(f"mask/bias shape {tuple(t.shape)} not broadcastable to {tuple(shape4)}")
    return (C.c_int64 * 4)(*out)


def softmax_fwd(x, bias=None, mask=None, scale=1.0, out=None):
    """softmax((x + bias) * scale + mask) over the last axis of x [B, H, Q, K]
    (engine.fused_softmax_mask_bias_raw with scale=1, engine.py:193-203)."""
    _cuda(x, bias, mask)
    if x.dim() != 4:
        xs = x.reshape((1,) * (4 - x.dim()) + tuple(x.shape))
    else:
        xs = x
    xs = xs.contiguous()
    B, H, Q, K = xs.shape
    if out is None:
        out = torch.empty_like(xs)
    bs = _strides4(bias, xs.shape)
    ms = _strides4(mask, xs.shape)
    bias_bytes = 0 if bias is None else bias.numel() * bias.element_size()
    mask_bytes = 0 if mask is None else mask.numel() * mask.element_size()
    call("evo_softmax_fwd", _p(xs), _dt(xs), _p(bias), _dt(bias) if bias is not None else 0, bs,
         _p(mask), _dt(mask) if mask is not None else 0, ms, _p(out), _dt(out), B, H, Q, K, float(scale),
         stream_handle(), work=(0, xs.numel() * (xs.element_size() + out.element_size()) + bias_bytes + mask_bytes))
    return out.view(x.shape)


def softmax_bwd(y, dy, scale=1.0, out=None):
    _cuda(y, dy)
    K = y.shape[-1]
    rows = y.numel() // K
    if out is None:
        out = torch.empty_like(dy)
    call("evo_softmax_bwd", _p(y), _dt(y), _p(dy), _dt(dy), _p(out), _dt(out), rows, K, float(scale),
         stream_handle())
    return out


def count_nonfinite(x) -> int:
    counter = torch.zeros(1, dtype=torch.int32, device=x.device)
    call("evo_count_nonfinite", _p(x), _dt(x), x.numel(), _p(counter), stream_handle())
    return int(counter.item())


# ------------------------------------------------------------------ attention

@dataclass
class Strided:
    """A [batch, position, channel] view: element (b, l, col) at t.data_ptr() + (b*sb + l*sl + col)."""
    t: torch.Tensor
    sb: int
    sl: int
    offset: int = 0  # element offset of channel 0

    def ptr(self):
        return self.t.data_ptr() + self.offset * self.t.element_size()


def attention_desc(q: Strided, k: Strided, v: Strided, g: Strided, og: Strided, orw: Strided, lse,
                   B, L, H, c, scale, bias=None, bias_s=(0, 0, 0, 0), bias_off=0, flags=0):
    """flags: EVO_ATTN_* kernel-selection hints (include/evo.h), 0 = automatic"""
    d = EvoAttnDesc()
    d.q, d.k, d.v, d.g = q.ptr(), k.ptr(), v.ptr(), g.ptr()
    d.q_sb, d.q_sl, d.k_sb, d.k_sl = q.sb, q.sl, k.sb, k.sl
    d.v_sb, d.v_sl, d.g_sb, d.g_sl = v.sb, v.sl, g.sb, g.sl
    d.bias = None if bias is None else bias.data_ptr() + bias_off * bias.element_size()
    d.bias_s = (C.c_int64 * 4)(*bias_s)
    d.o_gated, d.o_sb, d.o_sl = og.ptr(), og.sb, og.sl
    if orw is not None:
        d.o_raw, d.r_sb, d.r_sl = orw.ptr(), orw.sb, orw.sl
    d.lse = _p(lse)
    d.B, d.L, d.H, d.c, d.scale = B, L, H, c, float(scale)
    d.flags = int(flags)
    return d


def _attn_work(d: EvoAttnDesc, bwd=False):
    B, L, H, c = d.B, d.L, d.H, d.c
    io = B * L * H * c * 2
    bias = 0
    if d.bias:
        bias = (H * L * L * 2) if d.bias_s[2] != 0 else B * H * L * 2
    if not bwd:   # read q,k,v,g (+bias), write o_gated, o_raw, lse
        return 4 * B * H * L * L * c, 4 * io + bias + 2 * io + B * H * L * 4
    # read q,k,v,g,o_raw,dout,lse (+bias), write dq,dk,dv,dg (+dbias fp32)
    return 10 * B * H * L * L * c, 6 * io + bias + 4 * io + B * H * L * 4 + 2 * bias


def attention_fwd(desc: EvoAttnDesc):
    call("evo_gated_attention_fwd", C.byref(desc), stream_handle(), work=_attn_work(desc))


def key_bias_grad_cols(dbias, B, nh, L, dst: Strided, cols: int):
    """dst[b, l, h] = bf16(dbias[b, h, l]) for h < nh and 0 for nh <= h < cols (dbias fp32
    [B, nh, L] contiguous): the per-key bias gradient into the bias columns of dqkv."""
    _cuda(dbias)
    call("evo_key_bias_grad_cols", _p(dbias), B, nh, L, dst.ptr(), dst.sb, dst.sl, cols, stream_handle())
    return dst


def attention_bwd_workspace(B, L, H, c, batch_reduced_bias=False) -> int:
    return int(_lib.load().evo_gated_attention_bwd_workspace(B, L, H, c, int(batch_reduced_bias)))


def attention_bwd(fdesc: EvoAttnDesc, dout: Strided, dq: Strided, dk: Strided, dv: Strided, dg: Strided,
                  workspace: torch.Tensor, dbias=None, dbias_s=(0, 0, 0, 0)):
    d = EvoAttnBwdDesc()
    d.f = fdesc
    d.dout, d.do_sb, d.do_sl = dout.ptr(), dout.sb, dout.sl
    d.dq, d.dk, d.dv, d.dg = dq.ptr(), dk.ptr(), dv.ptr(), dg.ptr()
    d.dq_sb, d.dq_sl, d.dk_sb, d.dk_sl = dq.sb, dq.sl, dk.sb, dk.sl
    d.dv_sb, d.dv_sl, d.dg_sb, d.dg_sl = dv.sb, dv.sl, dg.sb, dg.sl
    d.dbias = _p(dbias)
    d.dbias_s = (C.c_int64 * 4)(*dbias_s)
    d.workspace = workspace.data_ptr()
    d.workspace_bytes = workspace.numel() * workspace.element_size()
    batch_reduced = (dbias is not None and fdesc.bias and dbias_s[0] == 0 and dbias_s[2] != 0
                     and fdesc.L % 8 == 0)
    nkt = (fdesc.L + 127) // 128
    # prep + main (+ dq finish when > 1 key tile), + bias transpose & dbias reduce, + dQ memset
    launches = 2 + (1 if nkt > 1 else 0) + (2 if batch_reduced else 0) + (1 if nkt > 4 else 0)
    call("evo_gated_attention_bwd", C.byref(d), stream_handle(), work=_attn_work(fdesc, bwd=True),
         launches=launches)


# ------------------------------------------------------------------ batched GEMM

BIG = 1 << 40


@dataclass
class Mat:
    """2-level strided matrix view for evo_bgemm (see EvoMat in include/evo.h).

    dim d of index i maps to (i // split[d]) * hi[d] + (i % split[d]) * lo[d];
    split = 0 means "no split" (plain stride lo)."""
    t: torch.Tensor
    lo: tuple
    split: tuple = (0, 0)
    hi: tuple = (0, 0)
    batch_stride: int = 0
    offset: int = 0

    def to_c(self) -> EvoMat:
        m = EvoMat()
        m.ptr = self.t.data_ptr() + self.offset * self.t.element_size()
        m.dtype = _dt(self.t)
        m.batch_stride = self.batch_stride
        m.split = (C.c_int64 * 2)(*[s if s else BIG for s in self.split])
        m.stride_hi = (C.c_int64 * 2)(*self.hi)
        m.stride_lo = (C.c_int64 * 2)(*self.lo)
        return m


def bgemm(A: Mat, B: Mat, Cm: Mat, batch, M, N, K, alpha=1.0, beta=0.0):
    """C[b] = alpha * A[b] . B[b]^T + beta * C[b] on tcgen05 (evo_bgemm)."""
    _cuda(A.t, B.t, Cm.t)
    a, b, c = A.to_c(), B.to_c(), Cm.to_c()
    work = (2 * batch * M * N * K, batch * (2 * M * K + 2 * N * K + Cm.t.element_size() * M * N))
    ws_bytes = int(_lib.load().evo_bgemm_workspace(batch, M, N, K))
    if ws_bytes:  # split-K (long K, few output tiles): fp32 partials + reduction
        ws = torch.empty(ws_bytes // 4, device=Cm.t.device, dtype=torch.float32)
        call("evo_bgemm_ws", C.byref(a), C.byref(b), C.byref(c), batch, M, N, K, float(alpha), float(beta),
             ws.data_ptr(), ws_bytes, stream_handle(), work=work)
        return
    call("evo_bgemm", C.byref(a), C.byref(b), C.byref(c), batch, M, N, K, float(alpha), float(beta),
         stream_handle(), work=work)


def opm_fused_supported(I, J, S, P, Hz) -> bool:
    return bool(_lib.load().evo_opm_fused_supported(I, J, S, P, Hz))


def opm_transpose(x, S, R, P, col0=0, both=False):
    """[S*R, ld] projection rows (s, r) -> sequence-contiguous [R, P, S] (and the next P channels
    as a second [R, P, S] when both) for the fused OPM (evo_opm_transpose)."""
    _cuda(x)
    out_a = torch.empty(R, P, S, device=x.device, dtype=torch.bfloat16)
    out_b = torch.empty_like(out_a) if both else None
    call("evo_opm_transpose", _p(x), x.stride(0), col0, S, R, P, _p(out_a), _p(out_b), stream_handle(),
         work=(0, 4 * S * R * P * (2 if both else 1)))
    return (out_a, out_b) if both else out_a


def opm_fused_fwd(a_t, b_t, w_o, I, J, S, P, Hz, alpha, y=None, o_save=None):
    """outer_product_mean contraction + output projection (evoformer.py:251-255) with o kept on chip:
    y[(i, j), c] = sum_{p,q} (alpha * sum_s a[s,i,p] b[s,j,q]) W_o[p*P+q, c]  (evo_opm_fused_fwd).
    a_t: [I, P, S], b_t: [J, P, S] bf16 contiguous (opm_transpose); w_o: [P*P, Hz] bf16.
    o_save: optional [I, J, P, P] bf16 output of o (kept for the backward)."""
    _cuda(a_t, b_t, w_o)
    if not (a_t.is_contiguous() and b_t.is_contiguous() and w_o.is_contiguous()):
        raise KernelError("opm_fused_fwd: a_t, b_t and w_o must be contiguous")
    if y is None:
        y = torch.empty(I * J, Hz, device=a_t.device, dtype=torch.bfloat16)
    call("evo_opm_fused_fwd", _p(a_t), _p(b_t), _p(w_o), _p(y), y.stride(0), _p(o_save), I, J, S, P, Hz,
         float(alpha), stream_handle(),
         work=(2 * I * J * P * P * (S + Hz), 2 * (S * I * P + S * J * P + P * P * Hz + I * J * Hz)))
    return y


def wgrad(x, dy, dw):
    """dw (fp32 [M, N], any row stride) += x^T @ dy for x [rows, M], dy [rows, N] bf16 (evo_wgrad)."""
    _cuda(x, dy, dw)
    rows, M = x.shape
    N = dy.shape[1]
    if x.stride(1) != 1 or dy.stride(1) != 1 or dw.stride(1) != 1 or dw.dtype != torch.float32:
        raise KernelError("wgrad: row-major bf16 x / dy and an fp32 dw are required")
    ws_bytes = int(_lib.load().evo_wgrad_workspace(rows, M, N))
    ws = torch.empty(max(ws_bytes // 4, 1), device=x.device, dtype=torch.float32)
    call("evo_wgrad", _p(x), x.stride(0), _p(dy), dy.stride(0), _p(dw), dw.stride(0), rows, M, N,
         _p(ws) if ws_bytes else None, ws_bytes, stream_handle(),
         work=(2 * rows * M * N, 2 * rows * (M + N) + 8 * M * N), launches=2 if ws_bytes else 1)
    return dw


def opm_bwd_supported(I, J, S, P, Hz) -> bool:
    return bool(_lib.load().evo_opm_bwd_supported(I, J, S, P, Hz))


def opm_bwd_factor(role, dy, w_o, other_t, X, Y, S, P, Hz, alpha, out, o_ss, o_sr, o_sx, x_split=None):
    """one factor gradient of the fused OPM (evo_opm_bwd_factor): role 0 -> da (x = i, other = b_t),
    role 1 -> db (x = j, other = a_t); out element (s, x, p) at
    out[s*o_ss + (x // x_split)*o_sr + (x % x_split)*o_sx + p] (out bf16 or fp32)."""
    _cuda(dy, w_o, other_t, out)
    ws_bytes = int(_lib.load().evo_opm_bwd_workspace(X))
    ws = torch.empty(ws_bytes // 4, device=dy.device, dtype=torch.float32)
    call("evo_opm_bwd_factor", role, _p(dy), dy.stride(0), _p(w_o), _p(other_t), X, Y, S, P, Hz, float(alpha),
         _p(out), 1 if out.dtype == torch.float32 else 0, o_ss, o_sr, o_sx, X if x_split is None else x_split,
         _p(ws), ws_bytes, stream_handle(),
         work=(4 * X * Y * P * P * (Hz + S), 2 * (X * Y * Hz * P // 4 + P * P * Hz + Y * P * S)))
    return out


# ------------------------------------------------------------------ elementwise epilogues

def tri_gate_fwd(y, rows, hz, p, a_cm, b_cm):
    call("evo_tri_gate_fwd", _p(y), rows, hz, p, _p(a_cm), _p(b_cm), stream_handle())


def tri_gate_bwd(y, da_cm, db_cm, rows, hz, p, dy, dsum=None):
    """dsum (fp32 [4p]): += fp32 column sums of dY[:, hz:] (the a/b projection bias gradient)"""
    call("evo_tri_gate_bwd", _p(y), _p(da_cm), _p(db_cm), _dt(da_cm), rows, hz, p, _p(dy), _p(dsum), stream_handle())


def gated_residual_fwd(res, y, bias, rows, cols, y_rs=None, gp=None, gp_rs=0, out=None):
    """out = res + sigmoid(gp) * (y + bias)   (gp None -> plain residual + bias)."""
    if out is None:
        out = torch.empty_like(res)
    call("evo_gated_residual_fwd", _p(res), _p(y), cols if y_rs is None else y_rs, _p(bias), _p(gp), gp_rs,
         _p(out), _dt(res), rows, cols, stream_handle())
    return out


def residual_layernorm_fwd(res, y, bias, rows, cols, gamma, beta, y_rs=None, gp=None, gp_rs=0, eps=1e-5):
    """out = res + [sigmoid(gp) *] (y + bias) and the next module's LayerNorm of out in one pass
    -> (out, ln, mean, rstd)"""
    _cuda(res, y, gamma, beta)
    y_rs = cols if y_rs is None else y_rs
    out = torch.empty(rows, cols, device=res.device, dtype=res.dtype)
    ln = torch.empty_like(out)
    mean = torch.empty(rows, device=res.device, dtype=torch.float32)
    rstd = torch.empty_like(mean)
    call("evo_residual_layernorm_fwd", _p(res), _p(y), y_rs, _p(bias), _p(gp), gp_rs, _p(out), _p(gamma), _p(beta),
         _p(ln), _p(mean), _p(rstd), rows, cols, eps, stream_handle(),
         work=(0, rows * cols * 2 * (4 + (1 if gp is not None else 0)) + 8 * rows))
    return out, ln, mean, rstd


def gated_residual_bwd(dout, rows, cols, y=None, y_rs=None, bias=None, gp=None, gp_rs=0, dy=None, dgp=None,
                       dgp_rs=0, dbias=None, dgp_sum=None):
    """dgp_sum (fp32 [cols]): += fp32 column sums of dgp (the gate projection's bias gradient)"""
    call("evo_gated_residual_bwd", _p(dout), _p(y), cols if y_rs is None else y_rs, _p(bias), _p(gp), gp_rs,
         _p(dy), _p(dgp), dgp_rs, _p(dbias), _p(dgp_sum), _dt(dout), rows, cols, stream_handle())


def bias_act_fwd(y, bias, rows, cols, relu=True):
    call("evo_bias_act_fwd", _p(y), _p(bias), rows, cols, 1 if relu else 0, _dt(y), stream_handle())
    return y


def bias_act_bwd(dh, h, rows, cols, dy=None, dbias=None, relu=True):
    if dy is None:
        dy = torch.empty_like(dh)
    call("evo_bias_act_bwd", _p(dh), _p(h), _p(dy), _p(dbias), rows, cols, 1 if relu else 0, _dt(dh),
         stream_handle())
    return dy


def gate_mul(gate, y=None, bias=None, act=1, rows=None, cols=None, gate_rs=None, y_rs=None, out=None):
    """out = act(gate) * (y + bias) over a [rows, cols] view (evo_gate_mul_fwd); gate or y may be None
    (factor 1).  act: 0 identity, 1 sigmoid, 2 ReLU."""
    ref = gate if gate is not None else y
    _cuda(ref, y, bias)
    rows = ref.shape[0] if rows is None else rows
    cols = ref.shape[-1] if cols is None else cols
    if out is None:
        out = torch.empty(rows, cols, device=ref.device, dtype=ref.dtype)
    for t in (gate, y):
        if t is not None and t.dtype != out.dtype:
            raise KernelError("gate_mul: gate / y / out must share a dtype")
    call("evo_gate_mul_fwd", _p(gate), gate.stride(0) if gate_rs is None and gate is not None else (gate_rs or 0),
         int(act), _p(y), y.stride(0) if y_rs is None and y is not None else (y_rs or 0), _p(bias), _p(out),
         out.stride(0), _dt(out), rows, cols, stream_handle())
    return out


def colsum(x, out, rows=None, cols=None, ld=None):
    """out (fp32) += column sums of the 2-D view x [rows, cols] (row stride ld)."""
    rows = x.shape[0] if rows is None else rows
    cols = x.shape[-1] if cols is None else cols
    ld = x.stride(0) if ld is None else ld
    call("evo_colsum", _p(x), _dt(x), ld, rows, cols, _p(out), stream_handle())
    return out
