"""Reference-precision forward of the Evoformer block: a parity mode far tighter than bf16.

The product path (``evoformer.py`` / ``block.py``) stores activations in bf16, so its parity
against the float64 reference is bounded by bf16 rounding (2e-2 relative).  This
module recomputes the same block, sub-module by sub-module in the reference's order
(evoformer.py:173-325), with fp32 storage and near-fp32 products, so a semantic bug that hides
under bf16 noise (a missing bias, a wrong eps, a transposed einsum) shows up at 1e-5:

* every dense contraction named by the north star runs on the sm_100a tcgen05 batched GEMM
  (``evo_bgemm``) as a **three-term bf16 split**: x = hi + lo with hi = bf16(x),
  lo = bf16(x - hi); A.B^T = hi.hi^T + hi.lo^T + lo.hi^T accumulated in fp32 (TMEM, then
  beta = 1 into the fp32 output).  Each operand keeps ~16 mantissa bits, the dropped lo.lo^T
  term is ~2^-16 of the product: QK^T and PV of every attention (evoformer.py:186, 192), the
  triangle einsums (276, 283) and the outer-product contraction (253);
* LayerNorm (``evo_layernorm_fwd``), the biased softmax (``evo_softmax_fwd``: softmax((x + bias)
  c^-1/2) with the bias broadcast through strides, engine.py:193-203), the sigmoid gates
  (``evo_gate_mul_fwd``), the ReLU (``evo_bias_act_fwd``) and the gated / plain residual adds
  (``evo_gated_residual_fwd``) are the same hand-written kernels as the product path, in their
  fp32 instantiation;
* plain projections are cuBLAS fp32 GEMMs with TF32 disabled.

Forward only (the product path's gradients are checked against the torch float64 autograd oracle,
tests/test_gpu_parity.py).  Layout reshuffles between the reference's axis orders are torch
copies: this mode is a checker of the composition, not a fast path.  Requires head dims, N_s,
N_r and hidden_proj that are multiples of 8 (the bgemm's 16-byte operand runs).

Tolerance (tests/test_gpu_precise.py): relative Frobenius error <= 2e-5 per sub-module output and
per block output, max-abs <= 1e-4 per block, against the float64 oracle; measured 1.1e-6 - 5.1e-6
relative and 2.6e-5 - 5.0e-5 max-abs over four configs and three seeds, where the bf16 product path
measures 4e-3 - 9e-3 (profiles/r02_precise_errors.txt).
"""

from __future__ import annotations

import math
from contextlib import contextmanager

import numpy as np
import torch

from . import ops
from .config import EvoConfig
from .errors import DimensionError, KernelError
from .ops import Mat

F32 = torch.float32
BF16 = torch.bfloat16

__all__ = ["evoformer_block", "msa_row_bias", "msa_row_attention", "msa_col_attention", "transition",
           "outer_product_mean", "tri_update_outgoing", "tri_update_incoming", "pair_attention_row",
           "pair_attention_col", "gemm_nt"]


@contextmanager
def _no_tf32():
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _dev(x):
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise KernelError("precise mode: tensors must live on the GPU (no CPU path)")
        return x.to(F32)
    return torch.as_tensor(np.asarray(x, dtype=np.float32), device="cuda")


def _split(x):
    hi = x.to(BF16)
    lo = (x - hi.to(F32)).to(BF16)
    return hi, lo


def gemm_nt(A, B, alpha=1.0):
    """C[b] = alpha * A[b] @ B[b]^T for fp32 A [b, M, K], B [b, N, K] -> fp32 [b, M, N], as three bf16
    tcgen05 products (hi.hi + hi.lo + lo.hi) accumulating in fp32 (evo_bgemm, beta = 1)."""
    if A.dim() == 2:
        return gemm_nt(A[None], B[None], alpha)[0]
    bt, M, K = A.shape
    N = B.shape[1]
    if B.shape[0] != bt or B.shape[2] != K:
        raise DimensionError(f"gemm_nt: A {tuple(A.shape)} and B {tuple(B.shape)} do not contract")
    if K % 8:
        raise DimensionError(f"gemm_nt: contraction extent {K} must be a multiple of 8")
    Ah, Al = _split(A.contiguous())
    Bh, Bl = _split(B.contiguous())
    C = torch.empty(bt, M, N, device=A.device, dtype=F32)
    Cm = Mat(C, (N, 1), batch_stride=M * N)
    for i, (a, b) in enumerate(((Al, Bh), (Ah, Bl), (Ah, Bh))):  # small terms first
        ops.bgemm(Mat(a, (K, 1), batch_stride=M * K), Mat(b, (K, 1), batch_stride=N * K), Cm, bt, M, N, K,
                  alpha=alpha, beta=0.0 if i == 0 else 1.0)
    return C


def _ln(x2d, p, prefix):
    """engine.layernorm_raw (engine.py:206-217) in fp32 (evo_layernorm_fwd)"""
    rows, cols = x2d.shape
    out, _, _ = ops.layernorm_fwd(x2d.contiguous(), _dev(p[f"{prefix}/g"]), _dev(p[f"{prefix}/b"]), rows, cols,
                                  save_stats=False)
    return out


def _lin(x2d, w, b=None):
    with _no_tf32():
        y = x2d @ _dev(w)
    return y if b is None else y + _dev(b)


def _residual(res2d, y2d, bias=None, gate_pre=None):
    """res + [sigmoid(gate_pre) *] (y + bias)   (evo_gated_residual_fwd, fp32)"""
    rows, cols = res2d.shape
    b = _dev(bias) if bias is not None else torch.zeros(cols, device=res2d.device, dtype=F32)
    gp = gate_pre.contiguous() if gate_pre is not None else None
    return ops.gated_residual_fwd(res2d.contiguous(), y2d.contiguous(), b, rows, cols, gp=gp,
                                  gp_rs=cols if gp is not None else 0)


def _attention_out(x, p, prefix, nh, c, bias=None):
    """_attention_core (evoformer.py:173-198) on x [B, L, H] fp32 -> the module output [B*L, H]
    (before the residual).  bias: tensor broadcastable to the logits [B, nh, L, L] (added before
    the c^-1/2 scale, G1) or None."""
    B, L, H = x.shape
    rows = B * L
    x2 = x.reshape(rows, H)
    ln = _ln(x2, p, f"{prefix}/ln")
    cat = lambda part, key: np.concatenate([np.asarray(p[f"{prefix}/{part}/{h}/{key}"]) for h in range(nh)],
                                           axis=-1)
    q, k, v = (_lin(ln, cat(t, "w"), cat(t, "b")) for t in ("q", "k", "v"))
    heads = lambda t: t.view(B, L, nh, c).permute(0, 2, 1, 3).reshape(B * nh, L, c)
    logits = gemm_nt(heads(q), heads(k)).view(B, nh, L, L)
    a = ops.softmax_fwd(logits, bias=bias, scale=1.0 / math.sqrt(c))
    o = gemm_nt(a.view(B * nh, L, L), heads(v).transpose(1, 2))  # (a @ v) per head
    o2 = o.view(B, nh, L, c).permute(0, 2, 1, 3).reshape(rows, nh * c).contiguous()
    gpre = _lin(x2, cat("g", "w"), cat("g", "b")).contiguous()  # the gate reads raw x (G2)
    og = ops.gate_mul(gpre, o2, act=1)
    return _lin(og, p[f"{prefix}/o/w"])  # + o/b in the residual kernel


def _check_msa(m, cfg):
    if tuple(m.shape) != (cfg.n_seq, cfg.n_res, cfg.h_msa):
        raise DimensionError(f"MSA tensor shape {tuple(m.shape)} does not match config")


def _check_pair(z, cfg):
    if tuple(z.shape) != (cfg.n_res, cfg.n_res, cfg.h_pair):
        raise DimensionError(f"pair tensor shape {tuple(z.shape)} does not match config")


def msa_row_bias(z, p, cfg: EvoConfig):
    """evoformer.py:201-207 -> [N_r, N_r, n_head] fp32"""
    z = _dev(z)
    R = z.shape[0]
    ln = _ln(z.reshape(R * R, -1), p, "msa_row/ln_z")
    w = np.stack([np.asarray(p[f"msa_row/bias/{h}/w"]) for h in range(cfg.n_head_msa)], axis=-1)
    return _lin(ln, w).view(R, R, cfg.n_head_msa)


def msa_row_attention(m, z, p, cfg: EvoConfig):
    """m + msa_row_attention(m, z) (evoformer.py:219-223 and the residual of 316)"""
    m, z = _dev(m), _dev(z)
    _check_msa(m, cfg)
    _check_pair(z, cfg)
    bias = msa_row_bias(z, p, cfg).permute(2, 0, 1)  # [nh, i, j], shared over sequences
    y = _attention_out(m, p, "msa_row", cfg.n_head_msa, cfg.c_msa, bias=bias)
    S, R, H = m.shape
    return _residual(m.reshape(-1, H), y, p["msa_row/o/b"]).view(S, R, H)


def msa_col_attention(m, p, cfg: EvoConfig):
    """m + msa_col_attention(m) (evoformer.py:226-234, no bias G5)"""
    m = _dev(m)
    _check_msa(m, cfg)
    S, R, H = m.shape
    mt = m.permute(1, 0, 2).contiguous()
    y = _attention_out(mt, p, "msa_col", cfg.n_head_msa, cfg.c_msa)
    y = y.view(R, S, H).permute(1, 0, 2).reshape(S * R, H)
    return _residual(m.reshape(-1, H), y, p["msa_col/o/b"]).view(S, R, H)


def transition(x, p, prefix: str):
    """x + transition(x) (evoformer.py:237-240): LN -> W1 + b1 -> ReLU -> W2 + b2"""
    x = _dev(x)
    shape = x.shape
    x2 = x.reshape(-1, shape[-1])
    h = _lin(_ln(x2, p, f"{prefix}/ln"), p[f"{prefix}/w1"]).contiguous()
    ops.bias_act_fwd(h, _dev(p[f"{prefix}/b1"]), h.shape[0], h.shape[1], relu=True)
    return _residual(x2, _lin(h, p[f"{prefix}/w2"]), p[f"{prefix}/b2"]).view(shape)


def outer_product_mean(m, z, p, cfg: EvoConfig):
    """z + outer_product_mean(m) (evoformer.py:243-255): o[i,j,p,q] = sum_s a[s,i,p] b[s,j,q] / N_s,
    flattened p-major (G6), then W_o + b_o"""
    m, z = _dev(m), _dev(z)
    _check_msa(m, cfg)
    S, R, H = m.shape
    P = cfg.hidden_proj
    ln = _ln(m.reshape(S * R, H), p, "opm/ln")
    a = _lin(ln, p["opm/a/w"], p["opm/a/b"]).view(S, R, P)
    b = _lin(ln, p["opm/b/w"], p["opm/b/b"]).view(S, R, P)
    ip = lambda t: t.permute(1, 2, 0).reshape(R * P, S)  # [(i, p), s]
    o = gemm_nt(ip(a), ip(b), alpha=1.0 / S).view(R, P, R, P).permute(0, 2, 1, 3).reshape(R * R, P * P)
    Hz = z.shape[-1]
    return _residual(z.reshape(-1, Hz), _lin(o, p["opm/o/w"]), p["opm/o/b"]).view(R, R, Hz)


def _triangle(z, p, prefix, incoming: bool):
    """z + tri_update_{outgoing,incoming}(z) (evoformer.py:258-284)"""
    R, _, Hz = z.shape
    z2 = z.reshape(R * R, Hz)
    ln = _ln(z2, p, f"{prefix}/ln")
    gpre = _lin(ln, p[f"{prefix}/g/w"], p[f"{prefix}/g/b"])

    def factor(name):
        sig = _lin(ln, p[f"{prefix}/{name}_sig/w"], p[f"{prefix}/{name}_sig/b"]).contiguous()
        lin = _lin(ln, p[f"{prefix}/{name}_lin/w"], p[f"{prefix}/{name}_lin/b"]).contiguous()
        return ops.gate_mul(sig, lin, act=1).view(R, R, -1)  # sigmoid(sig) * lin

    a, b = factor("a"), factor("b")
    P = a.shape[-1]
    if incoming:  # t[i,j,h] = sum_k a[k,i,h] b[k,j,h]
        A, B = a.permute(2, 1, 0), b.permute(2, 1, 0)
    else:  # t[i,j,h] = sum_k a[i,k,h] b[j,k,h]
        A, B = a.permute(2, 0, 1), b.permute(2, 0, 1)
    t = gemm_nt(A, B).permute(1, 2, 0).reshape(R * R, P)  # [h, i, j] -> [(i, j), h]
    y = _lin(_ln(t, p, f"{prefix}/ln2"), p[f"{prefix}/o/w"])
    return _residual(z2, y, p[f"{prefix}/o/b"], gate_pre=gpre).view(R, R, Hz)


def tri_update_outgoing(z, p, cfg: EvoConfig):
    z = _dev(z)
    _check_pair(z, cfg)
    return _triangle(z, p, "tri_out", incoming=False)


def tri_update_incoming(z, p, cfg: EvoConfig):
    z = _dev(z)
    _check_pair(z, cfg)
    return _triangle(z, p, "tri_in", incoming=True)


def _pair_attention(zt, p, prefix, cfg):
    """_attention_core with the per-key bias of the row's own LN (_pair_bias_fn, evoformer.py:287-292, G4)"""
    B, L, H = zt.shape
    nh = cfg.n_head_pair
    ln = _ln(zt.reshape(B * L, H), p, f"{prefix}/ln")
    w = np.stack([np.asarray(p[f"{prefix}/bias/{h}/w"]) for h in range(nh)], axis=-1)
    kb = _lin(ln, w).view(B, L, nh).permute(0, 2, 1)[:, :, None, :]  # [B, nh, 1, L(key)]
    return _attention_out(zt, p, prefix, nh, cfg.c_pair, bias=kb)


def pair_attention_row(z, p, cfg: EvoConfig):
    """z + pair_attention_row(z) (evoformer.py:295-299)"""
    z = _dev(z)
    _check_pair(z, cfg)
    R, _, Hz = z.shape
    y = _pair_attention(z, p, "pair_row", cfg)
    return _residual(z.reshape(-1, Hz), y, p["pair_row/o/b"]).view(R, R, Hz)


def pair_attention_col(z, p, cfg: EvoConfig):
    """z + pair_attention_col(z) (evoformer.py:302-311)"""
    z = _dev(z)
    _check_pair(z, cfg)
    R, _, Hz = z.shape
    y = _pair_attention(z.permute(1, 0, 2).contiguous(), p, "pair_col", cfg)
    y = y.view(R, R, Hz).permute(1, 0, 2).reshape(R * R, Hz)
    return _residual(z.reshape(-1, Hz), y, p["pair_col/o/b"]).view(R, R, Hz)


def evoformer_block(m, z, p, cfg: EvoConfig):
    """evoformer_block (evoformer.py:314-325) at reference precision: returns (m', z') as fp32 CUDA
    tensors; numpy inputs are accepted (float64 is rounded to fp32 on the way in)."""
    m, z = _dev(m), _dev(z)
    _check_msa(m, cfg)
    _check_pair(z, cfg)
    m = msa_row_attention(m, z, p, cfg)
    m = msa_col_attention(m, p, cfg)
    m = transition(m, p, "msa_trans")
    z = outer_product_mean(m, z, p, cfg)
    z = tri_update_outgoing(z, p, cfg)
    z = tri_update_incoming(z, p, cfg)
    z = pair_attention_row(z, p, cfg)
    z = pair_attention_col(z, p, cfg)
    z = transition(z, p, "pair_trans")
    return m, z
