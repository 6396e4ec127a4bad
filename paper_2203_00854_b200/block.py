"""Forward / backward of one Evoformer block on the GPU (bf16 activations, fp32
statistics and accumulation).

Each sub-module of ``evoformer_block`` (evoformer.py:314-325) is a pair
``<name>_fwd(bp, ..., save) -> x_new`` / ``<name>_bwd(bp, saved, dx_new) -> dx``
composed of libevo.so kernels (LayerNorm, fused attention, tcgen05 batched GEMM,
gating / residual epilogues) and cuBLAS for the plain projection GEMMs
(the "K7 merged projections" of SURVEY.md 2.1).  Residual adds are fused into
the epilogues, so every ``*_fwd`` returns the updated stream (x + f(x)) and
every ``*_bwd`` returns d(input) = d(output) + df/dx.

Activation layout in HBM: m = [N_s, N_r, H_m] and z = [N_r, N_r, H_z], bf16,
row-major; every sub-module works on the 2-D view [rows, channels].  The
transposed variants (msa_col, pair_col, tri_in) never copy: they hand the
kernels strides (attention) or MN-major operands (batched GEMM).
"""

from __future__ import annotations

import math

import torch

from . import ops
from .config import EvoConfig
from .ops import Mat, Strided
from .params import BlockParams

BF16 = torch.bfloat16
F32 = torch.float32


def _mm(a, b):
    return torch.mm(a, b)


class SideStream:
    """Parameter-gradient work (weight GEMMs, bias column sums) is off the critical
    path of the input-gradient chain: it is forked onto a side CUDA stream (event
    fork/join, also captured into CUDA graphs) so it fills the gaps left by the
    latency-bound kernels of the main stream.  ``join()`` before reading grads."""

    enabled = True
    stream = None

    @classmethod
    def run(cls, fn, *keep):
        if not (cls.enabled and keep and keep[0].is_cuda):
            return fn()
        if cls.stream is None:
            cls.stream = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        cls.stream.wait_stream(main)
        with torch.cuda.stream(cls.stream):
            fn()
        for t in keep:  # the main stream's allocator must not recycle these before the side work ran
            t.record_stream(cls.stream)

    @classmethod
    def join(cls):
        if cls.stream is not None and torch.cuda.is_available():
            torch.cuda.current_stream().wait_stream(cls.stream)


def _wgrad(x, dy, out):
    """out (fp32) += x^T @ dy with fp32 accumulation (side stream).  Every parameter gradient
    ACCUMULATES into bp.grad (micro-batch accumulation works; zero_grad() between steps)."""
    if x.is_cuda:  # cuBLAS, beta = 1: the fp32 result is added straight into the grad buffer view
        # (evo_wgrad, the tcgen05 split-K form, matches cuBLAS in isolation but measured 1 % slower in
        # the step: its all-SM grid competes with the main stream's kernels; profiles/r02_wgrad_*)
        SideStream.run(lambda: torch.addmm(out, x.t(), dy, out_dtype=F32, out=out), x, dy)
    else:  # CPU only in the host-logic tests (fake kernel backend)
        out += x.t().float() @ dy.float()


def _bgrad(dy, out):
    """bias gradient (accumulated into the zeroed fp32 grad view; side stream)"""
    if dy.is_cuda:
        SideStream.run(lambda: ops.colsum(dy, out), dy)
    else:  # CPU only in the host-logic tests (fake kernel backend)
        out += dy.float().sum(0)


def _dbias_only(dx_new, rows, cols, out):
    """dbias = column sums of the residual-stream gradient (side stream)"""
    if dx_new.is_cuda:
        SideStream.run(lambda: ops.colsum(dx_new, out, rows, cols), dx_new)
    else:
        ops.gated_residual_bwd(dx_new, rows, cols, dbias=out)


class Saved(dict):
    """activations saved by a forward for its backward"""


class LnChain:
    """The next module's LayerNorm parameters handed to a module's residual epilogue: the
    residual add and that LayerNorm run as one kernel (evo_residual_layernorm_fwd) and the
    result (ln, mean, rstd) is picked up by the next module instead of recomputing it."""

    def __init__(self, gamma, beta):
        self.gamma, self.beta, self.result = gamma, beta, None


def _layernorm_in(x2d, gamma, beta, rows, cols, pre_ln):
    """the module's input LayerNorm: the chained result when the previous epilogue made it"""
    if pre_ln is not None and pre_ln.result is not None:
        return pre_ln.result
    return ops.layernorm_fwd(x2d, gamma, beta, rows, cols)


def _residual_out(res, y, bias, rows, cols, next_ln, gp=None, gp_rs=0):
    """residual epilogue, fused with the next module's LayerNorm when chained"""
    if next_ln is not None and res.is_cuda and cols in (32, 64, 128, 256):
        out, ln, mean, rstd = ops.residual_layernorm_fwd(res, y, bias, rows, cols, next_ln.gamma, next_ln.beta, gp=gp,
                                                         gp_rs=gp_rs)
        next_ln.result = (ln, mean, rstd)
        return out
    return ops.gated_residual_fwd(res, y, bias, rows, cols, gp=gp, gp_rs=gp_rs)


# ----------------------------------------------------------------------------- attention
def _attn_geometry(kind: str, B: int, L: int):
    """rows of the [rows, C] view for attention batch b / position l:
    row = b*sb + l*sl  (row-wise: batch = leading axis; column-wise: transposed)."""
    return (L, 1) if kind == "row" else (1, B)


def attention_fwd(bp: BlockParams, mod: str, x2d, B: int, L: int, kind: str, bias=None, save=True, pre_ln=None,
                  next_ln=None, flags=0):
    """_attention_core (evoformer.py:173-198) + residual: returns x + attn(x).
    flags: EVO_ATTN_* kernel-selection hints (0 = automatic; tests force each variant).

    kind "row": attention along the second axis of [B, L, C]; "col": x2d is
    [L, B, C] and attention runs along the first axis (msa_col / pair_col).
    bias: None, ("full", tensor [nh, L, L]) shared over the batch (msa_row), or
    "pair" = per-key bias from the merged projection (pair_row / pair_col).
    """
    a = bp.layout.attn[mod]
    H, nh, c, ldq = a["H"], a["nh"], a["c"], a["ldq"]
    rows = B * L
    h, f = bp.h, bp.f
    ln, mean, rstd = _layernorm_in(x2d, f[f"{mod}.ln_g"], f[f"{mod}.ln_b"], rows, H, pre_ln)
    qkv = torch.addmm(h[f"{mod}.b_qkv"], ln, h[f"{mod}.w_qkv"])
    gpre = torch.addmm(h[f"{mod}.b_g"], x2d, h[f"{mod}.w_g"])
    og = torch.empty(rows, nh * c, device=x2d.device, dtype=BF16)
    orw = torch.empty_like(og)
    lse = torch.empty(B, nh, L, device=x2d.device, dtype=F32)
    sbr, slr = _attn_geometry(kind, B, L)
    S = lambda t, ld, off=0: Strided(t, sbr * ld, slr * ld, off)
    if callable(bias):  # deferred (e.g. a DAP all-gather completing while the GEMMs above ran)
        bias = bias()
    if bias is None:
        bt, bs, boff = None, (0, 0, 0, 0), 0
    elif isinstance(bias, str) and bias == "pair":
        bt, bs, boff = qkv, (sbr * ldq, 1, 0, slr * ldq), 3 * nh * c
    else:
        bt, bs, boff = bias, (0, L * L, L, 1), 0
    desc = ops.attention_desc(S(qkv, ldq, 0), S(qkv, ldq, nh * c), S(qkv, ldq, 2 * nh * c), S(gpre, nh * c),
                              S(og, nh * c), S(orw, nh * c), lse, B, L, nh, c, 1.0 / math.sqrt(c),
                              bias=bt, bias_s=bs, bias_off=boff, flags=flags)
    ops.attention_fwd(desc)
    y = _mm(og, h[f"{mod}.w_o"])
    out = _residual_out(x2d, y, f[f"{mod}.b_o"], rows, H, next_ln)
    sv = None
    if save:
        sv = Saved(x=x2d, ln=ln, mean=mean, rstd=rstd, qkv=qkv, gpre=gpre, og=og, orw=orw, lse=lse,
                   desc=desc, B=B, L=L, kind=kind, bias=bias, mod=mod)  # bias: resolved tensor / "pair" / None
    return out, sv


def attention_bwd(bp: BlockParams, sv: Saved, dx_new, next_db=None, db_done=False):
    """returns (dx, dbias) with dx = dx_new + d attn / dx; dbias fp32 for "full" bias.
    next_db: bias-gradient buffer of the module consuming dx (its column sums are fused into
    the final LayerNorm backward); db_done: this module's b_o gradient was already produced
    that way by the module that wrote dx_new."""
    mod, B, L, kind = sv["mod"], sv["B"], sv["L"], sv["kind"]
    a = bp.layout.attn[mod]
    H, nh, c, ldq = a["H"], a["nh"], a["c"], a["ldq"]
    rows = B * L
    h, f, g = bp.h, bp.f, bp.g
    dev = dx_new.device
    if not db_done:
        _dbias_only(dx_new, rows, H, g[f"{mod}.b_o"])  # db_o = sum_r dx_new
    dog = _mm(dx_new, h[f"{mod}.w_o"].t())
    _wgrad(sv["og"], dx_new, g[f"{mod}.w_o"])
    sbr, slr = _attn_geometry(kind, B, L)
    S = lambda t, ld, off=0: Strided(t, sbr * ld, slr * ld, off)
    dqkv = torch.empty(rows, ldq, device=dev, dtype=BF16)
    pair_bias = isinstance(sv["bias"], str) and sv["bias"] == "pair"
    if ldq > 3 * nh * c and not pair_bias:  # (pair: the padding is written with the bias columns)
        dqkv[:, 3 * nh * c:].zero_()
    dgpre = torch.empty(rows, nh * c, device=dev, dtype=BF16)
    bias = sv["bias"]
    if bias is None:
        dbias, dbs = None, (0, 0, 0, 0)
    elif isinstance(bias, str) and bias == "pair":
        dbias, dbs = torch.zeros(B, nh, L, device=dev, dtype=F32), (nh * L, L, 0, 1)
    else:
        dbias, dbs = torch.zeros(nh, L, L, device=dev, dtype=F32), (0, L * L, L, 1)
    full_bias = bias is not None and not isinstance(bias, str)
    ws = torch.empty(ops.attention_bwd_workspace(B, L, nh, c, batch_reduced_bias=full_bias),
                     device=dev, dtype=torch.uint8)
    ops.attention_bwd(sv["desc"], S(dog, nh * c), S(dqkv, ldq, 0), S(dqkv, ldq, nh * c), S(dqkv, ldq, 2 * nh * c),
                      S(dgpre, nh * c), ws, dbias=dbias, dbias_s=dbs)
    if pair_bias:
        # fp32 [B, nh, L] -> the bias columns of dqkv (bf16) + zeroed row padding, one pass
        ops.key_bias_grad_cols(dbias, B, nh, L, S(dqkv, ldq, 3 * nh * c), ldq - 3 * nh * c)
    _wgrad(sv["ln"], dqkv, g[f"{mod}.w_qkv"])
    _bgrad(dqkv, g[f"{mod}.b_qkv"])
    _wgrad(sv["x"], dgpre, g[f"{mod}.w_g"])
    _bgrad(dgpre, g[f"{mod}.b_g"])
    dx = torch.addmm(dx_new, dgpre, h[f"{mod}.w_g"].t())          # gate reads raw x (G2)
    dln = _mm(dqkv, h[f"{mod}.w_qkv"].t())
    ops.layernorm_bwd(dln, sv["x"], f[f"{mod}.ln_g"], sv["mean"], sv["rstd"], rows, H, dx=dx, accumulate=True,
                      dgamma=g[f"{mod}.ln_g"], dbeta=g[f"{mod}.ln_b"], dx_colsum=next_db)
    return dx, (dbias if full_bias else None)


# ----------------------------------------------------------------------------- msa_row bias
def msa_row_bias_fwd(bp: BlockParams, z2d, n_i: int, n_j: int | None = None, save=True):
    """msa_row_bias (evoformer.py:201-207) -> bias[h][i][j] bf16.  n_i rows of z (an i-shard
    under DAP).  LN_z on the lane-group LayerNorm kernel, then the 8 (padded) head dots as one
    GEMM producing the head-major layout directly: bias = W^T LN(z)^T  ([8, rows])."""
    cfg = bp.cfg
    n_j = n_i if n_j is None else n_j
    nh = cfg.n_head_msa
    rows = n_i * n_j
    ln, mean, rstd = ops.layernorm_fwd(z2d, bp.f["msa_row.lnz_g"], bp.f["msa_row.lnz_b"], rows, cfg.h_pair)
    if ln.is_cuda:
        out = torch.mm(bp.h["msa_row.w_bias"].t(), ln.t())            # [8, rows] bf16
    else:  # CPU host-logic tests (fake kernel backend)
        out = (bp.f["msa_row.w_bias"].t() @ ln.float().t()).to(ln.dtype)
    out = out.view(-1, n_i, n_j)
    sv = Saved(z=z2d, ln=ln, mean=mean, rstd=rstd) if save else None
    return out[:nh], sv


def msa_row_bias_bwd(bp: BlockParams, sv: Saved, dbias, dz):
    """dbias fp32 [nh, n_i, n_j]; returns dz + dLN/dz (bf16 [n_i*n_j, Hz]) as a NEW tensor:
    d LN = dbias^T W^T (one K = nh GEMM), dW = LN^T dbias^T (side stream), LN backward with
    the residual-stream add and dgamma / dbeta fused.  Out of place because dz may still be
    read by side-stream weight-gradient GEMMs (opm's w_o) issued earlier in the block."""
    cfg = bp.cfg
    nh, Hz = cfg.n_head_msa, cfg.h_pair
    rows = dbias[0].numel()
    db2 = dbias.reshape(nh, rows)
    w = bp.f["msa_row.w_bias"][:, :nh]                                   # fp32 [Hz, nh]
    if not dz.is_cuda:  # CPU host-logic tests (fake kernel backend)
        dln = db2.t() @ w.t()
        bp.g["msa_row.w_bias"][:, :nh] += sv["ln"].float().t() @ db2.t()
    else:
        dln = torch.mm(db2.t(), w.t())                                  # fp32 [rows, Hz]
        db2h = db2.to(torch.bfloat16)
        gw = bp.g["msa_row.w_bias"]
        SideStream.run(lambda: gw[:, :nh].add_(torch.mm(sv["ln"].t(), db2h.t(), out_dtype=F32)), sv["ln"], db2h)
    return ops.layernorm_bwd(dln, sv["z"], bp.f["msa_row.lnz_g"], sv["mean"], sv["rstd"], rows, Hz, res=dz,
                             dgamma=bp.g["msa_row.lnz_g"], dbeta=bp.g["msa_row.lnz_b"])


# ----------------------------------------------------------------------------- transition
def transition_fwd(bp: BlockParams, mod: str, x2d, rows: int, save=True, pre_ln=None, next_ln=None):
    """transition (evoformer.py:237-240) + residual."""
    H = x2d.shape[1]
    h, f = bp.h, bp.f
    ln, mean, rstd = _layernorm_in(x2d, f[f"{mod}.ln_g"], f[f"{mod}.ln_b"], rows, H, pre_ln)
    if ln.is_cuda:  # bias + ReLU in the cuBLASLt epilogue (RELU_BIAS): hid is written once
        hid = torch._addmm_activation(h[f"{mod}.b1"], ln, h[f"{mod}.w1"])
    else:
        hid = _mm(ln, h[f"{mod}.w1"])
        ops.bias_act_fwd(hid, f[f"{mod}.b1"], rows, hid.shape[1], relu=True)
    y = _mm(hid, h[f"{mod}.w2"])
    out = _residual_out(x2d, y, f[f"{mod}.b2"], rows, H, next_ln)
    sv = Saved(x=x2d, ln=ln, mean=mean, rstd=rstd, hid=hid, mod=mod) if save else None
    return out, sv


def transition_bwd(bp: BlockParams, sv: Saved, dx_new, next_db=None, db_done=False):
    mod = sv["mod"]
    rows, H = dx_new.shape
    h, f, g = bp.h, bp.f, bp.g
    if not db_done:
        _dbias_only(dx_new, rows, H, g[f"{mod}.b2"])
    _wgrad(sv["hid"], dx_new, g[f"{mod}.w2"])
    dhid = _mm(dx_new, h[f"{mod}.w2"].t())
    dpre = ops.bias_act_bwd(dhid, sv["hid"], rows, dhid.shape[1], dy=dhid, dbias=g[f"{mod}.b1"])
    _wgrad(sv["ln"], dpre, g[f"{mod}.w1"])
    dln = _mm(dpre, h[f"{mod}.w1"].t())
    dx = torch.empty_like(dx_new)
    ops.layernorm_bwd(dln, sv["x"], f[f"{mod}.ln_g"], sv["mean"], sv["rstd"], rows, H, dx=dx, res=dx_new,
                      dgamma=g[f"{mod}.ln_g"], dbeta=g[f"{mod}.ln_b"], dx_colsum=next_db)
    return dx


# ----------------------------------------------------------------------------- outer product mean
def opm_fwd(bp: BlockParams, m2d, z2d, S: int, R: int, save=True, b_full=None, Rj=None, gather=None, pre_ln=None,
            next_ln=None):
    """outer_product_mean (evoformer.py:243-255) + residual into z.

    Fused path (evo_opm_fused_fwd, P = 32, N_s <= 128, R % 32 == 0): the projections are turned
    sequence-contiguous ([R, P, S], evo_opm_transpose) and o[i][j][p][q] = sum_s a b / S is
    contracted with W_o tile by tile on chip; o reaches HBM only when ``save`` (the backward's
    operand).  Otherwise o is ONE tcgen05 GEMM (M = i*p, N = j*q, K = s) written straight into
    the [i][j][p][q] layout, then o @ W_o.
    Under DAP, a is local and b is all-gathered (rank-major [N_dev, R_loc, P, S] = [J, P, S] for
    the fused kernel, [N_dev, S, R_loc, P] otherwise), addressed without unpacking.
    """
    cfg = bp.cfg
    P, Hm, Hz = cfg.hidden_proj, cfg.h_msa, cfg.h_pair
    rows_m = S * R
    h, f = bp.h, bp.f
    ln, mean, rstd = _layernorm_in(m2d, f["opm.ln_g"], f["opm.ln_b"], rows_m, Hm, pre_ln)
    # evo_opm_fused_fwd when the extents allow it (J = N_dev * R is then a multiple of 8 as well)
    fused = ops.opm_fused_supported(R, R, S, P, Hz)
    if gather is None:
        ab = torch.addmm(h["opm.b_ab"], ln, h["opm.w_ab"])          # [S*R, 2P] = [a | b]
        pending = None
    else:
        # DAP: the right projection first; its all-gather is in flight on the communicator's
        # stream while the left projection runs (DAO).  a and b are separate
        # [S*R, P] buffers, so the overlapped and the synchronous schedules compute the same bits.
        bl = torch.addmm(h["opm.b_ab"][P:], ln, h["opm.w_ab"][:, P:])
        # the fused kernel reads b sequence-contiguous: the gathered blocks [R_loc][P][S] stack into [J][P][S]
        pending = gather(ops.opm_transpose(bl, S, R, P) if fused else bl, async_op=True)
        ab = torch.addmm(h["opm.b_ab"][:P], ln, h["opm.w_ab"][:, :P])   # a only
    if fused:
        if pending is None:
            a_t, b_t = ops.opm_transpose(ab, S, R, P, both=True)    # [R, P, S] each
            bsrc = None
        else:
            a_t = ops.opm_transpose(ab, S, R, P)
            b_t = pending().reshape(-1, P, S)                       # [J, P, S]
            bsrc = b_t
        Rj = b_t.shape[0]
        # evo_opm_fused_fwd: o stays on chip; training also stores it (bf16) for the backward
        o = torch.empty(R, Rj, P, P, device=m2d.device, dtype=BF16) if save else None
        y = ops.opm_fused_fwd(a_t, b_t, h["opm.w_o"], R, Rj, S, P, Hz, 1.0 / S, o_save=o)
    else:  # tcgen05 contraction into o [R, Rj, P, P], then o @ W_o
        if pending is None:
            A = Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0))
            Rj = R
            bsrc = ab
            B = Mat(ab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P)
        else:
            A = Mat(ab, lo=(1, R * P))
            bsrc = pending()
            Rj = bsrc.shape[0] * R
            B = Mat(bsrc, lo=(1, R * P), split=(R * P, 0), hi=(S * R * P, 0))
        o = torch.empty(R, Rj, P, P, device=m2d.device, dtype=BF16)
        Cm = Mat(o, lo=(P, 1), split=(P, P), hi=(Rj * P * P, P * P))
        ops.bgemm(A, B, Cm, 1, R * P, Rj * P, S, alpha=1.0 / S)
        y = _mm(o.view(R * Rj, P * P), h["opm.w_o"])
    out = _residual_out(z2d, y, f["opm.b_o"], R * Rj, Hz, next_ln)
    sv = Saved(m=m2d, ln=ln, mean=mean, rstd=rstd, ab=ab, bsrc=bsrc, o=o, S=S, R=R, Rj=Rj,
               gathered=gather is not None, b_seq=fused and gather is not None,
               a_t=a_t if fused else None, b_t=b_t if fused else None) if save else None
    return out, sv


def opm_contract(a2d, b2d, S: int, I: int, J: int, P: int):
    """o[i][j][p][q] = sum_s a[s, i, p] b[s, j, q] / S (evoformer.py:253) for separate projections
    a [S, I*P], b [S, J*P] (outer_product_mean_from_projections): one tcgen05 GEMM with M = (i,p),
    N = (j,q), K = s, both operands MN-major, written straight into the [i][j][p][q] layout."""
    o = torch.empty(I, J, P, P, device=a2d.device, dtype=BF16)
    A = Mat(a2d, lo=(1, a2d.stride(0)))
    B = Mat(b2d, lo=(1, b2d.stride(0)))
    Cm = Mat(o, lo=(P, 1), split=(P, P), hi=(J * P * P, P * P))
    ops.bgemm(A, B, Cm, 1, I * P, J * P, S, alpha=1.0 / S)
    return o


def opm_bwd(bp: BlockParams, sv: Saved, dz_new, dm, reduce_scatter=None, next_db=None, db_done=False):
    """returns dm + the OPM's input gradient as a NEW bf16 [S*R, Hm] tensor (dm is only read, so
    the caller's gradient needs no defensive copy); dz passes through.
    next_db: bias gradient of the module consuming dm (fused column sums of the final dm)."""
    cfg = bp.cfg
    P, Hm, Hz = cfg.hidden_proj, cfg.h_msa, cfg.h_pair
    S, R, Rj = sv["S"], sv["R"], sv["Rj"]
    h, f, g = bp.h, bp.f, bp.g
    if not db_done:
        _dbias_only(dz_new, R * Rj, Hz, g["opm.b_o"])
    _wgrad(sv["o"].view(R * Rj, P * P), dz_new, g["opm.w_o"])
    dab = torch.empty(S * R, 2 * P, device=dz_new.device, dtype=BF16)
    if sv.get("a_t") is not None and ops.opm_bwd_supported(R, Rj, S, P, Hz):
        # evo_opm_bwd_factor: da and db straight from dz and W_o - do = dz W_o^T is never materialised
        w_o = h["opm.w_o"]
        if not sv["gathered"]:
            ops.opm_bwd_factor(0, dz_new, w_o, sv["b_t"], R, Rj, S, P, Hz, 1.0 / S, dab, R * 2 * P, 0, 2 * P)
            ops.opm_bwd_factor(1, dz_new, w_o, sv["a_t"], Rj, R, S, P, Hz, 1.0 / S, dab[:, P:], R * 2 * P, 0, 2 * P)
        else:
            # the gathered factor's rank-major fp32 partial first: its reduce-scatter overlaps da
            nd = Rj // R
            dbf = torch.empty(nd, S, R, P, device=dz_new.device, dtype=F32)
            ops.opm_bwd_factor(1, dz_new, w_o, sv["a_t"], Rj, R, S, P, Hz, 1.0 / S, dbf, R * P, S * R * P, P,
                               x_split=R)
            pending = reduce_scatter(dbf, async_op=True)
            ops.opm_bwd_factor(0, dz_new, w_o, sv["b_t"], R, Rj, S, P, Hz, 1.0 / S, dab, R * 2 * P, 0, 2 * P)
            dab[:, P:].copy_(pending().view(S * R, P))
        return _opm_proj_bwd(bp, sv, dab, dm, next_db)
    do = _mm(dz_new, h["opm.w_o"].t())                               # [R*Rj, P*P] == [i][j][p][q]
    ab = sv["ab"]                                                    # [a | b], or a alone under DAP
    dO_A = Mat(do, lo=(P, 1), split=(P, P), hi=(Rj * P * P, P * P))
    Cda = Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0))
    dO_T = Mat(do, lo=(1, P), split=(P, P), hi=(P * P, Rj * P * P))
    if not sv["gathered"]:
        # da[s,i,p] = sum_{j,q} do[i,j,p,q] b[s,j,q] / S      (M = (i,p), N = s, K = (j,q))
        Bb = Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P), offset=P)
        ops.bgemm(dO_A, Bb, Cda, 1, R * P, S, Rj * P, alpha=1.0 / S)
        # db[s,j,q] = sum_{i,p} a[s,i,p] do[i,j,p,q] / S      (M = (j,q), N = s, K = (i,p))
        Ba = Mat(ab, lo=(R * 2 * P, 1), split=(0, P), hi=(0, 2 * P))
        Cdb = Mat(dab, lo=(1, R * 2 * P), split=(P, 0), hi=(2 * P, 0), offset=P)
        ops.bgemm(dO_T, Ba, Cdb, 1, Rj * P, S, R * P, alpha=1.0 / S)
    else:
        # the gathered factor's partial gradient first: its reduce-scatter overlaps the da GEMM
        nd = Rj // R
        dbf = torch.empty(nd, S, R, P, device=dz_new.device, dtype=F32)   # rank-major partials
        Cdb = Mat(dbf, lo=(1, R * P), split=(R * P, 0), hi=(S * R * P, 0))
        ops.bgemm(dO_T, Mat(ab, lo=(R * P, 1)), Cdb, 1, Rj * P, S, R * P, alpha=1.0 / S)
        pending = reduce_scatter(dbf, async_op=True)
        if sv["b_seq"]:  # gathered b sequence-contiguous [J][P][S] (fused forward): (n = s, k = (j, q))
            Bb = Mat(sv["bsrc"], lo=(1, S))
        else:
            Bb = Mat(sv["bsrc"], lo=(R * P, 1), split=(0, R * P), hi=(0, S * R * P))
        ops.bgemm(dO_A, Bb, Cda, 1, R * P, S, Rj * P, alpha=1.0 / S)
        dab[:, P:].copy_(pending().view(S * R, P))
    return _opm_proj_bwd(bp, sv, dab, dm, next_db)


def _opm_proj_bwd(bp: BlockParams, sv: Saved, dab, dm, next_db):
    """backward of the [a | b] projection and the OPM's input LayerNorm: returns dm + dLN/dm"""
    Hm, S, R = bp.cfg.h_msa, sv["S"], sv["R"]
    h, f, g = bp.h, bp.f, bp.g
    _wgrad(sv["ln"], dab, g["opm.w_ab"])
    _bgrad(dab, g["opm.b_ab"])
    dln = _mm(dab, h["opm.w_ab"].t())
    return ops.layernorm_bwd(dln, sv["m"], f["opm.ln_g"], sv["mean"], sv["rstd"], S * R, Hm, res=dm,
                             dgamma=g["opm.ln_g"], dbeta=g["opm.ln_b"], dx_colsum=next_db)


# ----------------------------------------------------------------------------- triangle update
def triangle_fwd(bp: BlockParams, mod: str, z2d, R: int, save=True, Rl=None, gather=None, pre_ln=None, next_ln=None):
    """tri_update_outgoing / incoming (evoformer.py:258-284) + residual.

    Y = LN(z) @ [W_g|W_as|W_al|W_bs|W_bl] + b (cuBLAS);  a, b = sigmoid gating
    written channel-major (one kernel);  t_h = a_h b_h^T (outgoing) or
    a_h^T b_h (incoming) as ONE batched tcgen05 GEMM over the p channels
    (MN-major operands for incoming, no transposes);  LN over channels read
    channel-major;  out = z + sigmoid(g) * (LN2(t) @ W_o + b_o) (one epilogue).
    Single GPU: Rl = R.  DAP (outgoing: z is an i-shard [Rl, R]; incoming: a
    j-shard stored as [R, Rl]): the other factor is all-gathered rank-major by
    ``gather`` and addressed in place.
    """
    cfg = bp.cfg
    P, Hz = cfg.hidden_proj, cfg.h_pair
    incoming = mod == "tri_in"
    Rl = R if Rl is None else Rl
    rows = R * Rl
    h, f = bp.h, bp.f
    ln, mean, rstd = _layernorm_in(z2d, f[f"{mod}.ln_g"], f[f"{mod}.ln_b"], rows, Hz, pre_ln)
    Y = torch.addmm(h[f"{mod}.b_proj"], ln, h[f"{mod}.w_proj"])       # [rows, Hz + 4P]
    a_cm = torch.empty(P, rows, device=z2d.device, dtype=BF16)
    b_cm = torch.empty_like(a_cm)
    ops.tri_gate_fwd(Y, rows, Hz, P, a_cm, b_cm)
    # local shapes: outgoing z-shard rows i (Rl), cols k (R); incoming rows k (R), cols j (Rl)
    if not incoming:
        A = Mat(a_cm, lo=(R, 1), batch_stride=rows)                   # A_h[i][k], K-major
        if gather is None:
            Bm, N = Mat(b_cm, lo=(R, 1), batch_stride=rows), R        # B_h[j][k], K-major
            bfull = b_cm
        else:
            bfull = gather(b_cm)                                      # [N, P, Rl, R]
            N = bfull.shape[0] * Rl
            Bm = Mat(bfull, lo=(R, 1), split=(Rl, 0), hi=(P * Rl * R, 0), batch_stride=Rl * R)
        M = Rl
        t_cm = torch.empty(P, M, N, device=z2d.device, dtype=BF16)
        ops.bgemm(A, Bm, Mat(t_cm, lo=(N, 1), batch_stride=M * N), P, M, N, R)
        afull = a_cm
    else:
        Bm = Mat(b_cm, lo=(1, Rl), batch_stride=rows)                 # B_h[j][k] = b[k][j], MN-major
        if gather is None:
            A, M = Mat(a_cm, lo=(1, R), batch_stride=rows), R          # A_h[i][k] = a[k][i], MN-major
            afull = a_cm
        else:
            afull = gather(a_cm)                                      # [N, P, R, Rl]  (cols i gathered)
            M = afull.shape[0] * Rl
            A = Mat(afull, lo=(1, Rl), split=(Rl, 0), hi=(P * R * Rl, 0), batch_stride=R * Rl)
        N = Rl
        t_cm = torch.empty(P, M, N, device=z2d.device, dtype=BF16)
        ops.bgemm(A, Bm, Mat(t_cm, lo=(N, 1), batch_stride=M * N), P, M, N, R)
        bfull = b_cm
    ln2, mean2, rstd2 = ops.layernorm_fwd(t_cm, f[f"{mod}.ln2_g"], f[f"{mod}.ln2_b"], rows, P, x_rs=1, x_cs=rows)
    y2 = _mm(ln2, h[f"{mod}.w_o"])
    out = _residual_out(z2d, y2, f[f"{mod}.b_o"], rows, Hz, next_ln, gp=Y, gp_rs=Hz + 4 * P)
    sv = Saved(z=z2d, ln=ln, mean=mean, rstd=rstd, Y=Y, a_cm=a_cm, b_cm=b_cm, afull=afull, bfull=bfull,
               t_cm=t_cm, ln2=ln2, mean2=mean2, rstd2=rstd2, y2=y2, mod=mod, R=R, Rl=Rl, M=M, N=N,
               gathered=gather is not None) if save else None
    return out, sv


def triangle_bwd(bp: BlockParams, sv: Saved, dz_new, reduce_scatter=None, next_db=None):
    cfg = bp.cfg
    P, Hz = cfg.hidden_proj, cfg.h_pair
    mod, R, Rl, M, N = sv["mod"], sv["R"], sv["Rl"], sv["M"], sv["N"]
    incoming = mod == "tri_in"
    rows = R * Rl
    h, f, g = bp.h, bp.f, bp.g
    dev = dz_new.device
    ld = Hz + 4 * P
    dY = torch.empty(rows, ld, device=dev, dtype=BF16)
    dy2 = torch.empty(rows, Hz, device=dev, dtype=BF16)
    # the merged projection's bias gradient comes out of the two epilogues in fp32 (before
    # dY is rounded to bf16): g part here, a/b part in tri_gate_bwd
    ops.gated_residual_bwd(dz_new, rows, Hz, y=sv["y2"], bias=f[f"{mod}.b_o"], gp=sv["Y"], gp_rs=ld, dy=dy2,
                           dgp=dY, dgp_rs=ld, dbias=g[f"{mod}.b_o"], dgp_sum=g[f"{mod}.b_proj"][:Hz])
    _wgrad(sv["ln2"], dy2, g[f"{mod}.w_o"])
    dln2 = _mm(dy2, h[f"{mod}.w_o"].t())                              # [rows, P]
    dt_cm = torch.empty(P, rows, device=dev, dtype=BF16)
    ops.layernorm_bwd(dln2, sv["t_cm"], f[f"{mod}.ln2_g"], sv["mean2"], sv["rstd2"], rows, P, x_rs=1, x_cs=rows,
                      dx=dt_cm, dgamma=g[f"{mod}.ln2_g"], dbeta=g[f"{mod}.ln2_b"])
    da_cm = torch.empty(P, rows, device=dev, dtype=BF16)
    db_cm = torch.empty(P, rows, device=dev, dtype=BF16)
    dT = Mat(dt_cm, lo=(N, 1), batch_stride=M * N)                    # dT_h[i][j] K-major over j
    dTt = Mat(dt_cm, lo=(1, N), batch_stride=M * N)                   # as [j][i]
    if not incoming:
        # t[i][j] = sum_k a[i][k] b[j][k]:  da = dT b,  db = dT^T a   (b gathered under DAP)
        bfull = sv["bfull"]
        if not sv["gathered"]:
            Bb = Mat(bfull, lo=(1, R), batch_stride=rows)             # [N=k][K=j] MN-major
        else:
            Bb = Mat(bfull, lo=(1, R), split=(0, Rl), hi=(0, P * Rl * R), batch_stride=Rl * R)
        Aa = Mat(sv["a_cm"], lo=(1, R), batch_stride=rows)            # [N=k][K=i] MN-major
        if not sv["gathered"]:
            ops.bgemm(dT, Bb, Mat(da_cm, lo=(R, 1), batch_stride=rows), P, M, R, N)
            ops.bgemm(dTt, Aa, Mat(db_cm, lo=(R, 1), batch_stride=rows), P, N, R, M)
        else:
            # the gathered factor's partial gradient first: its reduce-scatter overlaps the da GEMM
            nd = N // Rl
            dbf = torch.empty(nd, P, Rl, R, device=dev, dtype=F32)
            ops.bgemm(dTt, Aa, Mat(dbf, lo=(R, 1), split=(Rl, 0), hi=(P * Rl * R, 0), batch_stride=Rl * R),
                      P, N, R, M)
            pending = reduce_scatter(dbf, async_op=True)
            ops.bgemm(dT, Bb, Mat(da_cm, lo=(R, 1), batch_stride=rows), P, M, R, N)
            db_cm.copy_(pending().view(P, rows))
    else:
        # t[i][j] = sum_k a[k][i] b[k][j]:  da[k][i] = sum_j b[k][j] dT[i][j],  db[k][j] = sum_i a[k][i] dT[i][j]
        Ab = Mat(sv["b_cm"], lo=(Rl, 1), batch_stride=rows)           # [M=k][K=j] K-major
        if not sv["gathered"]:
            ops.bgemm(Ab, dT, Mat(da_cm, lo=(R, 1), batch_stride=rows), P, R, M, N)
            Aa = Mat(sv["afull"], lo=(R, 1), batch_stride=rows)
        else:
            nd = M // Rl
            daf = torch.empty(nd, P, R, Rl, device=dev, dtype=F32)
            ops.bgemm(Ab, dT, Mat(daf, lo=(Rl, 1), split=(0, Rl), hi=(0, P * R * Rl), batch_stride=R * Rl),
                      P, R, M, N)
            pending = reduce_scatter(daf, async_op=True)             # overlaps the db GEMM below
            Aa = Mat(sv["afull"], lo=(Rl, 1), split=(0, Rl), hi=(0, P * R * Rl), batch_stride=R * Rl)
        ops.bgemm(Aa, dTt, Mat(db_cm, lo=(Rl, 1), batch_stride=rows), P, R, N, M)
        if sv["gathered"]:
            da_cm.copy_(pending().view(P, rows))
    ops.tri_gate_bwd(sv["Y"], da_cm, db_cm, rows, Hz, P, dY, dsum=g[f"{mod}.b_proj"][Hz:])
    _wgrad(sv["ln"], dY, g[f"{mod}.w_proj"])
    dln = _mm(dY, h[f"{mod}.w_proj"].t())
    dz = torch.empty_like(dz_new)
    ops.layernorm_bwd(dln, sv["z"], f[f"{mod}.ln_g"], sv["mean"], sv["rstd"], rows, Hz, dx=dz, res=dz_new,
                      dgamma=g[f"{mod}.ln_g"], dbeta=g[f"{mod}.ln_b"], dx_colsum=next_db)
    return dz


# ----------------------------------------------------------------------------- block
def block_fwd(bp: BlockParams, m, z, save=True, attn_flags=0):
    """evoformer_block (evoformer.py:314-325) on bf16 device tensors m [S,R,Hm], z [R,R,Hz].
    attn_flags: EVO_ATTN_* hints for the four attention forwards (0 = automatic)."""
    cfg: EvoConfig = bp.cfg
    S, R = cfg.n_seq, cfg.n_res
    m2 = m.reshape(S * R, cfg.h_msa)
    z2 = z.reshape(R * R, cfg.h_pair)
    saved = [] if save else None
    # each residual epilogue also produces the next module's input LayerNorm (LnChain)
    f = bp.f
    c = {k: LnChain(f[f"{k}.ln_g"], f[f"{k}.ln_b"]) for k in
         ("msa_col", "msa_trans", "opm", "tri_out", "tri_in", "pair_row", "pair_col", "pair_trans")}
    bias, sv_b = msa_row_bias_fwd(bp, z2, R, R, save)
    m2, s1 = attention_fwd(bp, "msa_row", m2, S, R, "row", bias=bias, save=save, next_ln=c["msa_col"],
                           flags=attn_flags)
    m2, s2 = attention_fwd(bp, "msa_col", m2, R, S, "col", save=save, pre_ln=c["msa_col"], next_ln=c["msa_trans"],
                           flags=attn_flags)
    m2, s3 = transition_fwd(bp, "msa_trans", m2, S * R, save, pre_ln=c["msa_trans"], next_ln=c["opm"])
    z2, s4 = opm_fwd(bp, m2, z2, S, R, save, pre_ln=c["opm"], next_ln=c["tri_out"])
    z2, s5 = triangle_fwd(bp, "tri_out", z2, R, save, pre_ln=c["tri_out"], next_ln=c["tri_in"])
    z2, s6 = triangle_fwd(bp, "tri_in", z2, R, save, pre_ln=c["tri_in"], next_ln=c["pair_row"])
    z2, s7 = attention_fwd(bp, "pair_row", z2, R, R, "row", bias="pair", save=save, pre_ln=c["pair_row"],
                           next_ln=c["pair_col"], flags=attn_flags)
    z2, s8 = attention_fwd(bp, "pair_col", z2, R, R, "col", bias="pair", save=save, pre_ln=c["pair_col"],
                           next_ln=c["pair_trans"], flags=attn_flags)
    z2, s9 = transition_fwd(bp, "pair_trans", z2, R * R, save, pre_ln=c["pair_trans"])
    if save:
        saved.extend([sv_b, s1, s2, s3, s4, s5, s6, s7, s8, s9])
    return m2.view(S, R, cfg.h_msa), z2.view(R, R, cfg.h_pair), saved


def block_bwd(bp: BlockParams, saved, dm, dz, join=True):
    """gradients w.r.t. (m, z) of the block input; parameter grads accumulate into bp.grad."""
    cfg: EvoConfig = bp.cfg
    S, R = cfg.n_seq, cfg.n_res
    sv_b, s1, s2, s3, s4, s5, s6, s7, s8, s9 = saved
    dm2 = dm.reshape(S * R, cfg.h_msa).contiguous()
    dz2 = dz.reshape(R * R, cfg.h_pair).contiguous()
    # each module's output-bias gradient (column sums of its incoming gradient) is fused into
    # the final LayerNorm backward of the module that produced that gradient
    fuse = dz2.is_cuda and cfg.h_pair in (32, 64, 128, 256) and cfg.h_msa in (32, 64, 128, 256)
    g = bp.g
    nd = (lambda k: g[k]) if fuse else (lambda k: None)
    dz2 = transition_bwd(bp, s9, dz2, next_db=nd("pair_col.b_o"))
    dz2, _ = attention_bwd(bp, s8, dz2, next_db=nd("pair_row.b_o"), db_done=fuse)
    dz2, _ = attention_bwd(bp, s7, dz2, db_done=fuse)
    dz2 = triangle_bwd(bp, s6, dz2)
    dz2 = triangle_bwd(bp, s5, dz2, next_db=nd("opm.b_o"))
    dm2 = opm_bwd(bp, s4, dz2, dm2, next_db=nd("msa_trans.b2"), db_done=fuse)
    dm2 = transition_bwd(bp, s3, dm2, next_db=nd("msa_col.b_o"), db_done=fuse)
    dm2, _ = attention_bwd(bp, s2, dm2, next_db=nd("msa_row.b_o"), db_done=fuse)
    dm2, dbias = attention_bwd(bp, s1, dm2, db_done=fuse)
    dz2 = msa_row_bias_bwd(bp, sv_b, dbias, dz2)
    if join:  # a stack joins once after its last block: side work then overlaps the next block
        SideStream.join()
    return dm2.view(S, R, cfg.h_msa), dz2.view(R, R, cfg.h_pair)
