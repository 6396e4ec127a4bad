"""Reference-compatible Evoformer API on the B200 engine.

Same names and argument meaning as /root/reference/pkg/src/evoplan/evoformer.py:
``evoformer_block(m, z, p, cfg)`` (evoformer.py:314), the sub-modules
``msa_row_attention`` (219), ``msa_row_bias`` (201), ``msa_row_attention_with_bias``
(210), ``msa_col_attention`` (226), ``transition`` (237), ``outer_product_mean``
(243), ``tri_update_outgoing`` / ``tri_update_incoming`` (273 / 280),
``pair_attention_row`` / ``pair_attention_col`` (295 / 302), and the engine ops
``layernorm`` / ``fused_softmax_mask_bias`` (engine.py:206, 291).

Inputs may be numpy float64 (the reference's type: copied to the GPU, computed
in bf16 with fp32 accumulation, returned as float64 numpy) or torch CUDA
tensors (returned as torch).  Shape errors raise ``DimensionError`` exactly
where the reference does (evoformer.py:328-339).  There is no CPU path.

Training entry points (the reference has none): ``BlockParams``,
``block_forward_backward``, ``EvoformerStack`` (N blocks fwd+bwd) and the autograd
``EvoformerBlockFunction``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import block as _blk
from . import ops
from .config import EvoConfig
from .errors import DimensionError, DomainError, KernelError
from .params import BlockLayout, BlockParams

__all__ = ["evoformer_block", "msa_row_attention", "msa_row_bias", "msa_row_attention_with_bias",
           "msa_col_attention", "transition", "outer_product_mean", "tri_update_outgoing",
           "tri_update_incoming", "pair_attention_row", "pair_attention_col", "layernorm",
           "fused_softmax_mask_bias", "BlockParams", "block_forward_backward", "EvoformerStack",
           "EvoformerBlockFunction", "GraphedStep"]

_DEV = "cuda"


def _check_msa(m, cfg):
    if tuple(m.shape) != (cfg.n_seq, cfg.n_res, cfg.h_msa):
        raise DimensionError(f"MSA tensor shape {tuple(m.shape)} does not match config "
                             f"({cfg.n_seq}, {cfg.n_res}, {cfg.h_msa})")


def _check_pair(z, cfg):
    if tuple(z.shape) != (cfg.n_res, cfg.n_res, cfg.h_pair):
        raise DimensionError(f"pair tensor shape {tuple(z.shape)} does not match config "
                             f"({cfg.n_res}, {cfg.n_res}, {cfg.h_pair})")


def _require_cuda():
    if not torch.cuda.is_available():
        raise KernelError("the B200 Evoformer engine needs a CUDA device (no CPU fallback)")


def _to_dev(x):
    """-> (bf16 contiguous CUDA tensor, was_numpy)"""
    if isinstance(x, np.ndarray):
        _require_cuda()
        return torch.from_numpy(np.ascontiguousarray(x)).to(_DEV).to(torch.bfloat16), True
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise KernelError("torch inputs must be CUDA tensors (no CPU fallback)")
        return x.to(torch.bfloat16).contiguous(), False
    raise TypeError(f"unsupported input type {type(x)}")


def _out(t, was_np):
    return t.double().cpu().numpy() if was_np else t


_PARAM_CACHE: dict = {}


def _block_params(p, cfg: EvoConfig) -> BlockParams:
    if isinstance(p, BlockParams):
        return p
    key = (id(p), cfg)
    hit = _PARAM_CACHE.get(key)
    if hit is not None and hit[0] is p:
        return hit[1]
    _require_cuda()
    bp = BlockParams(p, cfg, device=_DEV)
    _PARAM_CACHE.clear()
    _PARAM_CACHE[key] = (p, bp)
    return bp


# ----------------------------------------------------------------------------- engine ops
def layernorm(x, gamma, beta, eps: float = 1e-5):
    """engine.layernorm (engine.py:206-217) on the GPU; returns the input's type."""
    xt, was_np = _to_dev(x) if isinstance(x, np.ndarray) else (x.contiguous(), False)
    if xt.dtype not in (torch.float32, torch.bfloat16):
        xt = xt.float()
    if tuple(np.shape(gamma)) != (xt.shape[-1],) or tuple(np.shape(beta)) != (xt.shape[-1],):
        raise DimensionError(f"layernorm params must match last extent {xt.shape[-1]}")
    if was_np:
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(_DEV).float()
    g = torch.as_tensor(np.asarray(gamma) if not isinstance(gamma, torch.Tensor) else gamma,
                        dtype=torch.float32, device=xt.device)
    b = torch.as_tensor(np.asarray(beta) if not isinstance(beta, torch.Tensor) else beta,
                        dtype=torch.float32, device=xt.device)
    C = xt.shape[-1]
    y, _, _ = ops.layernorm_fwd(xt, g, b, xt.numel() // C, C, eps=eps, save_stats=False)
    y = y.view(xt.shape)
    return _out(y, was_np)


def fused_softmax_mask_bias(x, mask, bias, axis: int = -1, check_finite: bool = True):
    """engine.fused_softmax_mask_bias (engine.py:291-298): softmax(x + mask + bias, axis).

    One fused kernel; the only allocation is the output.  Like the reference,
    non-finite input raises ``DomainError`` (checked on the device).
    """
    def dev(a):
        if isinstance(a, np.ndarray):
            _require_cuda()
            return torch.from_numpy(np.ascontiguousarray(a)).to(_DEV).float(), True
        return a, False

    xt, was_np = dev(x)
    mt, _ = dev(mask)
    bt, _ = dev(bias)
    try:
        shape = torch.broadcast_shapes(xt.shape, mt.shape, bt.shape)
    except RuntimeError as exc:
        raise DimensionError(f"mask/bias not broadcastable to {tuple(xt.shape)}") from exc
    if tuple(shape) != tuple(xt.shape):
        raise DimensionError(f"mask/bias broadcast would change the shape of x {tuple(xt.shape)}")
    nd = xt.dim()
    ax = axis % nd
    if ax != nd - 1:
        xt, mt, bt = (t.movedim(ax, -1) if t.dim() == nd else t for t in (xt, mt, bt))
    if check_finite and ops.count_nonfinite(xt.contiguous()) > 0:
        raise DomainError("softmax input contains non-finite values")
    lead = xt.shape[:-1]
    x4 = xt.contiguous().reshape((-1,) + (1, 1) + (xt.shape[-1],)) if len(lead) > 3 else xt
    if len(lead) > 3:
        raise DimensionError("fused_softmax_mask_bias supports rank <= 4")
    y = ops.softmax_fwd(x4, bt if bt.dim() <= 4 else None, mt if mt.dim() <= 4 else None, 1.0)
    if ax != nd - 1:
        y = y.movedim(-1, ax)
    return _out(y.float().contiguous(), was_np) if was_np else y


# ----------------------------------------------------------------------------- sub-modules
def msa_row_bias(z, p, cfg: EvoConfig):
    """evoformer.py:201-207 -> [N_r, N_r, n_head] (reference layout)."""
    _check_pair(z, cfg)
    zt, was_np = _to_dev(z)
    bp = _block_params(p, cfg)
    bias, _ = _blk.msa_row_bias_fwd(bp, zt.view(-1, cfg.h_pair), cfg.n_res, save=False)
    return _out(bias.permute(1, 2, 0).contiguous(), was_np)


def msa_row_attention_with_bias(m, bias, p, cfg: EvoConfig, return_weights: bool = False):
    """evoformer.py:210-216; bias [N_r, N_r, n_head] (reference layout)."""
    _check_msa(m, cfg)
    mt, was_np = _to_dev(m)
    bt, _ = _to_dev(bias)
    bp = _block_params(p, cfg)
    S, R = cfg.n_seq, cfg.n_res
    bh = bt.permute(2, 0, 1).contiguous()
    x2 = mt.view(S * R, cfg.h_msa)
    res = _update_exact(bp, "msa_row", x2, S, R, "row", bh)
    if return_weights:
        _, sv = _blk.attention_fwd(bp, "msa_row", x2, S, R, "row", bias=bh, save=True)
        return _out(res, was_np), _attention_weights(bp, sv)
    return _out(res, was_np)


def _update_exact(bp, mod, x2d, B, L, kind, bias):
    """the sub-module update f(x) itself (reference returns f(x), not x + f(x)):
    run with a zero residual so no bf16 cancellation happens."""
    a = bp.layout.attn[mod]
    out, _ = _attention_update(bp, mod, x2d, torch.zeros_like(x2d), B, L, kind, bias)
    if kind == "row":
        return out.view(B, L, a["H"])
    return out.view(L, B, a["H"])


def _attention_update(bp, mod, x2d, res, B, L, kind, bias):
    import math
    from .ops import Strided
    a = bp.layout.attn[mod]
    H, nh, c, ldq = a["H"], a["nh"], a["c"], a["ldq"]
    rows = B * L
    h, f = bp.h, bp.f
    ln, _, _ = ops.layernorm_fwd(x2d, f[f"{mod}.ln_g"], f[f"{mod}.ln_b"], rows, H, save_stats=False)
    qkv = torch.addmm(h[f"{mod}.b_qkv"], ln, h[f"{mod}.w_qkv"])
    gpre = torch.addmm(h[f"{mod}.b_g"], x2d, h[f"{mod}.w_g"])
    og = torch.empty(rows, nh * c, device=x2d.device, dtype=torch.bfloat16)
    sbr, slr = _blk._attn_geometry(kind, B, L)
    S_ = lambda t, ld, off=0: Strided(t, sbr * ld, slr * ld, off)
    if bias is None:
        bt, bs, boff = None, (0, 0, 0, 0), 0
    elif isinstance(bias, str):
        bt, bs, boff = qkv, (sbr * ldq, 1, 0, slr * ldq), 3 * nh * c
    else:
        bt, bs, boff = bias, (0, L * L, L, 1), 0
    desc = ops.attention_desc(S_(qkv, ldq, 0), S_(qkv, ldq, nh * c), S_(qkv, ldq, 2 * nh * c), S_(gpre, nh * c),
                              S_(og, nh * c), None, None, B, L, nh, c, 1.0 / math.sqrt(c),
                              bias=bt, bias_s=bs, bias_off=boff)
    ops.attention_fwd(desc)
    y = torch.mm(og, h[f"{mod}.w_o"])
    return ops.gated_residual_fwd(res, y, f[f"{mod}.b_o"], rows, H), None


def _attention_weights(bp, sv):
    """debug path for return_weights=True: softmax((qk^T + bias)/sqrt(c)) per head, materialised
    with the fused softmax kernel (the flash kernel never materialises them)."""
    import math
    mod, B, L, kind = sv["mod"], sv["B"], sv["L"], sv["kind"]
    a = bp.layout.attn[mod]
    nh, c, ldq = a["nh"], a["c"], a["ldq"]
    qkv = sv["qkv"].float()
    if kind == "row":
        qkv = qkv.view(B, L, ldq)
    else:
        qkv = qkv.view(L, B, ldq).transpose(0, 1)
    q = qkv[..., :nh * c].reshape(B, L, nh, c).permute(0, 2, 1, 3)
    k = qkv[..., nh * c:2 * nh * c].reshape(B, L, nh, c).permute(0, 2, 1, 3)
    logits = (q @ k.transpose(-1, -2)).contiguous()
    bias = sv["bias"]
    if bias is None:
        bt = None
    elif isinstance(bias, str):
        bt = qkv[..., 3 * nh * c:3 * nh * c + nh].permute(0, 2, 1)[:, :, None, :].contiguous()
    else:
        bt = bias.float()[None]
    w = ops.softmax_fwd(logits, bt, None, 1.0 / math.sqrt(c))
    return [w[:, hh].double().cpu().numpy() for hh in range(nh)]


def msa_row_attention(m, z, p, cfg: EvoConfig, return_weights: bool = False):
    """evoformer.py:219-223."""
    _check_msa(m, cfg)
    _check_pair(z, cfg)
    zt, _ = _to_dev(z)
    bp = _block_params(p, cfg)
    bias, _ = _blk.msa_row_bias_fwd(bp, zt.view(-1, cfg.h_pair), cfg.n_res, save=False)
    mt, was_np = _to_dev(m)
    S, R = cfg.n_seq, cfg.n_res
    x2 = mt.view(S * R, cfg.h_msa)
    res = _update_exact(bp, "msa_row", x2, S, R, "row", bias)
    if return_weights:
        _, sv = _blk.attention_fwd(bp, "msa_row", x2, S, R, "row", bias=bias, save=True)
        return _out(res, was_np), _attention_weights(bp, sv)
    return _out(res, was_np)


def msa_col_attention(m, p, cfg: EvoConfig, return_weights: bool = False):
    """evoformer.py:226-234 (no bias, G5); no transpose copy is made."""
    _check_msa(m, cfg)
    mt, was_np = _to_dev(m)
    bp = _block_params(p, cfg)
    S, R = cfg.n_seq, cfg.n_res
    x2 = mt.view(S * R, cfg.h_msa)
    res = _update_exact(bp, "msa_col", x2, R, S, "col", None)   # [S, R, H] already
    if return_weights:
        _, sv = _blk.attention_fwd(bp, "msa_col", x2, R, S, "col", save=True)
        return _out(res, was_np), _attention_weights(bp, sv)
    return _out(res, was_np)


def pair_attention_row(z, p, cfg: EvoConfig, return_weights: bool = False):
    """evoformer.py:295-299 (per-key self bias, G4)."""
    _check_pair(z, cfg)
    zt, was_np = _to_dev(z)
    bp = _block_params(p, cfg)
    R = cfg.n_res
    x2 = zt.view(R * R, cfg.h_pair)
    res = _update_exact(bp, "pair_row", x2, R, R, "row", "pair")
    if return_weights:
        _, sv = _blk.attention_fwd(bp, "pair_row", x2, R, R, "row", bias="pair", save=True)
        return _out(res, was_np), _attention_weights(bp, sv)
    return _out(res, was_np)


def pair_attention_col(z, p, cfg: EvoConfig, return_weights: bool = False):
    """evoformer.py:302-311."""
    _check_pair(z, cfg)
    zt, was_np = _to_dev(z)
    bp = _block_params(p, cfg)
    R = cfg.n_res
    x2 = zt.view(R * R, cfg.h_pair)
    res = _update_exact(bp, "pair_col", x2, R, R, "col", "pair")
    if return_weights:
        _, sv = _blk.attention_fwd(bp, "pair_col", x2, R, R, "col", bias="pair", save=True)
        return _out(res, was_np), _attention_weights(bp, sv)
    return _out(res, was_np)


def transition(x, p, prefix: str, cfg: EvoConfig | None = None):
    """evoformer.py:237-240.  cfg may be omitted when p is a reference dict."""
    xt, was_np = _to_dev(x)
    if cfg is None:
        cfg = _infer_cfg(p)
    bp = _block_params(p, cfg)
    H = xt.shape[-1]
    rows = xt.numel() // H
    x2 = xt.view(rows, H)
    f, h = bp.f, bp.h
    ln, _, _ = ops.layernorm_fwd(x2, f[f"{prefix}.ln_g"], f[f"{prefix}.ln_b"], rows, H, save_stats=False)
    hid = torch.mm(ln, h[f"{prefix}.w1"])
    ops.bias_act_fwd(hid, f[f"{prefix}.b1"], rows, hid.shape[1])
    y = torch.mm(hid, h[f"{prefix}.w2"])
    out = ops.gated_residual_fwd(torch.zeros_like(x2), y, f[f"{prefix}.b2"], rows, H)
    return _out(out.view(xt.shape), was_np)


def outer_product_mean(m, p, cfg: EvoConfig):
    """evoformer.py:243-255."""
    _check_msa(m, cfg)
    mt, was_np = _to_dev(m)
    bp = _block_params(p, cfg)
    S, R = cfg.n_seq, cfg.n_res
    zero = torch.zeros(R * R, cfg.h_pair, device=mt.device, dtype=torch.bfloat16)
    out, _ = _blk.opm_fwd(bp, mt.view(S * R, cfg.h_msa), zero, S, R, save=False)
    return _out(out.view(R, R, cfg.h_pair), was_np)


def _triangle(z, p, cfg, mod):
    _check_pair(z, cfg)
    zt, was_np = _to_dev(z)
    bp = _block_params(p, cfg)
    R = cfg.n_res
    x2 = zt.view(R * R, cfg.h_pair)
    # residual-free update: run the fused epilogue against a zero residual
    out, sv = _blk.triangle_fwd(bp, mod, x2, R, save=True)
    upd = ops.gated_residual_fwd(torch.zeros_like(x2), sv["y2"], bp.f[f"{mod}.b_o"], R * R, cfg.h_pair,
                                 gp=sv["Y"], gp_rs=cfg.h_pair + 4 * cfg.hidden_proj)
    return _out(upd.view(R, R, cfg.h_pair), was_np)


def tri_update_outgoing(z, p, cfg: EvoConfig):
    """evoformer.py:273-277."""
    return _triangle(z, p, cfg, "tri_out")


def tri_update_incoming(z, p, cfg: EvoConfig):
    """evoformer.py:280-284."""
    return _triangle(z, p, cfg, "tri_in")


def _infer_cfg(p) -> EvoConfig:
    if isinstance(p, BlockParams):
        return p.cfg
    raise DimensionError("pass cfg= when calling transition() with a plain parameter dict")


def evoformer_block(m, z, p, cfg: EvoConfig):
    """evoformer.py:314-325: (m, z) -> (m', z'), nine residual sub-modules."""
    _check_msa(m, cfg)
    _check_pair(z, cfg)
    mt, was_np = _to_dev(m)
    zt, _ = _to_dev(z)
    bp = _block_params(p, cfg)
    mo, zo, _ = _blk.block_fwd(bp, mt, zt, save=False)
    return _out(mo, was_np), _out(zo, was_np)


# ----------------------------------------------------------------------------- training API
def block_forward_backward(bp: BlockParams, m, z, gm, gz):
    """one block forward + backward of loss = <m', gm> + <z', gz> (the gradient
    oracle's loss, oracle/evoformer_torch.block_grads).  numpy in, numpy out:
    (m', z', dm, dz, dparams[reference keys])."""
    cfg = bp.cfg
    mt, _ = _to_dev(m)
    zt, _ = _to_dev(z)
    bp.zero_grad()
    mo, zo, saved = _blk.block_fwd(bp, mt, zt, save=True)
    dm, dz = _blk.block_bwd(bp, saved, _to_dev(gm)[0], _to_dev(gz)[0])
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()
    return f(mo), f(zo), f(dm), f(dz), bp.grads_to_reference()


class EvoformerStack:
    """N independent Evoformer blocks (block i <- init_block_params(cfg, seed + i),
    SURVEY.md 8d) with an explicit fwd / bwd engine (no autograd tape)."""

    def __init__(self, cfg: EvoConfig, n_blocks: int, seed: int = 0, device="cuda", params=None):
        self.cfg = cfg
        self.layout = BlockLayout(cfg)
        from .config import init_block_params
        self.blocks = []
        for i in range(n_blocks):
            p = params[i] if params is not None else init_block_params(cfg, seed + i)
            self.blocks.append(BlockParams(p, cfg, device=device, layout=self.layout))

    def zero_grad(self):
        for b in self.blocks:
            b.zero_grad()

    def forward(self, m, z, save=True):
        saved = []
        for b in self.blocks:
            m, z, s = _blk.block_fwd(b, m, z, save=save)
            saved.append(s)
        return m, z, saved

    def backward(self, saved, dm, dz):
        # parameter-gradient work of block i stays on the side stream while block i-1's
        # backward runs (block_bwd never writes a tensor in place that side work may still
        # read); one join at the end
        for b, s in zip(reversed(self.blocks), reversed(saved)):
            dm, dz = _blk.block_bwd(b, s, dm, dz, join=False)
        _blk.SideStream.join()
        return dm, dz

    def forward_backward(self, m, z, gm, gz):
        """loss = <m_out, gm> + <z_out, gz>; returns (loss fp32 device scalar, dm, dz)."""
        mo, zo, saved = self.forward(m, z, save=True)
        loss = (mo.float() * gm.float()).sum() + (zo.float() * gz.float()).sum()
        dm, dz = self.backward(saved, gm.to(torch.bfloat16), gz.to(torch.bfloat16))
        return loss, dm, dz


class GraphedStep:
    """One fwd+bwd step of a stack captured as a single CUDA graph (no host work per
    kernel at replay).  ``inputs`` are copied into static buffers; ``replay()`` returns
    the static loss tensor; gradients land in the stack's BlockParams.grad buffers and
    ``dm`` / ``dz``.  Works for EvoformerStack and dap.DapStack (NCCL collectives are
    capturable)."""

    def __init__(self, stack, m, z, gm, gz, warmup: int = 2):
        self.stack = stack
        self.m, self.z, self.gm, self.gz = (t.detach().clone() for t in (m, z, gm, gz))
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss, self.dm, self.dz = self._body()

    def _body(self):
        self.stack.zero_grad()
        return self.stack.forward_backward(self.m, self.z, self.gm, self.gz)

    def set_inputs(self, m=None, z=None, gm=None, gz=None):
        for dst, src in ((self.m, m), (self.z, z), (self.gm, gm), (self.gz, gz)):
            if src is not None:
                dst.copy_(src, non_blocking=True)

    def replay(self):
        self.graph.replay()
        return self.loss


class EvoformerBlockFunction(torch.autograd.Function):
    """autograd wrapper: (m, z, flat_params) -> (m', z'); backward fills flat_params.grad
    through the packed-gradient buffer of the BlockParams."""

    @staticmethod
    def forward(ctx, m, z, flat, bp):
        mo, zo, saved = _blk.block_fwd(bp, m.to(torch.bfloat16).contiguous(), z.to(torch.bfloat16).contiguous())
        ctx.bp, ctx.saved = bp, saved
        ctx.dtypes = (m.dtype, z.dtype)
        return mo.to(m.dtype), zo.to(z.dtype)

    @staticmethod
    def backward(ctx, gm, gz):
        bp = ctx.bp
        bp.zero_grad()
        dm, dz = _blk.block_bwd(bp, ctx.saved, gm.to(torch.bfloat16).contiguous(), gz.to(torch.bfloat16).contiguous())
        ctx.saved = None
        return dm.to(ctx.dtypes[0]), dz.to(ctx.dtypes[1]), bp.grad.clone(), None
