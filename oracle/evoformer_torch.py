"""torch float64 CPU restatement of the reference block (TEST ORACLE).

Same algorithm as ``oracle/evoformer_np.py`` (which cites
/root/reference/pkg/src/evoplan/evoformer.py line by line), written with torch
ops so that autograd provides the gradient oracle: the reference has no
backward pass.  Forward agreement with the numpy oracle is
asserted at <=1e-12 in tests/test_oracle_golden.py.

Every function also accepts float32 tensors; the GPU parity tests use the
float64 path only.
"""

from __future__ import annotations

import math

import torch

EPS = 1e-5


def layernorm(x, g, b, eps=EPS):
    """engine.py:206-217."""
    mu = x.mean(-1, keepdim=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdim=True)
    return xc / torch.sqrt(var + eps) * g + b


def _heads(p, mod, part, heads):
    w = torch.stack([p[f"{mod}/{part}/{h}/w"] for h in range(heads)], 0)
    b = torch.stack([p[f"{mod}/{part}/{h}/b"] for h in range(heads)], 0)
    return w, b


def gated_attention(x, p, mod, heads, bias=None):
    """evoformer.py:173-198; bias broadcastable to [B, H, L, L]."""
    ln = layernorm(x, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    wq, bq = _heads(p, mod, "q", heads)
    wk, bk = _heads(p, mod, "k", heads)
    wv, bv = _heads(p, mod, "v", heads)
    wg, bg = _heads(p, mod, "g", heads)
    c = wq.shape[-1]
    q = torch.einsum("blc,hcd->bhld", ln, wq) + bq[None, :, None, :]
    k = torch.einsum("blc,hcd->bhld", ln, wk) + bk[None, :, None, :]
    v = torch.einsum("blc,hcd->bhld", ln, wv) + bv[None, :, None, :]
    s = q @ k.transpose(-1, -2)
    if bias is not None:
        s = s + bias
    a = torch.softmax(s * (1.0 / math.sqrt(c)), -1)
    g = torch.sigmoid(torch.einsum("blc,hcd->bhld", x, wg) + bg[None, :, None, :])
    o = g * (a @ v)
    B, L = x.shape[:2]
    cat = o.permute(0, 2, 1, 3).reshape(B, L, heads * c)
    return cat @ p[f"{mod}/o/w"] + p[f"{mod}/o/b"]


def msa_row_bias(z, p, cfg):
    lz = layernorm(z, p["msa_row/ln_z/g"], p["msa_row/ln_z/b"])
    w = torch.stack([p[f"msa_row/bias/{h}/w"] for h in range(cfg.n_head_msa)], -1)
    return lz @ w


def msa_row_attention_with_bias(m, bias, p, cfg):
    return gated_attention(m, p, "msa_row", cfg.n_head_msa, bias.permute(2, 0, 1)[None])


def msa_row_attention(m, z, p, cfg):
    return msa_row_attention_with_bias(m, msa_row_bias(z, p, cfg), p, cfg)


def msa_col_attention(m, p, cfg):
    return gated_attention(m.transpose(0, 1), p, "msa_col", cfg.n_head_msa).transpose(0, 1)


def transition(x, p, mod, mask=None):
    """evoformer.py:237-240.  mask (bool, the hidden layer's shape): use this ReLU pattern
    instead of (pre > 0) - the mask-matched gradient oracle (see block_grads)."""
    ln = layernorm(x, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    pre = ln @ p[f"{mod}/w1"] + p[f"{mod}/b1"]
    hid = torch.relu(pre) if mask is None else pre * mask.to(pre.dtype)
    return hid @ p[f"{mod}/w2"] + p[f"{mod}/b2"]


def opm_projections(m, p):
    ln = layernorm(m, p["opm/ln/g"], p["opm/ln/b"])
    return ln @ p["opm/a/w"] + p["opm/a/b"], ln @ p["opm/b/w"] + p["opm/b/b"]


def opm_from_projections(a, b, p, n_seq):
    S, I, P = a.shape
    J = b.shape[1]
    o = (a.reshape(S, I * P).T @ b.reshape(S, J * P)) / n_seq
    o = o.reshape(I, P, J, P).permute(0, 2, 1, 3).reshape(I, J, P * P)
    return o @ p["opm/o/w"] + p["opm/o/b"]


def outer_product_mean(m, p, cfg):
    a, b = opm_projections(m, p)
    return opm_from_projections(a, b, p, cfg.n_seq)


def triangle_projections(z, p, mod):
    ln = layernorm(z, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    lin = lambda part: ln @ p[f"{mod}/{part}/w"] + p[f"{mod}/{part}/b"]
    return (torch.sigmoid(lin("g")), torch.sigmoid(lin("a_sig")) * lin("a_lin"),
            torch.sigmoid(lin("b_sig")) * lin("b_lin"))


def triangle_finish(g, t, p, mod):
    ln2 = layernorm(t, p[f"{mod}/ln2/g"], p[f"{mod}/ln2/b"])
    return g * (ln2 @ p[f"{mod}/o/w"] + p[f"{mod}/o/b"])


def tri_contract_outgoing(a, b):
    return torch.einsum("ikh,jkh->ijh", a, b)


def tri_contract_incoming(a, b):
    return torch.einsum("kih,kjh->ijh", a, b)


def tri_update_outgoing(z, p, cfg):
    g, a, b = triangle_projections(z, p, "tri_out")
    return triangle_finish(g, tri_contract_outgoing(a, b), p, "tri_out")


def tri_update_incoming(z, p, cfg):
    g, a, b = triangle_projections(z, p, "tri_in")
    return triangle_finish(g, tri_contract_incoming(a, b), p, "tri_in")


def pair_key_bias(x, p, mod, heads):
    ln = layernorm(x, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    w = torch.stack([p[f"{mod}/bias/{h}/w"] for h in range(heads)], -1)
    return (ln @ w).permute(0, 2, 1)[:, :, None, :]


def pair_attention_row(z, p, cfg):
    return gated_attention(z, p, "pair_row", cfg.n_head_pair,
                           pair_key_bias(z, p, "pair_row", cfg.n_head_pair))


def pair_attention_col(z, p, cfg):
    zt = z.transpose(0, 1)
    return gated_attention(zt, p, "pair_col", cfg.n_head_pair,
                           pair_key_bias(zt, p, "pair_col", cfg.n_head_pair)).transpose(0, 1)


def evoformer_block(m, z, p, cfg, masks=None):
    """evoformer.py:314-325.  masks: optional {"msa_trans": bool, "pair_trans": bool} ReLU
    patterns for the two transitions (mask-matched oracle)."""
    masks = masks or {}
    m = m + msa_row_attention(m, z, p, cfg)
    m = m + msa_col_attention(m, p, cfg)
    m = m + transition(m, p, "msa_trans", masks.get("msa_trans"))
    z = z + outer_product_mean(m, p, cfg)
    z = z + tri_update_outgoing(z, p, cfg)
    z = z + tri_update_incoming(z, p, cfg)
    z = z + pair_attention_row(z, p, cfg)
    z = z + pair_attention_col(z, p, cfg)
    z = z + transition(z, p, "pair_trans", masks.get("pair_trans"))
    return m, z


def block_grads(m, z, params, cfg, gm, gz, dtype=torch.float64, masks=None):
    """Gradient oracle: d/d(m, z, params) of <m', gm> + <z', gz>.

    Inputs are numpy or torch; returns (m', z', dm, dz, dparams) as float64 numpy.
    masks: the ReLU patterns the GPU run took in its two transitions.  A bf16 run flips the
    pattern of units whose pre-activation lies within rounding distance of 0; each flip is an
    O(1) change of that unit's gradient (~sqrt(fraction) relative error in dm/dz).  With the
    GPU's own pattern the oracle differentiates the same piecewise-linear branch, so the
    comparison measures the kernels' error, not the branch choice.  The forward is unchanged
    up to the flipped units' |pre| ~ bf16 rounding.
    """
    t = lambda a: torch.as_tensor(a, dtype=dtype).clone().requires_grad_(True)
    mt, zt = t(m), t(z)
    pt = {k: t(v) for k, v in params.items()}
    if masks is not None:
        masks = {k: torch.as_tensor(v).bool() for k, v in masks.items()}
    mo, zo = evoformer_block(mt, zt, pt, cfg, masks)
    loss = (mo * torch.as_tensor(gm, dtype=dtype)).sum() + (zo * torch.as_tensor(gz, dtype=dtype)).sum()
    keys = list(pt)
    grads = torch.autograd.grad(loss, [mt, zt] + [pt[k] for k in keys], allow_unused=True)
    npy = lambda x: x.detach().double().numpy()
    dparams = {k: (npy(g) if g is not None else torch.zeros_like(pt[k]).double().numpy())
               for k, g in zip(keys, grads[2:])}
    return npy(mo), npy(zo), npy(grads[0]), npy(grads[1]), dparams
