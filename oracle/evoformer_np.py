"""float64 numpy restatement of the reference Evoformer block (TEST ORACLE).

Reference: /root/reference/pkg/src/evoplan/evoformer.py (EVO) and engine.py (ENG).
Heads are processed as one batched tensor instead of the reference's Python
loop over heads (EVO:182); the arithmetic per element is the same.
Semantics kept exactly:
  G1 bias added before the 1/sqrt(c) scale           EVO:186-189
  G2 gate reads raw x, not LN(x)                      EVO:191
  G4 pair attention bias is per key, from own LN      EVO:287-292
  G5 msa_col has no bias                              EVO:226-234
  G6 OPM divides by n_seq, W_o rows indexed p*P+q     EVO:253-255
  G9 LN population variance, eps inside sqrt          ENG:206-217
"""

from __future__ import annotations

import math

import numpy as np

EPS = 1e-5
MASK_VALUE = -1e30  # ENG:31


class OracleDomainError(ValueError):
    pass


def layernorm(x, g, b, eps=EPS):
    """ENG:206-217 - population variance, eps inside the square root."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=-1, keepdims=True)
    return xc / np.sqrt(var + eps) * g + b


def softmax(x, axis=-1):
    """ENG:183-190 - max-shifted softmax; rejects non-finite input."""
    if not np.all(np.isfinite(x)):
        raise OracleDomainError("softmax input contains non-finite values")
    e = np.exp(x - x.max(axis=axis, keepdims=True))
    return e / e.sum(axis=axis, keepdims=True)


def fused_softmax_mask_bias(x, mask, bias, axis=-1):
    """ENG:193-203 - softmax(x + mask + bias) with numpy broadcasting."""
    np.broadcast_shapes(x.shape, mask.shape, bias.shape)
    return softmax(x + mask + bias, axis)


def sigmoid(x):
    """ENG:220-221 (scipy expit) - numerically stable logistic."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def _stack_heads(p, mod, part, heads):
    w = np.stack([p[f"{mod}/{part}/{h}/w"] for h in range(heads)], 0)  # [H, C, c]
    b = np.stack([p[f"{mod}/{part}/{h}/b"] for h in range(heads)], 0)  # [H, c]
    return w, b


def gated_attention(x, p, mod, heads, bias=None, return_weights=False):
    """EVO:173-198 (_attention_core) over axis 1 of x [B, L, C].

    bias: None or array broadcastable to [B, heads, L, L] (already per head).
    """
    ln = layernorm(x, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])                 # EVO:179
    wq, bq = _stack_heads(p, mod, "q", heads)
    wk, bk = _stack_heads(p, mod, "k", heads)
    wv, bv = _stack_heads(p, mod, "v", heads)
    wg, bg = _stack_heads(p, mod, "g", heads)
    c = wq.shape[-1]
    q = np.einsum("blc,hcd->bhld", ln, wq) + bq[None, :, None, :]         # EVO:183
    k = np.einsum("blc,hcd->bhld", ln, wk) + bk[None, :, None, :]         # EVO:184
    v = np.einsum("blc,hcd->bhld", ln, wv) + bv[None, :, None, :]         # EVO:185
    s = q @ np.swapaxes(k, -1, -2)                                         # EVO:186
    if bias is not None:
        s = s + bias                                                       # EVO:187-188
    a = softmax(s * (1.0 / math.sqrt(c)), -1)                             # EVO:189-190
    g = sigmoid(np.einsum("blc,hcd->bhld", x, wg) + bg[None, :, None, :])  # EVO:191 (raw x)
    o = g * (a @ v)                                                        # EVO:192
    B, L = x.shape[:2]
    cat = np.transpose(o, (0, 2, 1, 3)).reshape(B, L, heads * c)           # EVO:195 concat
    out = cat @ p[f"{mod}/o/w"] + p[f"{mod}/o/b"]
    return (out, a) if return_weights else out


def msa_row_bias(z, p, cfg):
    """EVO:201-207 - b[i,j,h] = LN_z(z)[i,j,:] . w_h (no bias term)."""
    lz = layernorm(z, p["msa_row/ln_z/g"], p["msa_row/ln_z/b"])
    w = np.stack([p[f"msa_row/bias/{h}/w"] for h in range(cfg.n_head_msa)], -1)
    return lz @ w                                                          # [N_r, N_r, H]


def msa_row_attention_with_bias(m, bias, p, cfg):
    """EVO:210-216 - bias [N_r, N_r, H] shared across sequences."""
    bh = np.transpose(bias, (2, 0, 1))[None]                               # [1, H, L, L]
    return gated_attention(m, p, "msa_row", cfg.n_head_msa, bh)


def msa_row_attention(m, z, p, cfg):
    """EVO:219-223."""
    return msa_row_attention_with_bias(m, msa_row_bias(z, p, cfg), p, cfg)


def msa_col_attention(m, p, cfg):
    """EVO:226-234 - attention over sequences per residue column, no bias."""
    mt = np.ascontiguousarray(np.transpose(m, (1, 0, 2)))
    return np.transpose(gated_attention(mt, p, "msa_col", cfg.n_head_msa), (1, 0, 2))


def transition(x, p, mod):
    """EVO:237-240 - LN -> W1 + b1 -> ReLU -> W2 + b2."""
    ln = layernorm(x, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    h = np.maximum(ln @ p[f"{mod}/w1"] + p[f"{mod}/b1"], 0.0)
    return h @ p[f"{mod}/w2"] + p[f"{mod}/b2"]


def opm_projections(m, p):
    """EVO:245-247."""
    ln = layernorm(m, p["opm/ln/g"], p["opm/ln/b"])
    return ln @ p["opm/a/w"] + p["opm/a/b"], ln @ p["opm/b/w"] + p["opm/b/b"]


def opm_from_projections(a, b, p, n_seq):
    """EVO:251-255 - o[i,j,p,q] = sum_s a[s,i,p] b[s,j,q] / n_seq; flatten p-major."""
    S, I, P = a.shape
    J = b.shape[1]
    o = (a.reshape(S, I * P).T @ b.reshape(S, J * P)) / n_seq              # [(i,p),(j,q)]
    o = o.reshape(I, P, J, P).transpose(0, 2, 1, 3).reshape(I, J, P * P)
    return o @ p["opm/o/w"] + p["opm/o/b"]


def outer_product_mean(m, p, cfg):
    a, b = opm_projections(m, p)
    return opm_from_projections(a, b, p, cfg.n_seq)


def triangle_projections(z, p, mod):
    """EVO:258-265 - g = sig(.), a = sig(.)*(.), b = sig(.)*(.) on LN(z)."""
    ln = layernorm(z, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    lin = lambda part: ln @ p[f"{mod}/{part}/w"] + p[f"{mod}/{part}/b"]
    g = sigmoid(lin("g"))
    a = sigmoid(lin("a_sig")) * lin("a_lin")
    b = sigmoid(lin("b_sig")) * lin("b_lin")
    return g, a, b


def triangle_finish(g, t, p, mod):
    """EVO:268-270 - g * (LN2(t) @ W_o + b_o)."""
    ln2 = layernorm(t, p[f"{mod}/ln2/g"], p[f"{mod}/ln2/b"])
    return g * (ln2 @ p[f"{mod}/o/w"] + p[f"{mod}/o/b"])


def tri_contract_outgoing(a, b):
    """EVO:276 - t[i,j,h] = sum_k a[i,k,h] b[j,k,h] (batched over h)."""
    return np.transpose(np.transpose(a, (2, 0, 1)) @ np.transpose(b, (2, 1, 0)), (1, 2, 0))


def tri_contract_incoming(a, b):
    """EVO:283 - t[i,j,h] = sum_k a[k,i,h] b[k,j,h]."""
    return np.transpose(np.transpose(a, (2, 1, 0)) @ np.transpose(b, (2, 0, 1)), (1, 2, 0))


def tri_update_outgoing(z, p, cfg):
    """EVO:273-277."""
    g, a, b = triangle_projections(z, p, "tri_out")
    return triangle_finish(g, tri_contract_outgoing(a, b), p, "tri_out")


def tri_update_incoming(z, p, cfg):
    """EVO:280-284."""
    g, a, b = triangle_projections(z, p, "tri_in")
    return triangle_finish(g, tri_contract_incoming(a, b), p, "tri_in")


def pair_key_bias(x, p, mod, heads):
    """EVO:287-292 - per-key bias from the attention's own LN, [B, H, 1, L]."""
    ln = layernorm(x, p[f"{mod}/ln/g"], p[f"{mod}/ln/b"])
    w = np.stack([p[f"{mod}/bias/{h}/w"] for h in range(heads)], -1)      # [C, H]
    return np.transpose(ln @ w, (0, 2, 1))[:, :, None, :]


def pair_attention_row(z, p, cfg):
    """EVO:295-299."""
    return gated_attention(z, p, "pair_row", cfg.n_head_pair,
                           pair_key_bias(z, p, "pair_row", cfg.n_head_pair))


def pair_attention_col(z, p, cfg):
    """EVO:302-311 - transpose, row attention with pair_col params, transpose back."""
    zt = np.ascontiguousarray(np.transpose(z, (1, 0, 2)))
    out = gated_attention(zt, p, "pair_col", cfg.n_head_pair,
                          pair_key_bias(zt, p, "pair_col", cfg.n_head_pair))
    return np.transpose(out, (1, 0, 2))


SUBMODULES = ("msa_row", "msa_col", "msa_trans", "opm", "tri_out", "tri_in",
              "pair_row", "pair_col", "pair_trans")


def evoformer_block(m, z, p, cfg, trace=None):
    """EVO:314-325 - nine residual sub-modules in fixed order.

    ``trace`` (optional dict) receives the state after each sub-module.
    """
    steps = [
        ("msa_row", lambda m, z: (m + msa_row_attention(m, z, p, cfg), z)),
        ("msa_col", lambda m, z: (m + msa_col_attention(m, p, cfg), z)),
        ("msa_trans", lambda m, z: (m + transition(m, p, "msa_trans"), z)),
        ("opm", lambda m, z: (m, z + outer_product_mean(m, p, cfg))),
        ("tri_out", lambda m, z: (m, z + tri_update_outgoing(z, p, cfg))),
        ("tri_in", lambda m, z: (m, z + tri_update_incoming(z, p, cfg))),
        ("pair_row", lambda m, z: (m, z + pair_attention_row(z, p, cfg))),
        ("pair_col", lambda m, z: (m, z + pair_attention_col(z, p, cfg))),
        ("pair_trans", lambda m, z: (m, z + transition(z, p, "pair_trans"))),
    ]
    for name, fn in steps:
        m, z = fn(m, z)
        if trace is not None:
            trace[name] = (m, z)
    return m, z
