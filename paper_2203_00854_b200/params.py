"""Device-resident, packed parameters of one Evoformer block.

The reference keeps one small matrix per head and per projection
(evoformer.py:66-126).  On the GPU they are packed once into merged GEMM
operands (the paper's merge-GEMM):

  attention  w_qkv [H, ldq] = [q_0..q_{n-1} | k_0.. | v_0.. | pair-bias w_0.. | 0-pad]
             (q, k, v read LN(x); the gate g reads raw x (G2), so w_g stays separate)
  msa_row    w_bias [Hz, n]  (LN_z(z) . w_h, evoformer.py:201-207)
  triangle   w_proj [Hz, Hz+4p] = [g | a_sig | a_lin | b_sig | b_lin]
  OPM        w_ab   [Hm, 2p]    = [a | b]

Master weights live in ONE fp32 flat buffer (``flat``) with named views; a bf16
copy (``flat_h``) feeds the tensor cores; gradients accumulate into ``grad``
(same layout).  ``to_reference`` / ``grads_to_reference`` map back to the
reference's key names, so parity tests compare per reference key.
"""

from __future__ import annotations

import numpy as np
import torch

from .config import EvoConfig, check_params


def _r8(n: int) -> int:
    return (n + 7) // 8 * 8


def _rowdot_k(n: int) -> int:
    """the fused LN + bias-dot kernel handles 8 heads (fewer are zero-padded)"""
    if n > 8:
        raise ValueError(f"msa heads {n} > 8 unsupported by the fused bias kernel")
    return 8


class BlockLayout:
    """Packed tensor names/shapes and their mapping to reference keys."""

    ATTN = ("msa_row", "msa_col", "pair_row", "pair_col")

    def __init__(self, cfg: EvoConfig):
        self.cfg = cfg
        c = cfg
        self.entries: list[tuple[str, tuple[int, ...]]] = []
        # maps: packed name -> list of (ref key, index expression builder)
        self.maps: dict[str, list] = {}
        p = c.hidden_proj
        self.attn = {}
        for mod, H, nh, ch, pair_bias in (("msa_row", c.h_msa, c.n_head_msa, c.c_msa, False),
                                          ("msa_col", c.h_msa, c.n_head_msa, c.c_msa, False),
                                          ("pair_row", c.h_pair, c.n_head_pair, c.c_pair, True),
                                          ("pair_col", c.h_pair, c.n_head_pair, c.c_pair, True)):
            ldq = _r8(3 * nh * ch + (nh if pair_bias else 0))
            self.attn[mod] = dict(H=H, nh=nh, c=ch, ldq=ldq, pair_bias=pair_bias)
            self._add(f"{mod}.ln_g", (H,), [(f"{mod}/ln/g", (slice(None),))])
            self._add(f"{mod}.ln_b", (H,), [(f"{mod}/ln/b", (slice(None),))])
            wq, bq = [], []
            for part_i, part in enumerate("qkv"):
                for h in range(nh):
                    col = slice(part_i * nh * ch + h * ch, part_i * nh * ch + (h + 1) * ch)
                    wq.append((f"{mod}/{part}/{h}/w", (slice(None), col)))
                    bq.append((f"{mod}/{part}/{h}/b", (col,)))
            if pair_bias:
                for h in range(nh):
                    wq.append((f"{mod}/bias/{h}/w", (slice(None), 3 * nh * ch + h)))
            self._add(f"{mod}.w_qkv", (H, ldq), wq)
            self._add(f"{mod}.b_qkv", (ldq,), bq)
            self._add(f"{mod}.w_g", (H, nh * ch),
                      [(f"{mod}/g/{h}/w", (slice(None), slice(h * ch, (h + 1) * ch))) for h in range(nh)])
            self._add(f"{mod}.b_g", (nh * ch,),
                      [(f"{mod}/g/{h}/b", (slice(h * ch, (h + 1) * ch),)) for h in range(nh)])
            self._add(f"{mod}.w_o", (nh * ch, H), [(f"{mod}/o/w", (slice(None), slice(None)))])
            self._add(f"{mod}.b_o", (H,), [(f"{mod}/o/b", (slice(None),))])
        nh = c.n_head_msa
        self.rowdot_k = _rowdot_k(nh)
        self._add("msa_row.lnz_g", (c.h_pair,), [("msa_row/ln_z/g", (slice(None),))])
        self._add("msa_row.lnz_b", (c.h_pair,), [("msa_row/ln_z/b", (slice(None),))])
        self._add("msa_row.w_bias", (c.h_pair, self.rowdot_k),
                  [(f"msa_row/bias/{h}/w", (slice(None), h)) for h in range(nh)])
        for mod, H in (("msa_trans", c.h_msa), ("pair_trans", c.h_pair)):
            F = c.transition_factor * H
            self._add(f"{mod}.ln_g", (H,), [(f"{mod}/ln/g", (slice(None),))])
            self._add(f"{mod}.ln_b", (H,), [(f"{mod}/ln/b", (slice(None),))])
            self._add(f"{mod}.w1", (H, F), [(f"{mod}/w1", (slice(None), slice(None)))])
            self._add(f"{mod}.b1", (F,), [(f"{mod}/b1", (slice(None),))])
            self._add(f"{mod}.w2", (F, H), [(f"{mod}/w2", (slice(None), slice(None)))])
            self._add(f"{mod}.b2", (H,), [(f"{mod}/b2", (slice(None),))])
        self._add("opm.ln_g", (c.h_msa,), [("opm/ln/g", (slice(None),))])
        self._add("opm.ln_b", (c.h_msa,), [("opm/ln/b", (slice(None),))])
        self._add("opm.w_ab", (c.h_msa, 2 * p), [("opm/a/w", (slice(None), slice(0, p))),
                                                ("opm/b/w", (slice(None), slice(p, 2 * p)))])
        self._add("opm.b_ab", (2 * p,), [("opm/a/b", (slice(0, p),)), ("opm/b/b", (slice(p, 2 * p),))])
        self._add("opm.w_o", (p * p, c.h_pair), [("opm/o/w", (slice(None), slice(None)))])
        self._add("opm.b_o", (c.h_pair,), [("opm/o/b", (slice(None),))])
        Hz = c.h_pair
        for mod in ("tri_out", "tri_in"):
            self._add(f"{mod}.ln_g", (Hz,), [(f"{mod}/ln/g", (slice(None),))])
            self._add(f"{mod}.ln_b", (Hz,), [(f"{mod}/ln/b", (slice(None),))])
            cols = [("g", 0, Hz), ("a_sig", Hz, p), ("a_lin", Hz + p, p), ("b_sig", Hz + 2 * p, p),
                    ("b_lin", Hz + 3 * p, p)]
            self._add(f"{mod}.w_proj", (Hz, Hz + 4 * p),
                      [(f"{mod}/{n}/w", (slice(None), slice(o, o + w))) for n, o, w in cols])
            self._add(f"{mod}.b_proj", (Hz + 4 * p,), [(f"{mod}/{n}/b", (slice(o, o + w),)) for n, o, w in cols])
            self._add(f"{mod}.ln2_g", (p,), [(f"{mod}/ln2/g", (slice(None),))])
            self._add(f"{mod}.ln2_b", (p,), [(f"{mod}/ln2/b", (slice(None),))])
            self._add(f"{mod}.w_o", (p, Hz), [(f"{mod}/o/w", (slice(None), slice(None)))])
            self._add(f"{mod}.b_o", (Hz,), [(f"{mod}/o/b", (slice(None),))])
        # offsets (16-byte aligned for bf16 views)
        self.offsets = {}
        off = 0
        for name, shape in self.entries:
            self.offsets[name] = off
            off += _r8(int(np.prod(shape)))
        self.numel = off

    def _add(self, name, shape, refs):
        self.entries.append((name, tuple(shape)))
        self.maps[name] = refs

    def pack(self, params, strict: bool = True) -> np.ndarray:
        """reference-keyed dict -> packed flat vector; strict=False leaves the entries of
        absent keys zero (a caller holding only one module's weights)."""
        flat = np.zeros(self.numel, dtype=np.float64)
        for name, shape in self.entries:
            view = np.zeros(shape)
            for key, idx in self.maps[name]:
                if not strict and key not in params:
                    continue
                view[idx] = np.asarray(params[key], dtype=np.float64)
            o = self.offsets[name]
            flat[o:o + view.size] = view.reshape(-1)
        return flat

    def unpack(self, flat) -> dict[str, np.ndarray]:
        """packed flat vector -> reference-keyed dict (each key lives in exactly one place)."""
        from .config import param_shapes
        flat = np.asarray(flat, dtype=np.float64)
        shapes = param_shapes(self.cfg)
        out = {}
        for name, shape in self.entries:
            o = self.offsets[name]
            view = flat[o:o + int(np.prod(shape))].reshape(shape)
            for key, idx in self.maps[name]:
                out[key] = np.array(view[idx]).reshape(shapes[key])
        return {k: out[k] for k in shapes}


class BlockParams:
    """Packed device parameters of one block (fp32 master, bf16 compute copy, fp32 grads)."""

    def __init__(self, params=None, cfg: EvoConfig | None = None, device="cuda", layout: BlockLayout | None = None,
                 flat: torch.Tensor | None = None, partial: bool = False):
        """partial=True: params may hold a subset of the block's keys (the reference's module
        functions only read their own prefix); absent entries are zero."""
        self.cfg = cfg
        self.layout = layout or BlockLayout(cfg)
        if flat is None:
            if not partial:
                check_params(params, cfg)
            flat = torch.from_numpy(self.layout.pack(params, strict=not partial)).to(device=device,
                                                                                    dtype=torch.float32)
        self.flat = flat
        self.device = flat.device
        self.flat_h = torch.empty(self.layout.numel, device=self.device, dtype=torch.bfloat16)
        self.grad = torch.zeros(self.layout.numel, device=self.device, dtype=torch.float32)
        self.f = self._views(self.flat)
        self.h = self._views(self.flat_h)
        self.g = self._views(self.grad)
        self.refresh()

    def _views(self, buf):
        return {name: buf[self.layout.offsets[name]:self.layout.offsets[name] + int(np.prod(shape))].view(shape)
                for name, shape in self.layout.entries}

    def refresh(self):
        """re-derive the bf16 tensor-core copy from the fp32 master weights."""
        self.flat_h.copy_(self.flat)

    def zero_grad(self):
        self.grad.zero_()

    def to_reference(self) -> dict[str, np.ndarray]:
        return self.layout.unpack(self.flat.detach().double().cpu().numpy())

    def grads_to_reference(self) -> dict[str, np.ndarray]:
        return self.layout.unpack(self.grad.detach().double().cpu().numpy())
