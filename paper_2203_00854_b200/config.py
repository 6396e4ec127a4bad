"""Block configuration and parameter layout.

Mirrors the reference's configuration / parameter API exactly, so weights
produced by ``evoplan.evoformer.init_block_params`` or ``params_to_json`` load
unchanged:

* ``EvoConfig``           - evoformer.py:29-58 (same fields, defaults, validation)
* ``param_shapes``        - evoformer.py:100-126 (same keys, same insertion order)
* ``init_block_params``   - evoformer.py:129-144 (same RNG draw order -> bit-identical)
* ``params_to_json`` / ``params_from_json`` - evoformer.py:147-165 (schema evoplan-params-v1)
"""

from __future__ import annotations

import base64
import json
import math
from dataclasses import dataclass

import numpy as np

from .errors import DimensionError

PARAMS_SCHEMA = "evoplan-params-v1"


@dataclass(frozen=True)
class EvoConfig:
    """Extents of one Evoformer block (evoformer.py:29-58)."""

    n_seq: int
    n_res: int
    h_msa: int = 16
    h_pair: int = 8
    n_head_msa: int = 2
    n_head_pair: int = 2
    hidden_proj: int = 4
    transition_factor: int = 4

    def __post_init__(self) -> None:
        for name in ("n_seq", "n_res", "h_msa", "h_pair", "n_head_msa",
                     "n_head_pair", "hidden_proj", "transition_factor"):
            if getattr(self, name) < 1:
                raise DimensionError(f"{name} must be positive")
        if self.h_msa % self.n_head_msa:
            raise DimensionError("h_msa must be divisible by n_head_msa")
        if self.h_pair % self.n_head_pair:
            raise DimensionError("h_pair must be divisible by n_head_pair")

    @property
    def c_msa(self) -> int:
        return self.h_msa // self.n_head_msa

    @property
    def c_pair(self) -> int:
        return self.h_pair // self.n_head_pair


# --------------------------------------------------------------------------
# parameter layout
# --------------------------------------------------------------------------

def _attn_keys(mod: str, width: int, head_dim: int, heads: int,
               bias_from: int | None) -> list[tuple[str, tuple[int, ...]]]:
    out = [(f"{mod}/ln/g", (width,)), (f"{mod}/ln/b", (width,))]
    for h in range(heads):
        for part in "qkvg":
            out.append((f"{mod}/{part}/{h}/w", (width, head_dim)))
            out.append((f"{mod}/{part}/{h}/b", (head_dim,)))
        if bias_from is not None:
            out.append((f"{mod}/bias/{h}/w", (bias_from,)))
    out.append((f"{mod}/o/w", (heads * head_dim, width)))
    out.append((f"{mod}/o/b", (width,)))
    return out


def _trans_keys(mod: str, width: int, factor: int):
    hid = factor * width
    return [(f"{mod}/ln/g", (width,)), (f"{mod}/ln/b", (width,)),
            (f"{mod}/w1", (width, hid)), (f"{mod}/b1", (hid,)),
            (f"{mod}/w2", (hid, width)), (f"{mod}/b2", (width,))]


def _tri_keys(mod: str, width: int, proj: int):
    out = [(f"{mod}/ln/g", (width,)), (f"{mod}/ln/b", (width,)),
           (f"{mod}/g/w", (width, width)), (f"{mod}/g/b", (width,))]
    for part in ("a_sig", "a_lin", "b_sig", "b_lin"):
        out += [(f"{mod}/{part}/w", (width, proj)), (f"{mod}/{part}/b", (proj,))]
    out += [(f"{mod}/ln2/g", (proj,)), (f"{mod}/ln2/b", (proj,)),
            (f"{mod}/o/w", (proj, width)), (f"{mod}/o/b", (width,))]
    return out


def param_shapes(cfg: EvoConfig) -> dict[str, tuple[int, ...]]:
    """Every weight of one block; key order is the RNG draw order."""
    p = cfg.hidden_proj
    items: list[tuple[str, tuple[int, ...]]] = []
    items += _attn_keys("msa_row", cfg.h_msa, cfg.c_msa, cfg.n_head_msa, cfg.h_pair)
    items += [("msa_row/ln_z/g", (cfg.h_pair,)), ("msa_row/ln_z/b", (cfg.h_pair,))]
    items += _attn_keys("msa_col", cfg.h_msa, cfg.c_msa, cfg.n_head_msa, None)
    items += _trans_keys("msa_trans", cfg.h_msa, cfg.transition_factor)
    items += [("opm/ln/g", (cfg.h_msa,)), ("opm/ln/b", (cfg.h_msa,)),
              ("opm/a/w", (cfg.h_msa, p)), ("opm/a/b", (p,)),
              ("opm/b/w", (cfg.h_msa, p)), ("opm/b/b", (p,)),
              ("opm/o/w", (p * p, cfg.h_pair)), ("opm/o/b", (cfg.h_pair,))]
    items += _tri_keys("tri_out", cfg.h_pair, p)
    items += _tri_keys("tri_in", cfg.h_pair, p)
    items += _attn_keys("pair_row", cfg.h_pair, cfg.c_pair, cfg.n_head_pair, cfg.h_pair)
    items += _attn_keys("pair_col", cfg.h_pair, cfg.c_pair, cfg.n_head_pair, cfg.h_pair)
    items += _trans_keys("pair_trans", cfg.h_pair, cfg.transition_factor)
    return dict(items)


_LN_GAIN = ("ln/g", "ln2/g", "ln_z/g")
_LN_SHIFT = ("ln/b", "ln2/b", "ln_z/b")


def init_block_params(cfg: EvoConfig, seed: int) -> dict[str, np.ndarray]:
    """Seeded float64 parameters, bit-identical to evoformer.py:129-144.

    LayerNorm gains/shifts are constants (no RNG draw); biases ~ N(0, 0.1);
    weights ~ N(0, 1/sqrt(fan_in)) with fan_in = leading extent.  One
    ``default_rng(seed)`` is consumed in ``param_shapes`` order.
    """
    rng = np.random.default_rng(seed)
    out: dict[str, np.ndarray] = {}
    for key, shape in param_shapes(cfg).items():
        if key.endswith(_LN_GAIN):
            out[key] = np.ones(shape)
        elif key.endswith(_LN_SHIFT):
            out[key] = np.zeros(shape)
        elif key.rsplit("/", 1)[-1] in ("b", "b1", "b2"):
            out[key] = rng.normal(0.0, 0.1, shape)
        else:
            out[key] = rng.normal(0.0, 1.0 / math.sqrt(shape[0]), shape)
    return out


def params_to_json(params: dict[str, np.ndarray]) -> str:
    """Bit-stable dump (schema ``evoplan-params-v1``, evoformer.py:147-156)."""
    body = {}
    for key in sorted(params):
        arr = np.ascontiguousarray(np.asarray(params[key]), dtype=np.float64)
        body[key] = {"shape": list(arr.shape),
                     "data": base64.b64encode(arr.tobytes()).decode("ascii")}
    return json.dumps({"schema": PARAMS_SCHEMA, "params": body}, sort_keys=True)


def params_from_json(text: str) -> dict[str, np.ndarray]:
    doc = json.loads(text)
    out = {}
    for key, ent in doc["params"].items():
        raw = base64.b64decode(ent["data"])
        out[key] = np.frombuffer(raw, dtype=np.float64).reshape(ent["shape"]).copy()
    return out


def check_params(params, cfg: EvoConfig) -> None:
    shapes = param_shapes(cfg)
    missing = [k for k in shapes if k not in params]
    if missing:
        raise DimensionError(f"params missing {len(missing)} keys, e.g. {missing[0]}")
    for k, s in shapes.items():
        if tuple(params[k].shape) != tuple(s):
            raise DimensionError(f"param {k} has shape {tuple(params[k].shape)}, want {s}")


def synthetic_inputs(cfg: EvoConfig, seed: int):
    """m then z from ``default_rng(seed)`` exactly as cli.py:112-114 draws them."""
    rng = np.random.default_rng(seed)
    m = rng.normal(size=(cfg.n_seq, cfg.n_res, cfg.h_msa))
    z = rng.normal(size=(cfg.n_res, cfg.n_res, cfg.h_pair))
    return m, z
