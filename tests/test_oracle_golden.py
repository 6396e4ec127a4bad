"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  Tolerances follow the reference's own tests
(test_evoformer.py:42-132: <=1e-12 per op, <=1e-11 per block)."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import evoformer_np as O
from oracle import evoformer_torch as T
from paper_2203_00854_b200.config import EvoConfig, init_block_params, synthetic_inputs

from conftest import GOLDEN


def _digest(params):
    h = hashlib.sha256()
    for k in sorted(params):
        h.update(k.encode())
        h.update(np.ascontiguousarray(params[k], dtype=np.float64).tobytes())
    return h.digest()


CFG3 = EvoConfig(n_seq=3, n_res=4, h_msa=4, h_pair=4, n_head_msa=2, n_head_pair=2, hidden_proj=2)
G3 = np.load(os.path.join(GOLDEN, "golden_cfg3.npz"))
GT = np.load(os.path.join(GOLDEN, "golden_tiny.npz"))
GS = np.load(os.path.join(GOLDEN, "golden_softmax.npz"))


@pytest.mark.parametrize("seed", range(20))
def test_params_bit_identical_to_reference(seed):
    p = init_block_params(CFG3, seed)
    assert _digest(p) == G3[f"s{seed}/params_sha256"].tobytes()


@pytest.mark.parametrize("seed", range(20))
def test_submodules_match_reference(seed):
    m, z = synthetic_inputs(CFG3, seed)
    p = init_block_params(CFG3, seed)
    got = {
        "msa_row": O.msa_row_attention(m, z, p, CFG3),
        "msa_row_bias": O.msa_row_bias(z, p, CFG3),
        "msa_col": O.msa_col_attention(m, p, CFG3),
        "msa_trans": O.transition(m, p, "msa_trans"),
        "pair_trans": O.transition(z, p, "pair_trans"),
        "opm": O.outer_product_mean(m, p, CFG3),
        "tri_out": O.tri_update_outgoing(z, p, CFG3),
        "tri_in": O.tri_update_incoming(z, p, CFG3),
        "pair_row": O.pair_attention_row(z, p, CFG3),
        "pair_col": O.pair_attention_col(z, p, CFG3),
    }
    for k, v in got.items():
        assert np.max(np.abs(v - G3[f"s{seed}/{k}"])) <= 1e-12, k
    mo, zo = O.evoformer_block(m, z, p, CFG3)
    assert np.max(np.abs(mo - G3[f"s{seed}/block_m"])) <= 1e-11
    assert np.max(np.abs(zo - G3[f"s{seed}/block_z"])) <= 1e-11


@pytest.mark.parametrize("name", ["c1_s7", "c1_s31", "h84_s101"])
def test_tiny_block_matches_reference(name):
    dims = [int(v) for v in GT[f"{name}/dims"]]
    cfg, seed = EvoConfig(*dims[:7]), dims[7]
    p = init_block_params(cfg, seed)
    assert _digest(p) == GT[f"{name}/params_sha256"].tobytes()
    m, z = synthetic_inputs(cfg, seed)
    mo, zo = O.evoformer_block(m, z, p, cfg)
    assert np.max(np.abs(mo - GT[f"{name}/m"])) <= 1e-11
    assert np.max(np.abs(zo - GT[f"{name}/z"])) <= 1e-11
    # torch float64 restatement (gradient oracle) agrees in the forward
    pt = {k: torch.tensor(v) for k, v in p.items()}
    mt, zt = T.evoformer_block(torch.tensor(m), torch.tensor(z), pt, cfg)
    assert np.max(np.abs(mt.numpy() - GT[f"{name}/m"])) <= 1e-11
    assert np.max(np.abs(zt.numpy() - GT[f"{name}/z"])) <= 1e-11


def test_fused_softmax_set_and_kats():
    for i in range(100):
        y = O.fused_softmax_mask_bias(GS[f"c{i}/x"], GS[f"c{i}/mask"], GS[f"c{i}/bias"])
        assert np.max(np.abs(y - GS[f"c{i}/y"])) <= 1e-12
    assert np.allclose(O.softmax(GS["kat/sm_in"]), [[0.5, 0.5], [2 / 3, 1 / 3]], atol=1e-12)
    assert np.max(np.abs(O.softmax(GS["kat/sm_in"]) - GS["kat/sm_out"])) <= 1e-15
    fs = O.fused_softmax_mask_bias(GS["kat/fs_x"], GS["kat/fs_mask"], np.zeros((1, 2)))
    assert np.max(np.abs(fs - GS["kat/fs_out"])) <= 1e-12 and abs(fs[0, 0] - 1) <= 1e-12
    ln = O.layernorm(GS["kat/ln_in"], np.ones(3), np.zeros(3))
    assert np.max(np.abs(ln - GS["kat/ln_out"])) <= 1e-12
    with pytest.raises(ValueError):
        O.softmax(np.array([1.0, np.inf]))


def test_torch_gradient_oracle_is_consistent():
    """Finite-difference check of the torch fp64 gradient oracle on CFG3."""
    m, z = synthetic_inputs(CFG3, 3)
    p = init_block_params(CFG3, 3)
    rng = np.random.default_rng(0)
    gm, gz = rng.normal(size=m.shape), rng.normal(size=z.shape)
    _, _, dm, dz, dp = T.block_grads(m, z, p, CFG3, gm, gz)

    def loss(m_, z_, p_):
        mo, zo = O.evoformer_block(m_, z_, p_, CFG3)
        return float((mo * gm).sum() + (zo * gz).sum())

    eps = 1e-6
    for idx in [(0, 0, 0), (2, 3, 1)]:
        mp, mm = m.copy(), m.copy()
        mp[idx] += eps
        mm[idx] -= eps
        fd = (loss(mp, z, p) - loss(mm, z, p)) / (2 * eps)
        assert abs(fd - dm[idx]) <= 1e-6 * max(1.0, abs(fd))
    for key in ["tri_in/a_lin/w", "msa_row/bias/1/w", "opm/o/w", "pair_col/ln/g"]:
        pp = {k: v.copy() for k, v in p.items()}
        pm = {k: v.copy() for k, v in p.items()}
        i0 = (0,) * p[key].ndim
        pp[key][i0] += eps
        pm[key][i0] -= eps
        fd = (loss(m, z, pp) - loss(m, z, pm)) / (2 * eps)
        assert abs(fd - dp[key][i0]) <= 1e-6 * max(1.0, abs(fd)), key


def test_predicted_ledger_golden():
    from paper_2203_00854_b200.dap import predict_block_ledger
    doc = json.load(open(os.path.join(GOLDEN, "golden_ledger.json")))
    for name, ent in doc["predicted"].items():
        cfg = EvoConfig(*ent["dims"])
        for n, want in ent["ledgers"].items():
            assert predict_block_ledger(cfg, int(n), 2) == want
