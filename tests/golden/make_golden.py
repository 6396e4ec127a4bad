"""Generate golden vectors by importing the REFERENCE itself (run in the build
container only: /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

Outputs (committed, small):
  golden_cfg3.npz     - test_evoformer.py CFG (3,4,4,4,2,2,2) seeds 0..19: every
                        sub-module output + full block (reference functions).
  golden_tiny.npz     - BASELINE config 1 (16,32,64,32,2,1,16) seeds 7,31 and the
                        heads-8/4 variant seed 101: full block outputs.
  golden_softmax.npz  - fused softmax set of test_acceptance.py:218-236 (seed 8,
                        100 cases) + the SPEC.md KATs, outputs from engine.py.
  golden_ledger.json  - dap_evoformer_block ledgers (simulated, reference) for
                        test_dap CFG at N=2,4,8 and predict_block_ledger at the
                        training shape, N=2,4,8.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from evoplan import engine
from evoplan import evoformer as R
from evoplan.commcost import predict_block_ledger
from evoplan.dap_block import dap_evoformer_block
from evoplan.sharding import CommLedger, DeviceMesh

HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(params):
    h = hashlib.sha256()
    for k in sorted(params):
        h.update(k.encode())
        h.update(np.ascontiguousarray(params[k], dtype=np.float64).tobytes())
    return h.hexdigest()


def _data(cfg, seed):
    rng = np.random.default_rng(seed)
    m = rng.normal(size=(cfg.n_seq, cfg.n_res, cfg.h_msa))
    z = rng.normal(size=(cfg.n_res, cfg.n_res, cfg.h_pair))
    return m, z, R.init_block_params(cfg, seed)


def cfg3():
    cfg = R.EvoConfig(n_seq=3, n_res=4, h_msa=4, h_pair=4, n_head_msa=2,
                      n_head_pair=2, hidden_proj=2)
    out = {}
    for seed in range(20):
        m, z, p = _data(cfg, seed)
        out[f"s{seed}/msa_row"] = R.msa_row_attention(m, z, p, cfg)
        out[f"s{seed}/msa_row_bias"] = R.msa_row_bias(z, p, cfg)
        out[f"s{seed}/msa_col"] = R.msa_col_attention(m, p, cfg)
        out[f"s{seed}/msa_trans"] = R.transition(m, p, "msa_trans")
        out[f"s{seed}/pair_trans"] = R.transition(z, p, "pair_trans")
        out[f"s{seed}/opm"] = R.outer_product_mean(m, p, cfg)
        out[f"s{seed}/tri_out"] = R.tri_update_outgoing(z, p, cfg)
        out[f"s{seed}/tri_in"] = R.tri_update_incoming(z, p, cfg)
        out[f"s{seed}/pair_row"] = R.pair_attention_row(z, p, cfg)
        out[f"s{seed}/pair_col"] = R.pair_attention_col(z, p, cfg)
        mo, zo = R.evoformer_block(m, z, p, cfg)
        out[f"s{seed}/block_m"] = mo
        out[f"s{seed}/block_z"] = zo
        out[f"s{seed}/params_sha256"] = np.frombuffer(
            bytes.fromhex(_digest(p)), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_cfg3.npz"), **out)


def tiny():
    out = {}
    cases = [("c1_s7", (16, 32, 64, 32, 2, 1, 16), 7),
             ("c1_s31", (16, 32, 64, 32, 2, 1, 16), 31),
             ("h84_s101", (16, 32, 64, 32, 8, 4, 8), 101)]
    for name, dims, seed in cases:
        cfg = R.EvoConfig(*dims)
        m, z, p = _data(cfg, seed)
        mo, zo = R.evoformer_block(m, z, p, cfg)
        out[f"{name}/dims"] = np.array(dims + (seed,), dtype=np.int64)
        out[f"{name}/m"] = mo
        out[f"{name}/z"] = zo
        out[f"{name}/params_sha256"] = np.frombuffer(bytes.fromhex(_digest(p)), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_tiny.npz"), **out)


def softmax_set():
    rng = np.random.default_rng(8)
    out = {}
    for i in range(100):
        b, l = int(rng.integers(1, 5)), int(rng.integers(2, 9))
        x = rng.normal(size=(b, l, l)) * 3
        mask = np.where(rng.random((1, 1, l)) < 0.3, -1e30, 0.0)
        bias = rng.normal(size=(1, l, l))
        out[f"c{i}/x"], out[f"c{i}/mask"], out[f"c{i}/bias"] = x, mask, bias
        out[f"c{i}/y"] = engine.fused_softmax_mask_bias_raw(x, mask, bias, -1)
    # SPEC.md:67-88 known answers
    out["kat/sm_in"] = np.array([[0.0, 0.0], [np.log(2.0), 0.0]])
    out["kat/sm_out"] = engine.softmax_raw(out["kat/sm_in"], -1)
    out["kat/fs_x"] = np.array([[1.0, 1.0]])
    out["kat/fs_mask"] = np.array([[0.0, -1e30]])
    out["kat/fs_out"] = engine.fused_softmax_mask_bias_raw(
        out["kat/fs_x"], out["kat/fs_mask"], np.zeros((1, 2)), -1)
    out["kat/ln_in"] = np.array([[5.0, 5.0, 5.0], [1.0, -1.0, 0.0]])[:, :3]
    out["kat/ln_out"] = engine.layernorm_raw(out["kat/ln_in"], np.ones(3), np.zeros(3))
    np.savez_compressed(os.path.join(HERE, "golden_softmax.npz"), **out)


def ledgers():
    doc = {"simulated": {}, "predicted": {}}
    cfg = R.EvoConfig(n_seq=8, n_res=16, h_msa=8, h_pair=4, n_head_msa=2, n_head_pair=2)
    for n in (2, 4, 8):
        m, z, p = _data(cfg, 31)
        led = CommLedger(n, element_size=2)
        dap_evoformer_block(m, z, p, cfg, DeviceMesh(n), led)
        doc["simulated"][str(n)] = json.loads(led.to_json())
    train = R.EvoConfig(128, 256, 256, 128, 8, 4, 32)
    for name, c in (("dap_cfg", cfg), ("training", train),
                    ("longseq1024", R.EvoConfig(128, 1024, 256, 128, 8, 4, 32))):
        doc["predicted"][name] = {
            "dims": [c.n_seq, c.n_res, c.h_msa, c.h_pair, c.n_head_msa, c.n_head_pair, c.hidden_proj],
            "ledgers": {str(n): predict_block_ledger(c, n, 2) for n in (1, 2, 4, 8)}}
    with open(os.path.join(HERE, "golden_ledger.json"), "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    cfg3()
    tiny()
    softmax_set()
    ledgers()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
