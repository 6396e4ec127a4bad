"""DAP on the GPU without a multi-GPU box: the mesh's ranks run as threads of one
process on cuda:0 (ThreadMesh), executing the same SPMD schedule as the NCCL path
(dap_block_fwd / dap_block_bwd).  Mirrors tests/test_dap.py of the reference
(test_dap.py:21-74): equivalence to the single-device block, collective counts,
byte-exact ledger vs predict_block_ledger, device-order invariance, ShardError."""

import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2203_00854_b200 as evo  # noqa: E402
from paper_2203_00854_b200 import block as B  # noqa: E402
from paper_2203_00854_b200.config import EvoConfig, init_block_params, synthetic_inputs  # noqa: E402
from paper_2203_00854_b200.dap import (CommLedger, DeviceMesh, ThreadComm, ThreadMesh, dap_block_bwd,  # noqa: E402
                                       dap_block_fwd, dap_evoformer_block, predict_block_ledger, shard_of)
from paper_2203_00854_b200.params import BlockParams  # noqa: E402

CFG = EvoConfig(16, 32, 64, 32, 2, 1, 16)


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("seed", [7, 31, 101])
def test_dap_matches_single_device(n, seed):
    p = init_block_params(CFG, seed)
    m, z = synthetic_inputs(CFG, seed)
    m1, z1 = evo.evoformer_block(m, z, p, CFG)
    mn, zn = dap_evoformer_block(m, z, p, CFG, DeviceMesh(n))
    # same bf16 kernels, different shard extents -> reduction-order differences only
    assert rel(mn, m1) <= 5e-3 and rel(zn, z1) <= 5e-3, (rel(mn, m1), rel(zn, z1))
    from oracle import evoformer_np as O
    rm, rz = O.evoformer_block(m, z, p, CFG)
    assert rel(mn, rm) <= 2e-2 and rel(zn, rz) <= 2e-2


@pytest.mark.parametrize("n", [2, 4])
def test_dap_ledger_is_byte_exact(n):
    p = init_block_params(CFG, 31)
    m, z = synthetic_inputs(CFG, 31)
    led = CommLedger(n, element_size=2)
    dap_evoformer_block(m, z, p, CFG, DeviceMesh(n), led)
    assert led.counts == {"all_to_all": 6, "all_gather": 3, "bias_gather": 1}
    assert led.summary() == predict_block_ledger(CFG, n, 2)


def test_device_order_invariance_and_shard_error():
    p = init_block_params(CFG, 7)
    m, z = synthetic_inputs(CFG, 7)
    ma, za = dap_evoformer_block(m, z, p, CFG, DeviceMesh(4))
    mb, zb = dap_evoformer_block(m, z, p, CFG, DeviceMesh(4, (2, 0, 3, 1)))
    assert np.array_equal(ma, mb) and np.array_equal(za, zb)
    with pytest.raises(evo.ShardError):
        dap_evoformer_block(m, z, p, CFG, DeviceMesh(3))


@pytest.mark.parametrize("n", [2, 4])
def test_dap_backward_matches_single_device(n):
    """fwd+bwd under DAP (all-gather^T = reduce-scatter, a2a^T = a2a, param grads summed)."""
    p = init_block_params(CFG, 11)
    m, z = synthetic_inputs(CFG, 11)
    rng = np.random.default_rng(2)
    gm, gz = rng.normal(size=m.shape), rng.normal(size=z.shape)
    dev = lambda a: torch.tensor(a, device="cuda").bfloat16()
    bp1 = BlockParams(p, CFG)
    bp1.zero_grad()
    mo, zo, sv = B.block_fwd(bp1, dev(m), dev(z))
    dm1, dz1 = B.block_bwd(bp1, sv, dev(gm), dev(gz))
    ref_grad = bp1.grad.clone()

    tm = ThreadMesh(n)
    bps = [BlockParams(p, CFG) for _ in range(n)]
    outs = [None] * n
    errs = []

    def run(r):
        try:
            comm = ThreadComm(tm, r)
            bp = bps[r]
            bp.zero_grad()
            ml, zl, s = dap_block_fwd(bp, comm, shard_of(dev(m), 0, comm), shard_of(dev(z), 0, comm))
            dm, dz = dap_block_bwd(bp, comm, s, shard_of(dev(gm), 0, comm), shard_of(dev(gz), 0, comm))
            comm.all_reduce_(bp.grad)
            outs[r] = (ml, zl, dm, dz)
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            tm.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(n)]
    [t.start() for t in th]
    [t.join() for t in th]
    if errs:
        raise errs[0]
    torch.cuda.synchronize()
    cat = lambda i: torch.cat([o[i] for o in outs], 0).double().cpu().numpy()
    assert rel(cat(0), mo.double().cpu()) <= 5e-3 and rel(cat(1), zo.double().cpu()) <= 5e-3
    assert rel(cat(2), dm1.double().cpu()) <= 2e-2, rel(cat(2), dm1.double().cpu())
    assert rel(cat(3), dz1.double().cpu()) <= 2e-2, rel(cat(3), dz1.double().cpu())
    assert rel(bps[0].grad.double().cpu(), ref_grad.double().cpu()) <= 2e-2
