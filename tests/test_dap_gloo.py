"""Multi-process DAP host logic on CPU: world_size 2 and 4 over gloo.

The real SPMD schedule (dap.dap_block_fwd / dap_block_bwd, DapComm over
torch.distributed) runs with the test-only CPU op stand-ins (tests/fake_ops.py)
in place of libevo.so.  Checked against the single-device composition with the
same stand-ins: outputs, input gradients, parameter gradients (after the
cross-rank all-reduce), the forward ledger vs predict_block_ledger
(commcost.py:126-158, byte-exact), and the collective counts of the backward
(every all-gather -> reduce-scatter, every all-to-all inverted).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_00854_b200.config import EvoConfig, init_block_params, synthetic_inputs

CFG = EvoConfig(16, 32, 64, 32, 2, 1, 16)
# hidden_proj 32 and R_loc % 32 == 0 at world 2: the OPM takes the fused-kernel host path (sequence-contiguous
# projections, gathered [J, P, S] b, the backward's b_seq operand)
CFG_FUSED_OPM = EvoConfig(16, 64, 64, 64, 2, 1, 32)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def _worker(rank, world, port, dims=None):
    CFG = EvoConfig(*dims) if dims else globals()["CFG"]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import fake_ops
        fake_ops.install()
        from paper_2203_00854_b200 import block as B
        from paper_2203_00854_b200.dap import (CommLedger, DapComm, dap_block_bwd, dap_block_fwd,
                                               predict_block_ledger, shard_of, switch_cols_to_rows,
                                               switch_rows_to_cols)
        from paper_2203_00854_b200.params import BlockParams

        # axis switches == reference re-shard semantics (sharding.py:130-159)
        comm = DapComm()
        x = torch.arange(8 * 12 * 3, dtype=torch.float32).view(8, 12, 3)
        sw = switch_rows_to_cols(comm, shard_of(x, 0, comm))
        assert torch.equal(sw, shard_of(x, 1, comm))
        assert torch.equal(switch_cols_to_rows(comm, sw), shard_of(x, 0, comm))

        p = init_block_params(CFG, 7)
        m, z = synthetic_inputs(CFG, 7)
        rng = np.random.default_rng(3)
        gm, gz = rng.normal(size=m.shape), rng.normal(size=z.shape)
        t = lambda a: torch.tensor(a).bfloat16()
        bp = BlockParams(p, CFG, device="cpu")
        bp.zero_grad()
        fwd_led = CommLedger(world, element_size=2)
        comm = DapComm(ledger=fwd_led)
        ml, zl, sv = dap_block_fwd(bp, comm, shard_of(t(m), 0, comm), shard_of(t(z), 0, comm))
        bwd_led = CommLedger(world, element_size=2)
        comm.ledger = bwd_led
        dm, dz = dap_block_bwd(bp, comm, sv, shard_of(t(gm), 0, comm), shard_of(t(gz), 0, comm))
        comm.all_reduce_(bp.grad)
        comm.ledger = None
        full = [comm.all_gather(a).flatten(0, 1) for a in (ml, zl, dm, dz)]
        # the overlapped (DAO) schedule == the synchronous one, bit for bit, same ledgers
        for overlap in (False, True):
            bq = BlockParams(p, CFG, device="cpu")
            bq.zero_grad()
            led_f, led_b = CommLedger(world, element_size=2), CommLedger(world, element_size=2)
            cq = DapComm(ledger=led_f, overlap=overlap)
            ml2, zl2, sv2 = dap_block_fwd(bq, cq, shard_of(t(m), 0, cq), shard_of(t(z), 0, cq))
            cq.ledger = led_b
            dm2, dz2 = dap_block_bwd(bq, cq, sv2, shard_of(t(gm), 0, cq), shard_of(t(gz), 0, cq))
            cq.all_reduce_(bq.grad, async_op=True).wait()
            for a, b_ in ((ml2, ml), (zl2, zl), (dm2, dm), (dz2, dz), (bq.grad, bp.grad)):
                assert torch.equal(a, b_), overlap
            assert led_f.to_json() == fwd_led.to_json() and led_b.to_json() == bwd_led.to_json()
        if rank == 0:
            assert fwd_led.summary() == predict_block_ledger(CFG, world, 2), fwd_led.summary()
            assert bwd_led.counts == {"all_to_all": 6, "reduce_scatter": 4, "grad_all_reduce": 1}, bwd_led.counts
            ref = BlockParams(p, CFG, device="cpu")
            ref.zero_grad()
            mo, zo, s1 = B.block_fwd(ref, t(m), t(z))
            dm1, dz1 = B.block_bwd(ref, s1, t(gm), t(gz))
            errs = [_rel(full[0], mo), _rel(full[1], zo), _rel(full[2], dm1), _rel(full[3], dz1),
                    _rel(bp.grad, ref.grad)]
            assert max(errs[:2]) <= 1e-2 and max(errs[2:]) <= 2e-2, errs
            if dims:  # the fused-OPM host path ran (sharded and single-device)
                assert fake_ops.CALLS["opm_fused_fwd"] >= 2 and fake_ops.CALLS["opm_bwd_factor"] >= 4, fake_ops.CALLS
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dap_block_gloo(world):
    mp.spawn(_worker, args=(world, _port()), nprocs=world, join=True)


def test_dap_block_gloo_fused_opm_layout():
    import dataclasses
    dims = tuple(dataclasses.astuple(CFG_FUSED_OPM))
    mp.spawn(_worker, args=(2, _port(), dims), nprocs=2, join=True)
